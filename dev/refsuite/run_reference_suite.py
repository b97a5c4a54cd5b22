#!/usr/bin/env python
"""Run the reference's own test suite (pkg/tests) against the drop-in.

    python dev/refsuite/run_reference_suite.py --stage      # here: copy the tests into baseline/_ref/tests
    python dev/refsuite/run_reference_suite.py --out FILE   # on the GPU box: run them, write a JSON summary

The tests are copied into the git-ignored baseline/_ref/ (next to the
pip-installed reference) so they travel to the GPU box with the snapshot;
nothing of the reference is committed.  refsuite_shim.py maps
``mcparareal`` onto ``paper_2310_11365_b200``.  Files that test only
subsystems outside the hot path (config, harness/CLI, analysis bounds) are
not collected.
"""

from __future__ import annotations

import argparse
import json
import os
import shutil
import subprocess
import sys
import xml.etree.ElementTree as ET

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
STAGED = os.path.join(ROOT, "baseline", "_ref", "tests")
SOURCE = "/root/reference/pkg/tests"
OUT_OF_SCOPE_FILES = {"test_config.py": "TOML config schema", "test_harness.py": "experiment harness and CLI",
                      "test_analysis.py": "analysis bounds and cost model"}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--stage", action="store_true")
    ap.add_argument("--tests", default=None)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "refsuite.json"))
    ap.add_argument("--timeout", type=int, default=1500)
    args = ap.parse_args()
    if args.stage:
        shutil.rmtree(STAGED, ignore_errors=True)
        shutil.copytree(SOURCE, STAGED)
        print(f"staged {SOURCE} -> {STAGED}")
        return 0
    tests = args.tests or (SOURCE if os.path.isdir(SOURCE) else STAGED)
    files = sorted(f for f in os.listdir(tests) if f.startswith("test_") and f.endswith(".py")
                   and f not in OUT_OF_SCOPE_FILES)
    xml = os.path.join(os.path.dirname(os.path.abspath(args.out)), "refsuite_junit.xml")
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([HERE, ROOT, os.environ.get("PYTHONPATH", "")]))
    cmd = [sys.executable, "-m", "pytest", "-p", "refsuite_shim", "-q", "-rfs", "--rootdir", tests,
           "-c", os.devnull, f"--junitxml={xml}", "-p", "no:cacheprovider"] + [os.path.join(tests, f) for f in files]
    proc = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=args.timeout)
    summary = {"command": " ".join(cmd[1:]), "returncode": proc.returncode, "files": {},
               "not_collected": OUT_OF_SCOPE_FILES, "failures": [], "skips": {}}
    root = ET.parse(xml).getroot()
    for case in root.iter("testcase"):
        f = (case.get("classname") or "").split(".")[0] + ".py"
        st = summary["files"].setdefault(f, {"passed": 0, "failed": 0, "skipped": 0})
        if case.find("failure") is not None or case.find("error") is not None:
            st["failed"] += 1
            node = case.find("failure") if case.find("failure") is not None else case.find("error")
            summary["failures"].append({"test": f"{f}::{case.get('name')}",
                                        "message": (node.get("message") or "")[:300]})
        elif case.find("skipped") is not None:
            st["skipped"] += 1
            msg = (case.find("skipped").get("message") or "")[:200]
            summary["skips"][f"{f}::{case.get('name')}"] = msg
        else:
            st["passed"] += 1
    tot = {k: sum(v[k] for v in summary["files"].values()) for k in ("passed", "failed", "skipped")}
    summary["totals"] = tot
    with open(args.out, "w") as fh:
        json.dump(summary, fh, indent=1)
    print(proc.stdout[-4000:])
    print(proc.stderr[-2000:], file=sys.stderr)
    print(json.dumps(tot))
    return 0


if __name__ == "__main__":
    sys.exit(main())
