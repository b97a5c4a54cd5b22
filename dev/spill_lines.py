"""Source lines of local-memory (spill) instructions of one kernel in a cubin
(development aid).  usage: python dev/spill_lines.py CUBIN SYMBOL_SUBSTRING"""
import re, subprocess, sys
lines = subprocess.run(["nvdisasm", "--print-line-info", sys.argv[1]], capture_output=True, text=True).stdout.split("\n")
func = cur = None
hits = {}
for l in lines:
    m = re.search(r"\.text\.(\S+):", l)
    if m:
        func = m.group(1)
        continue
    m = re.search(r"line (\d+)", l)
    if "//## File" in l and m:
        f = re.search(r'File "([^"]+)"', l)
        cur = (f.group(1).split("/")[-1], int(m.group(1)))
    if ("LDL" in l or "STL" in l) and func and sys.argv[2] in func:
        hits[cur] = hits.get(cur, 0) + 1
for k, v in sorted(hits.items()):
    print(k, v)
