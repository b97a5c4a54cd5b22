"""Opcode histogram of the fine step loop (from the stage-wait SYNCS to the
loop's backward branch) of one kernel in a cubin (development aid).
usage: python dev/loop_sass.py CUBIN MANGLED_SYMBOL"""
import re, subprocess, sys
from collections import Counter
sass = subprocess.run(["cuobjdump", "-sass", "-fun", sys.argv[2], sys.argv[1]], capture_output=True, text=True).stdout
ins = [l for l in sass.split("\n") if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l)]
addr = lambda l: int(re.search(r"/\*([0-9a-f]+)\*/", l).group(1), 16)
op = lambda l: re.sub(r"\s+", " ", l.split("*/")[1].split("/*")[0]).strip()
start = next(i for i, l in enumerate(ins) if "SYNCS.PHASECHK" in l and sum("DMUL" in x for x in ins[i:i + 150]) >= 20)
a0 = addr(ins[start])
end = None
for j in range(start, len(ins)):
    m = re.search(r"BRA (?:0x([0-9a-f]+))", op(ins[j]))
    if m and a0 - 0x800 < int(m.group(1), 16) <= a0:
        end = j
        break
body = [op(l) for l in ins[start - 12:(end or start + 600) + 1]]
c = Counter(b.split(" ")[0].lstrip("@!P0123456789 ") or b.split(" ")[1] for b in body)
print(len(body), "instructions;", "LDL/STL:", sum(("LDL" in b or "STL" in b) for b in body))
print(c.most_common(20))
