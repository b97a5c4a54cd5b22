"""Per-source-line instruction and stall-sample shares of one kernel from an
ncu report (SASS page) mapped through nvdisasm line info (development aid).
usage: python dev/ncu_lines.py REPORT.ncu-rep OBJ.cubin MANGLED_SYMBOL [top]"""
import csv, io, re, subprocess, sys
from collections import defaultdict

rep, cubin, sym = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
dis = subprocess.run(['nvdisasm', '--print-line-info', cubin], capture_output=True, text=True).stdout.split('\n')
start = next(i for i, l in enumerate(dis) if f'.text.{sym}' in l and 'section' in l)
cur, addr2line = None, {}
for l in dis[start + 1:]:
    if l.strip().startswith('.section') and 'text' in l:
        break
    m = re.search(r'line (\d+)', l)
    if '//## File' in l and m:
        f = re.search(r'File "([^"]+)"', l)
        cur = (f.group(1).split('/')[-1] if f else '?', int(m.group(1)))
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*)', l)
    if m and cur:
        addr2line[int(m.group(1), 16)] = cur
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'] + (['-k', 'regex:' + __import__('os').environ['NCU_KERNEL']] if __import__('os').environ.get('NCU_KERNEL') else []),
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
iA, iS, iE = h.index('Address'), h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
base = int(data[0][iA], 16)
agg = defaultdict(lambda: [0, 0])
tot = [0, 0]
for r in data:
    key = addr2line.get(int(r[iA], 16) - base, ('?', 0))
    s = int(r[iS]) if r[iS].isdigit() else 0
    e = int(r[iE]) if r[iE].isdigit() else 0
    agg[key][0] += s; agg[key][1] += e; tot[0] += s; tot[1] += e
print(f'samples {tot[0]}  warp instructions {tot[1]}')
for k, (s, e) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f'{k[0]}:{k[1]:<5d} stall {100 * s / tot[0]:5.1f}%  instr {100 * e / tot[1]:5.1f}%')
