"""Instruction mix + stall samples per SASS opcode of one kernel in an ncu report.

usage: python tools/sass_mix.py report.ncu-rep kernel_regex [top]
"""
import csv, io, subprocess, sys
from collections import Counter

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass', '-k', 'regex:' + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) > 5:
        data.append(r)
g = lambda r, i: int(r[i]) if r[i].strip().isdigit() else 0
samples, execd = Counter(), Counter()
for r in data:
    t = r[1].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith('@') else t[0]).split('.')[0]
    samples[op] += g(r, iS)
    execd[op] += g(r, iE)
ts, te = sum(samples.values()), sum(execd.values())
print(f"{rows[0][1][:100]}\ninstructions {te}  stall samples {ts}")
for op, n in execd.most_common(top):
    print(f"  {op:10s} {n:12d} {100.0 * n / te:6.2f}%   samples {samples[op]:7d} {100.0 * samples[op] / max(ts, 1):6.2f}%")
