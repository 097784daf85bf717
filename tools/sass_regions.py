"""Stall samples and executed instructions of one kernel in an ncu report, split into the chain loop
(the first backward branch whose body has FADD2) and everything else, plus the top stall PCs.

usage: python tools/sass_regions.py report.ncu-rep kernel_regex
"""
import csv
import io
import re
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass', '-k', 'regex:' + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iA, iS, iE = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) > 5:
        data.append(r)
g = lambda r, i: int(r[i]) if r[i].strip().isdigit() else 0
addr = [int(r[iA], 16) for r in data]
src = [r[1] for r in data]
lo = hi = None
for k, s in enumerate(src):
    m = re.search(r'BRA(\.U)? [^,]*?,? ?0x([0-9a-f]+)', s)
    if m:
        t = int(m.group(2), 16)
        if t < addr[k] and any('FADD2' in x for x in src[addr.index(t):k] if True) if t in addr else False:
            lo, hi = t, addr[k]
            break
tot_s = sum(g(r, iS) for r in data)
tot_e = sum(g(r, iE) for r in data)
in_s = sum(g(r, iS) for r, a in zip(data, addr) if lo is not None and lo <= a <= hi)
in_e = sum(g(r, iE) for r, a in zip(data, addr) if lo is not None and lo <= a <= hi)
print(f"loop {lo:#x}..{hi:#x}: samples {in_s}/{tot_s} ({100*in_s/max(tot_s,1):.1f}%), instructions {in_e}/{tot_e} ({100*in_e/max(tot_e,1):.1f}%)")
top = sorted(zip(data, addr), key=lambda t: -g(t[0], iS))[:25]
for r, a in top:
    print(f"  {a:#07x} {g(r, iS):7d}  {'loop' if lo is not None and lo <= a <= hi else 'out '}  {r[1][:70]}")
