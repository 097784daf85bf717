"""Executed SASS of one kernel in an ncu report: instructions with their execution counts (per launch),
filtered by an opcode regex.  usage: python tools/sass_exec.py report.ncu-rep kernel_regex [opcode_regex]"""
import csv
import io
import re
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
ore = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass', '-k', 'regex:' + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iA, iE, iS = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) <= 5:
        continue
    n = int(r[iE]) if r[iE].strip().isdigit() else 0
    if n == 0 or (ore and not ore.search(r[1])):
        continue
    print(f"{int(r[iA], 16) & 0xfffff:#07x} {n:10d} {r[iS]:>6s}  {r[1][:90]}")
