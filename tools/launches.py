"""Condense an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list.

usage: python tools/launches.py launches.csv out.csv "command that was profiled"
Writes id,kernel,grid,block,ns for every launch plus a per-kernel share summary
(cold-cache, serialised times: compare SHARES only) to stdout.
"""
import csv, sys
from collections import defaultdict

src, dst, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(open(src)) if len(r) > 10 and r[0].isdigit() and r[12] == "gpu__time_duration.sum"]
tot = defaultdict(float)
cnt = defaultdict(int)
with open(dst, "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 {cmd}\n")
    f.write("# cold-cache, serialised per-launch times (ns); compare SHARES only\n")
    f.write("id,kernel,grid,block,gpu__time_duration_ns\n")
    for r in rows:
        name = r[4] if len(r[4]) < 90 else r[4][:60] + "..."
        ns = float(r[14].replace(",", ""))
        f.write(f'{r[0]},"{name}",{r[8]},{r[7]},{int(ns)}\n')
        key = name.split("(")[0]
        tot[key] += ns
        cnt[key] += 1
all_ns = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{100 * v / all_ns:6.2f}%  {cnt[k]:5d} launches  {v / cnt[k] / 1e3:9.2f} us avg  {k}")
