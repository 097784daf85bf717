"""DRAM bytes (read + write) of one bench step from an `ncu --metrics dram__bytes_read.sum,
dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --csv` capture of tools/prof_case.py.

The capture covers whole steps at the end of the run: the last `per_step` hot-path launches (the
spinner / pass kernels, not torch's input generation) are one step.
usage: python tools/dram_traffic.py dram_<c>.csv per_step   -> prints JSON
"""
import collections
import csv
import io
import json
import sys

path, per_step = sys.argv[1], int(sys.argv[2])
lines = [ln for ln in open(path).read().splitlines() if ln.startswith('"')]
per = collections.OrderedDict()
for r in csv.DictReader(io.StringIO("\n".join(lines))):
    per.setdefault(r["ID"], {"kernel": r["Kernel Name"]})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
hot = [v for v in per.values() if "spinner_vec" in v["kernel"] or "pass" in v["kernel"] or "sketch_flow" in v["kernel"]]
step = hot[-per_step:]
rd = sum(v["dram__bytes_read.sum"] for v in step)
wr = sum(v["dram__bytes_write.sum"] for v in step)
ns = sum(v["gpu__time_duration.sum"] for v in step)
print(json.dumps({"launches": len(step), "dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes": rd + wr,
                  "serialised_ns": ns, "kernels": sorted({v["kernel"].split("(")[0] for v in step})}))
