#!/bin/bash
# c4 step time and DRAM bytes per step for env settings given on the command line (VAR=val ...)
# usage: tools/c4_dram.sh "SPN_FLOW_G=3" "SPN_FLOW_G=4 SPN_FLOW_WLAST=1" ...
mkdir -p gpurun_out
for cfg in "$@"; do
  ms=$(env $cfg timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), d.get("check",{}).get("pass"))')
  env $cfg timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none \
    --clock-control none -s 1 --csv --log-file gpurun_out/dram_c4_tmp.csv python tools/prof_case.py c4 256 > /dev/null 2>&1
  python - "$cfg" "$ms" <<'PY'
import csv, io, sys
lines = [l for l in open('gpurun_out/dram_c4_tmp.csv').read().splitlines() if l.startswith('"')]
per = {}
for r in csv.DictReader(io.StringIO("\n".join(lines))):
    if 'sketch_flow' in r['Kernel Name']:
        per.setdefault(r['ID'], {})[r['Metric Name']] = float(r['Metric Value'].replace(',', ''))
v = list(per.values())[-1]
print(f"{sys.argv[1]}: ms/check {sys.argv[2]}  DRAM read {v['dram__bytes_read.sum']/1e6:.1f} MB write {v['dram__bytes_write.sum']/1e6:.1f} MB")
PY
done
