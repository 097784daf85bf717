#!/bin/bash
# Round-end style bench pass: the reference arm, then ours (default flags), each timed by wall clock.
# usage: tools/gpu_bench.sh tag [extra bench args]
tag=${1:-x}; shift
mkdir -p gpurun_out
t0=$(date +%s); timeout 900 python bench.py --impl reference ${@} > gpurun_out/ref_$tag.json 2> gpurun_out/ref_$tag.err; echo "ref rc=$? wall=$(( $(date +%s) - t0 ))s"
t0=$(date +%s); timeout 1500 python bench.py ${@} > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$? wall=$(( $(date +%s) - t0 ))s"
tail -c 1500 gpurun_out/bench_$tag.err
python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
for f in (f"gpurun_out/ref_{tag}.json", f"gpurun_out/bench_{tag}.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f, d.get("impl", "ours"), "value", d["value"], "ms", d["ms_per_step"], "e2e", (d.get("e2e") or {}).get("value"))
    for k, v in (d.get("configs") or {}).items():
        print("  ", k, v["value"], (v.get("roofline") or {}).get("frac"), (v.get("e2e") or {}).get("value"), v.get("check"))
PY
