mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "sketch or c4 or Sketch or newton" > gpurun_out/pytest_r02c.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r02c.log
timeout 600 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/c4_disc.json 2> gpurun_out/c4_disc.err; echo "c4 rc=$?"; tail -1 gpurun_out/c4_disc.err
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none -s 8 --csv --log-file gpurun_out/dram_c4_disc.csv python tools/prof_case.py c4 256 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/dram_traffic.py gpurun_out/dram_c4_disc.csv 16
cat > /tmp/dense.py <<'PY'
import sys, os; sys.path.insert(0, os.getcwd())
import torch, paper_1610_06209_b200 as spn
sp = spn.StackedSpinner(spn.SpinnerVariant.gaussian_dense, 1024, 1024, 4096, 5)
x = torch.randn(4096, 1024, device="cuda")
for _ in range(3): y = sp.apply(x)
torch.cuda.synchronize(); print("ok")
PY
timeout 300 ncu --metrics gpu__time_duration.sum --csv --log-file gpurun_out/dense_launches.csv python /tmp/dense.py > /dev/null 2>&1; echo "dense ncu rc=$?"
grep -o '"[^"]*gemm[^"]*"\|"[^"]*Kernel[^"]*"\|"[^"]*sm100[^"]*"' gpurun_out/dense_launches.csv | sort | uniq -c | head
