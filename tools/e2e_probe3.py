"""Where does the config-3 host pipeline lose PCIe rate?  H2D of an 8 GiB pinned buffer in 128 MB chunks on
two streams: (i) copies only, (ii) copies + the hash kernel on each chunk, (iii) the library's host call."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1610_06209_b200 as spn
rows, n = 1 << 17, 16384
xh = torch.randn(rows, n).pin_memory()
h = spn.MultiTableHasher(spn.SpinnerVariant.hd3_hd2_hd1, n, n, 8, seed=3)
chunk = 2048
bufs = [torch.empty(chunk, n, device="cuda") for _ in range(2)]
sts = [torch.cuda.Stream() for _ in range(2)]
def run(kernel):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for c, r0 in enumerate(range(0, rows, chunk)):
        s = sts[c & 1]
        with torch.cuda.stream(s):
            bufs[c & 1].copy_(xh[r0:r0 + chunk], non_blocking=True)
            if kernel:
                h.hash_ids(bufs[c & 1], stream=s)
    torch.cuda.synchronize(); return rows * n * 4 / (time.perf_counter() - t0) / 1e9
run(True)
print(f"(i)  copies only        : {run(False):.1f} GB/s")
print(f"(ii) copies + hash      : {run(True):.1f} GB/s")
xn = xh.numpy()
h.plan.hash(xn[:4096])
t0 = time.perf_counter(); h.plan.hash(xn); dt = time.perf_counter() - t0
print(f"(iii) spn_hash_f32_host : {rows * n * 4 / dt / 1e9:.1f} GB/s")
# kernel alone on a 2048-row chunk
x = bufs[0]
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10): h.hash_ids(x)
torch.cuda.synchronize(); print(f"hash kernel on {chunk} rows: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms (copy of the chunk at 55 GB/s: {chunk * n * 4 / 55e9 * 1e3:.3f} ms)")
