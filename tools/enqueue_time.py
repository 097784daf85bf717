import time, torch, sys
sys.path.insert(0, '.')
import paper_1610_06209_b200 as spn
V = spn.SpinnerVariant
sp = spn.StackedSpinner(V.gauss3, 1 << 20, 1 << 20, 1 << 20, 13, scale=1.0)
x = torch.randn(256, 1 << 20, device="cuda"); y = torch.empty_like(x)
sk = spn.SketchOperator(V.hd3_hd2_hd1, 1 << 17, 2048, 11, mode="random", p_seed=77)
a = torch.randn(1 << 17, 256, device="cuda"); o = torch.empty(2048, 256, device="cuda")
for name, f in [("c5", lambda: sp.apply(x, relu=True, out=y)), ("c4", lambda: sk.apply(a, out=o))]:
    for _ in range(3): f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        torch.cuda._sleep(20_000_000)  # ~10 ms of GPU work queued first: pure host enqueue time
        t0 = time.perf_counter(); f(); t1 = time.perf_counter()
        torch.cuda.synchronize(); ts.append(t1 - t0)
    print(name, "host enqueue ms", [round(1e3 * t, 3) for t in ts])
