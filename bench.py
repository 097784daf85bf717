#!/usr/bin/env python3
"""Benchmark of the structured-spinner hot path on B200 (BASELINE.json metric:
"spinner vectors/sec (and GB/s as % of HBM roofline) at 1/2/4/8 B200 vs host-CPU ref").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step is one pass of the hot path over one batch of the config's synthetic input:
  c1  LSH, 1 table: 4096 x 1024 unit vectors -> int32 ids + fp32 y (scale 1)
  c2  (default; BASELINE configs[1]) Gaussian RFF: 60000 x 784 -> pad 1024, 4 blocks,
      k = 4096, sigma = 5 -> 60000 x 8192 fp32 features
  c3  LSH, 8 tables: 2^20 x 16384 unit vectors (64 GiB, generated on device) -> ids, + NCCL all-gather
  c4  sketch: A[131072][256] -> sqrt(N/m) P H D3 H D2 H D1 A, m = 2048 random rows
  c5  all-Gaussian diagonals + ReLU: 256 x 2^20 -> 256 x 2^20
Multi-GPU (torchrun, one process per GPU): weak scaling, each rank runs its own
full batch (different seeds); c3 additionally all-gathers the codes over NCCL.
`value` = vectors processed by all ranks / max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "spinner vectors/sec"
UNIT = "vectors/s"

CONFIGS = {
    "c1": dict(workload="BASELINE configs[0]: cross-polytope LSH, 1 table, 4096 x n=1024, ids + fp32 y (scale 1)",
               n=1024, batch=4096, bytes_per_vec=1024 * 4 * 2 + 4, flush=True),
    "c2": dict(workload="BASELINE configs[1]: Gaussian RFF, 60000 x 784 (zero-pad 1024), 4 HD3HD2HD1 blocks "
                        "(k=4096), sigma=5, out 60000 x 8192 fp32",
               n=1024, n_in=784, batch=60000, k=4096, sigma=5.0, bytes_per_vec=784 * 4 + 8192 * 4, flush=False),
    "c3": dict(workload="BASELINE configs[2]: cross-polytope LSH, 8 tables, 2^20 x n=16384 unit vectors -> int32 ids",
               n=16384, batch=1 << 20, tables=8, bytes_per_vec=16384 * 4 + 8 * 4, flush=False),
    "c4": dict(workload="BASELINE configs[3]: sketch sqrt(N/m) P H D3 H D2 H D1 A, A = 131072 x 256, m = 2048 "
                        "random rows", N=1 << 17, d=256, m=2048, bytes_per_vec=(1 << 17) * 4 + 2048 * 4, flush=True),
    "c5": dict(workload="BASELINE configs[4]: ReLU(H D3 H D2 H D1 x), Gaussian D's, 256 x n=2^20",
               n=1 << 20, batch=256, bytes_per_vec=(1 << 20) * 8, flush=False),
    "c7": dict(workload="SURVEY 8(f) rank 2: collision_curve of the HD3 family, n=256, m=64, 20000 pairs x 100 "
                        "trials (acceptance criterion 5 scale); units = hashed vectors (2 x pairs x trials)",
               n=256, m=64, pairs=20000, trials=100, bytes_per_vec=256 * 4, flush=False),
    "c6": dict(workload="SURVEY 8(f) rank 1: one sketched Newton iteration of solve() (fresh HD3 SketchOperator, "
                        "sketched_step, Armijo line search) for logistic regression on A = 131072 x 256, m = 2048",
               N=1 << 17, d=256, m=2048, bytes_per_vec=(1 << 17) * 4 * 6, flush=False),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ----------------------------------------------------------------- distributed
def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if os.environ.get("SPN_BENCH_BACKEND") == "gloo":
            # test mode only: exercise the multi-rank code path with every rank on the GPUs there
            # are (ranks share a device; timings are then contended and not a scaling result)
            local = local % max(1, torch.cuda.device_count())
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.samples, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ workloads
class Workload:
    """Device-resident inputs/outputs for one config + a `step()` that launches the hot path."""

    def __init__(self, name, cfg, rank, device, world=1):
        import torch
        import paper_1610_06209_b200 as spn
        self.spn, self.torch, self.name, self.cfg = spn, torch, name, cfg
        self.device = device
        g = torch.Generator(device="cuda")
        g.manual_seed(1234 + rank)
        V = spn.SpinnerVariant
        self.launches_per_step = 1
        if name == "c1":
            self.sp = spn.StackedSpinner(V.hd3_hd2_hd1, 1024, 1024, 1024, 42 + rank, scale=1.0)
            x = torch.randn((cfg["batch"], 1024), device="cuda", generator=g)
            self.x = x / x.norm(dim=1, keepdim=True)
            self.y = torch.empty_like(self.x)
            self.vectors = cfg["batch"]
        elif name == "c2":
            self.sp = spn.StackedSpinner(V.hd3_hd2_hd1, 1024, 1024, cfg["k"], 5 + rank)
            self.fm = spn.FeatureMap(self.sp, spn.KernelKind.gaussian(cfg["sigma"]))
            self.x = torch.rand((cfg["batch"], cfg["n_in"]), device="cuda", generator=g)
            self.out = torch.empty((cfg["batch"], 2 * cfg["k"]), device="cuda")
            self.vectors = cfg["batch"]
        elif name == "c3":
            self.h = spn.MultiTableHasher(V.hd3_hd2_hd1, cfg["n"], cfg["n"], cfg["tables"], seed=3)
            self.x = torch.empty((cfg["batch"], cfg["n"]), device="cuda")
            for r0 in range(0, cfg["batch"], 1 << 16):  # N(0,1) then L2-normalised, generated on device
                blk = torch.randn((min(1 << 16, cfg["batch"] - r0), cfg["n"]), device="cuda", generator=g)
                self.x[r0:r0 + blk.shape[0]] = blk / blk.norm(dim=1, keepdim=True)
                del blk
            self.ids = torch.empty((cfg["batch"], cfg["tables"]), device="cuda", dtype=torch.int32)
            self.vectors = cfg["batch"]
            # multi-GPU: the all-gather of the codes fused into the hash kernel (peer stores over
            # NVLink through CUDA IPC mappings); NCCL all_gather stays as the fallback
            self.pc, self.rank, self.exchange = None, rank, None
            if world > 1:
                try:
                    from paper_1610_06209_b200.shard import PeerCodes
                    self.pc = PeerCodes(world * cfg["batch"], cfg["tables"], world, rank, device)
                    self.exchange = "fused peer stores in the hash kernel (CUDA IPC / NVLink), one barrier"
                except Exception as exc:  # pragma: no cover - depends on the node's IPC support
                    self.exchange = f"nccl all_gather_into_tensor (peer mapping unavailable: {type(exc).__name__})"
        elif name == "c4":
            self.sk = spn.SketchOperator(V.hd3_hd2_hd1, cfg["N"], cfg["m"], 11 + rank, mode="random", p_seed=77)
            self.x = torch.randn((cfg["N"], cfg["d"]), device="cuda", generator=g)
            self.out = torch.empty((cfg["m"], cfg["d"]), device="cuda")
            self.vectors = cfg["d"]  # one column = one spinner vector
            lsa = (17 + 1) // 2
            groups = math.ceil(cfg["d"] / max(32, ((32 << 20) // (cfg["N"] * 4)) // 32 * 32))
            self.launches_per_step = 4 * groups
            del lsa
        elif name == "c6":
            from paper_1610_06209_b200 import newton
            self.newton = newton
            f = torch.randn((cfg["N"], cfg["d"]), device="cuda", generator=g)
            y = torch.where(torch.rand(cfg["N"], device="cuda", generator=g) < 0.5, -1.0, 1.0)
            self.prob = spn.LogisticProblem(f, y)
            self.prob.workspace(cfg["m"])
            self.xk = torch.full((cfg["d"],), 0.01, dtype=torch.float64, device="cuda")
            self.vectors = cfg["d"]  # columns sketched per iteration
            self.t = 0
            import concurrent.futures
            self.pool = concurrent.futures.ThreadPoolExecutor(1)  # next sketch realised during this step
            self.mk = lambda it: spn.SketchOperator(V.hd3_hd2_hd1, cfg["N"], cfg["m"], spn.mix_seed(3, it))  # noqa: E731
            self.pending = self.pool.submit(self.mk, 0)
            # pass over A + 4 sketch passes + line-search pass per iteration (launch count is a lower bound)
            self.launches_per_step = 16
        elif name == "c7":
            import numpy as np
            rng = np.random.default_rng(88 + rank)
            P, n = cfg["pairs"], cfg["n"]
            ang = np.pi * (np.arange(P) + 0.5) / P
            x = rng.standard_normal((P, n))
            u = rng.standard_normal((P, n))
            x /= np.linalg.norm(x, axis=1, keepdims=True)
            u -= np.sum(u * x, axis=1, keepdims=True) * x
            u /= np.linalg.norm(u, axis=1, keepdims=True)
            y = np.cos(ang)[:, None] * x + np.sin(ang)[:, None] * u
            self.cx = torch.from_numpy(x.astype(np.float32)).cuda()
            self.cy = torch.from_numpy(y.astype(np.float32)).cuda()
            self.cd = 2.0 * np.sin(ang / 2.0)
            self.fac = spn.make_hasher_factory(V.hd3_hd2_hd1, n, cfg["m"])
            self.vectors = 2 * P * cfg["trials"]
            self.t = 0
        elif name == "c5":
            self.sp = spn.StackedSpinner(V.gauss3, cfg["n"], cfg["n"], cfg["n"], 13 + rank, scale=1.0)
            self.x = torch.randn((cfg["batch"], cfg["n"]), device="cuda", generator=g)
            self.y = torch.empty_like(self.x)
            self.vectors = cfg["batch"]
            G = max(1, min(cfg["batch"], (24 << 20) // (cfg["n"] * 4)))
            self.launches_per_step = 4 * math.ceil(cfg["batch"] / G)
        torch.cuda.synchronize()

    def step(self, stream):
        if self.name == "c1":
            return self.sp.plan.hash(self.x, y_out=self.y, stream=stream)
        if self.name == "c2":
            return self.spn.embed(self.fm, self.x, out=self.out, stream=stream)
        if self.name == "c3":
            if self.pc is not None:
                return self.pc.hash(self.h, self.x, self.rank * self.cfg["batch"], stream=stream)
            return self.h.plan.hash(self.x, stream=stream)
        if self.name == "c4":
            return self.sk.apply(self.x, out=self.out, stream=stream)
        if self.name == "c7":  # lsh.cpp:38-74, fresh trial seeds every step
            self.t += 1
            return self.spn.collision_curve((self.cx, self.cy, self.cd), self.fac, self.cfg["trials"], 90 + self.t,
                                            stream=stream)
        if self.name == "c6":  # newton_sketch.cpp:155-170, one iteration
            cfg, nt = self.cfg, self.newton
            sk = self.pending.result()
            self.t += 1
            self.pending = self.pool.submit(self.mk, self.t)
            step, g, f = nt._step_dev(self.prob, self.xk, sk, stream)
            slope = float(self.torch.dot(g, step).item())
            s, _ = nt._backtrack(self.prob, self.xk, step, float(f.item()), slope, stream)
            self.xk = self.xk + s * step
            return self.xk
        return self.sp.apply(self.x, relu=True, out=self.y, stream=stream)


def run_ours(args, rank, world, local):
    import torch
    cfg = CONFIGS[args.config]
    w = Workload(args.config, cfg, rank, local, world)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if cfg["flush"] else None
    flush_sink = torch.zeros((), dtype=torch.int64, device="cuda")
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        # warm-up, continued (untimed) until nvidia-smi has seen the GPU under this load
        t_end = time.time() + 3.0
        i = 0
        # (multi-rank: a fixed count — steps may contain collectives, so every rank must run as many)
        while i < max(3, args.warmup) or (world == 1 and len(clk.samples) < 3 and time.time() < t_end):
            w.step(stream)
            i += 1
            if i >= max(3, args.warmup):
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        for i in range(args.steps):
            if flush is not None:
                # evict L2 outside the timed region: write 256 MB (> 126 MB L2), then read it back so
                # the lines left in L2 are clean (otherwise the timed kernel pays for write-backs of
                # the flush's own dirty lines)
                flush.fill_(i & 0xFF)
                flush_sink += flush.view(torch.int64).sum()
            # keep the device busy past the start event so it never times the host's launch latency
            torch.cuda._sleep(200_000)
            evs[i][0].record(stream)
            w.step(stream)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    ids = None
    if args.config == "c3" and world > 1 and w.pc is None:  # exchange step: NCCL all-gather of the codes
        from paper_1610_06209_b200.shard import gather_codes
        ids = w.step(stream)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        gather_codes(ids, world)
        t1.record(stream)
        torch.cuda.synchronize()
        total_ms += t0.elapsed_time(t1) * args.steps
    barrier(world)
    torch.cuda.synchronize()
    total_ms = max_over_ranks(total_ms, world)
    ms_per_step = total_ms / args.steps
    value = w.vectors * world * args.steps / (total_ms / 1e3)
    peak, peak_src = measured_peaks()
    kernel_ms = statistics.mean(step_ms) / w.launches_per_step  # dominant kernel = the whole step for c1-c3
    alg_bytes = cfg["bytes_per_vec"] * w.vectors
    achieved = alg_bytes / (statistics.mean(step_ms) / 1e3) / 1e9
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, BASELINE config shapes)",
        "config": {"workload": cfg["workload"], "name": args.config, "vectors_per_gpu_step": w.vectors,
                   "l2": "L2 flushed (256 MB write + read-back) between timed steps" if cfg["flush"]
                   else "inputs+outputs > 126 MB L2", "parallelism": f"dp{world} (independent shards)",
                   **({"exchange": w.exchange} if getattr(w, "exchange", None) else {})},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic_from_profiles(args.config), "peak_source": peak_src,
                     "algorithmic_bytes_per_step": alg_bytes, "mean_kernel_ms": kernel_ms},
        "clocks": clk.summary(),
        "gpu_launches": w.launches_per_step * args.steps,
    }
    result.update(secondary_rooflines(args.config, cfg, w, statistics.mean(step_ms), result["clocks"]))
    if args.config in ("c1", "c2") and not args.no_e2e:
        result["e2e"] = e2e_measure(args, w, world)
    return result, w


# Issue floors from the ncu instruction mix (tools/sass_mix.py on profiles/r01_<c>_ncu_full.json, DESIGN.md
# sections 3-4): warp-issue cycles per unit with FADD2 counted twice, at the clock the floor was computed for.
ISSUE_FLOOR = {
    "c2": {"ms": 0.356, "mhz": 1785.0, "model": "6.26 K issue cycles per sample (1536 FADD2 x2, 768 FADD, 432 sign "
           "flips, 555 LDS/STS, 416 FMUL, 256 MUFU, ~450 address/loop) over 60000 samples on 592 SMSPs"},
    "c3": {"ms": 205.6, "mhz": 1965.0, "model": "28.5 K warp-issue cycles per (vector, table) (9216 FADD2 x2, 3072 "
           "FADD, 1931 LOP3 + 192 R2P sign flips, 1925 LDS/STS transposes, 576 LDG, 754 IMAD, argmax) over "
           "2^20 x 8 items on 592 SMSPs"},
}


# L2-resident read-modify-write bandwidth measured on this pool's B200 (tools/microbench/mb.cu, in-place
# float4 r+w over a 32 MB buffer, 148 x 4 CTAs): 12.3-12.9 TB/s at 16-32 MB, 9.3 TB/s at 64 MB.  (A torch
# elementwise probe reaches only ~6.5 TB/s, its own kernel's limit, so it is not used as the roof.)
L2_RMW_GBS = 12877.8


def secondary_rooflines(name, cfg, w, step_ms, clocks):
    """The roofs that actually bind the configs whose HBM fraction is low by construction: the multi-pass
    configs (c4, c5) against the L2 read-modify-write rate (4 passes, each reading and writing the working
    set through L2), the issue-bound ones (c2, c3) against their instruction-count floor."""
    out = {}
    if name in ("c4", "c5"):
        if name == "c5":
            l2_bytes = 4 * 2 * w.vectors * cfg["n"] * 4
        else:  # passes 1-3 read + write A's columns, pass 4 reads them and writes the m gathered rows
            l2_bytes = 7 * cfg["N"] * cfg["d"] * 4 + cfg["m"] * cfg["d"] * 4
        peak = L2_RMW_GBS
        ach = l2_bytes / (step_ms * 1e-3) / 1e9
        out["roofline_l2"] = {"bound": "l2", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                              "traffic_model": "4 passes x (read + write) of the working set through L2",
                              "l2_bytes_per_step": l2_bytes,
                              "peak_source": "tools/microbench/mb.cu L2 rmw, 32 MB, this pool's B200"}
    if name in ISSUE_FLOOR:
        f = ISSUE_FLOOR[name]
        mhz = clocks.get("sm_mhz") or f["mhz"]
        floor = f["ms"] * f["mhz"] / mhz
        out["roofline_issue"] = {"bound": "issue", "floor_ms": floor, "measured_ms": step_ms,
                                 "frac": floor / step_ms, "sm_mhz": mhz, "model": f["model"]}
    return out


def traffic_from_profiles(config):
    """dram bytes/launch from the committed `ncu --set full` summary, if present."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(config)
    except Exception:
        return None


def e2e_measure(args, w, world):
    """Same metric through the public API with HOST buffers: pinned host input in,
    pinned host output back, the copies inside the timed region (spn_*_host)."""
    import torch
    cfg = CONFIGS[args.config]
    xh = w.x.cpu().pin_memory().numpy()
    if args.config == "c2":
        outh = torch.empty((cfg["batch"], 2 * cfg["k"]), dtype=torch.float32).pin_memory().numpy()
        run = lambda: w.spn.embed(w.fm, xh, out=outh)  # noqa: E731
        bi, bo = xh.nbytes, outh.nbytes
    else:
        outh = torch.empty((cfg["batch"], 1024), dtype=torch.float32).pin_memory().numpy()
        run = lambda: w.sp.plan.apply(xh, out=outh)  # noqa: E731
        bi, bo = xh.nbytes, outh.nbytes
    run()
    steps = max(3, min(args.steps, 10))
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(steps):
        run()
    dt = time.perf_counter() - t0
    dt = max_over_ranks(dt, world)
    return {"value": w.vectors * world * steps / dt, "unit": UNIT, "h2d_bytes_per_step": bi,
            "d2h_bytes_per_step": bo, "steps": steps, "api": "spn_embed_f32_host" if args.config == "c2"
            else "spn_apply_f32_host (the y projection only; the host API returns ids through spn_hash_f32_host)"}


# ---------------------------------------------------------------- CPU reference
def cpu_reference(config, budget_s=20.0, threads=None):
    """The reference's own CPU code (oracle/_ref: proj/src compiled unmodified) on the
    host cores, over a bounded sample of the same workload.  Returns (vectors/s, info)."""
    import numpy as np
    from oracle.oracle import HD3, Oracle, Reference
    threads = threads or os.cpu_count() or 1
    r, o = Reference(), Oracle()
    cfg = CONFIGS[config]
    rng = np.random.default_rng(0)

    def timed(fn, count):
        t0 = time.perf_counter()
        fn(count)
        return time.perf_counter() - t0

    if config == "c1":
        x = rng.standard_normal((cfg["batch"], 1024)).astype(np.float32)
        fn = lambda c: (r.hash(HD3, 1024, 1024, [42], x[:c], threads=threads),  # noqa: E731
                        r.apply(HD3, 1024, 1024, 1024, 42, 1.0, x[:c], threads=threads))
        total = cfg["batch"]
        what = "CrossPolytopeHasher::hash + StructuredSpinner::apply(scale 1)"
    elif config == "c2":
        x = rng.random((cfg["batch"], cfg["n_in"])).astype(np.float32)
        fn = lambda c: r.embed(HD3, 1024, cfg["k"], 5, 0, cfg["sigma"], x[:c], n_in=cfg["n_in"],  # noqa: E731
                               threads=threads)
        total = cfg["batch"]
        what = "embed(FeatureMap{StackedSpinner(HD3,1024,1024,4096)}, gaussian sigma=5)"
    elif config == "c3":
        x = rng.standard_normal((4096, cfg["n"])).astype(np.float32)
        seeds = [o.mix_seed(3, t) for t in range(cfg["tables"])]
        fn = lambda c: r.hash(HD3, cfg["n"], cfg["n"], seeds, x[:c], threads=threads)  # noqa: E731
        total = x.shape[0]
        what = "8 x CrossPolytopeHasher::hash (n=16384)"
    elif config == "c4":
        a = rng.standard_normal((cfg["N"], cfg["d"])).astype(np.float32)
        rows = o.sample_rows(cfg["N"], cfg["m"], 77)
        fn = lambda c: r.sketch(HD3, np.ascontiguousarray(a[:, :c]), cfg["m"], 11, row_list=rows,  # noqa: E731
                                threads=threads)
        total = cfg["d"]
        what = "SketchOperator::apply restated over the reference StackedSpinner, random P"
    elif config == "c7":  # the reference's collision_curve on 2 of the 100 trials (single-threaded driver)
        P, n = cfg["pairs"], cfg["n"]
        ang = np.pi * (np.arange(P) + 0.5) / P
        x = rng.standard_normal((P, n))
        u = rng.standard_normal((P, n))
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        u -= np.sum(u * x, axis=1, keepdims=True) * x
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        y = np.cos(ang)[:, None] * x + np.sin(ang)[:, None] * u
        d = 2.0 * np.sin(ang / 2.0)
        dt = timed(lambda c: r.collision_curve(HD3, n, cfg["m"], x, y, d, 2, 91), 1)
        return 2 * P * 2 / dt, {"kind": "reference", "cores": 1, "cpu_model": cpu_model(),
                                "sample": "collision_curve over all 20000 pairs x 2 trials (80000 hashed vectors); "
                                          "the reference's lsh.cpp driver, single-threaded"}
    elif config == "c6":  # one reference sketched_step (newton_sketch.cpp:103-122, single-threaded code)
        a = rng.standard_normal((cfg["N"], cfg["d"])).astype(np.float32).astype(np.float64)
        y = np.where(rng.random(cfg["N"]) < 0.5, -1.0, 1.0)
        x = np.full(cfg["d"], 0.01)
        dt = timed(lambda c: r.sketched_step(a, y, x, HD3, cfg["m"], o.mix_seed(3, 0)), 1)
        return cfg["d"] / dt, {"kind": "reference", "cores": 1, "cpu_model": cpu_model(),
                               "sample": "1 sketched_step (131072 x 256, m = 2048, HD3) of c6 = 256 sketched "
                                         "columns; the reference's newton_sketch.cpp, single-threaded"}
    else:
        n = cfg["n"]
        d = [a[0].astype(np.float32).astype(np.float64) for a in o.realize(100, n, n, n, 13)]
        x = rng.standard_normal((cfg["batch"], n)).astype(np.float32)
        fn = lambda c: r.chain(d[0], d[1], d[2], 1.0, x[:c], relu=True, threads=threads)  # noqa: E731
        total = cfg["batch"]
        what = "fwht_normalized/diag_matvec chain + ReLU, Gaussian D's"
    # size the sample: a small probe, then up to `budget_s` of work
    probe = max(1, min(total, threads))
    dt = timed(fn, probe)
    count = int(min(total, max(probe, probe * budget_s / max(dt, 1e-6) * 0.5)))
    dt = timed(fn, count)
    return count / dt, {"kind": "reference", "cores": threads, "cpu_model": cpu_model(),
                        "sample": f"{count} of {total} vectors of {config}: {what}; oracle/_ref on {threads} threads"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical CPUs)"
    except OSError:
        pass
    return None


def run_reference(args, rank, world):
    if rank != 0:
        return None
    cfg = CONFIGS[args.config]
    vals = []
    info = None
    for i in range(args.warmup + args.steps):
        v, info = cpu_reference(args.config, budget_s=4.0)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.mean(vals)
    per_step = cfg.get("batch", cfg.get("d"))  # vectors in one full step of this workload
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step / value * 1e3,
            "ms_per_step_note": "full-step time at the sampled rate (each step times a bounded sample)",
            "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"], "name": args.config},
            "cpu_baseline": dict(info, value=value, unit=UNIT),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    if args.impl == "reference":  # host-CPU arm: rank 0 only, no GPU work
        rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
        res = run_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    rank, world, local = dist_init()
    res, w = run_ours(args, rank, world, local)
    if rank == 0:
        if world == 1 and not args.no_cpu:
            v, info = cpu_reference(args.config)
            res["cpu_baseline"] = dict(info, value=v, unit=UNIT)
            if args.config in ("c1", "c2", "c3", "c4", "c5"):  # the reference's own contract: one thread
                v1, info1 = cpu_reference(args.config, budget_s=4.0, threads=1)
                res["cpu_baseline"]["value_1thread"] = v1
                res["cpu_baseline"]["sample_1thread"] = info1["sample"]
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
