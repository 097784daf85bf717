#!/usr/bin/env python3
"""Benchmark of the structured-spinner hot path on B200 (BASELINE.json metric:
"spinner vectors/sec (and GB/s as % of HBM roofline) at 1/2/4/8 B200 vs host-CPU ref").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config all|c1..c7] [--impl ours|reference]
                  [--scaling strong|weak] [--no-e2e] [--no-cpu] [--no-check]

A step is one pass of the hot path over one batch of a config's synthetic input (BASELINE.json):
  c1  LSH, 1 table: 4096 x 1024 unit vectors -> int32 ids + fp32 y (scale 1)
  c2  Gaussian RFF: 60000 x 784 -> pad 1024, 4 blocks, k = 4096, sigma = 5 -> 60000 x 8192 fp32
  c3  LSH, 8 tables: 2^20 x 16384 unit vectors (64 GiB, generated on device) -> int32 ids [2^20 x 8]
  c4  sketch: A[131072][256] -> sqrt(N/m) P H D3 H D2 H D1 A, m = 2048 random rows
  c5  all-Gaussian diagonals + ReLU: 256 x 2^20 -> 256 x 2^20
The default (--config all) prints ONE line whose headline is c3 — the largest configuration that fits
one GPU and the one the 1/2/4/8-GPU metric is quoted on — with c1, c2, c4 and c5 measured the same
way and nested under "configs".  Each config carries its own roofline, traffic, clocks, e2e (through
the host-buffer C-ABI entry points, copies inside the timed region) and CPU baseline (the reference
compiled from its own sources, oracle/_ref, timed on this box's host cores; rank 0, N = 1).

Multi-GPU (torchrun, one process per GPU): strong scaling by default, as BASELINE config 3 reads
("batch 2^20 ... sharded across 1/2/4/8 GPUs"): every config's batch (c4: its columns) is split with
shard_range, c3 additionally all-gathers the codes (fused into the hash kernel as peer stores, or NCCL).
--scaling weak gives every rank a full batch instead.  value = units of the whole job / max-over-ranks
device time.
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
HEADLINE = "c3"
NESTED = ("c1", "c2", "c4", "c5")

# Workload definitions: the SAME dicts go into both arms' `config` (ours and --impl reference).
CONFIGS = {
    "c1": dict(workload="BASELINE configs[0]: cross-polytope LSH, 1 table, 4096 x n=1024 unit vectors -> int32 ids "
                        "+ fp32 y (scale 1)", n=1024, batch=4096),
    "c2": dict(workload="BASELINE configs[1]: Gaussian RFF, 60000 x 784 uniform (zero-pad 1024), 4 HD3HD2HD1 blocks "
                        "(k=4096), sigma=5 -> 60000 x 8192 fp32", n=1024, n_in=784, batch=60000, k=4096, sigma=5.0),
    "c3": dict(workload="BASELINE configs[2]: cross-polytope LSH, 8 tables, 2^20 x n=16384 unit vectors -> int32 ids "
                        "[2^20 x 8]", n=16384, batch=1 << 20, tables=8),
    "c4": dict(workload="BASELINE configs[3]: sketch sqrt(N/m) P H D3 H D2 H D1 A, A = 131072 x 256 N(0,1), "
                        "m = 2048 random rows -> 2048 x 256", N=1 << 17, d=256, m=2048),
    "c5": dict(workload="BASELINE configs[4]: ReLU(H D3 H D2 H D1 x), N(0,1) diagonals, 256 x n=2^20", n=1 << 20,
               batch=256),
    "c6": dict(workload="SURVEY 8(f) rank 1: one sketched Newton iteration of solve() (fresh HD3 SketchOperator, "
                        "sketched_step, Armijo line search), logistic regression on A = 131072 x 256, m = 2048",
               N=1 << 17, d=256, m=2048),
    "c7": dict(workload="SURVEY 8(f) rank 2: collision_curve of the HD3 family, n=256, m=64, 20000 pairs x 100 "
                        "trials; units = hashed vectors (2 x pairs x trials)", n=256, m=64, pairs=20000, trials=100),
}
# algorithmic HBM bytes per unit (DESIGN.md §3 / SURVEY §8(d)): every input byte read once, every
# output byte written once
BYTES_PER_UNIT = {"c1": 1024 * 4 * 2 + 4, "c2": 784 * 4 + 8192 * 4, "c3": 16384 * 4 + 8 * 4,
                  "c4": (1 << 17) * 4 + 2048 * 4, "c5": (1 << 20) * 8, "c6": (1 << 17) * 4 * 6, "c7": 256 * 4}
# inputs smaller than L2 (126 MB): flush L2 between timed steps (c1's 16 MB, c4's 128 MB A)
FLUSH = {"c1": True, "c4": True}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="all", choices=["all"] + sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    return ap.parse_args()


def config_dict(name, world, scaling):
    """The workload description both arms print (identical dicts -> comparable records)."""
    c = CONFIGS[name]
    d = {"workload": c["workload"], "name": name}
    d.update({k: v for k, v in c.items() if k != "workload"})
    d["parallelism"] = f"dp{world} ({scaling} scaling: " + (
        "each rank a full batch)" if scaling == "weak" else
        ("columns sharded across ranks)" if name == "c4" else "batch sharded across ranks)")) + (
        " + all-gather of the codes" if name == "c3" and world > 1 else "")
    d["l2"] = ("L2 flushed (256 MB write + read-back) between timed steps" if FLUSH.get(name)
               else "inputs + outputs larger than the 126 MB L2")
    return d


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

    def mark(self):
        return len(self.samples)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, since=0):
        smp = self.samples[since:] or self.samples
        if not smp:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in smp if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in smp if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in smp for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(smp)}


# ------------------------------------------------------------------ workloads
class Workload:
    """Device-resident inputs/outputs for one config (this rank's shard) + `step()` (the hot path over
    one batch), `e2e()` (the same through the host-buffer C ABI) and `check()` (a sampled comparison
    of the last step's output with the reference)."""

    def __init__(self, name, rank, world, device, scaling):
        import torch
        import paper_1610_06209_b200 as spn
        from paper_1610_06209_b200.shard import shard_range
        self.spn, self.torch, self.name, self.cfg = spn, torch, name, CONFIGS[name]
        self.rank, self.world, self.device = rank, world, device
        cfg = self.cfg
        dev = torch.cuda.current_device()  # every plan on this rank's GPU (torch.cuda.set_device(LOCAL_RANK))
        strong = scaling == "strong"
        g = torch.Generator(device="cuda")
        g.manual_seed(1234 + (0 if strong else rank))
        V = spn.SpinnerVariant
        self.launches_per_step = 1
        self.pc = self.exchange = None

        def rows_of(total):  # this rank's shard of a batch (strong) or the full batch (weak)
            if not strong or world == 1:
                return 0, total
            return shard_range(total, rank, world)

        def gen(shape, kind):  # shard of a globally seeded tensor: generate the whole and slice
            x = torch.randn(shape, device="cuda", generator=g) if kind == "n" else \
                torch.rand(shape, device="cuda", generator=g)
            return x

        if name == "c1":
            self.r0, self.units = rows_of(cfg["batch"])
            self.sp = spn.StackedSpinner(V.hd3_hd2_hd1, 1024, 1024, 1024, 42, scale=1.0, device=dev)
            x = gen((cfg["batch"], 1024), "n")
            self.x = (x / x.norm(dim=1, keepdim=True))[self.r0:self.r0 + self.units].contiguous()
            self.y = torch.empty_like(self.x)
        elif name == "c2":
            self.r0, self.units = rows_of(cfg["batch"])
            self.sp = spn.StackedSpinner(V.hd3_hd2_hd1, 1024, 1024, cfg["k"], 5, device=dev)
            self.fm = spn.FeatureMap(self.sp, spn.KernelKind.gaussian(cfg["sigma"]))
            self.x = gen((cfg["batch"], cfg["n_in"]), "u")[self.r0:self.r0 + self.units].contiguous()
            self.out = torch.empty((self.units, 2 * cfg["k"]), device="cuda")
        elif name == "c3":
            self.r0, self.units = rows_of(cfg["batch"])
            self.h = spn.MultiTableHasher(V.hd3_hd2_hd1, cfg["n"], cfg["n"], cfg["tables"], seed=3, device=dev)
            self.x = torch.empty((self.units, cfg["n"]), device="cuda")
            # N(0,1) then L2-normalised, generated on device in 2^16-row blocks keyed by the global row
            blk_rows = 1 << 16
            for b0 in range(0, cfg["batch"], blk_rows):
                lo, hi = max(b0, self.r0), min(b0 + blk_rows, self.r0 + self.units)
                if lo >= hi:
                    continue
                gb = torch.Generator(device="cuda")
                gb.manual_seed(1000 + b0 // blk_rows + (0 if strong else 7919 * rank))
                blk = torch.randn((blk_rows, cfg["n"]), device="cuda", generator=gb)[lo - b0:hi - b0]
                self.x[lo - self.r0:hi - self.r0] = blk / blk.norm(dim=1, keepdim=True)
                del blk
            self.ids = None
            if world > 1:
                total = cfg["batch"] if strong else world * cfg["batch"]
                self.row0 = self.r0 if strong else rank * cfg["batch"]
                try:  # the all-gather fused into the hash kernel: peer stores over NVLink (CUDA IPC)
                    from paper_1610_06209_b200.shard import PeerCodes
                    self.pc = PeerCodes(total, cfg["tables"], world, rank, device)
                    self.exchange = "fused peer stores in the hash kernel (CUDA IPC / NVLink), one barrier"
                except Exception as exc:  # no peer access: NCCL all_gather_into_tensor
                    self.exchange = f"nccl all_gather (peer mapping unavailable: {type(exc).__name__}: {exc})"
                    self.gather_total = total
        elif name == "c4":
            self.c0, self.units = rows_of(cfg["d"])  # columns
            self.sk = spn.SketchOperator(V.hd3_hd2_hd1, cfg["N"], cfg["m"], 11, mode="random", p_seed=77, device=dev)
            a = gen((cfg["N"], cfg["d"]), "n")
            self.x = a[:, self.c0:self.c0 + self.units].contiguous()
            del a
            self.out = torch.empty((cfg["m"], self.units), device="cuda")
            if self.units % 32 == 0 and os.environ.get("SPN_FLOW", "1") != "0":
                self.launches_per_step = 1  # the dataflow sketch kernel (sketch_flow.cuh): the whole step
            else:  # grouped pass launches: 4 per column group
                groups = math.ceil(self.units / max(32, ((32 << 20) // (cfg["N"] * 4)) // 32 * 32))
                self.launches_per_step = 4 * groups
        elif name == "c5":
            self.r0, self.units = rows_of(cfg["batch"])
            self.sp = spn.StackedSpinner(V.gauss3, cfg["n"], cfg["n"], cfg["n"], 13, scale=1.0, device=dev)
            self.x = torch.empty((self.units, cfg["n"]), device="cuda")
            for r in range(self.units):  # row r of the global batch from its own seed
                gr = torch.Generator(device="cuda")
                gr.manual_seed(50000 + self.r0 + r + (0 if strong else 7919 * rank))
                self.x[r] = torch.randn(cfg["n"], device="cuda", generator=gr)
            self.y = torch.empty_like(self.x)
            G = max(1, min(self.units, (24 << 20) // (cfg["n"] * 4)))
            self.launches_per_step = 4 * math.ceil(self.units / G)
        elif name == "c6":
            from paper_1610_06209_b200 import newton
            self.newton = newton
            f = torch.randn((cfg["N"], cfg["d"]), device="cuda", generator=g)
            y = torch.where(torch.rand(cfg["N"], device="cuda", generator=g) < 0.5, -1.0, 1.0)
            self.prob = spn.LogisticProblem(f, y, device=dev)
            self.prob.workspace(cfg["m"])
            self.xk = torch.full((cfg["d"],), 0.01, dtype=torch.float64, device="cuda")
            self.units = cfg["d"]  # columns sketched per iteration
            self.t = 0
            import concurrent.futures
            self.pool = concurrent.futures.ThreadPoolExecutor(1)  # next sketch realised during this step
            self.mk = lambda it: spn.SketchOperator(V.hd3_hd2_hd1, cfg["N"], cfg["m"], spn.mix_seed(3, it), device=dev)  # noqa
            self.pending = self.pool.submit(self.mk, 0)
            self.launches_per_step = 16  # pass over A + 4 sketch passes + line search (a lower bound)
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
            self.fac = spn.make_hasher_factory(V.hd3_hd2_hd1, n, cfg["m"], device=dev)
            self.units = 2 * P * cfg["trials"]
            self.t = 0
        torch.cuda.synchronize()

    # ---- the hot path over one batch
    def step(self, stream):
        n = self.name
        if n == "c1":
            return self.sp.plan.hash(self.x, y_out=self.y, stream=stream)
        if n == "c2":
            return self.spn.embed(self.fm, self.x, out=self.out, stream=stream)
        if n == "c3":
            if self.pc is not None:
                self.ids = self.pc.hash(self.h, self.x, self.row0, stream=stream)
            else:
                self.ids = self.h.plan.hash(self.x, stream=stream)
                if self.world > 1:
                    from paper_1610_06209_b200.shard import gather_codes
                    self.ids = gather_codes(self.ids, self.world, self.gather_total)
            return self.ids
        if n == "c4":
            return self.sk.apply(self.x, out=self.out, stream=stream)
        if n == "c5":
            return self.sp.apply(self.x, relu=True, out=self.y, stream=stream)
        if n == "c7":  # lsh.cpp:38-74, fresh trial seeds every step
            self.t += 1
            return self.spn.collision_curve((self.cx, self.cy, self.cd), self.fac, self.cfg["trials"], 90 + self.t,
                                            stream=stream)
        # c6: newton_sketch.cpp:155-170, one iteration
        nt = self.newton
        sk = self.pending.result()
        self.t += 1
        self.pending = self.pool.submit(self.mk, self.t)
        stp, gr, f = nt._step_dev(self.prob, self.xk, sk, stream)
        slope = float(self.torch.dot(gr, stp).item())
        s, _ = nt._backtrack(self.prob, self.xk, stp, float(f.item()), slope, stream)
        self.xk = self.xk + s * stp
        return self.xk

    # ---- end to end through the public host-buffer API
    def e2e_prepare(self):
        """Pinned host copies of this rank's inputs and pinned outputs (outside any timing)."""
        import numpy as np
        torch = self.torch

        def pinned(shape, dtype=torch.float32):
            return torch.empty(shape, dtype=dtype, pin_memory=True).numpy()

        t0 = time.perf_counter()
        xt = torch.empty(tuple(self.x.shape), dtype=torch.float32, pin_memory=True)
        t1 = time.perf_counter()
        xt.copy_(self.x)  # straight into the pinned buffer
        xh = xt.numpy()
        self.e2e_note = {"pinned_alloc_s": round(t1 - t0, 2), "input_d2h_s": round(time.perf_counter() - t1, 2)}
        n = self.name
        if n == "c1":
            self.e2e_out = (pinned((self.units, 1)), pinned((self.units, 1024)))
            ids, y = self.e2e_out
            self.e2e_run = lambda: self.sp.plan.hash(xh, y_out=y)
            self.e2e_api = "spn_hash_project_f32_host (ids + y, pinned host buffers)"
            self.e2e_bytes = (xh.nbytes, self.units * 4 + y.nbytes)
        elif n == "c2":
            out = pinned((self.units, 2 * self.cfg["k"]))
            self.e2e_run = lambda: self.spn.embed(self.fm, xh, out=out)
            self.e2e_api = "spn_embed_f32_host (pinned host buffers)"
            self.e2e_bytes = (xh.nbytes, out.nbytes)
        elif n == "c3":
            self.e2e_run = lambda: self.h.plan.hash(xh)
            self.e2e_api = "spn_hash_f32_host (pinned 64 GiB host input, ids back to the host)"
            self.e2e_bytes = (xh.nbytes, self.units * self.cfg["tables"] * 4)
        elif n == "c4":
            out = pinned((self.cfg["m"], self.units))
            self.e2e_run = lambda: self.sk.apply(xh, out=out)
            self.e2e_api = "spn_sketch_f32_host (SketchOperator::apply value semantics, pinned host buffers)"
            self.e2e_bytes = (xh.nbytes, out.nbytes)
        elif n == "c5":
            out = pinned((self.units, self.cfg["n"]))
            self.e2e_run = lambda: self.sp.apply(xh, relu=True, out=out)
            self.e2e_api = "spn_apply_f32_host (pinned host buffers)"
            self.e2e_bytes = (xh.nbytes, out.nbytes)
        del np

    # ---- sampled check of the last step's output against the reference (test infrastructure)
    def check(self):
        import numpy as np
        from oracle.oracle import GAUSS3, HD3, Reference  # noqa: F401  (checker only, after timing)
        ref = Reference()
        thr = os.cpu_count() or 1
        rng = np.random.default_rng(99)
        torch = self.torch
        res = {"checked_against": "oracle/_ref (the reference compiled from its own sources)"}

        def rel(got, want):
            return float((np.linalg.norm(got - want, axis=-1) / np.linalg.norm(want, axis=-1)).max())

        def ids_gaps(y, k):
            a = np.abs(y)
            idx = np.argmax(a, axis=1)
            val = y[np.arange(y.shape[0]), idx]
            top2 = np.partition(a, -2, axis=1)[:, -2:]
            return (idx + np.where(val < 0.0, k, 0)).astype(np.int32), (top2[:, 1] - top2[:, 0]) / top2[:, 1]

        n = self.name
        if n in ("c1", "c3"):
            cfg = self.cfg
            nn = cfg["n"]
            rows = np.sort(rng.choice(self.units, min(self.units, 1024 if n == "c3" else 512), replace=False))
            xs = self.x[torch.from_numpy(rows).cuda()].cpu().numpy()
            if n == "c1":
                got = self.ids_last.cpu().numpy()[rows] if hasattr(self, "ids_last") else None
                seeds = [42]
                y = self.y[torch.from_numpy(rows).cuda()].cpu().numpy()
                y_ref = ref.apply(HD3, nn, nn, nn, 42, 1.0, xs, threads=thr)
                res["y_max_rel_l2"] = rel(y, y_ref)
                yr = [y_ref]
            else:
                glob = self.ids.cpu().numpy()
                got = glob[(self.row0 if self.pc is not None else (self.r0 if self.world > 1 else 0)) + rows]
                seeds = self.h.table_seeds
                yr = [ref.apply(HD3, nn, nn, nn, s, 0.0, xs, threads=thr) for s in seeds]
            want, gaps = zip(*[ids_gaps(y, nn) for y in yr])
            want, gaps = np.stack(want, 1), np.stack(gaps, 1)
            if got is not None:
                diff = got != want
                near = gaps < 1e-5
                res.update(rows=int(rows.size), ids=int(want.size), id_mismatches=int(diff.sum()),
                           near_ties=int(near.sum()), mismatches_outside_near_ties=int((diff & ~near).sum()))
        elif n == "c2":
            rows = np.sort(rng.choice(self.units, min(self.units, 2048), replace=False))
            rt = torch.from_numpy(rows).cuda()
            want = ref.embed(HD3, 1024, self.cfg["k"], 5, 0, self.cfg["sigma"], self.x[rt].cpu().numpy(),
                             n_in=self.cfg["n_in"], threads=thr)
            res.update(rows=int(rows.size), max_rel_l2=rel(self.out[rt].cpu().numpy(), want))
        elif n == "c4":
            a = self.x.cpu().numpy()
            want = ref.sketch(HD3, a, self.cfg["m"], 11, row_list=self.sk.row_list, threads=thr)
            res.update(columns=int(self.units), max_rel_l2=rel(self.out.cpu().numpy().T, want.T))
        elif n == "c5":
            rows = np.sort(rng.choice(self.units, min(self.units, 32), replace=False))
            d = [v[0].astype(np.float32).astype(np.float64) for v in self.sp.diagonals()]
            rt = torch.from_numpy(rows).cuda()
            want = ref.chain(d[0], d[1], d[2], 1.0, self.x[rt].cpu().numpy(), relu=True, threads=thr)
            res.update(rows=int(rows.size), max_rel_l2=rel(self.y[rt].cpu().numpy(), want))
        res["pass"] = bool(res.get("max_rel_l2", res.get("y_max_rel_l2", 0.0)) <= 1e-5 and
                           res.get("mismatches_outside_near_ties", 0) == 0)
        return res


# Issue floors from the ncu instruction mix (tools/sass_mix.py on the committed ncu reports):
# warp-issue cycles per unit with FADD2 counted twice, at the clock the floor was computed for.
ISSUE_FLOOR = {
    "c2": {"ms": 0.307, "mhz": 1965.0, "model": "5.95 K issue cycles per sample (1536 FADD2 x2, 768 FADD, 513 LOP3 + "
           "48 R2P sign flips, 96 STS + 75 LDS + 64 LDSM + 32 STSM, 416 FMUL, 256 MUFU, ~550 address/loop) over 60000 "
           "samples on 592 SMSPs (profiles/r02_c2_sass_mix.txt)"},
    "c3": {"ms": 192.8, "mhz": 1965.0, "model": "26.7 K warp-issue cycles per (vector, table) (9216 FADD2 x2, 3072 "
           "FADD, 1919 LOP3 + 192 R2P sign flips, 389 STS + 384 LDSM transposes, 576 LDG, 202 IMAD, argmax) over "
           "2^20 x 8 items on 592 SMSPs (profiles/r02_c3_sass_mix.txt)"},
    "c1": {"ms": 0.00527, "mhz": 1965.0, "model": "1.50 K issue cycles per vector (384 FADD2 x2, 192 FADD, 125 LOP3 + 12 "
           "R2P sign flips, 64 STS/LDS/LDSM/STSM, 8 LDG.128 + 8 STG.128 in permuted coordinates, argmax) over 4096 "
           "vectors on 592 SMSPs: one wave, bound by each warp's own chain latency (profiles/r02_c1_sass_mix.txt)"},
}

# L2-resident read-modify-write bandwidth measured on this pool's B200 (tools/microbench/mb.cu, in-place
# float4 r+w over a 32 MB buffer, 148 x 4 CTAs): 12.3-12.9 TB/s at 16-32 MB, 9.3 TB/s at 64 MB.
L2_RMW_GBS = 12877.8


def secondary_rooflines(name, cfg, units, step_ms, clocks):
    """The roofs that bind the configs whose HBM fraction is low by construction: the multi-pass configs
    (c4, c5) against the L2 read-modify-write rate (4 passes, each reading and writing the working set
    through L2), the issue-bound ones (c2, c3) against their instruction-count floor."""
    out = {}
    if name in ("c4", "c5"):
        if name == "c5":  # + D1, D2, D3 (fp32, n each) read by their pass for every vector (ncu: the three
            # passes with a diagonal move 2x the group's bytes from L2, profiles/r02_c5_ncu_full.json)
            l2_bytes = (4 * 2 + 3) * units * cfg["n"] * 4
            model = "4 passes x (read + write) of the working set + 3 diagonal reads per vector through L2"
        else:  # passes 1-3 read + write A's columns, pass 4 reads them and writes the m gathered rows
            l2_bytes = 7 * cfg["N"] * units * 4 + cfg["m"] * units * 4
            model = "4 passes x (read + write) of the working set through L2"
        ach = l2_bytes / (step_ms * 1e-3) / 1e9
        out["roofline_l2"] = {"bound": "l2", "achieved": ach, "peak": L2_RMW_GBS, "unit": "GB/s",
                              "frac": ach / L2_RMW_GBS,
                              "traffic_model": model,
                              "l2_bytes_per_step": l2_bytes,
                              "peak_source": "tools/microbench/mb.cu L2 rmw, 32 MB, this pool's B200"}
    if name == "c4":
        # shared-memory roof of the dataflow sketch kernel (sketch_flow.cuh): every 64 KB task moves its
        # tile through shared memory 6 times (TMA in, tile -> registers, one transpose = write + read,
        # registers -> tile, TMA store out) plus one more transpose for the two passes that apply two H's;
        # the last pass stores only the sampled rows (5 moves).  27 tile moves per element over the four
        # passes, against 128 B / clk / SM (tools/microbench/mb.cu measures 124).
        mhz = clocks.get("sm_mhz") or 1965.0
        smem_bytes = 27 * cfg["N"] * units * 4
        peak = 124.0 * 148 * mhz * 1e6 / 1e9
        ach = smem_bytes / (step_ms * 1e-3) / 1e9
        out["roofline_smem"] = {"bound": "shared memory", "achieved": ach, "peak": peak, "unit": "GB/s",
                                "frac": ach / peak, "smem_bytes_per_step": smem_bytes, "sm_mhz": mhz,
                                "model": "27 tile moves through shared memory per element over the 4 passes "
                                         "(6 + 8 + 8 + 5) at the measured 124 B/clk/SM; ncu l1tex throughput of "
                                         "the same kernel: profiles/r02_c4_ncu_full.json"}
    if name in ISSUE_FLOOR:
        f = ISSUE_FLOOR[name]
        mhz = clocks.get("sm_mhz") or f["mhz"]
        scale = units / CONFIGS[name]["batch"]
        floor = f["ms"] * f["mhz"] / mhz * scale
        out["roofline_issue"] = {"bound": "issue", "floor_ms": floor, "measured_ms": step_ms,
                                 "frac": floor / step_ms, "sm_mhz": mhz, "model": f["model"]}
    return out


# FP32 butterfly adds per unit (3 H's of n log2 n adds each per spinner block; c2 four blocks per sample,
# c3 eight tables per vector): the ALU roof of SURVEY §8(d), at 128 FP32 adds / clk / SM
FP32_ADDS_PER_UNIT = {"c1": 3 * 10 * 1024, "c2": 4 * 3 * 10 * 1024, "c3": 8 * 3 * 14 * 16384,
                      "c4": 3 * 17 * (1 << 17), "c5": 3 * 20 * (1 << 20)}


def fp32_roofline(name, units, step_ms, clocks):
    if name not in FP32_ADDS_PER_UNIT:
        return {}
    mhz = clocks.get("sm_mhz") or 1965.0
    adds = FP32_ADDS_PER_UNIT[name] * units
    floor = adds / (148 * 128 * mhz * 1e6) * 1e3
    out = {"roofline_fp32": {"bound": "fp32 add pipe", "adds_per_step": adds, "floor_ms": floor,
                             "measured_ms": step_ms, "frac": floor / step_ms, "sm_mhz": mhz,
                             "model": "FP32 butterfly adds (3 n log2 n per spinner block) at 128 adds/clk/SM"}}
    try:  # the pipe utilisation ncu measured for this config's kernel (committed capture)
        with open(os.path.join(ROOT, "profiles", f"r02_{name}_ncu_full.json")) as f:
            m = json.load(f)["launches"][0]["metrics"]
        out["roofline_fp32"]["ncu_fma_pipe_active_pct"] = float(
            m["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"][0])
        out["roofline_fp32"]["ncu_issue_active_pct"] = float(
            m["smsp__issue_active.avg.pct_of_peak_sustained_active"][0])
        out["roofline_fp32"]["ncu_source"] = f"profiles/r02_{name}_ncu_full.json"
    except Exception:
        pass
    return out


def traffic_from_profiles(config):
    """DRAM bytes (read + write) per step from the committed ncu captures (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            v = json.load(f).get(config)
        return v if isinstance(v, (int, float)) else None
    except Exception:
        return None


def timed_steps(w, steps, warmup, world, clk):
    """W untimed warm-up steps, then exactly `steps` steps each bracketed by CUDA events on the
    launching stream; barrier + synchronize on both sides.  Returns per-step ms (this rank)."""
    torch = w.torch
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if FLUSH.get(w.name) else None
    sink = torch.zeros((), dtype=torch.int64, device="cuda")
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    t_end = time.time() + 3.0
    i = 0
    # warm-up; single rank: continue (untimed) until nvidia-smi has sampled the GPU under this load
    while i < max(3, warmup) or (world == 1 and clk.mark() - w.clk0 < 3 and time.time() < t_end):
        w.step(stream)
        i += 1
        if i >= max(3, warmup):
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    w.clk0 = clk.mark()
    for k in range(steps):
        if flush is not None:
            # evict L2 outside the timed region: write 256 MB (> 126 MB L2), then read it back so the
            # lines left in L2 are clean (the timed kernel must not pay for the flush's write-backs)
            flush.fill_(k & 0xFF)
            sink += flush.view(torch.int64).sum()
        torch.cuda._sleep(200_000)  # keep the device busy past the start event (no host launch gap timed)
        evs[k][0].record(stream)
        out = w.step(stream)
        evs[k][1].record(stream)
        if w.name == "c1":
            w.ids_last = out
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def c1_steady_state(w, steps, peak):
    """Config 1 back to back (SURVEY §7 hard part 7): the one-wave hash + y launch is latency-bound
    when timed alone, so also report the throughput of many consecutive steps captured in one CUDA
    graph, over 8 distinct input/output batch buffers (8 x 32 MB > 126 MB L2: every step streams
    its 16 MB of x from HBM and its 16 MB of y back).  Not the headline number for c1 (that is the
    cold single launch above); this is the sustained rate of a stream of config-1 batches."""
    torch = w.torch
    nb, reps = 8, 4
    xs = [w.x.clone() for _ in range(nb)]
    ys = [torch.empty_like(w.y) for _ in range(nb)]
    ids = [None] * nb
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm (plan layouts, occupancy caches) before capture
        for b in range(nb):
            ids[b] = w.sp.plan.hash(xs[b], y_out=ys[b], stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            for b in range(nb):
                w.sp.plan.hash(xs[b], y_out=ys[b], stream=s)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rounds = max(3, steps // 4)
    e0.record()
    for _ in range(rounds):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = rounds * reps * nb
    per_ms = ms / launches
    ach = BYTES_PER_UNIT["c1"] * w.units / (per_ms / 1e3) / 1e9
    # the graph's outputs equal a plain launch's (same kernel, same inputs)
    ok = bool(torch.equal(ys[0], ys[1]) and torch.equal(ys[0], w.y))
    return {"value": w.units / (per_ms / 1e3), "unit": UNIT, "ms_per_step": per_ms, "launches": launches,
            "hbm": {"achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak},
            "how": f"{reps} x {nb} distinct 32 MB batches per CUDA graph, {rounds} replays, CUDA events",
            "outputs_match_single_launch": ok}


def e2e_measure(w, steps, world):
    """The metric through the host-buffer C ABI: pinned host input in, host output back, both copies
    inside the timed region, every step."""
    w.e2e_prepare()
    w.e2e_run()  # warm (allocates the pipeline's staging buffers)
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(steps):
        w.e2e_run()
    dt = max_over_ranks(time.perf_counter() - t0, world)
    return {"value": w.units * world * steps / dt, "unit": UNIT, "h2d_bytes_per_step": w.e2e_bytes[0] * world,
            "d2h_bytes_per_step": w.e2e_bytes[1] * world, "steps": steps, "api": w.e2e_api, **w.e2e_note}


def measure_config(name, args, rank, world, local, clk):
    """One config's line: timed device steps, rooflines, clocks, e2e and (rank 0) the sampled check."""
    torch_mod = __import__("torch")
    w = Workload(name, rank, world, local, args.scaling)
    w.clk0 = clk.mark()
    step_ms = timed_steps(w, args.steps, args.warmup, world, clk)
    clocks = clk.summary(w.clk0)
    total_ms = max_over_ranks(sum(step_ms), world)
    ms_per_step = total_ms / args.steps
    job_units = w.units * world  # strong: the shards add up to the batch; weak: world full batches
    value = job_units * args.steps / (total_ms / 1e3)
    peak, peak_src = measured_peaks()
    mean_ms = statistics.mean(step_ms)
    alg_bytes = BYTES_PER_UNIT[name] * w.units
    achieved = alg_bytes / (mean_ms / 1e3) / 1e9
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "ms_per_step": ms_per_step,
        "units_per_step": job_units,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic_from_profiles(name) if world == 1 and args.scaling == "strong" else None,
                     "peak_source": peak_src, "algorithmic_bytes_per_step": alg_bytes,
                     "algorithmic_bytes_per_unit": BYTES_PER_UNIT[name], "mean_step_ms": mean_ms,
                     "launches_per_step": w.launches_per_step},
        "clocks": clocks,
        "gpu_launches": w.launches_per_step * args.steps,
        "l2_policy": "L2 flushed (256 MB write + read-back) between timed steps" if FLUSH.get(name)
        else "inputs + outputs > 126 MB L2",
    }
    if w.exchange:
        res["exchange"] = w.exchange
    res.update(secondary_rooflines(name, CONFIGS[name], w.units, mean_ms, clocks))
    res.update(fp32_roofline(name, w.units, mean_ms, clocks))
    if name == "c1":
        res["steady_state"] = c1_steady_state(w, args.steps, peak)
    if not args.no_e2e and name in ("c1", "c2", "c3", "c4", "c5"):
        res["e2e"] = e2e_measure(w, 3 if name in ("c2", "c3", "c5") else max(3, min(args.steps, 10)), world)
    if rank == 0 and world == 1 and not args.no_check and name in ("c1", "c2", "c3", "c4", "c5"):
        res["check"] = w.check()
    del w
    torch_mod.cuda.empty_cache()
    return res


# ---------------------------------------------------------------- CPU reference
def cpu_reference(config, budget_s=10.0, threads=None):
    """The reference's own CPU code (oracle/_ref: proj/src compiled unmodified) on the host cores,
    over a bounded sample of the same workload.  Returns (vectors/s, info)."""
    import numpy as np
    from oracle.oracle import Oracle, Reference
    HD3 = 0
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
        x = rng.standard_normal((2048, cfg["n"])).astype(np.float32)
        seeds = [o.mix_seed(3, t) for t in range(cfg["tables"])]
        fn = lambda c: r.hash(HD3, cfg["n"], cfg["n"], seeds, x[:c], threads=threads)  # noqa: E731
        total = cfg["batch"]
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
    else:  # c5
        n = cfg["n"]
        d = [v[0].astype(np.float32).astype(np.float64) for v in o.realize(100, n, n, n, 13)]
        x = rng.standard_normal((min(cfg["batch"], 64), n)).astype(np.float32)
        fn = lambda c: r.chain(d[0], d[1], d[2], 1.0, x[:c], relu=True, threads=threads)  # noqa: E731
        total = cfg["batch"]
        what = "fwht_normalized/diag_matvec chain + ReLU, Gaussian D's"
    avail = a.shape[1] if config == "c4" else x.shape[0]
    if avail < total:  # fewer distinct rows than the batch: process them cyclically
        rows, base = avail, fn
        fn = lambda c: [base(min(rows, c - i)) for i in range(0, c, rows)]  # noqa: E731
    # size the sample: a probe of one row per thread, then up to `budget_s` of work
    probe = max(1, min(total, threads))
    dt = timed(fn, probe)
    count = int(min(total, max(probe, probe * budget_s / max(dt, 1e-6) * 0.8)))
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


def cpu_baseline(name, budget_s):
    v, info = cpu_reference(name, budget_s=budget_s)
    out = dict(info, value=v, unit=UNIT)
    if name in ("c1", "c2", "c3", "c4", "c5"):  # the reference's own contract: one thread
        v1, info1 = cpu_reference(name, budget_s=min(4.0, budget_s), threads=1)
        out["value_1thread"] = v1
        out["sample_1thread"] = info1["sample"]
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation (oracle/_ref) on all host cores, same
    config dict / metric / unit as our arm; each step a bounded sample.  Rank 0 only."""
    if rank != 0:
        return None
    names = [HEADLINE] + list(NESTED) if args.config == "all" else [args.config]
    lines = {}
    for name in names:
        vals, info = [], None
        head = name == names[0]
        reps = (args.warmup + args.steps) if head else 2
        for i in range(reps):
            v, info = cpu_reference(name, budget_s=1.5 if head else 3.0)
            if i >= (args.warmup if head else 1):
                vals.append(v)
        value = statistics.mean(vals)
        units = CONFIGS[name].get("batch", CONFIGS[name].get("d"))
        lines[name] = {"metric": METRIC, "value": value, "unit": UNIT, "ms_per_step": units / value * 1e3,
                       "ms_per_step_note": "full-step time at the sampled rate (each step times a bounded sample)",
                       "config": config_dict(name, world, args.scaling),
                       "cpu_baseline": dict(info, value=value, unit=UNIT),
                       "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    head = lines.pop(names[0])
    res = {"impl": "reference", **head, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded, BASELINE config shapes and distributions)"}
    if lines:
        res["configs"] = lines
    return res


def main():
    args = parse()
    if args.impl == "reference":  # host-CPU arm: rank 0 only, no GPU work
        rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
        res = run_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    rank, world, local = dist_init()
    import torch
    names = [HEADLINE] + list(NESTED) if args.config == "all" else [args.config]
    lines = {}
    with ClockSampler(local) as clk:
        for name in names:
            lines[name] = measure_config(name, args, rank, world, local, clk)
            if rank == 0:
                lines[name]["config"] = config_dict(name, world, args.scaling)
                print(f"[bench] {name}: {lines[name]['value']:.4g} {UNIT}, {lines[name]['ms_per_step']:.4g} ms/step",
                      file=sys.stderr, flush=True)
    if rank == 0:
        if world == 1 and not args.no_cpu:
            for name in names:
                lines[name]["cpu_baseline"] = cpu_baseline(name, 10.0 if name == names[0] else 6.0)
        head = lines.pop(names[0])
        res = {"metric": METRIC, "value": head.pop("value"), "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": max(3, args.warmup), "ms_per_step": head.pop("ms_per_step"), "higher_is_better": True,
               "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
               "data": "synthetic (seeded, BASELINE config shapes and distributions)",
               "config": head.pop("config"), **head}
        if lines:
            res["configs"] = lines
        print(json.dumps(res), flush=True)
    if world > 1:
        import gc
        import torch.distributed as dist
        gc.collect()
        torch.cuda.ipc_collect()  # release the peer tables mapped from the other ranks (PeerCodes)
        barrier(world)  # ... on every rank before any producer exits
        dist.destroy_process_group()
    del torch


if __name__ == "__main__":
    main()
