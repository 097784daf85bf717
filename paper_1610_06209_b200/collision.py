"""Batched LSH drivers on the device — Python mirror of collision_curve /
compare_families (proj/include/spinners/lsh.hpp:38-75, proj/src/lsh.cpp:38-96).

All `trials` hashers of a curve (make_hasher_factory(v, n, m)(mix_seed(seed, t)),
lsh.cpp:56) are the tables of ONE multi-table plan, so every pair vector is
hashed under every trial in one fused launch; a device kernel then counts, per
pair, the trials with hash(x) == hash(y) and accumulates them into the pair's
distance bucket (spn_collision_hits_f32).  Bucketing, counts and probabilities
follow the reference exactly (same double arithmetic, NaN for empty buckets).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
from typing import List, Sequence

import numpy as np

from . import (DimensionError, DomainError, MultiTableHasher, _check, _i64, _sig, _stream_ptr, _torch, _vp,
               check_rows)

_hits = _sig("spn_collision_hits_f32", C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _vp, _vp])


@dataclasses.dataclass
class HashedPair:
    """lsh.hpp:38-44."""
    x: Sequence[float]
    y: Sequence[float]
    distance: float = 0.0


@dataclasses.dataclass
class CollisionCurve:
    """lsh.hpp:46-50."""
    bucket_edges: List[float]
    probabilities: List[float]
    counts: List[int]


@dataclasses.dataclass
class FamilyComparison:
    """lsh.hpp:68-73."""
    curve_a: CollisionCurve
    curve_b: CollisionCurve
    bucket_differences: List[float]
    sup_difference: float


def _pair_arrays(pairs):
    if isinstance(pairs, tuple) and len(pairs) == 3:
        xs, ys, dist = pairs
        return xs, ys, np.asarray(dist, dtype=np.float64).reshape(-1)
    xs = np.array([np.asarray(p.x, dtype=np.float64) for p in pairs])
    ys = np.array([np.asarray(p.y, dtype=np.float64) for p in pairs])
    return xs, ys, np.array([float(p.distance) for p in pairs], dtype=np.float64)


def collision_curve(pairs, factory, trials: int, seed: int, buckets: int = 25, max_distance: float = 2.0,
                    stream=None) -> CollisionCurve:
    """lsh.cpp:38-74.  `pairs`: a sequence of HashedPair, or (X [P, n], Y [P, n], distances [P])
    (host arrays or CUDA tensors); `factory`: a make_hasher_factory(...) callable."""
    torch = _torch()
    if trials < 1:
        raise DimensionError("collision_curve: trials must be >= 1")
    if buckets < 1:
        raise DimensionError("collision_curve: need at least one bucket")
    for attr in ("variant", "n", "m"):
        if not hasattr(factory, attr):
            raise DomainError("collision_curve: factory must come from make_hasher_factory")
    xs, ys, dist = _pair_arrays(pairs)
    P = dist.size
    width = max_distance / float(buckets)
    if P and (not bool(np.all(np.isfinite(dist))) or bool(np.any(dist < 0.0))):
        raise DomainError("collision_curve: distances must be finite and nonnegative")
    # size_t(d / width) clamped to the last bucket (lsh.cpp:46-51), same double arithmetic
    bucket_of = np.minimum((dist / width).astype(np.int64), buckets - 1).astype(np.int32)
    counts = np.bincount(bucket_of, minlength=buckets).astype(np.int64) * trials
    hits = np.zeros(buckets, dtype=np.int64)
    if P > 0:
        dev = factory.device
        X = xs if isinstance(xs, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(xs, dtype=np.float32))
        Y = ys if isinstance(ys, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(ys, dtype=np.float32))
        X = X.to(device=f"cuda:{dev}", dtype=torch.float32)
        Y = Y.to(device=f"cuda:{dev}", dtype=torch.float32)
        if X.dim() != 2 or X.shape != Y.shape or X.shape[0] != P:
            raise DimensionError("collision_curve: pair shapes mismatch")
        if X.shape[1] != factory.n:
            raise DimensionError("CrossPolytopeHasher::hash: dimension mismatch")
        xy = torch.stack((X, Y), dim=1).reshape(2 * P, factory.n).contiguous()
        if bool((check_rows(xy) != 0).any()):  # hash() rejects non-finite / all-zero inputs (lsh.cpp:23-30)
            raise DomainError("CrossPolytopeHasher::hash: non-finite or zero input")
        h = MultiTableHasher(factory.variant, factory.n, factory.m, trials, seed=seed, device=dev)
        b_dev = torch.from_numpy(bucket_of).to(xy.device)
        hits_dev = torch.zeros(buckets, dtype=torch.int64, device=xy.device)
        _check(_hits(h.plan._h, xy.data_ptr(), P, xy.stride(0), factory.n, b_dev.data_ptr(), buckets,
                     hits_dev.data_ptr(), _stream_ptr(stream)))
        hits = hits_dev.cpu().numpy()
    edges = [width * float(b) for b in range(buckets + 1)]
    probs = [float("nan") if counts[b] == 0 else float(hits[b]) / float(counts[b]) for b in range(buckets)]
    return CollisionCurve(edges, probs, [int(c) for c in counts])


def compare_families(pairs, family_a, family_b, trials: int, seed_a: int, seed_b: int, buckets: int = 25,
                     max_distance: float = 2.0, stream=None) -> FamilyComparison:
    """lsh.cpp:76-96."""
    ca = collision_curve(pairs, family_a, trials, seed_a, buckets, max_distance, stream)
    cb = collision_curve(pairs, family_b, trials, seed_b, buckets, max_distance, stream)
    diffs, sup = [], 0.0
    for b in range(buckets):
        pa, pb = ca.probabilities[b], cb.probabilities[b]
        if math.isnan(pa) or math.isnan(pb):
            diffs.append(float("nan"))
        else:
            diffs.append(abs(pa - pb))
            sup = max(sup, diffs[-1])
    return FamilyComparison(ca, cb, diffs, sup)


__all__ = ["HashedPair", "CollisionCurve", "FamilyComparison", "collision_curve", "compare_families"]
