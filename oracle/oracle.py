"""TEST INFRASTRUCTURE ONLY — ctypes front end for the CPU oracles.

* ``Oracle``   : the plain-C fp64 restatement (oracle/spinner_oracle.c).
* ``Reference``: the reference's own sources compiled into oracle/_ref
  (oracle/ref_api.cpp binds proj/src/{transforms,spinner,lsh,kernels,newton_sketch}.cpp).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
``--impl reference`` legs import this module, and only as the checker or the
timed CPU baseline.  The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspinners_ref.so")

_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
i64, u64, dbl, cint = C.c_int64, C.c_uint64, C.c_double, C.c_int

HD3, HDG, GAUSS3 = 0, 1, 100


def build(ref: bool = True) -> None:
    """Compile the C restatement (and the reference, when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _load(path):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle` (and `make -C oracle ref`)")
    return C.CDLL(path)


def _f32rows(x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim == 1:
        x = x[None, :]
    return x


class Oracle:
    """fp64 restatement of the reference hot path (spinner_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        L = self.lib = _load(path)
        L.orc_mix_seed.restype = u64
        L.orc_mix_seed.argtypes = [u64, u64]
        L.orc_realize_stacked.restype = i64
        L.orc_realize_stacked.argtypes = [cint, i64, i64, i64, u64, _f64p, _f64p, _f64p]
        L.orc_fwht_normalized.argtypes = [_f64p, i64]
        L.orc_signed_argmax.argtypes = [_f64p, i64, C.POINTER(i64), C.POINTER(cint)]
        L.orc_batch_apply.argtypes = [i64, i64, i64, dbl, _f64p, _f64p, _f64p, _f32p, i64, i64, i64, cint, _f64p]
        L.orc_batch_hash.argtypes = [i64, i64, i64, i64, dbl, _f64p, _f64p, _f64p, _f32p, i64, i64, i64,
                                     _i32p, _f64p]
        L.orc_batch_embed.argtypes = [i64, i64, i64, dbl, _f64p, _f64p, _f64p, cint, dbl, _f32p, i64, i64,
                                      i64, _f64p]
        L.orc_sketch.argtypes = [i64, dbl, dbl, _f64p, _f64p, _f64p, _f32p, i64, i64, i64, C.c_void_p, i64,
                                 _f64p]
        L.orc_sample_rows.argtypes = [i64, i64, u64, _i64p]
        L.orc_rng_fill.argtypes = [u64, cint, i64, _f64p]
        L.orc_realize_block.argtypes = [cint, i64, u64, _f64p, _f64p, _f64p]
        L.orc_block_apply.argtypes = [i64, i64, dbl, _f64p, _f64p, _f64p, _f64p, _f64p]
        L.orc_rng_init.argtypes = [C.c_void_p, u64]
        L.orc_rng_next.restype = u64
        L.orc_rng_next.argtypes = [C.c_void_p]
        for f in ("orc_rng_uniform01", "orc_rng_gaussian", "orc_rng_rademacher"):
            getattr(L, f).restype = dbl
            getattr(L, f).argtypes = [C.c_void_p]

    def mix_seed(self, base: int, stream: int) -> int:
        return int(self.lib.orc_mix_seed(base, stream))

    def rng_fill(self, seed: int, kind: str, count: int) -> np.ndarray:
        out = np.zeros(count)
        self.lib.orc_rng_fill(seed, {"uniform01": 1, "gaussian": 2, "rademacher": 3}[kind], count, out)
        return out

    # ---- seeded synthetic inputs (shapes/distributions of BASELINE.json configs)
    def gaussian_rows(self, seed: int, batch: int, n: int, unit: bool = False) -> np.ndarray:
        """Rows of iid N(0,1) from Rng(seed) (row-major), optionally L2-normalised in
        fp64 before the fp32 rounding (configs 1, 3)."""
        x = self.rng_fill(seed, "gaussian", batch * n).reshape(batch, n)
        if unit:
            x /= np.linalg.norm(x, axis=1, keepdims=True)
        return x.astype(np.float32)

    def uniform_rows(self, seed: int, batch: int, n: int) -> np.ndarray:
        """Rows of Rng::uniform01 (0,1] (config 2's [0,1] pixels)."""
        return self.rng_fill(seed, "uniform01", batch * n).reshape(batch, n).astype(np.float32)

    def rng_stream(self, seed: int, count: int, kind: str):
        st = C.create_string_buffer(312 * 8 + 64)
        self.lib.orc_rng_init(st, seed)
        f = {"u64": self.lib.orc_rng_next, "uniform01": self.lib.orc_rng_uniform01,
             "gaussian": self.lib.orc_rng_gaussian, "rademacher": self.lib.orc_rng_rademacher}[kind]
        vals = [f(st) for _ in range(count)]
        return np.array(vals, dtype=np.uint64 if kind == "u64" else np.float64)

    def realize(self, variant: int, n: int, m: int, k: int, seed: int):
        blocks = -(-k // m)
        d1, d2, d3 = (np.zeros(blocks * n) for _ in range(3))
        self.lib.orc_realize_stacked(variant, n, m, k, seed, d1, d2, d3)
        return d1.reshape(blocks, n), d2.reshape(blocks, n), d3.reshape(blocks, n)

    def realize_block(self, variant: int, n: int, spec_seed: int):
        d = [np.zeros(n) for _ in range(3)]
        self.lib.orc_realize_block(variant, n, spec_seed, *d)
        return tuple(d)

    def fwht(self, x):
        y = np.array(x, dtype=np.float64, copy=True)
        self.lib.orc_fwht_normalized(y, y.size)
        return y

    def signed_argmax(self, y):
        y = np.ascontiguousarray(y, dtype=np.float64)
        idx, sg = i64(), cint()
        self.lib.orc_signed_argmax(y, y.size, C.byref(idx), C.byref(sg))
        return int(idx.value), int(sg.value)

    @staticmethod
    def _diag(d):
        return np.ascontiguousarray(d, dtype=np.float64).reshape(-1)

    def apply(self, d1, d2, d3, n, m, k, scale, x, n_in=None, relu=False):
        x = _f32rows(x)
        n_in = x.shape[1] if n_in is None else n_in
        y = np.zeros((x.shape[0], k))
        self.lib.orc_batch_apply(n, m, k, scale, self._diag(d1), self._diag(d2), self._diag(d3), x,
                                 x.shape[0], x.shape[1], n_in, int(relu), y)
        return y

    def hash(self, d1, d2, d3, n, m, k, tables, scale, x, n_in=None):
        x = _f32rows(x)
        n_in = x.shape[1] if n_in is None else n_in
        ids = np.zeros((x.shape[0], tables), dtype=np.int32)
        gaps = np.zeros((x.shape[0], tables))
        self.lib.orc_batch_hash(n, m, k, tables, scale, self._diag(d1), self._diag(d2), self._diag(d3), x,
                                x.shape[0], x.shape[1], n_in, ids, gaps)
        return ids, gaps

    def embed(self, d1, d2, d3, n, m, k, scale, kind, sigma, x, n_in=None):
        x = _f32rows(x)
        n_in = x.shape[1] if n_in is None else n_in
        w = k if kind == 1 else 2 * k
        out = np.zeros((x.shape[0], w))
        self.lib.orc_batch_embed(n, m, k, scale, self._diag(d1), self._diag(d2), self._diag(d3), kind, sigma,
                                 x, x.shape[0], x.shape[1], n_in, out)
        return out

    def sketch(self, d1, d2, d3, n, scale, norm, a, m_out, rows=None):
        a = np.ascontiguousarray(a, dtype=np.float32)
        out = np.zeros((m_out, a.shape[1]))
        rl = None
        if rows is not None:
            rows = np.ascontiguousarray(rows, dtype=np.int64)
            rl = rows.ctypes.data
        self.lib.orc_sketch(n, scale, norm, self._diag(d1), self._diag(d2), self._diag(d3), a, a.shape[0],
                            a.shape[1], a.shape[1], rl, m_out, out)
        return out

    def sample_rows(self, N, m, seed):
        out = np.zeros(m, dtype=np.int64)
        self.lib.orc_sample_rows(N, m, seed, out)
        return out

    # ---- sketched Newton (newton_sketch.cpp)
    def ar1_problem(self, n, d, seed):
        a, y = np.zeros((n, d)), np.zeros(n)
        self.lib.orc_ar1_problem(i64(n), i64(d), u64(seed), a.ctypes.data_as(C.c_void_p),
                                 y.ctypes.data_as(C.c_void_p))
        return a, y

    def _ay(self, a, y):
        return np.ascontiguousarray(a, dtype=np.float64), np.ascontiguousarray(y, dtype=np.float64)

    def logistic(self, a, y, x):
        """(loss, gradient, hessian_sqrt) at x."""
        a, y = self._ay(a, y)
        x = np.ascontiguousarray(x, dtype=np.float64)
        n, d = a.shape
        L = self.lib
        L.orc_logistic_loss.restype = dbl
        vp = lambda v: v.ctypes.data_as(C.c_void_p)  # noqa: E731
        f = L.orc_logistic_loss(vp(a), vp(y), i64(n), i64(d), vp(x))
        g = np.zeros(d)
        L.orc_logistic_gradient(vp(a), vp(y), i64(n), i64(d), vp(x), vp(g))
        h = np.zeros((n, d))
        L.orc_hessian_sqrt(vp(a), i64(n), i64(d), vp(x), vp(h))
        return float(f), g, h

    def sketched_step(self, a, y, x, N=None, m=None, scale=None, norm=None, diags=None):
        """Exact step when diags is None, else first-m of one block (d1, d2, d3) over N."""
        a, y = self._ay(a, y)
        x = np.ascontiguousarray(x, dtype=np.float64)
        n, d = a.shape
        step = np.zeros(d)
        vp = lambda v: v.ctypes.data_as(C.c_void_p) if v is not None else None  # noqa: E731
        if diags is None:
            rc = self.lib.orc_sketched_step(vp(a), vp(y), i64(n), i64(d), vp(x), i64(0), i64(0), dbl(0), dbl(0),
                                            None, None, None, vp(step))
        else:
            d1, d2, d3 = (np.ascontiguousarray(v, dtype=np.float64).reshape(-1) for v in diags)
            rc = self.lib.orc_sketched_step(vp(a), vp(y), i64(n), i64(d), vp(x), i64(N), i64(m), dbl(scale),
                                            dbl(norm), vp(d1), vp(d2), vp(d3), vp(step))
        return int(rc), step


class ReferenceError_(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"reference error {code}: {msg}")
        self.code = code


class Reference:
    """The reference's own code (oracle/_ref/libspinners_ref.so)."""

    def __init__(self, path: str = REF_SO):
        L = self.lib = _load(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_mix_seed.restype = u64
        L.ref_mix_seed.argtypes = [u64, u64]
        L.ref_rng_stream.argtypes = [u64, i64, cint, C.c_void_p, C.c_void_p]
        L.ref_fwht.argtypes = [_f64p, i64]
        L.ref_signed_argmax.argtypes = [_f64p, i64, C.POINTER(i64), C.POINTER(cint)]
        L.ref_realize_stacked.restype = i64
        L.ref_realize_stacked.argtypes = [cint, i64, i64, i64, u64, _f64p, _f64p, _f64p]
        L.ref_batch_apply.argtypes = [cint, i64, i64, i64, u64, dbl, _f32p, i64, i64, i64, cint, _f64p, cint]
        L.ref_batch_hash.argtypes = [cint, i64, i64, i64, _u64p, _f32p, i64, i64, i64, _i32p, cint]
        L.ref_batch_embed.argtypes = [cint, i64, i64, u64, cint, dbl, _f32p, i64, i64, i64, _f64p, cint]
        L.ref_sketch.argtypes = [cint, i64, i64, u64, _f32p, i64, i64, C.c_void_p, _f64p, cint]
        L.ref_batch_chain.argtypes = [i64, _f64p, _f64p, _f64p, dbl, _f32p, i64, i64, cint, _f64p, cint]

    def _check(self, rc):
        if rc != 0:
            raise ReferenceError_(rc, self.lib.ref_last_error().decode())

    def mix_seed(self, base, stream):
        return int(self.lib.ref_mix_seed(base, stream))

    def rng_stream(self, seed, count, kind):
        k = {"u64": 0, "uniform01": 1, "gaussian": 2, "rademacher": 3}[kind]
        if k == 0:
            out = np.zeros(count, dtype=np.uint64)
            self.lib.ref_rng_stream(seed, count, 0, None, out.ctypes.data)
        else:
            out = np.zeros(count)
            self.lib.ref_rng_stream(seed, count, k, out.ctypes.data, None)
        return out

    def fwht(self, x):
        y = np.array(x, dtype=np.float64, copy=True)
        self._check(self.lib.ref_fwht(y, y.size))
        return y

    def signed_argmax(self, y):
        y = np.ascontiguousarray(y, dtype=np.float64)
        idx, sg = i64(), cint()
        self._check(self.lib.ref_signed_argmax(y, y.size, C.byref(idx), C.byref(sg)))
        return int(idx.value), int(sg.value)

    def realize(self, variant, n, m, k, seed):
        blocks = -(-k // m)
        d1, d2, d3 = (np.zeros(blocks * n) for _ in range(3))
        rc = self.lib.ref_realize_stacked(variant, n, m, k, seed, d1, d2, d3)
        if rc < 0:
            self._check(-rc)
        return d1.reshape(blocks, n), d2.reshape(blocks, n), d3.reshape(blocks, n)

    def apply(self, variant, n, m, k, seed, scale, x, n_in=None, relu=False, threads=1):
        x = _f32rows(x)
        n_in = x.shape[1] if n_in is None else n_in
        y = np.zeros((x.shape[0], k))
        self._check(self.lib.ref_batch_apply(variant, n, m, k, seed, scale, x, x.shape[0], x.shape[1], n_in,
                                             int(relu), y, threads))
        return y

    def hash(self, variant, n, m, table_seeds, x, n_in=None, threads=1):
        x = _f32rows(x)
        n_in = x.shape[1] if n_in is None else n_in
        seeds = np.ascontiguousarray(table_seeds, dtype=np.uint64)
        ids = np.zeros((x.shape[0], seeds.size), dtype=np.int32)
        self._check(self.lib.ref_batch_hash(variant, n, m, seeds.size, seeds, x, x.shape[0], x.shape[1], n_in,
                                            ids, threads))
        return ids

    def embed(self, variant, n, dprime, seed, kind, sigma, x, n_in=None, threads=1):
        x = _f32rows(x)
        n_in = x.shape[1] if n_in is None else n_in
        out = np.zeros((x.shape[0], dprime if kind == 1 else 2 * dprime))
        self._check(self.lib.ref_batch_embed(variant, n, dprime, seed, kind, sigma, x, x.shape[0], x.shape[1],
                                             n_in, out, threads))
        return out

    def sketch(self, variant, a, rows, seed, row_list=None, threads=1):
        a = np.ascontiguousarray(a, dtype=np.float32)
        out = np.zeros((rows, a.shape[1]))
        rl = None
        if row_list is not None:
            row_list = np.ascontiguousarray(row_list, dtype=np.int64)
            rl = row_list.ctypes.data
        self._check(self.lib.ref_sketch(variant, a.shape[0], rows, seed, a, a.shape[1], a.shape[1], rl, out,
                                        threads))
        return out

    def block_resampled(self, variant, n, m, spec_seed, mode, tail_seed=0, tail=None, x=None):
        """StructuredSpinner::build(spec) -> resample_last_block (0) / resample_tail (1) /
        with_tail_vector (2), applied to rows of x; returns (y, d1, d2, d3)."""
        x = _f32rows(np.zeros((0, n)) if x is None else x)
        y = np.zeros((x.shape[0], m))
        d = [np.zeros(n) for _ in range(3)]
        tv = None if tail is None else np.ascontiguousarray(tail, dtype=np.float64)
        vp = lambda v: None if v is None else v.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._check(self.lib.ref_block_resampled(cint(variant), i64(n), i64(m), u64(spec_seed), cint(mode),
                                                 u64(tail_seed), vp(tv), vp(x), i64(x.shape[0]), vp(y), vp(d[0]),
                                                 vp(d[1]), vp(d[2])))
        return y, d[0], d[1], d[2]

    def gram_exact(self, points, kind, sigma=1.0):
        p = np.ascontiguousarray(points, dtype=np.float32)
        out = np.zeros((p.shape[0], p.shape[0]))
        self._check(self.lib.ref_gram_exact(p.ctypes.data_as(C.c_void_p), i64(p.shape[0]), i64(p.shape[1]),
                                            cint(kind), dbl(sigma), out.ctypes.data_as(C.c_void_p)))
        return out

    def gram_approx(self, variant, n, dprime, seed, kind, sigma, points):
        p = np.ascontiguousarray(points, dtype=np.float32)
        out = np.zeros((p.shape[0], p.shape[0]))
        self._check(self.lib.ref_gram_approx(cint(variant), i64(n), i64(dprime), u64(seed), cint(kind), dbl(sigma),
                                             p.ctypes.data_as(C.c_void_p), i64(p.shape[0]),
                                             out.ctypes.data_as(C.c_void_p)))
        return out

    def gram_error(self, exact, approx):
        a = np.ascontiguousarray(exact, dtype=np.float64)
        b = np.ascontiguousarray(approx, dtype=np.float64)
        err = C.c_double()
        self._check(self.lib.ref_gram_error(a.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
                                            i64(a.shape[0]), C.byref(err)))
        return err.value

    def collision_curve(self, variant, n, m, xs, ys, dist, trials, seed, buckets=25, max_distance=2.0):
        """lsh.cpp:38-74 (the reference's own collision_curve + make_hasher_factory)."""
        xs = np.ascontiguousarray(xs, dtype=np.float32)
        ys = np.ascontiguousarray(ys, dtype=np.float32)
        dist = np.ascontiguousarray(dist, dtype=np.float64)
        edges, probs = np.zeros(buckets + 1), np.zeros(buckets)
        counts = np.zeros(buckets, dtype=np.uint64)
        vp = lambda v: v.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._check(self.lib.ref_collision_curve(cint(variant), i64(n), i64(m), vp(xs), vp(ys), vp(dist),
                                                 i64(xs.shape[0]), i64(trials), u64(seed), i64(buckets),
                                                 dbl(max_distance), vp(edges), vp(probs), vp(counts)))
        return {"bucket_edges": edges, "probabilities": probs, "counts": counts}

    # ---- sketched Newton: the reference's own newton_sketch.cpp
    def ar1_problem(self, n, d, seed):
        a, y = np.zeros((n, d)), np.zeros(n)
        self._check(self.lib.ref_ar1_problem(i64(n), i64(d), u64(seed), a.ctypes.data_as(C.c_void_p),
                                             y.ctypes.data_as(C.c_void_p)))
        return a, y

    def logistic(self, a, y, x):
        a = np.ascontiguousarray(a, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        n, d = a.shape
        f, g, h = C.c_double(), np.zeros(d), np.zeros((n, d))
        vp = lambda v: v.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._check(self.lib.ref_logistic(vp(a), vp(y), i64(n), i64(d), vp(x), C.byref(f), vp(g), vp(h)))
        return f.value, g, h

    def sketched_step(self, a, y, x, variant=-1, rows=0, seed=0):
        """variant < 0: exact step; else SketchOperator(variant, n, rows, seed) (first-m rows)."""
        a = np.ascontiguousarray(a, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        n, d = a.shape
        step = np.zeros(d)
        vp = lambda v: v.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._check(self.lib.ref_sketched_step(vp(a), vp(y), i64(n), i64(d), vp(x), cint(variant), i64(rows),
                                               u64(seed), vp(step)))
        return step

    def solve(self, a, y, variant=-1, rows=0, max_iters=50, gap_tol=1e-10, line_search=True, seed=0):
        a = np.ascontiguousarray(a, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        n, d = a.shape
        it, fs, cv = i64(), C.c_double(), cint()
        losses, gaps, xf = np.zeros(max_iters), np.zeros(max_iters), np.zeros(d)
        vp = lambda v: v.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._check(self.lib.ref_solve(vp(a), vp(y), i64(n), i64(d), cint(variant), i64(rows), i64(max_iters),
                                       dbl(gap_tol), cint(int(line_search)), u64(seed), C.byref(it), vp(losses),
                                       vp(gaps), vp(xf), C.byref(fs), C.byref(cv)))
        k = it.value
        return {"losses": losses[:k], "gaps": gaps[:k], "x": xf, "f_star": fs.value, "converged": bool(cv.value)}

    def chain(self, d1, d2, d3, scale, x, relu=False, threads=1):
        x = _f32rows(x)
        n = x.shape[1]
        y = np.zeros(x.shape)
        f = lambda d: np.ascontiguousarray(d, dtype=np.float64).reshape(-1)  # noqa: E731
        self._check(self.lib.ref_batch_chain(n, f(d1), f(d2), f(d3), scale, x, x.shape[0], x.shape[1], int(relu),
                                             y, threads))
        return y
