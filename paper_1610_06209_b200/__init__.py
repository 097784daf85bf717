"""B200-native structured spinners (arxiv 1610.06209) — Python host mirror.

A thin ctypes layer over the C ABI in ``include/spinners_b200.h`` whose classes
mirror the reference's C++ entry points (``proj/include/spinners/*.hpp``):

=========================  ==============================================================
this module                reference
=========================  ==============================================================
``SpinnerVariant``         ``SpinnerVariant`` (spinner.hpp:18-25)
``StructuredSpinner``      ``StructuredSpinner::build/apply`` (spinner.hpp:56-104)
``StackedSpinner``         ``StackedSpinner(v,n,m,k,seed)/apply`` (spinner.hpp:108-123)
``signed_argmax``          ``signed_argmax`` (lsh.hpp:21) — host helper on a projection
``CrossPolytopeHasher``    ``CrossPolytopeHasher::hash`` (lsh.hpp:26-36)
``make_hasher_factory``    ``make_hasher_factory`` (lsh.hpp:66, lsh.cpp:32-36)
``MultiTableHasher``       L tables at once (builder-defined, BASELINE config 3)
``KernelKind/FeatureMap``  ``KernelKind``/``FeatureMap`` (kernels.hpp:11-28)
``embed``                  ``embed`` (kernels.hpp:33, kernels.cpp:17-36)
``SketchOperator``         ``SketchOperator`` (newton_sketch.hpp:50-71)
``mix_seed``               ``mix_seed`` (common.hpp:51-56)
=========================  ==============================================================

Inputs may be CUDA ``torch.Tensor`` s (device path: stream-ordered kernels, no
copies) or host arrays (numpy / CPU tensors: the ``spn_*_host`` entry points,
which pipeline the host<->device copies with the kernels).  All arithmetic runs
in the sm_100a kernels of ``_lib/libspinners_b200.so``; there is no CPU
fallback — importing this module without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPN_LIB") or os.path.join(_HERE, "_lib", "libspinners_b200.so")  # SPN_LIB: A/B variants

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the sm_100a extension first "
        "(python paper_1610_06209_b200/build_ext.py, or __graft_entry__.build(), from the repo root)")

_lib = C.CDLL(LIB_PATH)

# ----------------------------------------------------------------------------- ABI
_i64, _u64, _i32, _dbl, _vp = C.c_int64, C.c_uint64, C.c_int32, C.c_double, C.c_void_p


class _Desc(C.Structure):
    _fields_ = [("variant", _i32), ("n", _i64), ("m", _i64), ("k", _i64), ("tables", _i64),
                ("table_seeds", C.POINTER(_u64)), ("seed", _u64), ("scale", _dbl), ("device", _i32)]


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_status_string = _sig("spn_status_string", C.c_char_p, [C.c_int])
_last_error = _sig("spn_last_error", C.c_char_p, [])
_version = _sig("spn_version", C.c_char_p, [])
_plan_create = _sig("spn_plan_create", C.c_int, [C.POINTER(_vp), C.POINTER(_Desc)])
_plan_create_block = _sig("spn_plan_create_block", C.c_int, [C.POINTER(_vp), _i32, _i64, _i64, _u64, _dbl, _i32])
_plan_create_explicit = _sig("spn_plan_create_explicit", C.c_int,
                             [C.POINTER(_vp), _i64, _i64, _i64, _i64, _vp, _vp, _vp, _dbl, _i32])
_plan_destroy = _sig("spn_plan_destroy", C.c_int, [_vp])
_plan_query = _sig("spn_plan_query", C.c_int, [_vp] + [C.POINTER(_i64)] * 5 + [C.POINTER(_dbl)])
_plan_diagonals = _sig("spn_plan_diagonals", C.c_int, [_vp, _vp, _vp, _vp])
_apply = _sig("spn_apply_f32", C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _i32, _vp])
_hash = _sig("spn_hash_f32", C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp])
_hash_peers = _sig("spn_hash_f32_peers", C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i32, _i64, _i64, _vp])
_enable_peer = _sig("spn_enable_peer_access", C.c_int, [_i32, _i32])
_embed = _sig("spn_embed_f32", C.c_int, [_vp, _i32, _dbl, _vp, _i64, _i64, _i64, _vp, _i64, _vp])
_sketch = _sig("spn_sketch_f32", C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _dbl, _vp, _i64, _vp])
_apply_host = _sig("spn_apply_f32_host", C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _i32])
_hash_host = _sig("spn_hash_f32_host", C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp])
_embed_host = _sig("spn_embed_f32_host", C.c_int, [_vp, _i32, _dbl, _vp, _i64, _i64, _i64, _vp, _i64])
_hash_project_host = _sig("spn_hash_project_f32_host", C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _i64])
_sketch_host = _sig("spn_sketch_f32_host", C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _dbl, _vp, _i64])
_plan_resample = _sig("spn_plan_resample", C.c_int, [C.POINTER(_vp), _vp, _i32, _u64])
_plan_with_tail = _sig("spn_plan_with_tail", C.c_int, [C.POINTER(_vp), _vp, _vp])
_sample_rows = _sig("spn_sample_rows", C.c_int, [_i64, _i64, _u64, _vp])
_mix_seed = _sig("spn_mix_seed", _u64, [_u64, _u64])
_check_rows = _sig("spn_check_rows_f32", C.c_int, [_vp, _i64, _i64, _i64, _vp, _vp])
_fwht = _sig("spn_fwht_f32", C.c_int, [_i64, _vp, _i64, _i64, _vp, _i64, _i32, _vp])
_fwht_host = _sig("spn_fwht_f32_host", C.c_int, [_i64, _vp, _i64, _i64, _vp, _i64, _i32])
_diag = _sig("spn_diag_f32", C.c_int, [_i64, _vp, _vp, _i64, _i64, _vp, _i64, _vp])
_diag_host = _sig("spn_diag_f32_host", C.c_int, [_i64, _vp, _vp, _i64, _i64, _vp, _i64, _i32])
_circ_create = _sig("spn_circulant_create", C.c_int, [C.POINTER(_vp), _i32, _i64, _vp, _vp, _i32])
_circ_destroy = _sig("spn_circulant_destroy", C.c_int, [_vp])
_circ_apply = _sig("spn_circulant_apply_f32", C.c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _vp])
_circ_apply_host = _sig("spn_circulant_apply_f32_host", C.c_int, [_vp, _vp, _i64, _i64, _vp, _i64])

SPN_OK, SPN_EDIM, SPN_EDOMAIN, SPN_ECUDA, SPN_ENOMEM, SPN_EUNSUPPORTED, SPN_EINVAL, SPN_ESINGULAR = range(8)
ABI_SYMBOLS = ("spn_status_string", "spn_last_error", "spn_version", "spn_plan_create", "spn_plan_create_block",
               "spn_plan_create_explicit", "spn_plan_destroy", "spn_plan_query", "spn_plan_diagonals",
               "spn_apply_f32", "spn_hash_f32", "spn_embed_f32", "spn_sketch_f32", "spn_apply_f32_host",
               "spn_hash_f32_host", "spn_embed_f32_host", "spn_sample_rows", "spn_mix_seed",
               "spn_check_rows_f32", "spn_realize_block", "spn_newton_create", "spn_newton_destroy",
               "spn_logistic_eval_f32", "spn_hessian_sqrt_f32", "spn_sketched_step_f32", "spn_logistic_line_f32",
               "spn_ar1_problem", "spn_newton_set_problem", "spn_logistic_eval_host", "spn_hessian_sqrt_host",
               "spn_sketched_step_host", "spn_logistic_line_host", "spn_collision_hits_f32", "spn_gram_exact_f32",
               "spn_gram_approx_f32", "spn_gram_error", "spn_gram_exact_host", "spn_gram_approx_host",
               "spn_gram_error_host", "spn_hash_f32_peers", "spn_fwht_f32", "spn_fwht_f32_host", "spn_diag_f32",
               "spn_diag_f32_host", "spn_circulant_create", "spn_circulant_destroy", "spn_circulant_apply_f32",
               "spn_circulant_apply_f32_host", "spn_hash_project_f32_host", "spn_sketch_f32_host", "spn_plan_resample",
               "spn_plan_with_tail", "spn_enable_peer_access")


# ----------------------------------------------------------------------- errors
class SpinnerError(RuntimeError):
    """CUDA / resource / unsupported-request failure (status >= 3)."""


class DimensionError(ValueError):
    """Mirrors spinners::DimensionError (common.hpp:15-17)."""


class DomainError(ValueError):
    """Mirrors spinners::DomainError (common.hpp:19-21)."""


class SingularSystemError(RuntimeError):
    """Mirrors spinners::SingularSystemError (common.hpp:25-27)."""


def _check(status: int) -> None:
    if status == SPN_OK:
        return
    msg = f"{_status_string(status).decode()}: {_last_error().decode()}"
    if status == SPN_EDIM:
        raise DimensionError(msg)
    if status == SPN_EDOMAIN:
        raise DomainError(msg)
    if status == SPN_ESINGULAR:
        raise SingularSystemError(msg)
    raise SpinnerError(msg)


def version() -> str:
    return _version().decode()


def mix_seed(base: int, stream: int) -> int:
    """splitmix64 seed derivation (common.hpp:51-56)."""
    return int(_mix_seed(base & (2**64 - 1), stream & (2**64 - 1)))


def sample_rows(N: int, m: int, seed: int) -> np.ndarray:
    """Builder-defined coordinate sampler P: m distinct sorted indices of [0, N)."""
    out = np.zeros(m, dtype=np.int64)
    _check(_sample_rows(N, m, seed & (2**64 - 1), out.ctypes.data))
    return out


class SpinnerVariant(enum.IntEnum):
    """spinner.hpp:18-25 (the full family) + the builder-defined all-Gaussian config-5 variant."""
    hd3_hd2_hd1 = 0
    hdg_hd2_hd1 = 1
    gcirc_d2_hd1 = 2
    gtoeplitz_d2_hd1 = 3
    gskew_circ_d2_hd1 = 4
    gaussian_dense = 5
    gauss3 = 100  # builder-defined: D1..D3 iid N(0,1)


_VARIANT_NAMES = {"HD3HD2HD1": SpinnerVariant.hd3_hd2_hd1, "HDgHD2HD1": SpinnerVariant.hdg_hd2_hd1,
                  "GcircD2HD1": SpinnerVariant.gcirc_d2_hd1, "GToeplitzD2HD1": SpinnerVariant.gtoeplitz_d2_hd1,
                  "GSkewCircD2HD1": SpinnerVariant.gskew_circ_d2_hd1,
                  "GaussianDense": SpinnerVariant.gaussian_dense, "Gauss3": SpinnerVariant.gauss3}


def variant_to_string(v) -> str:
    """spinner.cpp:9-19."""
    for k, val in _VARIANT_NAMES.items():
        if val == v:
            return k
    raise DomainError("to_string: unknown variant")


def variant_from_string(s: str) -> SpinnerVariant:
    """spinner.cpp:21-25 (only the variants this hot path implements)."""
    try:
        return _VARIANT_NAMES[s]
    except KeyError:
        raise DomainError(f"unknown spinner variant: {s}") from None


def all_variants():
    """spinner.cpp:27-31 (the reference's six; the builder-defined gauss3 is not listed)."""
    return [SpinnerVariant.hd3_hd2_hd1, SpinnerVariant.hdg_hd2_hd1, SpinnerVariant.gcirc_d2_hd1,
            SpinnerVariant.gtoeplitz_d2_hd1, SpinnerVariant.gskew_circ_d2_hd1, SpinnerVariant.gaussian_dense]


def structured_variants():
    """spinner.cpp:33-37."""
    return all_variants()[:5]


def has_hadamard(v) -> bool:
    """spinner.cpp:38."""
    return SpinnerVariant(v) != SpinnerVariant.gaussian_dense


# ------------------------------------------------------------------ buffers
def _torch():
    import torch
    return torch


def _is_cuda(x) -> bool:
    try:
        torch = _torch()
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


def _stream_ptr(stream):
    if stream is None:
        return _torch().cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _rows2d(x):
    one = x.ndim == 1
    if one:
        x = x.reshape(1, -1)
    if x.ndim != 2:
        raise DimensionError("expected a vector or a [batch, n] matrix")
    return x, one


class _Plan:
    """Owns one spn_plan* (device-resident realised diagonals)."""

    def __init__(self, handle: int, device: int):
        self._h = _vp(handle)
        self.device = device
        n, m, k, t, b, sc = _i64(), _i64(), _i64(), _i64(), _i64(), _dbl()
        _check(_plan_query(self._h, C.byref(n), C.byref(m), C.byref(k), C.byref(t), C.byref(b), C.byref(sc)))
        self.n, self.m, self.k, self.tables, self.blocks, self.scale = (
            n.value, m.value, k.value, t.value, b.value, sc.value)

    @classmethod
    def create(cls, variant, n, m, k, tables=1, table_seeds=None, seed=0, scale=0.0, device=0):
        d = _Desc()
        d.variant, d.n, d.m, d.k, d.tables = int(variant), n, m, k, tables
        seeds = None
        if table_seeds is not None:
            seeds = (_u64 * len(table_seeds))(*[int(s) & (2**64 - 1) for s in table_seeds])
            d.table_seeds = C.cast(seeds, C.POINTER(_u64))
        d.seed, d.scale, d.device = int(seed) & (2**64 - 1), float(scale), int(device)
        h = _vp()
        _check(_plan_create(C.byref(h), C.byref(d)))
        return cls(h.value, device)

    @classmethod
    def create_explicit(cls, d1, d2, d3, n, m, k, tables=1, scale=0.0, device=0):
        arrs = [np.ascontiguousarray(a, dtype=np.float64).reshape(-1) for a in (d1, d2, d3)]
        h = _vp()
        _check(_plan_create_explicit(C.byref(h), n, m, k, tables, arrs[0].ctypes.data, arrs[1].ctypes.data,
                                     arrs[2].ctypes.data, float(scale), int(device)))
        return cls(h.value, device)

    def diagonals(self):
        size = self.tables * self.blocks * self.n
        out = [np.zeros(size) for _ in range(3)]
        _check(_plan_diagonals(self._h, out[0].ctypes.data, out[1].ctypes.data, out[2].ctypes.data))
        shape = (self.tables, self.blocks, self.n)
        return tuple(o.reshape(shape) for o in out)

    def __del__(self):
        h = getattr(self, "_h", None)
        destroy = _plan_destroy  # None once the module is torn down at interpreter exit
        if h is not None and h.value and destroy is not None:
            destroy(h)
            self._h = None

    # ---- device / host dispatch helpers
    def _device_in(self, x):
        torch = _torch()
        if x.dtype != torch.float32:
            raise DomainError("device inputs must be float32")
        if (x.device.index or 0) != self.device:
            raise SpinnerError(f"input on cuda:{x.device.index or 0}, plan on cuda:{self.device}")
        x, one = _rows2d(x)
        if x.stride(1) != 1:
            x = x.contiguous()
        if x.shape[1] > self.n:
            raise DimensionError(f"expected length <= {self.n}, got {x.shape[1]}")
        return x, one

    @staticmethod
    def _host_in(x):
        x = np.asarray(x)
        if x.dtype != np.float32:
            x = x.astype(np.float32)
        x, one = _rows2d(x)
        return np.ascontiguousarray(x), one

    def _device_out(self, out, rows, cols, dtype=None, what="out"):
        """Caller-supplied device output: `dtype`, on the plan's device, >= rows x cols, unit stride
        along the last dim.  Returns (tensor, leading dimension)."""
        torch = _torch()
        dtype = dtype or torch.float32
        if not _is_cuda(out):
            raise SpinnerError(f"{what} must be a CUDA tensor for a device input")
        if out.dtype != dtype:
            raise DomainError(f"{what} must be {dtype}, got {out.dtype}")
        if (out.device.index or 0) != self.device:
            raise SpinnerError(f"{what} on cuda:{out.device.index or 0}, plan on cuda:{self.device}")
        o2 = out.reshape(1, -1) if out.dim() == 1 else out
        if o2.dim() != 2 or o2.shape[0] < rows or o2.shape[1] < cols or (o2.shape[1] > 1 and o2.stride(1) != 1):
            raise DimensionError(f"{what} must be at least [{rows}, {cols}] with unit stride along dim 1, "
                                 f"got shape {tuple(out.shape)} stride {tuple(out.stride())}")
        return o2, o2.stride(0)

    @staticmethod
    def _host_out(out, rows, cols, dtype=np.float32, what="out"):
        """Caller-supplied host output: a writable numpy array of `dtype`, >= rows x cols, unit
        stride along the last dim.  Returns (array, leading dimension in elements)."""
        if not isinstance(out, np.ndarray):
            raise SpinnerError(f"{what} must be a numpy array for a host input")
        if out.dtype != dtype:
            raise DomainError(f"{what} must be {np.dtype(dtype)}, got {out.dtype}")
        o2 = out.reshape(1, -1) if out.ndim == 1 else out
        isz = o2.itemsize
        if (o2.ndim != 2 or o2.shape[0] < rows or o2.shape[1] < cols or not o2.flags.writeable
                or (o2.shape[1] > 1 and o2.strides[1] != isz) or o2.strides[0] % isz or o2.strides[0] < cols * isz):
            raise DimensionError(f"{what} must be a writable array of at least [{rows}, {cols}] with packed rows, "
                                 f"got shape {out.shape} strides {out.strides}")
        return o2, o2.strides[0] // isz

    def apply(self, x, relu=False, out=None, stream=None):
        if _is_cuda(x):
            torch = _torch()
            x, one = self._device_in(x)
            y = out if out is not None else torch.empty((x.shape[0], self.k), device=x.device, dtype=torch.float32)
            y2, ldy = self._device_out(y, x.shape[0], self.k)
            _check(_apply(self._h, x.data_ptr(), x.shape[0], x.stride(0), x.shape[1], y2.data_ptr(), ldy,
                          int(relu), _stream_ptr(stream)))
            return y[0] if one and out is None else y
        x, one = self._host_in(x)
        y = out if out is not None else np.empty((x.shape[0], self.k), dtype=np.float32)
        y2, ldy = self._host_out(y, x.shape[0], self.k)
        _check(_apply_host(self._h, x.ctypes.data, x.shape[0], x.shape[1], x.shape[1], y2.ctypes.data, ldy,
                           int(relu)))
        return y[0] if one and out is None else y

    def hash(self, x, y_out=None, stream=None):
        """int32 ids [batch, tables]; with y_out (single-table plans) also the projection."""
        if y_out is not None and self.tables != 1:
            raise SpinnerError("y output needs a single-table plan")
        if _is_cuda(x):
            torch = _torch()
            x, one = self._device_in(x)
            ids = torch.empty((x.shape[0], self.tables), device=x.device, dtype=torch.int32)
            yp, ldy = None, 0
            if y_out is not None:
                y2, ldy = self._device_out(y_out, x.shape[0], self.k, what="y_out")
                yp = y2.data_ptr()
            _check(_hash(self._h, x.data_ptr(), x.shape[0], x.stride(0), x.shape[1], ids.data_ptr(), yp, ldy,
                         _stream_ptr(stream)))
            return ids[0] if one else ids
        x, one = self._host_in(x)
        ids = np.empty((x.shape[0], self.tables), dtype=np.int32)
        if y_out is not None:
            y2, ldy = self._host_out(y_out, x.shape[0], self.k, what="y_out")
            _check(_hash_project_host(self._h, x.ctypes.data, x.shape[0], x.shape[1], x.shape[1], ids.ctypes.data,
                                      y2.ctypes.data, ldy))
        else:
            _check(_hash_host(self._h, x.ctypes.data, x.shape[0], x.shape[1], x.shape[1], ids.ctypes.data))
        return ids[0] if one else ids

    def embed(self, kind, sigma, x, out=None, stream=None):
        w = 2 * self.k if kind == 0 else self.k
        if _is_cuda(x):
            torch = _torch()
            x, one = self._device_in(x)
            o = out if out is not None else torch.empty((x.shape[0], w), device=x.device, dtype=torch.float32)
            o2, ldo = self._device_out(o, x.shape[0], w)
            _check(_embed(self._h, kind, float(sigma), x.data_ptr(), x.shape[0], x.stride(0), x.shape[1],
                          o2.data_ptr(), ldo, _stream_ptr(stream)))
            return o[0] if one and out is None else o
        x, one = self._host_in(x)
        o = out if out is not None else np.empty((x.shape[0], w), dtype=np.float32)
        o2, ldo = self._host_out(o, x.shape[0], w)
        _check(_embed_host(self._h, kind, float(sigma), x.ctypes.data, x.shape[0], x.shape[1], x.shape[1],
                           o2.ctypes.data, ldo))
        return o[0] if one and out is None else o

    def sketch(self, a, m_out, norm, rows=None, out=None, stream=None):
        """Device A (CUDA tensor [n_in, d]) -> device sketch; host A (numpy) -> host sketch through
        spn_sketch_f32_host (the reference's value semantics)."""
        rl = None
        if rows is not None:
            rows = np.ascontiguousarray(rows, dtype=np.int64)
            if rows.size != m_out:
                raise DimensionError("rows must have m_out entries")
            rl = rows.ctypes.data
        if not _is_cuda(a):
            a = np.asarray(a)
            if a.ndim != 2:
                raise DimensionError("expected a [n_in, d] matrix")
            if a.dtype != np.float32 or a.strides[1] != 4 or a.strides[0] % 4:
                a = np.ascontiguousarray(a, dtype=np.float32)
            o = out if out is not None else np.empty((m_out, a.shape[1]), dtype=np.float32)
            o2, ldo = self._host_out(o, m_out, a.shape[1])
            _check(_sketch_host(self._h, a.ctypes.data, a.shape[0], a.shape[1], a.strides[0] // 4, rl, m_out,
                                float(norm), o2.ctypes.data, ldo))
            return o
        torch = _torch()
        if a.dtype != torch.float32:
            raise DomainError("device inputs must be float32")
        if (a.device.index or 0) != self.device:
            raise SpinnerError(f"input on cuda:{a.device.index or 0}, plan on cuda:{self.device}")
        if a.dim() != 2 or a.stride(1) != 1:
            a = a.reshape(a.shape[0], -1).contiguous()
        o = out if out is not None else torch.empty((m_out, a.shape[1]), device=a.device, dtype=torch.float32)
        o2, ldo = self._device_out(o, m_out, a.shape[1])
        _check(_sketch(self._h, a.data_ptr(), a.shape[0], a.shape[1], a.stride(0), rl, m_out, float(norm),
                       o2.data_ptr(), ldo, _stream_ptr(stream)))
        return o


def check_rows(x, stream=None):
    """Device finiteness / zero-row flags (bit0 non-finite, bit1 all-zero)."""
    torch = _torch()
    x, _ = _rows2d(x)
    flags = torch.empty(x.shape[0], dtype=torch.int32, device=x.device)
    _check(_check_rows(x.data_ptr(), x.shape[0], x.stride(0), x.shape[1], flags.data_ptr(), _stream_ptr(stream)))
    return flags


# ------------------------------------------------------------ reference mirror
class SpinnerSpec:
    """spinner.hpp:40-53 — (variant, n, m, seed, scale); scale 0 => default sqrt(n)."""

    def __init__(self, variant=SpinnerVariant.hd3_hd2_hd1, n=0, m=0, seed=0, scale=0.0):
        self.variant, self.n, self.m, self.seed, self.scale = SpinnerVariant(variant), n, m, seed, scale

    @staticmethod
    def make(variant, n, m, seed):
        s = SpinnerSpec(variant, n, m, seed, 0.0)
        s.validate()
        return s

    def validate(self):  # spinner.cpp:59-67
        if self.n < 1:
            raise DimensionError("SpinnerSpec: n must be >= 1")
        if self.m < 1 or self.m > self.n:
            raise DimensionError("SpinnerSpec: need 1 <= m <= n")
        if self.variant != SpinnerVariant.gaussian_dense and self.n & (self.n - 1):
            raise DimensionError(
                f"SpinnerSpec: Hadamard-bearing variant requires power-of-two n, got {self.n}")
        if self.scale != 0.0 and not math.isfinite(self.scale):
            raise DomainError("SpinnerSpec: non-finite scale")

    def to_json(self) -> dict:  # spinner.cpp:72-78 (the wire format of specs)
        return {"variant": variant_to_string(self.variant), "n": self.n, "m": self.m, "seed": self.seed,
                "scale": self.effective_scale()}

    @staticmethod
    def from_json(j: dict) -> "SpinnerSpec":  # spinner.cpp:80-89
        s = SpinnerSpec(variant_from_string(j["variant"]), int(j["n"]), int(j["m"]), int(j["seed"]),
                        float(j.get("scale", 0.0)))
        s.validate()
        return s

    def effective_scale(self):  # spinner.cpp:40-45,69-71
        if self.scale != 0.0:
            return self.scale
        hadamard_only = self.variant in (SpinnerVariant.hd3_hd2_hd1, SpinnerVariant.hdg_hd2_hd1, SpinnerVariant.gauss3)
        return math.sqrt(self.n) if hadamard_only else 1.0


class StackedSpinner:
    """k x n operator of ceil(k/m) independently seeded blocks (spinner.cpp:248-283).

    ``scale`` overrides every block's SpinnerSpec.scale (0 = default sqrt(n))."""

    def __init__(self, variant, n, m, k, seed, scale=0.0, device=0, _plan=None):
        if k < 1:
            raise DimensionError("StackedSpinner: k must be >= 1")
        self.variant = SpinnerVariant(variant) if variant is not None else None
        self._p = _plan or _Plan.create(variant, n, m, k, seed=seed, scale=scale, device=device)
        self.seed = seed

    @classmethod
    def from_diagonals(cls, d1, d2, d3, n, m, k, scale=0.0, device=0):
        return cls(None, n, m, k, 0, _plan=_Plan.create_explicit(d1, d2, d3, n, m, k, 1, scale, device))

    def rows(self):
        return self._p.k

    def input_dim(self):
        return self._p.n

    @property
    def plan(self):
        return self._p

    def diagonals(self):
        """Realised fp64 (d1, d2, d3) as [blocks][n] arrays (d3 = g for HDg)."""
        d1, d2, d3 = self._p.diagonals()
        return d1[0], d2[0], d3[0]

    def apply(self, x, relu=False, out=None, stream=None):
        """y = scale * stacked(x); x shorter than n is zero padded.  ReLU optional."""
        return self._p.apply(x, relu=relu, out=out, stream=stream)


class StructuredSpinner(StackedSpinner):
    """One m x n block (spinner.hpp:56-104): StructuredSpinner.build(spec).

    The block's diagonals come from spec.seed directly (spinner.cpp:137-151),
    realised by the library's host generator (spn_realize_block)."""

    @classmethod
    def build(cls, spec: SpinnerSpec, device=0):
        spec.validate()
        h = _vp()  # every variant, drawn from spec.seed itself (spinner.cpp:137-151)
        _check(_plan_create_block(C.byref(h), int(spec.variant), spec.n, spec.m, int(spec.seed) & (2**64 - 1),
                                  float(spec.scale), device))
        return cls._wrap(h, spec, device)

    @classmethod
    def _wrap(cls, h, spec, device):
        obj = cls(None, spec.n, spec.m, spec.m, spec.seed, _plan=_Plan(h.value, device))
        obj.variant = spec.variant
        obj.spec = spec
        obj.device = device
        obj._front = None
        return obj

    def resample_last_block(self, tail_seed):
        """spinner.hpp:67-69 / spinner.cpp:153-158: same M1, M2; the last block's randomness (D3, g,
        the circulant generator or the dense matrix) redrawn from Rng(mix_seed(tail_seed, 2))."""
        h = _vp()
        _check(_plan_resample(C.byref(h), self._p._h, 0, int(tail_seed) & (2**64 - 1)))
        return StructuredSpinner._wrap(h, self.spec, self.device)

    def resample_tail(self, tail_seed):
        """spinner.hpp:71-73 / spinner.cpp:160-166: D2 and the last block redrawn from
        Rng(mix_seed(tail_seed, 3)); M1 stays fixed."""
        h = _vp()
        _check(_plan_resample(C.byref(h), self._p._h, 1, int(tail_seed) & (2**64 - 1)))
        return StructuredSpinner._wrap(h, self.spec, self.device)

    def with_tail_vector(self, r):
        """spinner.hpp:75-77 / spinner.cpp:168-184: D3 (HD3) or g (HDg) replaced by r."""
        rv = np.ascontiguousarray(np.asarray(r, dtype=np.float64).reshape(-1))
        if rv.size != self.spec.n:
            raise DimensionError("with_tail_vector: length mismatch")
        h = _vp()
        _check(_plan_with_tail(C.byref(h), self._p._h, rv.ctypes.data))
        return StructuredSpinner._wrap(h, self.spec, self.device)

    def d1(self):
        return self.diagonals()[0]

    def d2(self):
        return self.diagonals()[1]

    def d3(self):
        return self.diagonals()[2]

    g_diag = d3

    def apply_front_blocks(self, x):
        """M2 M1 x (spinner.cpp:186-198): H D2 H D1 x for the Hadamard-only variants, D2 H D1 x for the
        circulant family (on the device: the D2 H D1 chain, plus one normalised FWHT), on the device
        the spinner was built on."""
        if self.variant == SpinnerVariant.gaussian_dense:
            raise DomainError("apply_front_blocks: dense baseline has no block structure")
        n = self.spec.n
        if self._front is None:  # D2 H D1 as a plan with D3 = 1 and scale 1 (H 1 H D2 H D1 = D2 H D1)
            d1, d2, _ = (a[0, 0] for a in self._p.diagonals())
            self._front = StackedSpinner.from_diagonals(d1, d2, np.ones(n), n, n, n, scale=1.0, device=self.device)
        hadamard_only = self.variant in (SpinnerVariant.hd3_hd2_hd1, SpinnerVariant.hdg_hd2_hd1, SpinnerVariant.gauss3)
        if _is_cuda(x):
            y = self._front.apply(x)
            return fwht_normalized(y, device=self.device) if hadamard_only else y
        xv = np.asarray(x, dtype=np.float64)
        if xv.shape[-1] != n:
            raise DimensionError("apply_front_blocks: length mismatch")
        if not np.all(np.isfinite(xv)):
            raise DomainError("apply_front_blocks: non-finite entry")
        y = self._front.apply(xv)
        if hadamard_only:
            y = fwht_normalized(y, device=self.device)
        return np.asarray(y, dtype=np.float64)


_realize_block = _sig("spn_realize_block", C.c_int, [_i32, _i64, _u64, _vp, _vp, _vp])


def realize_block(variant, n, spec_seed):
    """(d1, d2, d3) of one block realised from spec seed `spec_seed` with the
    reference's generator (d3 is g for HDg, all three Gaussian for gauss3)."""
    d = [np.zeros(n) for _ in range(3)]
    _check(_realize_block(int(variant), n, int(spec_seed) & (2**64 - 1), *(a.ctypes.data for a in d)))
    return tuple(d)


def signed_argmax(y) -> tuple[int, int]:
    """lsh.cpp:9-21 on a host vector (ties -> smallest index, sign(0) = +1)."""
    y = np.asarray(y, dtype=np.float64).reshape(-1)
    if y.size == 0:
        raise DimensionError("signed_argmax: empty vector")
    a = np.abs(y)
    i = int(np.argmax(a))  # numpy returns the first maximal index
    return i, (-1 if y[i] < 0.0 else 1)


def _host_rows(x):
    """fp64 host values -> contiguous fp32 rows (the reference's checks on the fp64 input first)."""
    xv = np.asarray(x, dtype=np.float64)
    one = xv.ndim == 1
    xv = xv.reshape(1, -1) if one else xv
    if xv.ndim != 2:
        raise DimensionError("expected a vector or a [batch, n] matrix")
    return np.ascontiguousarray(xv, dtype=np.float32), one


def fwht_normalized(x, out=None, stream=None, device=0):
    """transforms.hpp:13 / transforms.cpp:52-71: H_n x with the orthonormal Walsh-Hadamard H_n, for a
    vector or every row of a [batch, n] array.  Host input follows the reference (fp64 values,
    DimensionError for a non-power-of-two length, DomainError for a non-finite entry) and returns fp64;
    a CUDA tensor is transformed on the device on `stream` (fp32)."""
    if _is_cuda(x):
        torch = _torch()
        x2, one = _rows2d(x)
        if x2.dtype != torch.float32 or x2.stride(-1) != 1:
            x2 = x2.to(torch.float32).contiguous()
        o = out if out is not None else torch.empty_like(x2)
        _check(_fwht(x2.shape[1], x2.data_ptr(), x2.shape[0], x2.stride(0), o.data_ptr(), o.stride(0),
                     x2.device.index or 0, _stream_ptr(stream)))
        return o[0] if one else o
    xf, one = _host_rows(x)
    n = xf.shape[1]
    if n == 0 or n & (n - 1):
        raise DimensionError(f"fwht_normalized: length must be a power of two, got {n}")
    if not np.all(np.isfinite(np.asarray(x, dtype=np.float64))):
        raise DomainError("fwht_normalized: non-finite entry")
    o = np.empty_like(xf)
    _check(_fwht_host(n, xf.ctypes.data, xf.shape[0], n, o.ctypes.data, n, device))
    o = o.astype(np.float64)
    return o[0] if one else o


def diag_matvec(d, x, out=None, stream=None, device=0):
    """transforms.hpp:59 / transforms.cpp:228-235: d (.) x for a vector or every row of x.  Host input
    keeps the reference's length and finiteness checks; CUDA tensors run on the device."""
    if _is_cuda(x):
        torch = _torch()
        x2, one = _rows2d(x)
        if x2.dtype != torch.float32 or x2.stride(-1) != 1:
            x2 = x2.to(torch.float32).contiguous()
        dv = d.to(device=x2.device, dtype=torch.float32).contiguous() if _is_cuda(d) else \
            torch.from_numpy(np.ascontiguousarray(d, dtype=np.float32)).to(x2.device)
        if dv.numel() != x2.shape[1]:
            raise DimensionError("diag_matvec: length mismatch")
        o = out if out is not None else torch.empty_like(x2)
        _check(_diag(x2.shape[1], dv.data_ptr(), x2.data_ptr(), x2.shape[0], x2.stride(0), o.data_ptr(),
                     o.stride(0), _stream_ptr(stream)))
        return o[0] if one else o
    dv = np.asarray(d, dtype=np.float64).reshape(-1)
    xf, one = _host_rows(x)
    if dv.size != xf.shape[1]:
        raise DimensionError("diag_matvec: length mismatch")
    if not np.all(np.isfinite(dv)) or not np.all(np.isfinite(np.asarray(x, dtype=np.float64))):
        raise DomainError("diag_matvec: non-finite entry")
    df = np.ascontiguousarray(dv, dtype=np.float32)
    o = np.empty_like(xf)
    _check(_diag_host(xf.shape[1], df.ctypes.data, xf.ctypes.data, xf.shape[0], xf.shape[1], o.ctypes.data,
                      xf.shape[1], device))
    o = o.astype(np.float64)
    return o[0] if one else o


class CirculantKind(enum.IntEnum):
    """transforms.hpp:15."""
    circulant = 0
    toeplitz = 1
    skew_circulant = 2


class CirculantSpec:
    """transforms.hpp:22-35: generating data of a circulant-family matrix (validated like
    CirculantSpec::validate, transforms.cpp:98-110)."""

    def __init__(self, kind, first_row, first_col=None):
        self.kind = CirculantKind(kind)
        self.first_row = np.asarray(first_row, dtype=np.float64).reshape(-1)
        self.first_col = None if first_col is None else np.asarray(first_col, dtype=np.float64).reshape(-1)
        self.validate()

    @staticmethod
    def circulant(r):
        return CirculantSpec(CirculantKind.circulant, r)

    @staticmethod
    def toeplitz(col, row):
        return CirculantSpec(CirculantKind.toeplitz, row, col)

    @staticmethod
    def skew_circulant(r):
        return CirculantSpec(CirculantKind.skew_circulant, r)

    def dim(self):
        return self.first_row.size

    def validate(self):
        if self.first_row.size == 0:
            raise DimensionError("CirculantSpec: n must be >= 1")
        if not np.all(np.isfinite(self.first_row)):
            raise DomainError("CirculantSpec.first_row: non-finite entry")
        if self.kind == CirculantKind.toeplitz:
            if self.first_col is None or self.first_col.size != self.first_row.size:
                raise DimensionError("CirculantSpec: toeplitz first_col/first_row length mismatch")
            if not np.all(np.isfinite(self.first_col)):
                raise DomainError("CirculantSpec.first_col: non-finite entry")
            if self.first_col[0] != self.first_row[0]:
                raise DomainError("CirculantSpec: toeplitz corner entry mismatch")
        elif self.first_col is not None and self.first_col.size:
            raise DimensionError("CirculantSpec: first_col only valid for toeplitz")


class CirculantOperator:
    """transforms.hpp:37-51: the spectrum is computed once (on the host, as the reference does) and
    apply runs the fp64 correlation on the device.  apply(x): one vector (fp64 in / out, the
    reference's checks) or a [batch, n] CUDA tensor (fp32, stream-ordered)."""

    def __init__(self, spec: CirculantSpec, device=0):
        self._h = None
        spec.validate()
        self._spec, self.device = spec, device
        row = np.ascontiguousarray(spec.first_row)
        col = None if spec.kind != CirculantKind.toeplitz else np.ascontiguousarray(spec.first_col)
        h = _vp()
        _check(_circ_create(C.byref(h), int(spec.kind), row.size, row.ctypes.data,
                            None if col is None else col.ctypes.data, device))
        self._h = h

    def spec(self):
        return self._spec

    def apply(self, x, out=None, stream=None):
        n = self._spec.dim()
        if _is_cuda(x):
            torch = _torch()
            x2, one = _rows2d(x)
            if x2.shape[1] != n:
                raise DimensionError(f"CirculantOperator::apply: expected length {n}, got {x2.shape[1]}")
            if x2.dtype != torch.float32 or x2.stride(-1) != 1:
                x2 = x2.to(torch.float32).contiguous()
            o = out if out is not None else torch.empty_like(x2)
            _check(_circ_apply(self._h, x2.data_ptr(), x2.shape[0], x2.stride(0), o.data_ptr(), o.stride(0),
                               _stream_ptr(stream)))
            return o[0] if one else o
        xv = np.asarray(x, dtype=np.float64)
        xf, one = _host_rows(xv)
        if xf.shape[1] != n:
            raise DimensionError(f"CirculantOperator::apply: expected length {n}, got {xf.shape[1]}")
        if not np.all(np.isfinite(xv)):
            raise DomainError("CirculantOperator::apply: non-finite entry")
        o = np.empty_like(xf)
        _check(_circ_apply_host(self._h, xf.ctypes.data, xf.shape[0], n, o.ctypes.data, n))
        o = o.astype(np.float64)
        return o[0] if one else o

    def __del__(self):
        h = getattr(self, "_h", None)
        destroy = _circ_destroy
        if h is not None and h.value and destroy is not None:
            destroy(h)
            self._h = None


def circulant_matvec(spec: CirculantSpec, x):
    """transforms.cpp:210-214."""
    if spec.kind != CirculantKind.circulant:
        raise DomainError("circulant_matvec: spec is not circulant")
    return CirculantOperator(spec).apply(x)


def toeplitz_matvec(spec: CirculantSpec, x):
    """transforms.cpp:216-220."""
    if spec.kind != CirculantKind.toeplitz:
        raise DomainError("toeplitz_matvec: spec is not toeplitz")
    return CirculantOperator(spec).apply(x)


def skew_circulant_matvec(spec: CirculantSpec, x):
    """transforms.cpp:222-226."""
    if spec.kind != CirculantKind.skew_circulant:
        raise DomainError("skew_circulant_matvec: spec is not skew-circulant")
    return CirculantOperator(spec).apply(x)


def decode_id(bucket: int, k: int) -> tuple[int, int]:
    """int32 bucket id -> (index, sign): id = index + (sign < 0 ? k : 0)."""
    return (int(bucket) - k, -1) if bucket >= k else (int(bucket), 1)


class CrossPolytopeHasher:
    """lsh.hpp:26-36: signed argmax over a stacked spinner's rows."""

    def __init__(self, projector: StackedSpinner):
        self._proj = projector

    @property
    def projector(self):
        return self._proj

    def hash_ids(self, x, stream=None):
        """Batch: int32 bucket ids (index + k if the sign is negative)."""
        ids = self._proj.plan.hash(x, stream=stream)
        return ids[..., 0] if not hasattr(ids, "shape") or ids.ndim else ids

    def hash(self, x):
        """Single vector -> (index, sign), like CrossPolytopeHasher::hash.  Rejects
        non-finite and all-zero input as the reference does (lsh.cpp:24-28)."""
        xv = np.asarray(x.detach().cpu() if _is_cuda(x) else x, dtype=np.float64).reshape(-1)
        if not np.all(np.isfinite(xv)):
            raise DomainError("CrossPolytopeHasher::hash: non-finite entry")
        if not np.any(xv != 0.0):
            raise DomainError("CrossPolytopeHasher::hash: zero vector")
        bucket = int(np.asarray(self._proj.plan.hash(xv.astype(np.float32)[None, :]))[0, 0])
        return decode_id(bucket, self._proj.rows())


def make_hasher_factory(variant, n, m, device=0):
    """lsh.cpp:32-36: seed -> CrossPolytopeHasher(StackedSpinner(v, n, min(m,n), m, seed)).
    The returned callable also carries (variant, n, m, device) so the batched drivers
    (collision_curve) can build all trials' tables in one plan."""
    def factory(seed):
        return CrossPolytopeHasher(StackedSpinner(variant, n, min(m, n), m, seed, device=device))
    factory.variant, factory.n, factory.m, factory.device = variant, n, m, device
    return factory


class MultiTableHasher:
    """L independent cross-polytope tables evaluated in one fused launch.

    Table t is make_hasher_factory(variant, n, m)(table_seeds[t]); by default
    table_seeds[t] = mix_seed(seed, t) (the per-trial derivation of lsh.cpp:56)."""

    def __init__(self, variant, n, m, tables, seed=0, table_seeds: Optional[Sequence[int]] = None, device=0):
        if table_seeds is None:
            table_seeds = [mix_seed(seed, t) for t in range(tables)]
        self.table_seeds = [int(s) for s in table_seeds]
        self.k = m
        self._p = _Plan.create(variant, n, min(m, n), m, tables=len(self.table_seeds),
                               table_seeds=self.table_seeds, device=device)

    @property
    def plan(self):
        return self._p

    def hash_ids(self, x, stream=None):
        return self._p.hash(x, stream=stream)


class KernelKind:
    """kernels.hpp:11-24."""
    gaussian_tag, angular_tag = 0, 1

    def __init__(self, tag, sigma):
        self.tag, self.sigma = tag, sigma

    @staticmethod
    def gaussian(sigma):
        if not sigma > 0.0:
            raise DomainError("KernelKind: sigma must be positive")
        return KernelKind(0, float(sigma))

    @staticmethod
    def angular():
        return KernelKind(1, 0.0)


class FeatureMap:
    """kernels.hpp:26-30: a projector plus a kernel recipe."""

    def __init__(self, projector: StackedSpinner, kind: KernelKind):
        self.projector, self.kind = projector, kind


def embed(fm: FeatureMap, x, out=None, stream=None):
    """kernels.cpp:17-36.  Gaussian -> [cos(z/sigma) || sin(z/sigma)] / sqrt(d');
    angular -> sign(z) with sign(0) = +1.  Batch or single vector."""
    return fm.projector.plan.embed(fm.kind.tag, fm.kind.sigma, x, out=out, stream=stream)


_gram_exact = _sig("spn_gram_exact_f32", C.c_int, [_vp, _i64, _i64, _i64, _i32, _dbl, _vp, _i64, _vp])
_gram_approx = _sig("spn_gram_approx_f32", C.c_int, [_vp, _i64, _i64, _i64, _i32, _i64, _vp, _i64, _vp])
_gram_error = _sig("spn_gram_error", C.c_int, [_vp, _vp, _i64, _i64, C.POINTER(_dbl), _vp])


def _points_dev(points, device=0):
    torch = _torch()
    host = not _is_cuda(points)
    t = points if not host else torch.from_numpy(np.ascontiguousarray(np.asarray(points, dtype=np.float32)))
    t = t.to(device=f"cuda:{device}" if host else t.device, dtype=torch.float32)
    if t.dim() != 2:
        raise DimensionError("expected a [count, dim] point set")
    return t.contiguous(), host


def gram_exact(points, kind: KernelKind, stream=None):
    """kernels.cpp:38-76: exact kernel matrix (fp64 [count, count]) of fp32 points."""
    torch = _torch()
    p, host = _points_dev(points)
    if p.shape[0] < 1:
        raise DimensionError("gram_exact: empty dataset")
    if kind.tag == KernelKind.angular_tag and bool(((check_rows(p) & 2) != 0).any()):
        raise DomainError("gram_exact: angular kernel undefined at the zero vector")
    if bool(((check_rows(p) & 1) != 0).any()):
        raise DomainError("gram_exact: non-finite entry")
    g = torch.empty((p.shape[0], p.shape[0]), dtype=torch.float64, device=p.device)
    _check(_gram_exact(p.data_ptr(), p.shape[0], p.shape[1], p.stride(0), kind.tag, kind.sigma, g.data_ptr(),
                       g.stride(0), _stream_ptr(stream)))
    return g.cpu().numpy() if host else g


def gram_approx(fm: FeatureMap, points, stream=None):
    """kernels.cpp:78-103: features = embed(fm, points) on the device, then F F^T
    (gaussian) or 1/2 + F F^T / (2 d') (angular), diagonal 1, in fp64."""
    torch = _torch()
    p, host = _points_dev(points, fm.projector.plan.device)
    if p.shape[0] < 1:
        raise DimensionError("gram_approx: empty dataset")
    f = embed(fm, p, stream=stream)
    g = torch.empty((p.shape[0], p.shape[0]), dtype=torch.float64, device=p.device)
    _check(_gram_approx(f.data_ptr(), f.shape[0], f.shape[1], f.stride(0), fm.kind.tag, fm.projector.plan.k,
                        g.data_ptr(), g.stride(0), _stream_ptr(stream)))
    return g.cpu().numpy() if host else g


def gram_error(exact, approx, stream=None) -> float:
    """kernels.cpp:105-112: ||K - K_approx||_F / ||K||_F."""
    torch = _torch()
    a = exact if _is_cuda(exact) else torch.from_numpy(np.ascontiguousarray(exact, dtype=np.float64)).cuda()
    b = approx if _is_cuda(approx) else torch.from_numpy(np.ascontiguousarray(approx, dtype=np.float64)).cuda()
    a = a.to(torch.float64).contiguous()
    b = b.to(device=a.device, dtype=torch.float64).contiguous()
    if a.shape != b.shape or a.dim() != 2 or a.shape[0] != a.shape[1]:
        raise DimensionError("gram_error: shape mismatch")
    err = _dbl()
    _check(_gram_error(a.data_ptr(), b.data_ptr(), a.shape[0], a.stride(0), C.byref(err), _stream_ptr(stream)))
    return err.value


class SketchOperator:
    """newton_sketch.hpp:50-71 (the spinner sketch; `rows` output rows).

    mode "first" reproduces the reference (first `rows` rows of the padded
    StackedSpinner); mode "random" is the builder-defined P = sample_rows(...)
    of BASELINE config 4.  Output = sqrt(padded)/sqrt(rows) * P H D3 H D2 H D1 a_c."""

    def __init__(self, variant=None, input_dim=None, rows=None, seed=0, mode="first", p_seed=None, device=0):
        self._p = None
        if variant is None:  # SketchOperator() = the exact (identity) operator (newton_sketch.hpp:55-56)
            self.input_dim = self.padded = self.m = None
            self.norm, self.row_list = 1.0, None
            return
        padded = 1 << max(0, (input_dim - 1).bit_length())
        if mode == "random" and rows > padded:
            raise DimensionError("SketchOperator: a sampled P needs rows <= padded dimension")
        # rows > padded: ceil(rows / padded) stacked blocks (newton_sketch.cpp:77-79)
        self.input_dim, self.padded, self.m = input_dim, padded, rows
        self.norm = 1.0 / math.sqrt(rows)
        self._p = _Plan.create(variant, padded, min(rows, padded), rows, seed=seed, device=device)
        self.row_list = None
        if mode == "random":
            self.row_list = sample_rows(padded, rows, seed if p_seed is None else p_seed)
        elif mode != "first":
            raise DomainError(f"unknown sketch mode {mode}")

    @property
    def plan(self):
        return self._p

    def is_exact(self) -> bool:
        return self._p is None

    def rows(self, input_dim=None):
        return input_dim if self.is_exact() else self.m

    def apply(self, columns, out=None, stream=None):
        """columns: [input_dim, d] (row-major; the sketch runs along axis 0).  A CUDA tensor is
        sketched on the device (stream-ordered); a host array goes through spn_sketch_f32_host
        and the result comes back as a host array (newton_sketch.cpp:87-101)."""
        if self.is_exact():
            return columns
        if columns.shape[0] != self.input_dim:
            raise DimensionError("SketchOperator::apply: row count mismatch")
        return self._p.sketch(columns, self.m, self.norm, rows=self.row_list, out=out, stream=stream)


__all__ = [
    "SpinnerVariant", "SpinnerSpec", "StructuredSpinner", "StackedSpinner", "CrossPolytopeHasher",
    "MultiTableHasher", "make_hasher_factory", "signed_argmax", "decode_id", "KernelKind", "FeatureMap",
    "embed", "SketchOperator", "mix_seed", "sample_rows", "realize_block", "check_rows", "DimensionError", "DomainError",
    "fwht_normalized", "diag_matvec", "CirculantKind", "CirculantSpec", "CirculantOperator", "circulant_matvec",
    "toeplitz_matvec", "skew_circulant_matvec",
    "SpinnerError", "SingularSystemError", "variant_from_string", "all_variants", "structured_variants",
    "has_hadamard", "version", "LIB_PATH", "ABI_SYMBOLS",
    "LogisticProblem", "SketchConfig", "NewtonTrace", "loss", "gradient", "hessian_sqrt", "sketched_step", "solve",
    "generate_ar1_problem", "variant_to_string", "HashedPair", "CollisionCurve", "FamilyComparison", "collision_curve",
    "compare_families", "gram_exact", "gram_approx", "gram_error",
]

from .collision import (CollisionCurve, FamilyComparison, HashedPair, collision_curve,  # noqa: E402
                        compare_families)
from .newton import (LogisticProblem, NewtonTrace, SketchConfig, generate_ar1_problem, gradient,  # noqa: E402
                     hessian_sqrt, loss, sketched_step, solve)
from . import wire  # noqa: E402,F401  (result-table wire format of the reference CLI)
