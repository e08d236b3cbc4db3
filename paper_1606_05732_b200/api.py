"""Python mirror of the reference's CountGauss API, running on the B200 through libcgx.

Same names, argument meaning and error behaviour as the reference C++ library
(``/root/reference/proj/include/countgauss/{rng,sketch,nmf}.hpp``):

=====================================  ==============================================
reference (C++)                        here
=====================================  ==============================================
``SeededRng`` (rng.hpp:23-59)          :class:`SeededRng` (host-side seed plumbing)
``mix64`` (rng.hpp:12-17)              :func:`mix64`
``inverse_normal_cdf`` (rng.hpp:62)    :func:`inverse_normal_cdf` (GPU kernel)
``CountSketchMap`` (sketch.hpp:15-21)  :class:`CountSketchMap`
``countsketch_new`` (sketch.cpp:12)    :func:`countsketch_new`
``countsketch_injective`` (:30)        :func:`countsketch_injective`
``countsketch_apply`` x2 (:52, :68)    :func:`countsketch_apply`
``CountGaussTransform`` (:42-47)       :class:`CountGaussTransform`
``countgauss_new`` x2 (:115, :128)     :func:`countgauss_new`
``countgauss_apply`` x2 (:132, :136)   :func:`countgauss_apply`
``cg_nmf`` x2 (nmf.cpp:141-153)        :func:`cg_nmf` -> :class:`AnchorSet`
``SparseMatrix`` (matrix.hpp:45-61)    :class:`SparseMatrix`
=====================================  ==============================================

``std::invalid_argument`` surfaces as :class:`ValueError` with the reference's message.
Dense matrices are numpy arrays (host; results come back as numpy, column-major like the
reference's ``DenseMatrix``) or CUDA torch tensors (device-resident; results stay on the
device, stream-ordered on torch's current stream).  Every computation runs in libcgx's
sm_100a kernels; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field
from typing import Any, Optional

import numpy as np

from . import _lib
from ._lib import (CGX_COL_MAJOR, CGX_F32, CGX_F64, CGX_I32, CGX_I64, CGX_MEM_DEVICE, CGX_MEM_HOST,
                   CGX_ROW_MAJOR, check, lib)

GAMMA = 0x9E3779B97F4A7C15
_MASK = (1 << 64) - 1


# ----------------------------------------------------------------------------- RNG
def mix64(a: int, b: int) -> int:
    """Child-seed mixer (rng.hpp:12-17)."""
    return int(lib.cgx_mix64(a & _MASK, b & _MASK))


class SeededRng:
    """SplitMix64 stream (rng.hpp:23-59).  Host-side: it only carries seeds into the GPU."""

    kAlgorithm = "splitmix64/inverse-cdf-normal"

    def __init__(self, seed: int):
        self._seed = seed & _MASK
        self._state = seed & _MASK

    def seed(self) -> int:
        return self._seed

    def next_u64(self) -> int:
        self._state = (self._state + GAMMA) & _MASK
        z = self._state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def next_uniform(self) -> float:
        return ((self.next_u64() >> 11) + 0.5) * 2.0 ** -53

    def next_below(self, bound: int) -> int:
        return self.next_u64() % bound

    def next_normal(self) -> float:
        return inverse_normal_cdf(self.next_uniform())

    def split(self) -> "SeededRng":
        return SeededRng(self.next_u64())


# ------------------------------------------------------------------------- context
class Context:
    """One GPU: a libcgx context (stream, scratch, launch counter)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib.cgx_init(int(device), C.byref(h)))
        self.h = h
        self.device = int(device)

    def close(self):
        if self.h:
            lib.cgx_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(lib.cgx_launch_count(self.h))

    def set_option(self, key: str, value: int):
        check(lib.cgx_set_option(self.h, key.encode(), int(value)))

    def synchronize(self, stream=None):
        check(lib.cgx_synchronize(self.h, stream))

    def trim(self):
        """Release the scratch and pooled device memory kept between calls (cgx_trim)."""
        check(lib.cgx_trim(self.h))

    # profiling of stage 1 (sketch) / stage 2 (gemm) with CUDA events on the launch stream
    def profile(self, on: bool = True):
        check(lib.cgx_profile_enable(self.h, int(on)))

    def profile_read(self, stage: int):
        ms, n = C.c_double(), C.c_int64()
        check(lib.cgx_profile_read(self.h, stage, C.byref(ms), C.byref(n)))
        return ms.value, n.value


_ctx_lock = threading.Lock()
_contexts: dict[int, Context] = {}


def context(device: Optional[int] = None) -> Context:
    """The process-wide context of `device` (default: torch's current device, else 0)."""
    if device is None:
        device = 0
        try:
            import torch

            if torch.cuda.is_available():
                device = torch.cuda.current_device()
        except ImportError:
            pass
    with _ctx_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = _contexts[device] = Context(device)
        return ctx


def inverse_normal_cdf(p: float) -> float:
    """Standard normal quantile (rng.cpp:45-55), evaluated by the GPU kernel."""
    a = np.array([p], np.float64)
    out = np.empty(1, np.float64)
    check(lib.cgx_inverse_normal_cdf(context().h, a.ctypes.data, out.ctypes.data, 1, CGX_MEM_HOST, None))
    return float(out[0])


def inverse_normal_cdf_array(p: np.ndarray) -> np.ndarray:
    p = np.ascontiguousarray(p, np.float64)
    out = np.empty_like(p)
    check(lib.cgx_inverse_normal_cdf(context().h, p.ctypes.data, out.ctypes.data, p.size, CGX_MEM_HOST, None))
    return out


# ---------------------------------------------------------------------- transforms
class _Xform:
    """Owns one cgx_xform (freed when the last Python view goes away)."""

    def __init__(self, ctx: Context, h: C.c_void_p):
        self.ctx, self.h = ctx, h

    def __del__(self):
        try:
            lib.cgx_xform_free(self.h)
        except Exception:
            pass

    def info(self):
        t, ms, gs = C.c_uint64(), C.c_uint64(), C.c_uint64()
        m, B, n = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.cgx_xform_info(self.h, C.byref(t), C.byref(ms), C.byref(gs), C.byref(m), C.byref(B),
                                 C.byref(n)))
        return dict(t_seed=t.value, map_seed=ms.value, g_seed=gs.value, m=m.value, B=B.value, n=n.value)


class CountSketchMap:
    """buckets x input_dim CountSketch (sketch.hpp:15-21).  ``hash``/``sign`` are
    materialized from the GPU on first access; the apply kernels never need them."""

    def __init__(self, xf: _Xform):
        self._xf = xf
        inf = xf.info()
        self.buckets = inf["B"]
        self.input_dim = inf["n"]
        self.seed = inf["map_seed"]
        self._hash = self._sign = None

    @classmethod
    def from_arrays(cls, buckets: int, hash_, sign, ctx: Optional[Context] = None) -> "CountSketchMap":
        """A hand-built map (the reference fills the struct fields directly,
        test_sketch.cpp:72-78)."""
        ctx = ctx or context()
        hash_ = np.ascontiguousarray(hash_, np.int64)
        sign = np.ascontiguousarray(sign, np.float64)
        if hash_.shape != sign.shape:
            raise ValueError("countsketch map: hash and sign lengths differ")
        h = C.c_void_p()
        check(lib.cgx_countsketch_explicit(ctx.h, int(buckets), int(hash_.size), hash_.ctypes.data,
                                           sign.ctypes.data, CGX_MEM_HOST, C.byref(h)))
        return cls(_Xform(ctx, h))

    def _materialize(self):
        if self._hash is None:
            h = np.empty(self.input_dim, np.int64)
            s = np.empty(self.input_dim, np.float64)
            check(lib.cgx_fill_hash_sign(self._xf.ctx.h, self._xf.h, h.ctypes.data, s.ctypes.data,
                                         CGX_MEM_HOST, None))
            self._hash, self._sign = h, s

    @property
    def hash(self) -> np.ndarray:
        self._materialize()
        return self._hash

    @property
    def sign(self) -> np.ndarray:
        self._materialize()
        return self._sign


class CountGaussTransform:
    """T = G.S with G m x buckets (sketch.hpp:42-47).  G lives on the device (materialized by
    countgauss_new, like the reference's t.g); ``g`` copies it to the host on demand."""

    def __init__(self, xf: _Xform):
        self._xf = xf
        inf = xf.info()
        self.cs = CountSketchMap(xf)
        self.m = inf["m"]
        self.seed = inf["t_seed"]
        self._g = None

    @property
    def g(self) -> np.ndarray:
        if self._g is None:
            g = np.empty((self.cs.buckets, self.m), np.float64)  # col-major m x B
            check(lib.cgx_fill_gaussian(self._xf.ctx.h, self._xf.h, g.ctypes.data, CGX_MEM_HOST, None))
            self._g = g.T
        return self._g

    def materialize(self) -> np.ndarray:
        """T = G.S (m x n): the projection svm-check forms as gemm(t.g, materialize(t.cs))
        (tools/countgauss_main.cpp:660-668); column i is sign_i * G(:, hash_i)."""
        t = np.empty((self.cs.input_dim, self.m), np.float64)  # col-major m x n
        check(lib.cgx_countgauss_materialize(self._xf.ctx.h, self._xf.h, t.ctypes.data, CGX_MEM_HOST, None))
        return t.T


def countsketch_new(buckets: int, input_dim: int, rng: SeededRng, ctx: Optional[Context] = None) -> CountSketchMap:
    """sketch.cpp:12-28: map.seed = rng.next_u64(); hash/sign are index functions of it."""
    if buckets < 1 or input_dim < 1:
        raise ValueError("countsketch_new: buckets and input_dim must be >= 1")
    ctx = ctx or context()
    h = C.c_void_p()
    check(lib.cgx_countsketch_new(ctx.h, rng.next_u64(), int(buckets), int(input_dim), C.byref(h)))
    return CountSketchMap(_Xform(ctx, h))


def countsketch_injective(buckets: int, input_dim: int, rng: SeededRng,
                          ctx: Optional[Context] = None) -> CountSketchMap:
    """sketch.cpp:30-50 (distinct buckets; requires buckets >= input_dim)."""
    if buckets < input_dim:
        raise ValueError("countsketch_injective: needs buckets >= input_dim")
    ctx = ctx or context()
    h = C.c_void_p()
    check(lib.cgx_countsketch_injective(ctx.h, rng.next_u64(), int(buckets), int(input_dim), C.byref(h)))
    return CountSketchMap(_Xform(ctx, h))


def countgauss_new(m: int, *args, ctx: Optional[Context] = None) -> CountGaussTransform:
    """``countgauss_new(m, buckets, input_dim, rng)`` (sketch.cpp:115-126) or
    ``countgauss_new(m, input_dim, rng)`` with buckets = 5m (sketch.cpp:128-130)."""
    if len(args) == 3:
        buckets, input_dim, rng = args
    elif len(args) == 2:
        input_dim, rng = args
        buckets = 5 * m
    else:
        raise TypeError("countgauss_new(m, buckets, input_dim, rng) or countgauss_new(m, input_dim, rng)")
    if m < 1 or buckets < 1 or input_dim < 1:
        raise ValueError("countgauss_new: m, buckets and input_dim must be >= 1")
    ctx = ctx or context()
    h = C.c_void_p()
    check(lib.cgx_countgauss_new(ctx.h, rng.next_u64(), int(m), int(buckets), int(input_dim), C.byref(h)))
    return CountGaussTransform(_Xform(ctx, h))


def countgauss_new_shard(m: int, buckets: int, input_dim: int, row0: int, rows: int, t_seed: int,
                         ctx: Optional[Context] = None) -> CountGaussTransform:
    """Rows [row0, row0+rows) of the transform countgauss_new(m, buckets, input_dim, .)
    whose t.seed is `t_seed` (multi-GPU row sharding: every rank derives S and G from the
    shared seed -- the paper's seed sharing)."""
    if m < 1 or buckets < 1 or input_dim < 1:
        raise ValueError("countgauss_new: m, buckets and input_dim must be >= 1")
    ctx = ctx or context()
    h = C.c_void_p()
    check(lib.cgx_countgauss_new_shard(ctx.h, t_seed & _MASK, int(m), int(buckets), int(input_dim), int(row0),
                                       int(rows), C.byref(h)))
    return CountGaussTransform(_Xform(ctx, h))


def countgauss_bucket_shard(m: int, buckets: int, input_dim: int, b0: int, b1: int, t_seed: int,
                            ctx: Optional[Context] = None) -> CountGaussTransform:
    """Buckets [b0, b1) of countgauss_new(m, buckets, input_dim, .) with t.seed `t_seed`, as
    their own transform (hash-partitioned row placement, SURVEY 8e ablation C): its rows are
    the rows hashing into [b0, b1), in (bucket, row) order (``rows()``), its S.X is rows
    [b0, b1) of the full S.X and its G is G[:, b0:b1), so its apply is the split-K partial Z."""
    if m < 1 or buckets < 1 or input_dim < 1:
        raise ValueError("countgauss_new: m, buckets and input_dim must be >= 1")
    ctx = ctx or context()
    h = C.c_void_p()
    check(lib.cgx_countgauss_bucket_shard(ctx.h, t_seed & _MASK, int(m), int(buckets), int(input_dim), int(b0),
                                          int(b1), C.byref(h)))
    return CountGaussTransform(_Xform(ctx, h))


def xform_rows(t, device=None):
    """Global row index of each of the transform's rows (int64): numpy, or a CUDA tensor
    when `device` is given."""
    xf = (t.cs if isinstance(t, CountGaussTransform) else t)._xf
    n = xf.info()["n"]
    if device is not None:
        import torch

        rows = torch.empty(n, dtype=torch.int64, device=device)
        check(lib.cgx_xform_rows(xf.ctx.h, xf.h, rows.data_ptr(), CGX_MEM_DEVICE,
                                 C.c_void_p(torch.cuda.current_stream(rows.device).cuda_stream or 1)))
        return rows
    rows = np.empty(n, np.int64)
    check(lib.cgx_xform_rows(xf.ctx.h, xf.h, rows.ctypes.data, CGX_MEM_HOST, None))
    return rows


# ------------------------------------------------------------------------ matrices
def _to_host(a):
    if _is_torch(a):
        return a.detach().cpu().numpy()
    return np.asarray(a)


@dataclass
class SparseMatrix:
    """CSR matrix (matrix.hpp:45-61): int64 row offsets, column indices strictly
    increasing per row (int64 or int32), values (float64 or float32).  Arrays may be
    numpy (host) or CUDA torch tensors (device)."""

    rows: int
    cols: int
    row_offsets: Any
    col_indices: Any
    values: Any

    def nnz(self) -> int:
        return int(self.values.shape[0])

    @staticmethod
    def from_dense(x: np.ndarray, drop_tol: float = 0.0) -> "SparseMatrix":
        """SparseMatrix::from_dense (matrix.cpp:69-84)."""
        x = np.asarray(x, np.float64)
        mask = np.abs(x) > drop_tol
        rows, cols = np.nonzero(mask)
        counts = np.bincount(rows, minlength=x.shape[0])
        rp = np.zeros(x.shape[0] + 1, np.int64)
        np.cumsum(counts, out=rp[1:])
        return SparseMatrix(x.shape[0], x.shape[1], rp, cols.astype(np.int64), x[rows, cols])

    def save(self, path: str) -> None:
        """Write the binary CSR container (cgx_csr_save, include/cgx.h): the ingestion format
        that replaces the reference's text readers (io.cpp:72-136, 159-214)."""
        rp = np.ascontiguousarray(_to_host(self.row_offsets), np.int64)
        ci = np.ascontiguousarray(_to_host(self.col_indices))
        v = np.ascontiguousarray(_to_host(self.values))
        it = CGX_I32 if ci.dtype == np.int32 else CGX_I64
        if it == CGX_I64:
            ci = ci.astype(np.int64, copy=False)
        dt = CGX_F32 if v.dtype == np.float32 else CGX_F64
        if dt == CGX_F64:
            v = v.astype(np.float64, copy=False)
        check(lib.cgx_csr_save(os.fsencode(path), rp.ctypes.data, ci.ctypes.data, it, v.ctypes.data, dt, self.rows,
                               self.cols, v.shape[0]))

    @staticmethod
    def load(path: str, device=None, ctx: Optional[Context] = None) -> "SparseMatrix":
        """Read a binary CSR container; with `device` the arrays are streamed straight into
        HBM through pinned double buffers (cgx_csr_load) and come back as CUDA tensors."""
        n, d, nnz, it, dt = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int(), C.c_int()
        check(lib.cgx_csr_info(os.fsencode(path), C.byref(n), C.byref(d), C.byref(nnz), C.byref(it), C.byref(dt)))
        n, d, nnz = n.value, d.value, nnz.value
        if device is None:
            rp = np.empty(n + 1, np.int64)
            ci = np.empty(nnz, np.int32 if it.value == CGX_I32 else np.int64)
            v = np.empty(nnz, np.float32 if dt.value == CGX_F32 else np.float64)
            check(lib.cgx_csr_load(None, os.fsencode(path), rp.ctypes.data, ci.ctypes.data, v.ctypes.data,
                                   CGX_MEM_HOST, None))
            return SparseMatrix(n, d, rp, ci, v)
        import torch

        dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        ctx = ctx or context(dev.index if dev.index is not None else 0)
        rp = torch.empty(n + 1, dtype=torch.int64, device=dev)
        ci = torch.empty(nnz, dtype=torch.int32 if it.value == CGX_I32 else torch.int64, device=dev)
        v = torch.empty(nnz, dtype=torch.float32 if dt.value == CGX_F32 else torch.float64, device=dev)
        check(lib.cgx_csr_load(ctx.h, os.fsencode(path), rp.data_ptr(), ci.data_ptr(), v.data_ptr(), CGX_MEM_DEVICE,
                               _stream_of(v)))
        return SparseMatrix(n, d, rp, ci, v)

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.rows, self.cols), np.float64, order="F")
        rp = np.asarray(self.row_offsets)
        r = np.repeat(np.arange(self.rows), np.diff(rp))
        out[r, np.asarray(self.col_indices)] = np.asarray(self.values)
        return out


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _stream_of(x):
    """torch's current stream on x's device as a cudaStream_t.  torch's default stream is
    the legacy stream (handle 0); pass cudaStreamLegacy (0x1) for it, since a NULL stream
    means the context's own stream at the C-ABI."""
    import torch

    h = torch.cuda.current_stream(x.device).cuda_stream
    return C.c_void_p(h if h else 1)


def _dense_args(x):
    """(ptr, dtype, layout, ld, n, d, mem, keepalive, is_torch)."""
    if _is_torch(x):
        import torch

        if x.dim() != 2:
            raise ValueError("countsketch_apply: X must be a matrix")
        if x.dtype not in (torch.float32, torch.float64):
            x = x.to(torch.float64)
        if not x.is_cuda:
            x = x.numpy()
            return _dense_args(x)
        n, d = x.shape
        es = x.element_size()
        if x.stride(1) == 1 and (x.stride(0) >= max(d, 1) or n <= 1):
            layout, ld = CGX_ROW_MAJOR, max(x.stride(0), d, 1)
        elif x.stride(0) == 1 and (x.stride(1) >= max(n, 1) or d <= 1):
            layout, ld = CGX_COL_MAJOR, max(x.stride(1), n, 1)
        else:
            x = x.contiguous()
            layout, ld = CGX_ROW_MAJOR, max(d, 1)
        dt = CGX_F32 if x.dtype == torch.float32 else CGX_F64
        del es
        return x.data_ptr(), dt, layout, ld, n, d, CGX_MEM_DEVICE, x, True
    x = np.asarray(x)
    if x.ndim != 2:
        raise ValueError("countsketch_apply: X must be a matrix")
    if x.dtype not in (np.float32, np.float64):
        x = x.astype(np.float64)
    n, d = x.shape
    es = x.itemsize
    s0, s1 = x.strides
    if x.flags.c_contiguous:
        layout, ld = CGX_ROW_MAJOR, max(d, 1)
    elif x.flags.f_contiguous:
        layout, ld = CGX_COL_MAJOR, max(n, 1)
    elif s0 == es and s1 > 0 and s1 % es == 0 and s1 // es >= n:
        layout, ld = CGX_COL_MAJOR, s1 // es  # a row block of a column-major matrix: no copy
    elif s1 == es and s0 > 0 and s0 % es == 0 and s0 // es >= d:
        layout, ld = CGX_ROW_MAJOR, s0 // es  # a column block of a row-major matrix
    else:
        x = np.ascontiguousarray(x)
        layout, ld = CGX_ROW_MAJOR, max(d, 1)
    dt = CGX_F32 if x.dtype == np.float32 else CGX_F64
    return x.ctypes.data, dt, layout, ld, n, d, CGX_MEM_HOST, x, False


def _csr_args(x: SparseMatrix):
    if _is_torch(x.values) and x.values.is_cuda:
        import torch

        rp = x.row_offsets.to(torch.int64).contiguous()
        ci = x.col_indices
        if ci.dtype not in (torch.int32, torch.int64):
            ci = ci.to(torch.int64)
        ci = ci.contiguous()
        v = x.values
        if v.dtype not in (torch.float32, torch.float64):
            v = v.to(torch.float64)
        v = v.contiguous()
        return (rp.data_ptr(), ci.data_ptr(), CGX_I32 if ci.dtype == torch.int32 else CGX_I64, v.data_ptr(),
                CGX_F32 if v.dtype == torch.float32 else CGX_F64, CGX_MEM_DEVICE, (rp, ci, v), True)
    rp = np.ascontiguousarray(np.asarray(x.row_offsets), np.int64)
    ci = np.asarray(x.col_indices)
    if ci.dtype not in (np.int32, np.int64):
        ci = ci.astype(np.int64)
    ci = np.ascontiguousarray(ci)
    v = np.asarray(x.values)
    if v.dtype not in (np.float32, np.float64):
        v = v.astype(np.float64)
    v = np.ascontiguousarray(v)
    if rp.shape[0] != x.rows + 1:
        raise ValueError("SparseMatrix: row_offsets length must be rows+1")
    return (rp.ctypes.data, ci.ctypes.data, CGX_I32 if ci.dtype == np.int32 else CGX_I64, v.ctypes.data,
            CGX_F32 if v.dtype == np.float32 else CGX_F64, CGX_MEM_HOST, (rp, ci, v), False)


def _out(rows: int, cols: int, on_device: bool, like=None):
    """Column-major rows x cols float64 result (numpy F-order or a transposed torch view)."""
    if on_device:
        import torch

        buf = torch.empty((cols, rows), dtype=torch.float64, device=like.device)
        return buf.t(), buf.data_ptr()
    arr = np.empty((rows, cols), np.float64, order="F")
    return arr, arr.ctypes.data


def countsketch_apply(cs: CountSketchMap, x):
    """S.X (sketch.cpp:52-113): buckets x d, bit-identical to the reference."""
    if isinstance(cs, CountGaussTransform):
        cs = cs.cs
    xf = cs._xf
    if isinstance(x, SparseMatrix):
        rp, ci, it, v, dt, mem, keep, dev = _csr_args(x)
        out, optr = _out(cs.buckets, x.cols, dev, x.values)
        check(lib.cgx_countsketch_apply_csr(xf.ctx.h, xf.h, rp, ci, it, v, dt, x.rows, x.cols, x.nnz(), mem,
                                            optr, CGX_COL_MAJOR, mem, _stream_of(x.values) if dev else None))
        return out
    ptr, dt, layout, ld, n, d, mem, keep, dev = _dense_args(x)
    out, optr = _out(cs.buckets, d, dev, keep)
    check(lib.cgx_countsketch_apply_dense(xf.ctx.h, xf.h, ptr, dt, layout, ld, n, d, mem, optr, CGX_COL_MAJOR, mem,
                                          _stream_of(keep) if dev else None))
    return out


def countgauss_apply(t: CountGaussTransform, x):
    """Z = G.(S.X) (sketch.cpp:132-138): m x d."""
    xf = t._xf
    if isinstance(x, SparseMatrix):
        rp, ci, it, v, dt, mem, keep, dev = _csr_args(x)
        out, optr = _out(t.m, x.cols, dev, x.values)
        check(lib.cgx_countgauss_apply_csr(xf.ctx.h, xf.h, rp, ci, it, v, dt, x.rows, x.cols, x.nnz(), mem, optr,
                                           mem, _stream_of(x.values) if dev else None))
        return out
    ptr, dt, layout, ld, n, d, mem, keep, dev = _dense_args(x)
    out, optr = _out(t.m, d, dev, keep)
    check(lib.cgx_countgauss_apply_dense(xf.ctx.h, xf.h, ptr, dt, layout, ld, n, d, mem, optr, mem,
                                         _stream_of(keep) if dev else None))
    return out


def countgauss_apply_into(t: CountGaussTransform, x, z):
    """Device-resident countgauss_apply writing into a preallocated column-major m x d
    CUDA tensor `z` (e.g. ``torch.empty((d, m)).t()``) -- no allocation per call."""
    xf = t._xf
    assert z.stride(0) == 1 and z.shape[0] == t.m, "z must be column-major m x d"
    if isinstance(x, SparseMatrix):
        rp, ci, it, v, dt, mem, keep, dev = _csr_args(x)
        if not dev:
            raise ValueError("countgauss_apply_into: device inputs only")
        check(lib.cgx_countgauss_apply_csr(xf.ctx.h, xf.h, rp, ci, it, v, dt, x.rows, x.cols, x.nnz(), mem,
                                           z.data_ptr(), CGX_MEM_DEVICE, _stream_of(x.values)))
        return z
    ptr, dt, layout, ld, n, d, mem, keep, dev = _dense_args(x)
    if not dev:
        raise ValueError("countgauss_apply_into: device inputs only")
    check(lib.cgx_countgauss_apply_dense(xf.ctx.h, xf.h, ptr, dt, layout, ld, n, d, mem, z.data_ptr(),
                                         CGX_MEM_DEVICE, _stream_of(keep)))
    return z


def countsketch_apply_into(cs, x, sx):
    """Device-resident countsketch_apply writing into a preallocated CUDA tensor `sx`
    (buckets x d, row-major -- ``torch.empty((B, d))`` -- or column-major): the partial
    sketch a multi-GPU combine reduces."""
    if isinstance(cs, CountGaussTransform):
        cs = cs.cs
    xf = cs._xf
    if sx.stride(1) == 1 and sx.is_contiguous():
        out_layout = CGX_ROW_MAJOR
    elif sx.stride(0) == 1:
        out_layout = CGX_COL_MAJOR
    else:
        raise ValueError("countsketch_apply_into: sx must be row- or column-major")
    if isinstance(x, SparseMatrix):
        rp, ci, it, v, dt, mem, keep, dev = _csr_args(x)
        if not dev:
            raise ValueError("countsketch_apply_into: device inputs only")
        check(lib.cgx_countsketch_apply_csr(xf.ctx.h, xf.h, rp, ci, it, v, dt, x.rows, x.cols, x.nnz(), mem,
                                            sx.data_ptr(), out_layout, CGX_MEM_DEVICE, _stream_of(x.values)))
        return sx
    ptr, dt, layout, ld, n, d, mem, keep, dev = _dense_args(x)
    if not dev:
        raise ValueError("countsketch_apply_into: device inputs only")
    check(lib.cgx_countsketch_apply_dense(xf.ctx.h, xf.h, ptr, dt, layout, ld, n, d, mem, sx.data_ptr(), out_layout,
                                          CGX_MEM_DEVICE, _stream_of(keep)))
    return sx


def countsketch_apply_to(cs, x, bases, per: int):
    """countsketch_apply with the finished rows stored by bucket range into caller-supplied
    device destinations: bucket b's row goes to ``bases[b // per] + (b % per) * d`` (doubles).
    `bases` are device addresses (ints), e.g. this rank's slots in the other ranks' landing
    buffers (distributed.PeerLanding).  Device inputs; stream-ordered."""
    if isinstance(cs, CountGaussTransform):
        cs = cs.cs
    xf = cs._xf
    arr = (C.c_void_p * len(bases))(*bases)
    if isinstance(x, SparseMatrix):
        rp, ci, it, v, dt, mem, keep, dev = _csr_args(x)
        if not dev:
            raise ValueError("countsketch_apply_to: device inputs only")
        check(lib.cgx_countsketch_apply_csr_to(xf.ctx.h, xf.h, rp, ci, it, v, dt, x.rows, x.cols, x.nnz(), mem,
                                               arr, len(bases), per, _stream_of(x.values)))
        return
    ptr, dt, layout, ld, n, d, mem, keep, dev = _dense_args(x)
    if not dev:
        raise ValueError("countsketch_apply_to: device inputs only")
    check(lib.cgx_countsketch_apply_dense_to(xf.ctx.h, xf.h, ptr, dt, layout, ld, n, d, mem, arr, len(bases), per,
                                             _stream_of(keep)))


def sum_slots(ctx: Context, slots_ptr: int, nslots: int, stride: int, count: int, out):
    """out[i] = ((slot_0[i] + slot_1[i]) + ...) for i < count (rank order); `out` a CUDA tensor."""
    check(lib.cgx_sum_slots(ctx.h, C.c_void_p(slots_ptr), nslots, stride, count, C.c_void_p(out.data_ptr()),
                            _stream_of(out)))
    return out


def _sx_rows_args(sx):
    """Row-major float64 S.X (numpy or CUDA torch): (ptr, d, mem, keepalive, is_torch)."""
    if _is_torch(sx):
        import torch

        if not sx.is_cuda:
            return _sx_rows_args(sx.numpy())
        sx = sx.to(torch.float64).contiguous()
        return sx.data_ptr(), sx.shape[1], CGX_MEM_DEVICE, sx, True
    sx = np.ascontiguousarray(sx, dtype=np.float64)
    return sx.ctypes.data, sx.shape[1], CGX_MEM_HOST, sx, False


def gauss_gemm(t: CountGaussTransform, sx, z=None):
    """Stage 2 alone, Z = G . sx for a buckets x d S.X (numpy or CUDA torch, row- or
    column-major, packed); m x d column-major (into `z` when given).  With a column block
    of S.X this is the "cols" combine's split-N piece."""
    xf = t._xf
    if _is_torch(sx) and sx.is_cuda:
        import torch

        sx = sx.to(torch.float64)
        if sx.dim() != 2 or sx.shape[0] != t.cs.buckets:
            raise ValueError("gauss_gemm: sx must be buckets x d")
        if sx.stride(0) == 1 and sx.t().is_contiguous():
            layout = CGX_COL_MAJOR
        else:
            sx = sx.contiguous()
            layout = CGX_ROW_MAJOR
        mem, keep, dev = CGX_MEM_DEVICE, sx, True
        ptr = sx.data_ptr()
    else:
        sx = np.asarray(sx.numpy() if _is_torch(sx) else sx, dtype=np.float64)
        if sx.ndim != 2 or sx.shape[0] != t.cs.buckets:
            raise ValueError("gauss_gemm: sx must be buckets x d")
        if sx.flags.f_contiguous:
            layout = CGX_COL_MAJOR
        else:
            sx = np.ascontiguousarray(sx)
            layout = CGX_ROW_MAJOR
        mem, keep, dev = CGX_MEM_HOST, sx, False
        ptr = sx.ctypes.data
    d = sx.shape[1]
    if z is None:
        z, zptr = _out(t.m, d, dev, keep)
    else:
        zptr = z.data_ptr()
    check(lib.cgx_gauss_gemm(xf.ctx.h, xf.h, ptr, layout, d, mem, zptr, mem, _stream_of(keep) if dev else None))
    return z


def gauss_gemm_range(t: CountGaussTransform, sx_rows, b0: int, b1: int, z=None):
    """Split-K piece of stage 2 (the "sx" combine): G[:, b0:b1) . sx_rows for the row-major
    (b1-b0) x d slice of S.X; m x d column-major (into `z` when given)."""
    xf = t._xf
    ptr, d, mem, keep, dev = _sx_rows_args(sx_rows)
    if keep.shape[0] != b1 - b0:
        raise ValueError("gauss_gemm_range: sx_rows must have b1-b0 rows")
    if z is None:
        z, zptr = _out(t.m, d, dev, keep)
    else:
        zptr = z.data_ptr()
    check(lib.cgx_gauss_gemm_range(xf.ctx.h, xf.h, ptr, b0, b1, d, mem, zptr, mem,
                                   _stream_of(keep) if dev else None))
    return z


def gauss_gemm_rows(t: CountGaussTransform, sx, r0: int, r1: int, z=None):
    """Rows [r0, r1) of Z = G.(S.X) from the full row-major buckets x d S.X (the "g" combine:
    G's m rows split across ranks); (r1-r0) x d column-major (into `z` when given)."""
    xf = t._xf
    ptr, d, mem, keep, dev = _sx_rows_args(sx)
    if keep.shape[0] != t.cs.buckets:
        raise ValueError("gauss_gemm_rows: sx must be buckets x d")
    if z is None:
        z, zptr = _out(r1 - r0, d, dev, keep)
    else:
        zptr = z.data_ptr()
    check(lib.cgx_gauss_gemm_rows(xf.ctx.h, xf.h, ptr, d, r0, r1, mem, zptr, mem, _stream_of(keep) if dev else None))
    return z


# --------------------------------------------------------------------------- NMF
@dataclass
class AnchorSet:
    """nmf.hpp:38-46."""

    i_max: list = field(default_factory=list)
    i_min: list = field(default_factory=list)
    unioned: list = field(default_factory=list)
    tie_rows: int = 0

    def contains_all(self, wanted) -> bool:
        return all(w in self.unioned for w in wanted)

    def subset_of(self, allowed) -> bool:
        allowed = set(allowed)
        return all(u in allowed for u in self.unioned)


def select_extremes(z, ctx: Optional[Context] = None) -> AnchorSet:
    """Per-row argmax/argmin of Z (nmf.cpp:99-132) on the GPU; sorted-unique sets."""
    ctx = ctx or context()
    if _is_torch(z) and z.is_cuda:
        zz = z.t().contiguous().t() if not (z.stride(0) == 1) else z  # column-major
        m, d = zz.shape
        import torch

        amax = torch.empty(m, dtype=torch.int64, device=z.device)
        amin = torch.empty(m, dtype=torch.int64, device=z.device)
        ties = C.c_int64()
        check(lib.cgx_select_extremes(ctx.h, zz.data_ptr(), m, d, CGX_MEM_DEVICE, amax.data_ptr(), amin.data_ptr(),
                                      C.byref(ties), _stream_of(z)))
        amax, amin = amax.cpu().numpy(), amin.cpu().numpy()
    else:
        zz = np.asfortranarray(z, np.float64)
        m, d = zz.shape
        amax = np.empty(m, np.int64)
        amin = np.empty(m, np.int64)
        ties = C.c_int64()
        check(lib.cgx_select_extremes(ctx.h, zz.ctypes.data, m, d, CGX_MEM_HOST, amax.ctypes.data, amin.ctypes.data,
                                      C.byref(ties), None))
    i_max = sorted(set(int(a) for a in amax))
    i_min = sorted(set(int(a) for a in amin))
    return AnchorSet(i_max, i_min, sorted(set(i_max) | set(i_min)), int(ties.value))


def gaussian_project(x, m: int, rng: SeededRng, ctx: Optional[Context] = None):
    """Dense-Gaussian baseline Z = G~.X with G~ = gaussian_matrix(m, n, rng) (matrix.cpp:199-207,
    the product gp_nmf forms, nmf.cpp:155-159).  G~ is generated on the GPU in L2-sized
    chunks (never stored whole); rng advances by m*n draws exactly as in the reference.
    A SparseMatrix X takes the CSR kernel (the bench's naive loop; Z to rounding)."""
    if m < 1:
        raise ValueError("anchor extraction: m must be >= 1")
    ctx = ctx or context()
    if isinstance(x, SparseMatrix):  # the reference bench's O(nnz*m) loop (countgauss_main.cpp:535-547)
        rp, ci, it, v, dt, mem, keep, dev = _csr_args(x)
        out, optr = _out(m, x.cols, dev, x.values)
        check(lib.cgx_gaussian_project_csr(ctx.h, rng._state, int(m), rp, ci, it, v, dt, x.rows, x.cols, x.nnz(), mem,
                                           optr, mem, _stream_of(x.values) if dev else None))
        rng._state = (rng._state + m * x.rows * GAMMA) & _MASK
        return out
    ptr, dt, layout, ld, n, d, mem, keep, dev = _dense_args(x)
    if d < 1:
        raise ValueError("anchor extraction: X must have at least one column")
    out, optr = _out(m, d, dev, keep)
    check(lib.cgx_gaussian_project_dense(ctx.h, rng._state, int(m), ptr, dt, layout, ld, n, d, mem, optr, mem,
                                         _stream_of(keep) if dev else None))
    rng._state = (rng._state + m * n * GAMMA) & _MASK
    return out


def countsketch_batch_gram(u, buckets: int, trials: int, master: int, t0: int = 0, want_su: bool = False,
                           ctx: Optional[Context] = None):
    """distcheck's trial loop in one launch (distcheck.cpp:107-113): for t in [t0, t0+trials),
    map = countsketch_new(buckets, n, SeededRng(mix64(master, t))), su = S_t.U, gram(su).
    u: n x d float64 (host array or CUDA tensor).  Returns gram (trials x d x d) and, with
    want_su, su (trials x buckets x d) -- each trial's matrices in the reference layout,
    bit-identical to the reference."""
    import numpy as np

    ctx = ctx or context()
    if _is_torch(u) and u.is_cuda:
        import torch

        if u.dtype != torch.float64:
            raise ValueError("countsketch_batch_gram: U must be float64")
        ut = u.t().contiguous().t() if not (u.stride(0) == 1) else u  # column-major
        n, d = ut.shape
        ld = ut.stride(1) if d > 1 else n
        gram = torch.empty((trials, d, d), dtype=torch.float64, device=u.device)
        su = torch.empty((trials, d, buckets), dtype=torch.float64, device=u.device) if want_su else None
        check(lib.cgx_countsketch_batch_gram(ctx.h, master, t0, trials, buckets, ut.data_ptr(), ld, n, d, CGX_MEM_DEVICE,
                                             su.data_ptr() if want_su else None, gram.data_ptr(), CGX_MEM_DEVICE,
                                             _stream_of(ut)))
        gram = gram.transpose(1, 2)
        return (gram, su.transpose(1, 2)) if want_su else gram
    ua = np.asfortranarray(np.asarray(u, dtype=np.float64))
    n, d = ua.shape
    gram = np.empty((trials, d, d), dtype=np.float64)
    su = np.empty((trials, d, buckets), dtype=np.float64) if want_su else None
    check(lib.cgx_countsketch_batch_gram(ctx.h, master, t0, trials, buckets, ua.ctypes.data, n, n, d, CGX_MEM_HOST,
                                         su.ctypes.data if want_su else None, gram.ctypes.data, CGX_MEM_HOST, None))
    gram = gram.transpose(0, 2, 1)
    return (gram, su.transpose(0, 2, 1)) if want_su else gram


def gp_nmf(x, m: int, rng: SeededRng, ctx: Optional[Context] = None) -> AnchorSet:
    """Gaussian-projection anchor extraction (nmf.cpp:155-159): extremes of G~.X."""
    n, d = x.shape
    if m < 1:
        raise ValueError("anchor extraction: m must be >= 1")
    if d < 1:
        raise ValueError("anchor extraction: X must have at least one column")
    ctx = ctx or context()
    return select_extremes(gaussian_project(x, m, rng, ctx=ctx), ctx=ctx)


def cg_nmf(x, m: int, buckets: int, rng: SeededRng, ctx: Optional[Context] = None) -> AnchorSet:
    """CountGauss anchor extraction (nmf.cpp:141-153): Z = G.(S.X) with a fresh transform
    from rng, then per-row extremes.  buckets < 1 selects 5m."""
    if isinstance(x, SparseMatrix):
        n, d = x.rows, x.cols
    else:
        n, d = x.shape
    if m < 1:
        raise ValueError("anchor extraction: m must be >= 1")
    if d < 1:
        raise ValueError("anchor extraction: X must have at least one column")
    if buckets < 1:
        buckets = 5 * m
    t = countgauss_new(m, buckets, n, rng, ctx=ctx)
    return select_extremes(countgauss_apply(t, x), ctx=t._xf.ctx)
