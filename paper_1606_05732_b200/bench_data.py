"""Seeded synthetic inputs for the BASELINE configs, generated directly in HBM by libcgx's
generator kernels (csrc/datagen.cu) into torch-allocated device tensors.

The reference measures on no public dataset (BASELINE.json "published": {}); these
stand in with the configs' shapes and value distributions.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import CGX_F32, CGX_F64, CGX_ROW_MAJOR, CGX_COL_MAJOR, check, lib
from .api import context


def dense_normal(n: int, d: int, seed: int, dtype=None, layout: str = "row", device=None, row0: int = 0):
    """Rows [row0, row0+n) of an N(0,1) matrix with d columns (fp32 quantiles of
    SplitMix64 uniforms, entry (i, j) = draw i*d + j), row- or column-major."""
    import torch

    dtype = dtype or torch.float32
    ctx = context(device)
    dev = torch.device("cuda", ctx.device)
    if layout == "row":
        x = torch.empty((n, d), dtype=dtype, device=dev)
        lay = CGX_ROW_MAJOR
    else:
        x = torch.empty((d, n), dtype=dtype, device=dev).t()
        lay = CGX_COL_MAJOR
    dt = CGX_F32 if dtype == torch.float32 else CGX_F64
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream or 1)  # 1 = cudaStreamLegacy
    check(lib.cgx_gen_dense_normal(ctx.h, seed, row0, n, d, dt, lay, x.data_ptr(), stream))
    return x


def dense_normal_rows(rows, d: int, seed: int, dtype=None, device=None):
    """dense_normal's values for an arbitrary list of global rows (a CUDA int64 tensor, e.g.
    api.xform_rows of a bucket shard), row-major len(rows) x d."""
    import torch

    dtype = dtype or torch.float32
    ctx = context(device)
    dev = torch.device("cuda", ctx.device)
    rows = rows.to(device=dev, dtype=torch.int64).contiguous()
    n = rows.numel()
    x = torch.empty((n, d), dtype=dtype, device=dev)
    dt = CGX_F32 if dtype == torch.float32 else CGX_F64
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream or 1)
    check(lib.cgx_gen_dense_normal_rows(ctx.h, seed, rows.data_ptr(), n, d, dt, CGX_ROW_MAJOR, x.data_ptr(), stream))
    return x


def csr_zipf(n: int, d: int, seed: int, s_len: float = 1.5, cap: int = 512, s_col: float = 1.1, device=None):
    """Config-5 style heavy-tailed CSR (see cgx_gen_csr_zipf): Zipf(s_len) target row
    lengths capped at `cap`, Zipf(s_col)-skewed columns, fp32 N(0,1) values."""
    import torch

    from .api import SparseMatrix

    ctx = context(device)
    dev = torch.device("cuda", ctx.device)
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream or 1)  # 1 = cudaStreamLegacy
    rp = torch.empty(n + 1, dtype=torch.int64, device=dev)
    nnz = C.c_int64()
    check(lib.cgx_gen_csr_zipf(ctx.h, seed, n, d, s_len, cap, s_col, rp.data_ptr(), None, None, C.byref(nnz),
                               stream))
    cols = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)[: nnz.value]
    vals = torch.empty(max(nnz.value, 1), dtype=torch.float32, device=dev)[: nnz.value]
    check(lib.cgx_gen_csr_zipf(ctx.h, seed, n, d, s_len, cap, s_col, rp.data_ptr(), cols.data_ptr(),
                               vals.data_ptr(), None, stream))
    return SparseMatrix(n, d, rp, cols, vals)


def csr_bernoulli(n: int, d: int, density: float, seed: int, device=None):
    """CSR n x d, each entry present with probability `density` (sorted distinct columns,
    int32 columns, fp32 N(0,1) values, int64 row offsets).  Returns a SparseMatrix of
    device tensors."""
    import torch

    from .api import SparseMatrix

    ctx = context(device)
    dev = torch.device("cuda", ctx.device)
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream or 1)  # 1 = cudaStreamLegacy
    rp = torch.empty(n + 1, dtype=torch.int64, device=dev)
    nnz = C.c_int64()
    check(lib.cgx_gen_csr_bernoulli(ctx.h, seed, n, d, density, rp.data_ptr(), None, None, C.byref(nnz), stream))
    cols = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)[: nnz.value]
    vals = torch.empty(max(nnz.value, 1), dtype=torch.float32, device=dev)[: nnz.value]
    check(lib.cgx_gen_csr_bernoulli(ctx.h, seed, n, d, density, rp.data_ptr(), cols.data_ptr(), vals.data_ptr(),
                                    None, stream))
    return SparseMatrix(n, d, rp, cols, vals)


def separable_mixing(seed: int, r: int, cols: int, alpha: float = 0.5):
    """The config-4 mixing weights H (r x cols, fp64): Dirichlet(alpha) columns
    (cgx_separable_mixing; host only)."""
    h = np.empty((cols, r), np.float64)
    check(lib.cgx_separable_mixing(seed, r, cols, alpha, h.ctypes.data if h.size else None))
    return h.T


def dense_separable(n: int, d: int, seed: int, r: int = 16, alpha: float = 0.5, sigma: float = 0.01, dtype=None,
                    layout: str = "row", device=None, row0: int = 0):
    """Rows [row0, row0+n) of config 4's near-separable nonnegative X (BASELINE configs[3]):
    X = max(A.[I_r | H] + sigma*N(0,1), 0), A uniform on [0,1), H's columns Dirichlet(alpha).
    The anchor columns are 0..r-1."""
    import torch

    dtype = dtype or torch.float32
    ctx = context(device)
    dev = torch.device("cuda", ctx.device)
    if layout == "row":
        x = torch.empty((n, d), dtype=dtype, device=dev)
        lay = CGX_ROW_MAJOR
    else:
        x = torch.empty((d, n), dtype=dtype, device=dev).t()
        lay = CGX_COL_MAJOR
    dt = CGX_F32 if dtype == torch.float32 else CGX_F64
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream or 1)
    check(lib.cgx_gen_separable(ctx.h, seed, row0, n, d, r, alpha, sigma, dt, lay, x.data_ptr(), stream))
    return x
