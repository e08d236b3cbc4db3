"""Device groups (group.cu): the C-ABI multi-GPU path -- row shards built from the shared
seed, partials combined over NCCL (CGX_COMBINE_G / _SX / _Z) or over peer memory with the
reduce-scatter fused into the sketch kernels (CGX_COMBINE_P2P, second half of this file).  One
GPU is available to the tests.  The NCCL modes run on a one-rank group: the plumbing (NCCL
communicator, collectives, shard bookkeeping, host and device-sharded inputs) runs for real and
Z must equal the single-context apply within the Z bar; their multi-rank combine arithmetic is
covered on CPU by tests/test_distributed_cpu.py (gloo, world 2-4).  The peer-memory mode runs
with 1, 2 and 3 ranks that share device 0."""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_1606_05732_b200._lib import (CGX_COL_MAJOR, CGX_COMBINE_G, CGX_COMBINE_SX, CGX_COMBINE_Z, CGX_F32, CGX_F64,
                                        CGX_I32, CGX_I64, CGX_MEM_DEVICE, CGX_MEM_HOST, CGX_ROW_MAJOR, lib)

pytestmark = pytest.mark.gpu
Z_TOL = 1e-12
MODES = [CGX_COMBINE_G, CGX_COMBINE_SX, CGX_COMBINE_Z]


@pytest.fixture(scope="module")
def group(cg):
    g = C.c_void_p()
    devs = (C.c_int * 1)(0)
    assert lib.cgx_group_init(1, devs, C.byref(g)) == 0, lib.cgx_last_error()
    assert lib.cgx_group_size(g) == 1
    yield g
    assert lib.cgx_group_free(g) == 0


def _gx(group, m, B, n, seed):
    t = C.c_void_p()
    t_seed = oracle.draw(seed, 0)
    assert lib.cgx_group_countgauss_new(group, t_seed, m, B, n, C.byref(t)) == 0, lib.cgx_last_error()
    r0, rows = C.c_int64(), C.c_int64()
    assert lib.cgx_gxform_shard(t, 0, C.byref(r0), C.byref(rows)) == 0
    assert (r0.value, rows.value) == (0, n)
    return t


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("mode", MODES)
def test_group_dense_host_input(cg, group, restatement, mode):
    n, d, B, m, seed = 50000, 24, 4099, 20, 2024
    t = _gx(group, m, B, n, seed)
    x = restatement.gen_dense_f32(5, n, d).astype(np.float64)
    z_ref, _ = restatement.countgauss(seed, m, B, x=x)
    for arr, dt, lay in [(np.asfortranarray(x), CGX_F64, CGX_COL_MAJOR),
                         (np.ascontiguousarray(x.astype(np.float32)), CGX_F32, CGX_ROW_MAJOR)]:
        z = np.zeros((d, m), np.float64)  # column-major m x d
        ld = n if lay == CGX_COL_MAJOR else d
        rc = lib.cgx_group_countgauss_apply_dense(group, t, arr.ctypes.data, dt, lay, ld, n, d, CGX_MEM_HOST,
                                                  z.ctypes.data, CGX_MEM_HOST, mode)
        assert rc == 0, lib.cgx_last_error()
        assert rel(z.T, z_ref) <= Z_TOL
    assert lib.cgx_gxform_free(t) == 0


@pytest.mark.parametrize("mode", MODES)
def test_group_dense_device_shards(cg, group, mode):
    import torch

    from paper_1606_05732_b200 import bench_data

    n, d, B, m, seed = 1 << 20, 32, 65536, 64, 7
    t = _gx(group, m, B, n, seed)
    x = bench_data.dense_normal(n, d, seed=3)
    xs = (C.c_void_p * 1)(x.data_ptr())
    zd = torch.empty((d, m), dtype=torch.float64, device="cuda")
    zs = (C.c_void_p * 1)(zd.data_ptr())
    torch.cuda.synchronize()
    rc = lib.cgx_group_countgauss_apply_dense(group, t, xs, CGX_F32, CGX_ROW_MAJOR, d, n, d, CGX_MEM_DEVICE, zs,
                                              CGX_MEM_DEVICE, mode)
    assert rc == 0, lib.cgx_last_error()
    tt = cg.countgauss_new(m, B, n, cg.SeededRng(seed))
    z1 = cg.countgauss_apply(tt, x)
    torch.cuda.synchronize()
    assert (torch.linalg.norm(zd.t() - z1) / torch.linalg.norm(z1)).item() <= Z_TOL
    assert lib.cgx_gxform_free(t) == 0


@pytest.mark.parametrize("mode", MODES)
def test_group_csr_host_input(cg, group, restatement, mode):
    n, d, B, m, seed = 60000, 300, 5000, 16, 99
    t = _gx(group, m, B, n, seed)
    rng = np.random.default_rng(4)
    lens = rng.integers(0, 12, n)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    cols = np.concatenate([np.sort(rng.choice(d, k, replace=False)) for k in lens]).astype(np.int64)
    vals = rng.standard_normal(rp[-1])
    z_ref, _ = restatement.countgauss(seed, m, B, csr=(rp, cols, vals, d))
    for ci, it in [(cols, CGX_I64), (cols.astype(np.int32), CGX_I32)]:
        z = np.zeros((d, m), np.float64)
        rc = lib.cgx_group_countgauss_apply_csr(group, t, rp.ctypes.data, ci.ctypes.data, it, vals.ctypes.data, CGX_F64,
                                                n, d, int(rp[-1]), z.ctypes.data, CGX_MEM_HOST, mode)
        assert rc == 0, lib.cgx_last_error()
        assert rel(z.T, z_ref) <= Z_TOL
    assert lib.cgx_gxform_free(t) == 0


def test_group_errors(cg, group):
    t = _gx(group, 4, 64, 100, 1)
    x = np.zeros((100, 3))
    z = np.zeros((3, 4))
    assert lib.cgx_group_countgauss_apply_dense(group, t, x.ctypes.data, CGX_F64, CGX_ROW_MAJOR, 3, 100, 3,
                                                CGX_MEM_HOST, z.ctypes.data, CGX_MEM_HOST, 7) == 1
    assert lib.cgx_group_countgauss_apply_dense(group, t, x.ctypes.data, CGX_F64, CGX_ROW_MAJOR, 3, 99, 3,
                                                CGX_MEM_HOST, z.ctypes.data, CGX_MEM_HOST, CGX_COMBINE_G) == 1
    assert "rows" in lib.cgx_last_error().decode()
    bad = C.c_void_p()
    assert lib.cgx_group_init(0, None, C.byref(bad)) == 1
    assert lib.cgx_gxform_free(t) == 0


# ---- CGX_COMBINE_P2P: the reduce-scatter fused into the sketch kernels over peer memory ------
# One GPU here, so the ranks of these groups share device 0 (a device listed twice is allowed
# for this mode): every rank has its own context, stream, shard transform and landing buffers,
# and the "peer" pointers the kernels store through are plain local ones.  What runs is the
# real path: segmented stores from the gather kernels, the slot sums in rank order, the
# split-K stage 2 per bucket range, the Z exchange.  No kernel waits on another rank's kernel
# (the ranks' streams are ordered by events).
from paper_1606_05732_b200._lib import CGX_COMBINE_P2P  # noqa: E402


@pytest.fixture(scope="module", params=[1, 2, 3])
def pgroup(cg, request):
    P = request.param
    g = C.c_void_p()
    devs = (C.c_int * P)(*([0] * P))
    assert lib.cgx_group_init(P, devs, C.byref(g)) == 0, lib.cgx_last_error()
    assert lib.cgx_group_size(g) == P
    yield g, P
    assert lib.cgx_group_free(g) == 0


def _stats(g):
    f, c = C.c_int64(), C.c_int64()
    assert lib.cgx_group_stats(g, C.byref(f), C.byref(c)) == 0
    return f.value, c.value


def _pgx(g, m, B, n, seed):
    t = C.c_void_p()
    assert lib.cgx_group_countgauss_new(g, oracle.draw(seed, 0), m, B, n, C.byref(t)) == 0, lib.cgx_last_error()
    return t


@pytest.mark.parametrize("d", [24, 132, 130, 7])
def test_p2p_dense_host_input(cg, pgroup, restatement, d):
    g, P = pgroup
    n, B, m, seed = 50001, 4099, 20, 2024
    t = _pgx(g, m, B, n, seed)
    x = restatement.gen_dense_f32(5, n, d).astype(np.float64)
    z_ref, _ = restatement.countgauss(seed, m, B, x=x)
    f0, c0 = _stats(g)
    for arr, dt, lay in [(np.asfortranarray(x), CGX_F64, CGX_COL_MAJOR),
                         (np.ascontiguousarray(x.astype(np.float32)), CGX_F32, CGX_ROW_MAJOR)]:
        z = np.zeros((d, m), np.float64)
        ld = n if lay == CGX_COL_MAJOR else d
        rc = lib.cgx_group_countgauss_apply_dense(g, t, arr.ctypes.data, dt, lay, ld, n, d, CGX_MEM_HOST,
                                                  z.ctypes.data, CGX_MEM_HOST, CGX_COMBINE_P2P)
        assert rc == 0, lib.cgx_last_error()
        assert rel(z.T, z_ref) <= Z_TOL
    f1, c1 = _stats(g)
    # (the fp64 input holds fp32-representable values, so both travel and are sketched as fp32)
    # d = 24, 132: rows of whole 16 B pieces -> the cp.async gather stores into the peers' slots;
    # d = 130 (520 B rows) and d = 7 (sub-warp kernel): local S.X, then copies
    assert (f1 - f0, c1 - c0) == {24: (2 * P, 0), 132: (2 * P, 0), 130: (0, 2 * P), 7: (0, 2 * P)}[d]
    assert lib.cgx_gxform_free(t) == 0


def test_p2p_dense_device_shards_same_bits_on_every_rank(cg, pgroup):
    import torch

    from paper_1606_05732_b200 import bench_data

    g, P = pgroup
    n, d, B, m, seed = (1 << 20) + 5, 32, 65536, 64, 7
    t = _pgx(g, m, B, n, seed)
    x = bench_data.dense_normal(n, d, seed=3)
    shards = []
    for p in range(P):
        r0, rows = C.c_int64(), C.c_int64()
        assert lib.cgx_gxform_shard(t, p, C.byref(r0), C.byref(rows)) == 0
        shards.append(x[r0.value:r0.value + rows.value])
    xs = (C.c_void_p * P)(*[s.data_ptr() for s in shards])
    zd = [torch.empty((d, m), dtype=torch.float64, device="cuda") for _ in range(P)]
    zs = (C.c_void_p * P)(*[z.data_ptr() for z in zd])
    torch.cuda.synchronize()
    outs = []
    for _ in range(3):  # repeated: landing buffers are reused, the result must not move
        rc = lib.cgx_group_countgauss_apply_dense(g, t, xs, CGX_F32, CGX_ROW_MAJOR, d, n, d, CGX_MEM_DEVICE, zs,
                                                  CGX_MEM_DEVICE, CGX_COMBINE_P2P)
        assert rc == 0, lib.cgx_last_error()
        torch.cuda.synchronize()
        outs.append(zd[0].clone())
        for p in range(1, P):
            assert torch.equal(zd[p], zd[0])
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    tt = cg.countgauss_new(m, B, n, cg.SeededRng(seed))
    z1 = cg.countgauss_apply(tt, x)
    torch.cuda.synchronize()
    assert (torch.linalg.norm(zd[0].t() - z1) / torch.linalg.norm(z1)).item() <= Z_TOL
    assert lib.cgx_gxform_free(t) == 0


@pytest.mark.parametrize("shape", [
    (60000, 300, 5000, 16, 12, 0),     # lean gather: stores from sketch_csr_lean
    (60000, 40, 1000, 16, 12, 0),      # B.d <= 2^16: the chunked branch (local S.X + copies)
    (400000, 256, 8192, 128, 4, 3),    # the record path forced (local S.X + copies), tcgen05 stage 2
])
def test_p2p_csr_host_input(cg, pgroup, restatement, shape):
    g, P = pgroup
    n, d, B, m, maxlen, csr_mode = shape
    seed = 99
    t = _pgx(g, m, B, n, seed)
    for p in range(P):
        c = C.c_void_p()
        assert lib.cgx_group_context(g, p, C.byref(c)) == 0
        assert lib.cgx_set_option(c, b"csr_mode", csr_mode) == 0
    rng = np.random.default_rng(4)
    lens = rng.integers(0, maxlen, n)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    cols = rng.integers(0, d, rp[-1]).astype(np.int64)   # duplicates within a row allowed
    vals = rng.standard_normal(rp[-1]).astype(np.float32).astype(np.float64)  # (travels as fp32)
    z_ref, _ = restatement.countgauss(seed, m, B, csr=(rp, cols, vals, d))
    f0, c0 = _stats(g)
    for ci, it in [(cols, CGX_I64), (cols.astype(np.int32), CGX_I32)]:
        z = np.zeros((d, m), np.float64)
        rc = lib.cgx_group_countgauss_apply_csr(g, t, rp.ctypes.data, ci.ctypes.data, it, vals.ctypes.data, CGX_F64,
                                                n, d, int(rp[-1]), z.ctypes.data, CGX_MEM_HOST, CGX_COMBINE_P2P)
        assert rc == 0, lib.cgx_last_error()
        assert rel(z.T, z_ref) <= Z_TOL
    f1, c1 = _stats(g)
    assert (f1 - f0, c1 - c0) == ((2 * P, 0) if (B * d > 65536 and csr_mode == 0) else (0, 2 * P))
    for p in range(P):
        c = C.c_void_p()
        assert lib.cgx_group_context(g, p, C.byref(c)) == 0
        assert lib.cgx_set_option(c, b"csr_mode", 0) == 0
    assert lib.cgx_gxform_free(t) == 0


def test_p2p_more_ranks_than_buckets_and_nccl_modes_refused(cg, pgroup, restatement):
    g, P = pgroup
    n, d, B, m, seed = 3000, 20, 2, 5, 11   # B = 2 < P = 3: the last rank owns no bucket
    t = _pgx(g, m, B, n, seed)
    x = restatement.gen_dense_f32(9, n, d).astype(np.float64)
    z_ref, _ = restatement.countgauss(seed, m, B, x=x)
    z = np.zeros((d, m), np.float64)
    xr = np.ascontiguousarray(x)
    rc = lib.cgx_group_countgauss_apply_dense(g, t, xr.ctypes.data, CGX_F64, CGX_ROW_MAJOR, d, n, d, CGX_MEM_HOST,
                                              z.ctypes.data, CGX_MEM_HOST, CGX_COMBINE_P2P)
    assert rc == 0, lib.cgx_last_error()
    assert rel(z.T, z_ref) <= Z_TOL
    if P > 1:  # a device listed twice: NCCL has no communicator for it
        rc = lib.cgx_group_countgauss_apply_dense(g, t, xr.ctypes.data, CGX_F64, CGX_ROW_MAJOR, d, n, d, CGX_MEM_HOST,
                                                  z.ctypes.data, CGX_MEM_HOST, CGX_COMBINE_SX)
        assert rc != 0 and b"twice" in lib.cgx_last_error()
    assert lib.cgx_gxform_free(t) == 0
