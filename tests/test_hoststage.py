"""Host-input staging (csrc/hoststage.cu): pageable host arrays reach the device through a
ring of pinned 32 MiB chunks, with fp64 chunks whose values all round-trip through fp32 (and
int64 index chunks that fit int32) sent at half width.  Whatever the mix of narrowed and
full-width chunks, the device must see exactly the caller's values: S.X from host arrays is
checked bit-for-bit against S.X from the same values already on the device (and against the
oracle), including NaN / -0.0 / subnormal / non-fp32 values placed in later chunks, padded
(strided) column-major row blocks, and CSR with fp64 values."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _sx_host_and_device(cg, t, x):
    import torch

    sx_host = cg.countsketch_apply(t, x)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    sx_dev = cg.countsketch_apply(t, xd).cpu().numpy()
    return sx_host, sx_dev


def test_mixed_narrowed_and_full_width_chunks(cg, restatement):
    n, d, B = 600000, 16, 4096  # 76.8 MB of fp64: three 32 MiB chunks
    x = restatement.gen_dense_f32(41, n, d).astype(np.float64)  # every value fp32-exact
    x[300000, 5] = 1.0 / 3.0      # second chunk (row-major order) no longer narrows ...
    x[310000, 2] = np.nan         # ... nor would this
    x[10, 1] = -0.0               # first chunk still narrows: -0.0 keeps its sign
    t = cg.countgauss_new(8, B, n, cg.SeededRng(3))
    for arr in (np.ascontiguousarray(x), np.asfortranarray(x)):
        sx_h, sx_d = _sx_host_and_device(cg, t, arr)
        assert np.array_equal(sx_h, sx_d, equal_nan=True)
    _, cs, _ = restatement.countgauss_seeds(3)
    h, s = restatement.hash_sign(cs, B, n)
    assert np.array_equal(sx_h, restatement.sketch_dense(h, s, B, x), equal_nan=True)


def test_subnormal_and_signed_zero_values_survive(cg, restatement):
    n, d, B = 300000, 8, 1024
    rng = np.random.default_rng(5)
    x = rng.standard_normal((n, d))
    x[::7, 0] = -0.0
    x[::11, 1] = 5e-324          # subnormal fp64: sent at full width
    x[::13, 2] = np.float32(1e-40)  # subnormal fp32 value, exactly representable in fp32
    t = cg.countgauss_new(8, B, n, cg.SeededRng(4))
    sx_h, sx_d = _sx_host_and_device(cg, t, x)
    assert np.array_equal(sx_h, sx_d)


def test_padded_column_major_row_block(cg, restatement):
    """A row block of a larger column-major matrix (ld > rows): staged as its column
    segments, exactly."""
    n_all, d, B = 900000, 12, 2048
    big = np.asfortranarray(restatement.gen_dense_f32(43, n_all, d).astype(np.float64))
    r0, rows = 123457, 500000
    block = big[r0:r0 + rows]  # F-order view with ld = n_all
    assert not block.flags.f_contiguous and block.strides[0] == 8
    t = cg.countgauss_new(8, B, rows, cg.SeededRng(6))
    sx_h = cg.countsketch_apply(t, block)
    _, cs, _ = restatement.countgauss_seeds(6)
    h, s = restatement.hash_sign(cs, B, rows)
    assert np.array_equal(sx_h, restatement.sketch_dense(h, s, B, np.ascontiguousarray(block)))


@pytest.mark.parametrize("fp32_exact", [True, False])
def test_csr_host_fp64_values_and_int64_columns(cg, restatement, fp32_exact):
    n, d, B = 400000, 300, 8192
    rng = np.random.default_rng(7)
    lens = rng.integers(0, 20, n)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    cols = np.concatenate([np.sort(rng.choice(d, k, replace=False)) for k in lens]).astype(np.int64)
    vals = rng.standard_normal(int(rp[-1]))
    if fp32_exact:
        vals = vals.astype(np.float32).astype(np.float64)
    t = cg.countgauss_new(8, B, n, cg.SeededRng(8))
    sx = cg.countsketch_apply(t, cg.SparseMatrix(n, d, rp, cols, vals))
    _, cs, _ = restatement.countgauss_seeds(8)
    h, s = restatement.hash_sign(cs, B, n)
    assert np.array_equal(sx, restatement.sketch_csr(h, s, B, rp, cols, vals, n, d))
