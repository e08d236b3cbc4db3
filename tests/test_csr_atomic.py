"""The CSR record path (csrc/csr_atomic.cu, option csr_mode=3; the default for short-row CSR
of >= 4M nonzeros): bucket-range partitioned records + L2-resident fp64 atomics.  Its adds
into one (bucket, column) entry run in no fixed order, so S.X is checked against the oracle
within a floating-point bar rather than bit-for-bit:
  * S.X: relative Frobenius <= 1e-14, and every entry within 64 ulp of the entry's absolute
    sum of terms (|dS| <= 64 * eps * sum|s_i x_ij|);
  * Z = G.(S.X): relative Frobenius <= 1e-12 (the reference's own bar is 1e-8).
Shapes cover int32/int64 columns, B not a power of two, row shards (row0 > 0), empty rows,
tiles whose records overflow the shared-memory staging (long rows), one bucket, and d not a
power of two.  The gather (csr_mode=1) stays bit-exact on the same inputs."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps


@pytest.fixture
def mode3(cg):
    ctx = cg.context()
    ctx.set_option("csr_mode", 3)
    yield ctx
    ctx.set_option("csr_mode", 0)


def _csr(n, d, lens, seed, idx=np.int32):
    rng = np.random.default_rng(seed)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    cols = np.concatenate([np.sort(rng.choice(d, k, replace=False)) for k in lens] or [np.zeros(0)]).astype(idx)
    vals = rng.standard_normal(int(rp[-1])).astype(np.float32)
    return rp, cols, vals


def _check(cg, restatement, m, B, n, d, rp, cols, vals, seed=7, row0=0):
    from paper_1606_05732_b200 import SparseMatrix

    x = SparseMatrix(n, d, rp, cols, vals)
    if row0:
        t = cg.api.countgauss_new_shard(m, B, row0 + n, row0, n, oracle.draw(seed, 0))
    else:
        t = cg.countgauss_new(m, B, n, cg.SeededRng(seed))
    sx = cg.countsketch_apply(t, x)
    z = cg.countgauss_apply(t, x)
    _, cs, gs = restatement.countgauss_seeds(seed)
    h, s = restatement.hash_sign(cs, B, n, i0=row0)
    sx_ref = restatement.sketch_csr(h, s, B, rp, cols, vals, n, d)
    absx = restatement.sketch_csr(h, np.ones_like(s), B, rp, cols, np.abs(vals), n, d)
    assert np.linalg.norm(sx - sx_ref) <= 1e-14 * np.linalg.norm(sx_ref)
    assert np.all(np.abs(sx - sx_ref) <= 64 * EPS * absx)
    z_ref = restatement.gemm(restatement.gaussian(gs, m, B), sx_ref)
    assert np.linalg.norm(z - z_ref) <= 1e-12 * np.linalg.norm(z_ref)
    return sx, sx_ref


@pytest.mark.parametrize("idx", [np.int32, np.int64])
@pytest.mark.parametrize("B,d", [(4096, 256), (5003, 100), (1, 37), (65536, 1)])
def test_record_path_matches_oracle(cg, restatement, mode3, idx, B, d):
    n = 300000
    rng = np.random.default_rng(B + d)
    lens = np.minimum(rng.poisson(2.5, n), d)
    lens[::97] = 0  # empty rows
    lens[5000:5100] = 0  # a run of empty rows
    rp, cols, vals = _csr(n, d, lens, 1, idx)
    _check(cg, restatement, 16, B, n, d, rp, cols, vals)


def test_record_path_mixed_tiles(cg, restatement, mode3):
    """Tiles of 1024 rows around the staging limit (4096 records): some staged, some stored
    directly, and rows of a few hundred nonzeros."""
    n, d, B = 16 * 1024, 300, 3001
    rng = np.random.default_rng(8)
    lens = rng.integers(0, 8, n)
    lens[1024:2048] = 4  # exactly 4096 items: staged
    lens[2048:3072] = 4
    lens[2048] = 5  # 4097 items: direct
    lens[4096:4100] = 290  # rows spanning many bitmap words
    rp, cols, vals = _csr(n, d, lens, 3)
    _check(cg, restatement, 8, B, n, d, rp, cols, vals)


def test_record_path_long_rows_overflow_staging(cg, restatement, mode3):
    n, d, B = 20000, 4096, 2048
    rng = np.random.default_rng(3)
    lens = rng.integers(0, 12, n)
    lens[1000:1400] = 3000  # a tile with ~1.2M records: more than the staging area holds
    rp, cols, vals = _csr(n, d, lens, 2)
    _check(cg, restatement, 8, B, n, d, rp, cols, vals)


def test_record_path_row_shard(cg, restatement, mode3):
    n, d, B = 100000, 64, 1000
    rp, cols, vals = _csr(n, d, np.random.default_rng(5).integers(0, 6, n), 4)
    _check(cg, restatement, 8, B, n, d, rp, cols, vals, row0=123457)


def test_record_path_is_default_for_short_rows_and_gather_stays_exact(cg, restatement):
    """c3-like shape at reduced n: the default (record path) within the bar, the gather
    bit-exact."""
    from paper_1606_05732_b200 import bench_data

    n, d, B, m = 1 << 22, 256, 16384, 32
    x = bench_data.csr_bernoulli(n, d, 0.01, seed=11)
    rp, cols, vals = (a.cpu().numpy() for a in (x.row_offsets, x.col_indices, x.values))
    sx, sx_ref = _check(cg, restatement, m, B, n, d, rp, cols, vals, seed=9)
    ctx = cg.context()
    ctx.set_option("csr_mode", 1)
    try:
        t = cg.countgauss_new(m, B, n, cg.SeededRng(9))
        assert np.array_equal(cg.countsketch_apply(t, x).cpu().numpy(), sx_ref)
    finally:
        ctx.set_option("csr_mode", 0)


def test_record_path_key_all_ones(cg, restatement, mode3):
    """bucket bits + column bits = 32: the record of (bucket B-1, column d-1) has key
    0xffffffff, which must be added like any other (it once doubled as the accumulate's
    empty-slot sentinel).  S.X is 2^22 x 1024 (32 GB) and stays on the device."""
    import torch

    from paper_1606_05732_b200 import SparseMatrix

    n, d, B, seed = 200000, 1024, 1 << 22, 29  # seed 29: row 152986 hashes to bucket B-1
    _, cs, _ = restatement.countgauss_seeds(seed)
    h, s = restatement.hash_sign(cs, B, n)
    hot = np.flatnonzero(h == B - 1)
    if len(hot) == 0:
        pytest.skip("no row hashes to the last bucket for this seed")
    lens = np.random.default_rng(1).integers(0, 3, n)
    lens[hot] = 2
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    rng = np.random.default_rng(2)
    cols = np.concatenate([np.sort(rng.choice(d - 1, k, replace=False)) for k in lens]).astype(np.int32)
    cols[rp[hot] + 1] = d - 1  # every hot row's second nonzero in the last column
    vals = rng.standard_normal(int(rp[-1])).astype(np.float32)
    dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    x = SparseMatrix(n, d, dev(rp), dev(cols), dev(vals))
    t = cg.countgauss_new(4, B, n, cg.SeededRng(seed))
    sx = cg.countsketch_apply(t, x)
    want = 0.0
    for i in hot:  # ascending rows; one or two terms, so any order gives the same sum
        want += s[i] * float(vals[rp[i] + 1])
    assert float(sx[B - 1, d - 1]) == want
    del sx
    torch.cuda.empty_cache()
