"""GPU parity: the sm_100a path (through the C-ABI, via the Python mirror) against the
oracle on identical inputs.  Modeled on the reference's own tests (test_sketch.cpp,
test_rng.cpp, test_determinism.cpp, acceptance.cpp criteria 5/6).

Bars (stated here, checked below):
  * hash, sign, S.X (every dtype/layout/branch), anchors, tie_rows: bit-exact.
  * G: |G_gpu - G_ref| <= 1e-9 absolute and <= 1e-13 relative Frobenius (CUDA's erfc/exp/
    log are not glibc's; SURVEY.md 8c measured 1-4 ulp erfc changes move draws by <2e-10).
  * Z = G.(S.X): relative Frobenius <= 1e-12 (the reference's own bar is 1e-8,
    test_sketch.cpp:192-209, acceptance.cpp:146-164).
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

Z_TOL = 1e-12


@pytest.fixture(params=[1, 0], ids=["G-resident", "G-generated"])
def g_mode(request, cg):
    """Transforms built with G materialized at construction (the default, like the
    reference's CountGaussTransform::g) and with G generated inside the apply kernels."""
    ctx = cg.context()
    ctx.set_option("g_resident", request.param)
    yield request.param
    ctx.set_option("g_resident", 1)


def rel_fro(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = max(np.linalg.norm(b), 1e-300)
    return float(np.linalg.norm(a - b) / den)


# ------------------------------------------------------------------- construction
@pytest.mark.parametrize("m,B,n,seed", [(16, 2048, 65536, 12345), (3, 7, 1000, 31), (1, 1, 10, 1),
                                        (5, 1000003, 50000, 77), (4, 300, 123457, 2 ** 63 + 5)])
def test_hash_sign_bit_exact(cg, restatement, m, B, n, seed):
    t = cg.countgauss_new(m, B, n, cg.SeededRng(seed))
    ts, cs, gs = restatement.countgauss_seeds(seed)
    assert t.seed == ts and t.cs.seed == cs
    h, s = restatement.hash_sign(cs, B, n)
    assert np.array_equal(t.cs.hash, h)
    assert np.array_equal(t.cs.sign, s)


def test_single_bucket_and_default_buckets(cg):
    r = cg.SeededRng(1)
    one = cg.countsketch_new(1, 10, r)  # test_sketch.cpp:27-30
    assert np.all(one.hash == 0)
    t = cg.countgauss_new(4, 100, cg.SeededRng(32))  # B = 5m (test_sketch.cpp:187-189)
    assert t.cs.buckets == 20 and t.g.shape == (4, 20)
    a, b = cg.SeededRng(9), cg.SeededRng(9)
    m1, m2 = cg.countsketch_new(16, 100, a), cg.countsketch_new(16, 100, b)
    assert np.array_equal(m1.hash, m2.hash) and np.array_equal(m1.sign, m2.sign)


def test_countsketch_new_consumes_one_draw(cg, reference):
    m = cg.countsketch_new(37, 500, cg.SeededRng(4))
    ref = reference.countsketch_new(37, 500, 4)
    h, s = ref.hash_sign()
    assert m.seed == ref.cs_seed
    assert np.array_equal(m.hash, h) and np.array_equal(m.sign, s)


def test_hash_uniformity_and_sign_balance(cg):
    # test_sketch.cpp:51-70 (chi-square at 1 - 1e-6, Wilson-Hilferty threshold)
    B, n = 64, 100000
    mp = cg.countsketch_new(B, n, cg.SeededRng(12))
    counts = np.bincount(mp.hash, minlength=B)
    e = n / B
    chi2 = float(((counts - e) ** 2 / e).sum())
    z = cg.inverse_normal_cdf(1 - 1e-6)
    df = 63.0
    thr = df * (1 - 2 / (9 * df) + z * np.sqrt(2 / (9 * df))) ** 3
    assert chi2 < thr
    assert abs(mp.sign.sum()) < z * np.sqrt(n)


def test_injective_map(cg, reference):
    mp = cg.countsketch_injective(32, 10, cg.SeededRng(16))
    ref = reference.countsketch_injective(32, 10, 16)
    h, s = ref.hash_sign()
    assert np.array_equal(mp.hash, h) and np.array_equal(mp.sign, s)
    assert len(set(mp.hash.tolist())) == 10  # S^T S = I
    x = np.random.default_rng(0).standard_normal((10, 3))
    y = cg.countsketch_apply(mp, x)
    for i in range(10):
        assert np.array_equal(y[mp.hash[i]], mp.sign[i] * x[i])


# ------------------------------------------------------------------------------ G
@pytest.mark.parametrize("m,B,seed", [(16, 2048, 12345), (64, 65536, 12345), (7, 33, 5)])
def test_gaussian_within_tolerance(cg, restatement, m, B, seed, g_mode):
    t = cg.countgauss_new(m, B, 10, cg.SeededRng(seed))
    _, _, gs = restatement.countgauss_seeds(seed)
    ref = restatement.gaussian(gs, m, B)
    g = t.g
    assert np.abs(g - ref).max() <= 1e-9
    assert rel_fro(g, ref) <= 1e-13
    exact = float(np.mean(g == ref))
    print(f"G bit-exact fraction {exact:.3f}, max |dG| {np.abs(g - ref).max():.2e}")


def test_inverse_normal_cdf_known_quantiles(cg, golden):
    # test_rng.cpp:39-45
    assert abs(cg.inverse_normal_cdf(0.5)) <= 1e-12
    assert abs(cg.inverse_normal_cdf(0.975) - 1.959963984540054) <= 1e-10 * 1.96
    assert abs(cg.inverse_normal_cdf(0.0013498980316300945) + 3.0) <= 1e-9 * 3
    got = cg.inverse_normal_cdf_array(golden["quantile_p"])
    assert np.allclose(got, golden["quantile_x"], rtol=1e-13, atol=1e-13)
    for bad in (0.0, 1.0, -0.5, float("nan")):
        with pytest.raises(ValueError, match=r"\(0,1\)"):
            cg.inverse_normal_cdf(bad)


def test_inverse_normal_cdf_tails_and_region_edges(cg, restatement):
    # The device starts Halley from an fp32 Acklam value; the refined quantile must agree
    # with the reference's (fp64 Acklam start) to erfc resolution over the whole (0,1),
    # including the extreme draws uniform53 can produce and both sides of p_low.
    lo = 0.5 * 2.0 ** -53
    p = np.concatenate([
        np.array([lo, 3 * lo, 1e-15, 1e-12, 1e-9, 1e-6, 1e-3, 0.02425, np.nextafter(0.02425, 0),
                  np.nextafter(0.02425, 1), 0.3, 0.5 - 2 ** -40, 0.5, 0.5 + 2 ** -40, 0.97575,
                  np.nextafter(0.97575, 0), np.nextafter(0.97575, 1), 1 - 1e-6, 1 - 1e-9, 1 - 1e-12,
                  1 - 2.0 ** -52, 1 - 2.0 ** -53]),
        np.random.default_rng(3).random(4000),
        np.exp(-np.random.default_rng(4).uniform(0, 36, 2000)),
    ])
    got = cg.inverse_normal_cdf_array(p)
    ref = np.array([restatement.inverse_normal_cdf(float(v)) for v in p])
    # The reference's Halley residual e = 0.5*erfc(-x/sqrt2) - p is rounded at ulp(p), so
    # its own x is resolved only to ~ulp(p)/phi(x) (1e-10 near p = 1 - 1e-6): a different
    # start value may land anywhere inside that band.
    phi = np.exp(-0.5 * ref * ref) / np.sqrt(2 * np.pi)
    tol = 4e-15 + 1e-13 * np.abs(ref) + 4 * np.spacing(p) / phi
    excess = np.abs(got - ref) - tol
    assert np.all(excess <= 0), (float(p[np.argmax(excess)]), float(excess.max()))


def test_normal_moments(cg):
    # test_rng.cpp:23-37 on the GPU generator (1e6 draws)
    t = cg.countgauss_new(1000, 1000, 10, cg.SeededRng(2024))
    g = t.g.ravel()
    assert abs(g.mean()) < 5 / np.sqrt(g.size)
    assert abs(g.var() - 1) < 5 * np.sqrt(2 / g.size)


# ---------------------------------------------------------------------- dense S.X
def test_definition_case(cg):
    # test_sketch.cpp:72-92
    mp = cg.CountSketchMap.from_arrays(2, [0, 1, 0], [1.0, -1.0, 1.0])
    y = cg.countsketch_apply(mp, np.array([[1.0], [2.0], [3.0]]))
    assert y[0, 0] == 4.0 and y[1, 0] == -2.0
    assert np.abs(cg.countsketch_apply(mp, np.zeros((3, 4)))).max() == 0.0
    with pytest.raises(ValueError, match="X has 4 rows, sketch expects 3"):
        cg.countsketch_apply(mp, np.zeros((4, 1)))
    with pytest.raises(ValueError):
        cg.CountSketchMap.from_arrays(2, [0, 2, 0], [1.0, -1.0, 1.0])
    with pytest.raises(ValueError):
        cg.CountSketchMap.from_arrays(2, [0, 1, 0], [1.0, -0.5, 1.0])


def test_dense_golden(cg, golden, g_mode):
    n, d, B, m, seed = (int(v) for v in golden["dense_params"])
    t = cg.countgauss_new(m, B, n, cg.SeededRng(seed))
    x = golden["dense_x"]
    assert np.array_equal(cg.countsketch_apply(t, x), golden["dense_sx"])
    assert rel_fro(cg.countgauss_apply(t, x), golden["dense_z"]) <= Z_TOL


@pytest.mark.parametrize("d", [1, 2, 3, 5, 8, 13, 16, 17, 31, 32, 33, 64, 96, 100, 128, 130, 257])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("order", ["C", "F"])
def test_dense_bit_exact_shapes(cg, restatement, d, dtype, order):
    rng = np.random.default_rng(d * 7 + (dtype == np.float32))
    n, B, m = 3001, 97, 5
    x = np.asarray(rng.standard_normal((n, d)), dtype=dtype, order=order)
    seed = 1000 + d
    t = cg.countgauss_new(m, B, n, cg.SeededRng(seed))
    z_ref, sx_ref = restatement.countgauss(seed, m, B, x=x)
    assert np.array_equal(cg.countsketch_apply(t, x), sx_ref)
    assert rel_fro(cg.countgauss_apply(t, x), z_ref) <= Z_TOL


def test_integer_exactness_and_linearity(cg, reference):
    # test_sketch.cpp:94-127, acceptance.cpp:124-145
    rng = np.random.default_rng(13)
    for trial in range(50):
        n = int(rng.integers(2, 31))
        d = int(rng.integers(1, 31))
        B = int(rng.integers(1, 13))
        x = np.floor(11 * rng.uniform(size=(n, d))) - 5
        x[rng.uniform(size=(n, d)) >= 0.35] = 0
        seed = int(rng.integers(0, 2 ** 62))
        mp = cg.countsketch_new(B, n, cg.SeededRng(seed))
        ref = reference.countsketch_new(B, n, seed)
        slow = ref.materialized_sketch(x)
        assert np.array_equal(cg.countsketch_apply(mp, x), slow)
        sp = cg.SparseMatrix.from_dense(x)
        assert np.array_equal(cg.countsketch_apply(mp, sp), slow)
    mp = cg.countsketch_new(6, 20, cg.SeededRng(14))
    xa = np.floor(10 * rng.uniform(size=(20, 4))) - 4
    ya = np.floor(10 * rng.uniform(size=(20, 4))) - 4
    lhs = cg.countsketch_apply(mp, 3.0 * xa + ya)
    assert np.array_equal(lhs, 3.0 * cg.countsketch_apply(mp, xa) + cg.countsketch_apply(mp, ya))


def test_composite_vs_explicit(cg, reference):
    # test_sketch.cpp:192-209: |fast - (G.S).X| <= 1e-8 * max(1, max|slow|)
    rng = np.random.default_rng(18)
    for _ in range(20):
        n = 8 + int(rng.integers(0, 20))
        d = 1 + int(rng.integers(0, 6))
        x = rng.standard_normal((n, d)) * (rng.uniform(size=(n, d)) < 0.3)
        seed = int(rng.integers(0, 2 ** 62))
        t = cg.countgauss_new(2, 6, n, cg.SeededRng(seed))
        ref = reference.countgauss_new(2, 6, n, seed)
        h, s = ref.hash_sign()
        S = np.zeros((6, n))
        S[h, np.arange(n)] = s
        slow = (ref.g() @ S) @ x
        fast = cg.countgauss_apply(t, x)
        assert np.abs(fast - slow).max() <= 1e-8 * max(1.0, np.abs(slow).max())
    t = cg.countgauss_new(2, 5, 10, cg.SeededRng(3))
    assert np.abs(cg.countgauss_apply(t, cg.SparseMatrix.from_dense(np.zeros((10, 3))))).max() == 0.0


# ------------------------------------------------------------------------ CSR S.X
@pytest.mark.parametrize("case", ["csr", "chunk"])
def test_csr_golden(cg, golden, case):
    n, d, B, m, seed = (int(v) for v in golden[f"{case}_params"])
    t = cg.countgauss_new(m, B, n, cg.SeededRng(seed))
    x = cg.SparseMatrix(n, d, golden[f"{case}_rowptr"], golden[f"{case}_cols"], golden[f"{case}_vals"])
    assert np.array_equal(cg.countsketch_apply(t, x), golden[f"{case}_sx"])
    assert rel_fro(cg.countgauss_apply(t, x), golden[f"{case}_z"]) <= Z_TOL


def _random_csr(rng, n, d, density, idx, val):
    mask = rng.uniform(size=(n, d)) < density
    counts = mask.sum(1)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=rp[1:])
    r, c = np.nonzero(mask)
    v = rng.standard_normal(len(c)).astype(val)
    return rp, c.astype(idx), v


@pytest.mark.parametrize("n,d,B,density", [(5000, 256, 4099, 0.01), (3000, 7, 10, 0.5), (20000, 16, 80, 0.3),
                                           (1000, 600, 50, 0.2), (777, 40, 1, 0.1), (9000, 3, 2, 0.0)])
@pytest.mark.parametrize("idx", [np.int32, np.int64])
@pytest.mark.parametrize("val", [np.float32, np.float64])
def test_csr_bit_exact_shapes(cg, restatement, n, d, B, density, idx, val, g_mode):
    rng = np.random.default_rng(n + d + B)
    rp, c, v = _random_csr(rng, n, d, density, idx, val)
    seed = 17 + n
    t = cg.countgauss_new(6, B, n, cg.SeededRng(seed))
    z_ref, sx_ref = restatement.countgauss(seed, 6, B, csr=(rp, c, v, d))
    x = cg.SparseMatrix(n, d, rp, c, v)
    assert np.array_equal(cg.countsketch_apply(t, x), sx_ref)
    assert rel_fro(cg.countgauss_apply(t, x), z_ref) <= Z_TOL or np.abs(z_ref).max() == 0


def _csr_with_dups(rng, n, d, mean_len):
    """Rows of Poisson(mean_len) nonzeros with repeated and unsorted columns (legal CSR
    the reference accumulates in stored order)."""
    lens = rng.poisson(mean_len, n)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    c = rng.integers(0, d, int(rp[-1]))
    v = rng.standard_normal(int(rp[-1]))
    return rp, c, v


@pytest.mark.parametrize("n,d,B,mean_len,idx,val", [
    (60000, 256, 262144, 2.5, np.int32, np.float32),   # c3-like: B >> n/B, short rows
    (40000, 256, 4099, 2.5, np.int64, np.float64),
    (50000, 512, 1 << 16, 10.0, np.int32, np.float32),  # c5-like widths
    (30000, 1, 300, 1.0, np.int32, np.float64),
    (30000, 3, 70000, 2.0, np.int64, np.float32),
    (20000, 40, 5, 6.0, np.int32, np.float32),         # few buckets: long runs per bin
    (25000, 1000, 33333, 3.0, np.int32, np.float64),   # d not a power of two, padded slices
])
def test_csr_gather_bit_exact(cg, restatement, n, d, B, mean_len, idx, val):
    """The bucket-ordered row gather (csr_mode 1): S.X bit-exact against the oracle, including
    duplicate columns inside a row and empty rows (the record path, csr_mode 3, has its own
    tests in test_csr_atomic.py)."""
    rng = np.random.default_rng(n + d + B)
    rp, c, v = _csr_with_dups(rng, n, d, mean_len)
    c, v = c.astype(idx), v.astype(val)
    seed = 5 + d
    ctx = cg.context()
    ctx.set_option("csr_mode", 1)
    try:
        t = cg.countgauss_new(8, B, n, cg.SeededRng(seed))
        x = cg.SparseMatrix(n, d, rp, c, v)
        sx = cg.countsketch_apply(t, x)
        z = cg.countgauss_apply(t, x)
        # explicit map with the same hash/sign
        mp = cg.CountSketchMap.from_arrays(B, t.cs.hash, t.cs.sign)
        sx_explicit = cg.countsketch_apply(mp, x)
    finally:
        ctx.set_option("csr_mode", 0)
    z_ref, sx_ref = restatement.countgauss(seed, 8, B, csr=(rp, c, v, d))
    assert np.array_equal(sx, sx_ref)
    assert np.array_equal(sx_explicit, sx_ref)
    assert rel_fro(z, z_ref) <= Z_TOL


def test_csr_long_rows(cg, restatement):
    # heavy-tailed rows (config 5 shape): rows up to 2000 nnz
    rng = np.random.default_rng(3)
    n, d, B = 3000, 2048, 300
    lens = np.minimum((rng.pareto(0.8, n) + 1).astype(np.int64), d)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    cols = np.concatenate([np.sort(rng.choice(d, size=k, replace=False)) for k in lens]).astype(np.int32)
    vals = rng.standard_normal(rp[-1]).astype(np.float32)
    t = cg.countgauss_new(8, B, n, cg.SeededRng(5))
    z_ref, sx_ref = restatement.countgauss(5, 8, B, csr=(rp, cols, vals, d))
    assert np.array_equal(cg.countsketch_apply(t, cg.SparseMatrix(n, d, rp, cols, vals)), sx_ref)


def test_csr_zipf_config5_shape(cg, restatement):
    """Config-5 generator (heavy-tailed rows, skewed columns) at reduced n, full d/cap:
    CSR invariants, realized mean row length, S.X bit-exact, Z within tolerance."""
    from paper_1606_05732_b200 import bench_data

    n, d, B, m = 60000, 512, 4096, 32
    x = bench_data.csr_zipf(n, d, seed=99)
    rp = x.row_offsets.cpu().numpy()
    c = x.col_indices.cpu().numpy()
    v = x.values.cpu().numpy()
    lens = np.diff(rp)
    assert rp[0] == 0 and rp[-1] == len(c) and (lens >= 0).all() and lens.max() <= d
    for i in range(0, n, 997):  # sorted distinct columns within each row
        seg = c[rp[i]:rp[i + 1]]
        assert (np.diff(seg) > 0).all() and (seg >= 0).all() and (seg < d).all()
    assert abs(lens.mean() - 17.36) < 1.0  # E[L] of Zipf(1.5) on [1, 512]: rows hit L in expectation
    assert np.bincount(c, minlength=d)[:8].sum() > np.bincount(c, minlength=d)[-8:].sum()  # skewed columns
    t = cg.countgauss_new(m, B, n, cg.SeededRng(5))
    z_ref, sx_ref = restatement.countgauss(5, m, B, csr=(rp, c, v, d))
    assert np.array_equal(cg.countsketch_apply(t, x).cpu().numpy(), sx_ref)
    assert rel_fro(cg.countgauss_apply(t, x).cpu().numpy(), z_ref) <= Z_TOL


@pytest.fixture
def dmma_stage2(cg):
    """The DMMA stage 2 (large Z otherwise goes to the tensor-core path, ozgemm.cu)."""
    ctx = cg.context()
    ctx.set_option("oz_slices", 0)
    yield
    ctx.set_option("oz_slices", 7)


@pytest.mark.parametrize("m,d,B", [(96, 300, 20011), (256, 512, 40000), (130, 70, 9000), (64, 129, 33333),
                                   (128, 256, 30000)])
def test_stage2_large_z(cg, restatement, m, d, B, g_mode, dmma_stage2):
    """Stage 2 on its own (gemm(t.g, SX), matrix.cpp:111-129) for Z shapes that take the
    G-super-chunk + pipelined DMMA path, with G seeded (generated) and explicit."""
    import ctypes as C

    from paper_1606_05732_b200._lib import CGX_COL_MAJOR, CGX_MEM_HOST, check, lib

    rng = np.random.default_rng(m + d)
    sx = np.asfortranarray(rng.standard_normal((B, d)))
    t = cg.countgauss_new(m, B, 10, cg.SeededRng(m * d))
    _, _, gs = restatement.countgauss_seeds(m * d)
    G = restatement.gaussian(gs, m, B)
    ref = restatement.gemm(G, sx)
    ctx = cg.context()
    z = np.empty((m, d), np.float64, order="F")
    check(lib.cgx_gauss_gemm(ctx.h, t._xf.h, sx.ctypes.data, CGX_COL_MAJOR, d, CGX_MEM_HOST, z.ctypes.data,
                             CGX_MEM_HOST, None))
    assert rel_fro(z, ref) <= Z_TOL
    Gf = np.asfortranarray(G)
    check(lib.cgx_xform_set_gaussian_explicit(ctx.h, t._xf.h, m, Gf.ctypes.data, CGX_MEM_HOST))
    z2 = np.empty((m, d), np.float64, order="F")
    check(lib.cgx_gauss_gemm(ctx.h, t._xf.h, sx.ctypes.data, CGX_COL_MAJOR, d, CGX_MEM_HOST, z2.ctypes.data,
                             CGX_MEM_HOST, None))
    assert rel_fro(z2, ref) <= 1e-14


@pytest.fixture
def ozaki(cg):
    """Stage 2 on the tcgen05 int8 tensor cores (ozgemm.cu), S digit planes."""
    ctx = cg.context()

    def use(S, staged=1):
        ctx.set_option("oz_slices", S)
        ctx.set_option("oz_staged", staged)
        ctx.set_option("oz_min_z", 0)  # every Z shape, not only the large ones it is chosen for

    yield use
    ctx.set_option("oz_slices", 7)
    ctx.set_option("oz_staged", 1)
    ctx.set_option("oz_min_z", 16384)


# S = 7 planes of 8-bit balanced digits carry 54 bits per operand: Z to the DMMA path's bar.
# Fewer planes trade accuracy for speed; the bars below hold with 10x margin on Gaussian G.
OZ_TOL = {7: Z_TOL, 6: 1e-11, 5: 1e-8}


@pytest.mark.parametrize("m,d,B", [(96, 300, 20011), (256, 512, 40000), (130, 70, 9000), (64, 129, 33333),
                                   (128, 256, 30000), (1, 1, 37), (300, 1, 1000), (5, 66, 65)])
@pytest.mark.parametrize("S,staged", [(7, 1), (7, 0), (6, 1), (5, 1)])
def test_stage2_tensor_core_ozaki(cg, restatement, m, d, B, S, staged, ozaki):
    """Stage 2 (gemm(t.g, SX), matrix.cpp:111-129) through tcgen05.mma kind::i8 with FP64
    emulated by digit slicing: against the oracle's gemm, for resident seeded G and for an
    explicit G (whose cached digit image must be dropped when G is replaced)."""
    from paper_1606_05732_b200._lib import CGX_COL_MAJOR, CGX_MEM_HOST, check, lib

    ozaki(S, staged)
    rng = np.random.default_rng(m + d + B)
    sx = np.asfortranarray(rng.standard_normal((B, d)))
    sx[:, 0] = 0.0  # an all-zero column (scale 2^0, all digits 0)
    t = cg.countgauss_new(m, B, 10, cg.SeededRng(m * d + 1))
    _, _, gs = restatement.countgauss_seeds(m * d + 1)
    G = restatement.gaussian(gs, m, B)
    ctx = cg.context()
    z = np.empty((m, d), np.float64, order="F")
    for _ in range(2):  # second call reuses the transform's cached image of G
        check(lib.cgx_gauss_gemm(ctx.h, t._xf.h, sx.ctypes.data, CGX_COL_MAJOR, d, CGX_MEM_HOST, z.ctypes.data,
                                 CGX_MEM_HOST, None))
        assert rel_fro(z, restatement.gemm(G, sx)) <= OZ_TOL[S]
    G2 = np.asfortranarray(G * np.linspace(1e-3, 1e3, B)[None, :])  # new G, wide column range
    check(lib.cgx_xform_set_gaussian_explicit(ctx.h, t._xf.h, m, G2.ctypes.data, CGX_MEM_HOST))
    check(lib.cgx_gauss_gemm(ctx.h, t._xf.h, sx.ctypes.data, CGX_COL_MAJOR, d, CGX_MEM_HOST, z.ctypes.data,
                             CGX_MEM_HOST, None))
    assert rel_fro(z, restatement.gemm(G2, sx)) <= OZ_TOL[S]


@pytest.mark.parametrize("cluster,rs,st", [(1, 2, 0), (2, 2, 0), (4, 2, 0), (8, 6, 2), (2, 1, 4)])
def test_stage2_ozaki_cluster_and_rings(cg, restatement, cluster, rs, st, ozaki):
    """The tensor-core stage 2 with G's planes multicast across 1/2/4/8-CTA clusters and other
    ring depths: same Z (the partial sums do not depend on the launch shape's sharing)."""
    from paper_1606_05732_b200._lib import CGX_MEM_HOST, check, lib

    ozaki(7)
    ctx = cg.context()
    ctx.set_option("oz_cluster", cluster)
    ctx.set_option("oz_rs", rs)
    ctx.set_option("oz_st", st)
    try:
        m, d, B = 256, 512, 30011
        sx = np.random.default_rng(cluster).standard_normal((B, d))
        t = cg.countgauss_new(m, B, 10, cg.SeededRng(11))
        _, _, gs = restatement.countgauss_seeds(11)
        G = restatement.gaussian(gs, m, B)
        z = np.empty((m, d), order="F")
        check(lib.cgx_gauss_gemm_range(ctx.h, t._xf.h, np.ascontiguousarray(sx).ctypes.data, 0, B, d, CGX_MEM_HOST,
                                       z.ctypes.data, CGX_MEM_HOST, None))
        assert rel_fro(z, restatement.gemm(G, sx)) <= Z_TOL
    finally:
        ctx.set_option("oz_cluster", 2)
        ctx.set_option("oz_rs", 4)
        ctx.set_option("oz_st", 0)


@pytest.mark.parametrize("m,d,B", [(256, 512, 30011), (512, 64, 5000), (256, 70, 999)])
@pytest.mark.parametrize("S,staged", [(7, 1), (7, 0), (5, 1)])
def test_stage2_ozaki_mpair(cg, restatement, m, d, B, S, staged, ozaki):
    """M-tile pairs (option oz_mpair, the default for an even number of 128-row M tiles): each
    CTA of a pair converts half of every S.X tile and sends its half of the digit planes to the
    peer over DSMEM.  The digits and the integer products are the same, so Z is bit-identical
    to the unpaired kernel's, and within the bar of the oracle."""
    from paper_1606_05732_b200._lib import CGX_MEM_HOST, check, lib

    ozaki(S, staged)
    ctx = cg.context()
    sx = np.random.default_rng(m + d).standard_normal((B, d))
    sx[:, 1] *= 1e-200  # a column at the bottom of the scale range
    t = cg.countgauss_new(m, B, 10, cg.SeededRng(17))
    _, _, gs = restatement.countgauss_seeds(17)
    G = restatement.gaussian(gs, m, B)
    zs = []
    try:
        for mp in (0, 1):
            ctx.set_option("oz_mpair", mp)
            z = np.empty((m, d), order="F")
            check(lib.cgx_gauss_gemm_range(ctx.h, t._xf.h, np.ascontiguousarray(sx).ctypes.data, 0, B, d,
                                           CGX_MEM_HOST, z.ctypes.data, CGX_MEM_HOST, None))
            zs.append(z)
    finally:
        ctx.set_option("oz_mpair", 1)
    assert np.array_equal(zs[0], zs[1])
    assert rel_fro(zs[1], restatement.gemm(G, sx)) <= OZ_TOL[S]


@pytest.mark.parametrize("b0,b1", [(0, 4096), (64, 3000), (33, 4000), (4001, 4096)])
def test_stage2_ozaki_bucket_ranges(cg, restatement, b0, b1, ozaki):
    """Stage 2 over a bucket slice (the multi-GPU "sx" combine): aligned slices read the
    transform's cached digit image at a k-block offset, unaligned ones slice their own."""
    from paper_1606_05732_b200._lib import CGX_MEM_HOST, check, lib

    ozaki(7)
    m, d, B = 130, 70, 4096
    rng = np.random.default_rng(b0)
    sx = rng.standard_normal((B, d))
    t = cg.countgauss_new(m, B, 10, cg.SeededRng(99))
    _, _, gs = restatement.countgauss_seeds(99)
    G = restatement.gaussian(gs, m, B)
    ctx = cg.context()
    sl = np.ascontiguousarray(sx[b0:b1])
    z = np.empty((m, d), order="F")
    check(lib.cgx_gauss_gemm_range(ctx.h, t._xf.h, sl.ctypes.data, b0, b1, d, CGX_MEM_HOST, z.ctypes.data,
                                   CGX_MEM_HOST, None))
    assert rel_fro(z, restatement.gemm(np.asfortranarray(G[:, b0:b1]), sl)) <= Z_TOL


@pytest.mark.parametrize("r0,r1", [(0, 130), (64, 130), (3, 100)])
def test_stage2_ozaki_g_rows(cg, restatement, r0, r1, ozaki):
    """Rows [r0, r1) of Z (the multi-GPU "g" combine) through the tensor-core stage 2: the rows
    of G form a temporary view whose digit image is built per call, never cached on the
    transform (which keeps its own image of all of G)."""
    ozaki(7)
    m, d, B = 130, 200, 5000
    sx = np.random.default_rng(r0).standard_normal((B, d))
    t = cg.countgauss_new(m, B, 10, cg.SeededRng(7))
    _, _, gs = restatement.countgauss_seeds(7)
    G = restatement.gaussian(gs, m, B)
    zr = cg.api.gauss_gemm_rows(t, sx, r0, r1)
    assert rel_fro(zr, restatement.gemm(np.asfortranarray(G[r0:r1]), sx)) <= Z_TOL
    z = cg.api.gauss_gemm(t, sx)  # the full Z afterwards still uses the full G
    assert rel_fro(z, restatement.gemm(G, sx)) <= Z_TOL


def test_ozaki_full_apply_csr(cg, restatement, ozaki):
    """countgauss_apply on CSR X with stage 2 on the tensor cores: S.X stays bit-exact (the
    sketch is untouched) and Z meets the bar."""
    ozaki(7)
    rng = np.random.default_rng(5)
    n, d, B, m = 30000, 256, 4099, 128
    rp, c, v = _random_csr(rng, n, d, 0.02, np.int32, np.float32)
    t = cg.countgauss_new(m, B, n, cg.SeededRng(2024))
    x = cg.SparseMatrix(n, d, rp, c, v)
    z_ref, sx_ref = restatement.countgauss(2024, m, B, csr=(rp, c, v, d))
    assert np.array_equal(cg.countsketch_apply(t, x), sx_ref)
    assert rel_fro(cg.countgauss_apply(t, x), z_ref) <= Z_TOL
    # the gather's column maxima belong to its own call: a later stage 2 on other (larger)
    # S.X must compute its own scales
    cg.countsketch_apply(t, x)
    big = np.random.default_rng(6).standard_normal((B, d)) * 1e6
    _, _, gs = restatement.countgauss_seeds(2024)
    assert rel_fro(cg.api.gauss_gemm(t, big), restatement.gemm(restatement.gaussian(gs, m, B), big)) <= Z_TOL


@pytest.mark.parametrize("n,d,m,dtype", [(5000, 24, 16, np.float64), (70000, 32, 64, np.float32),
                                         (3000, 200, 40, np.float64)])
def test_dense_gaussian_projection(cg, restatement, n, d, m, dtype):
    """Dense-Gaussian baseline G~.X (gaussian_matrix(m, n, rng), matrix.cpp:199-207) vs the
    oracle, and the rng advancing by exactly m*n draws."""
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, d)).astype(dtype)
    r = cg.SeededRng(77)
    state0 = r._state
    z = cg.gaussian_project(x, m, r)
    G = restatement.gaussian(state0, m, n)  # draws of the stream continuing from state0
    ref = restatement.gemm(G, x.astype(np.float64))
    assert rel_fro(z, ref) <= Z_TOL
    assert r.next_u64() == oracle.draw(77, m * n)  # next draw after m*n normals


def test_gp_nmf_vs_reference(cg, reference):
    for trial in range(3):
        x = reference.generate_separable(80, 50, 6, 300 + trial)
        ref = reference.gp_nmf(reference.dense(x), 20, 400 + trial)
        got = cg.gp_nmf(np.asfortranarray(x), 20, cg.SeededRng(400 + trial))
        assert got.i_max == list(ref["i_max"]) and got.i_min == list(ref["i_min"])
        assert got.tie_rows == ref["tie_rows"]


# ------------------------------------------------------------------------- anchors
def test_cg_nmf_golden(cg, golden):
    a = cg.cg_nmf(np.asfortranarray(golden["nmf_x"]), 12, 60, cg.SeededRng(7006))
    assert a.i_max == list(golden["nmf_i_max"])
    assert a.i_min == list(golden["nmf_i_min"])
    assert a.unioned == list(golden["nmf_unioned"])
    assert a.tie_rows == int(golden["nmf_tie_rows"])


def test_select_extremes_ties_nan(cg, restatement):
    z = np.array([[1.0, 3.0, 3.0, 0.0], [2.0, 2.0, 1.0, 1.0], [np.nan, 5.0, -1.0, 2.0], [0.0, -0.0, 1.0, np.nan]])
    a = cg.select_extremes(z)
    e = restatement.select_extremes(z)
    assert a.i_max == list(e["i_max"]) and a.i_min == list(e["i_min"]) and a.tie_rows == e["tie_rows"]
    rng = np.random.default_rng(2)
    z = np.round(rng.standard_normal((300, 1000)), 1)  # many exact ties
    a = cg.select_extremes(z)
    e = restatement.select_extremes(z)
    assert a.i_max == list(e["i_max"]) and a.i_min == list(e["i_min"]) and a.tie_rows == e["tie_rows"]


def test_cg_nmf_random_vs_reference(cg, reference):
    rng = np.random.default_rng(8)
    for trial in range(5):
        x = reference.generate_separable(80, 50, 6, 100 + trial)
        ref = reference.cg_nmf(reference.dense(x), 20, 100, 200 + trial)
        got = cg.cg_nmf(np.asfortranarray(x), 20, 100, cg.SeededRng(200 + trial))
        assert got.i_max == list(ref["i_max"]) and got.i_min == list(ref["i_min"])
        assert got.tie_rows == ref["tie_rows"]


# -------------------------------------------------------------- device residency
def test_device_tensors_match_host(cg, restatement):
    import torch

    rng = np.random.default_rng(11)
    n, d, B, m = 20000, 32, 512, 16
    x = rng.standard_normal((n, d)).astype(np.float32)
    t = cg.countgauss_new(m, B, n, cg.SeededRng(99))
    xd = torch.from_numpy(x).cuda()
    sx_dev = cg.countsketch_apply(t, xd)
    z_dev = cg.countgauss_apply(t, xd)
    torch.cuda.synchronize()
    assert np.array_equal(sx_dev.cpu().numpy(), cg.countsketch_apply(t, x))
    assert np.array_equal(z_dev.cpu().numpy(), cg.countgauss_apply(t, x))
    # column-major device view
    xf = torch.from_numpy(np.asfortranarray(x)).cuda()
    xf = xf.t().contiguous().t()
    assert np.array_equal(cg.countsketch_apply(t, xf).cpu().numpy(), cg.countsketch_apply(t, x))
    rp, c, v = _random_csr(rng, n, d, 0.1, np.int32, np.float32)
    xs = cg.SparseMatrix(n, d, torch.from_numpy(rp).cuda(), torch.from_numpy(c).cuda(), torch.from_numpy(v).cuda())
    _, sx_ref = restatement.countgauss(99, m, B, csr=(rp, c, v, d))
    assert np.array_equal(cg.countsketch_apply(t, xs).cpu().numpy(), sx_ref)


@pytest.mark.parametrize("d,m,dtype", [(32, 64, np.float32), (24, 16, np.float32), (64, 32, np.float32),
                                       (128, 32, np.float32), (100, 8, np.float32), (32, 64, np.float64),
                                       (64, 64, np.float64), (40, 100, np.float32), (33, 5, np.float64)])
@pytest.mark.parametrize("mode", [1, 2])
def test_fused_matches_two_stage(cg, restatement, d, m, dtype, mode, g_mode):
    """The one-pass kernels (sketch + G + contraction; mode 1 all-warps, mode 2
    warp-specialized) vs the two-stage path and the oracle."""
    import torch

    rng = np.random.default_rng(d * 1000 + m)
    n, B = 40000, 777
    x = rng.standard_normal((n, d)).astype(dtype)
    t = cg.countgauss_new(m, B, n, cg.SeededRng(d + m))
    ctx = cg.context()
    xd = torch.from_numpy(x).cuda()
    ctx.set_option("fuse_mode", mode)
    ctx.set_option("fuse", 2)  # one-pass kernel even when G is resident
    try:
        z_fused = cg.countgauss_apply(t, xd).cpu().numpy()
        z_again = cg.countgauss_apply(t, xd).cpu().numpy()
    finally:
        ctx.set_option("fuse_mode", 2)
        ctx.set_option("fuse", 1)
    ctx.set_option("fuse", 0)
    try:
        z_two = cg.countgauss_apply(t, xd).cpu().numpy()
    finally:
        ctx.set_option("fuse", 1)
    z_ref, _ = restatement.countgauss(d + m, m, B, x=x)
    assert np.array_equal(z_fused, z_again)  # deterministic
    assert rel_fro(z_fused, z_ref) <= Z_TOL
    assert rel_fro(z_two, z_ref) <= Z_TOL
    assert rel_fro(z_fused, z_two) <= Z_TOL


@pytest.mark.parametrize("d,dtype,offset", [(32, np.float32, 0), (40, np.float32, 0), (100, np.float32, 0),
                                            (128, np.float32, 0), (256, np.float32, 0), (32, np.float64, 0),
                                            (64, np.float64, 0), (36, np.float32, 0), (32, np.float32, 1),
                                            (48, np.float64, 0)])
@pytest.mark.parametrize("stages", [0, 2, 3, 4])
def test_async_gather_ring(cg, restatement, d, dtype, offset, stages):
    """Row gather through the cp.async shared-memory ring (option async_stages) vs register
    batches (0): S.X bit-exact against the oracle for every ring depth and row width --
    partial last column chunks, and a misaligned base (offset) that must fall back -- and
    the one-pass Z deterministic and within tolerance."""
    import torch

    rng = np.random.default_rng(d * 10 + stages)
    n, B, m = 30000, 501, 16
    xfull = rng.standard_normal((n, d + offset)).astype(dtype)
    x = np.ascontiguousarray(xfull[:, offset:]) if offset == 0 else xfull[:, offset:]
    t = cg.countgauss_new(m, B, n, cg.SeededRng(d + 7))
    ctx = cg.context()
    xt = torch.from_numpy(xfull).cuda()
    xd = xt[:, offset:] if offset else xt
    ctx.set_option("async_stages", stages)
    try:
        sx = cg.countsketch_apply(t, xd).cpu().numpy()
        z1 = cg.countgauss_apply(t, xd).cpu().numpy()
        z2 = cg.countgauss_apply(t, xd).cpu().numpy()
    finally:
        ctx.set_option("async_stages", 2)
    z_ref, sx_ref = restatement.countgauss(d + 7, m, B, x=np.ascontiguousarray(x))
    assert np.array_equal(sx, sx_ref)
    assert np.array_equal(z1, z2)
    assert rel_fro(z1, z_ref) <= Z_TOL


def test_deterministic_across_runs(cg):
    rng = np.random.default_rng(12)
    x = rng.standard_normal((50000, 24))
    t = cg.countgauss_new(32, 1000, 50000, cg.SeededRng(1))
    z1 = cg.countgauss_apply(t, x)
    z2 = cg.countgauss_apply(t, x)
    t2 = cg.countgauss_new(32, 1000, 50000, cg.SeededRng(1))
    z3 = cg.countgauss_apply(t2, x)
    assert np.array_equal(z1, z2) and np.array_equal(z1, z3)


# ---------------------------------------------------- BASELINE config 2, full size
def test_config2_full_size_bit_exact(cg, restatement):
    """c2: n = 2^24 rows x 32 fp32, B = 65536, m = 64.  X generated on the GPU, copied to
    the host for the oracle; S.X bit-exact, Z within Z_TOL."""
    import torch

    from paper_1606_05732_b200 import bench_data

    n, d, B, m = 1 << 24, 32, 65536, 64
    x = bench_data.dense_normal(n, d, seed=oracle.mix64(12345, 2), dtype=torch.float32)
    t = cg.countgauss_new(m, B, n, cg.SeededRng(12345))
    sx = cg.countsketch_apply(t, x).cpu().numpy()
    z = cg.countgauss_apply(t, x).cpu().numpy()
    xh = x.cpu().numpy()
    del x
    z_ref, sx_ref = restatement.countgauss(12345, m, B, x=xh)
    assert np.array_equal(sx, sx_ref)
    assert rel_fro(z, z_ref) <= Z_TOL


# ------------------------------------------------------------- batched tiny sketches
@pytest.mark.parametrize("n,d,B,trials,t0", [(200, 5, 40, 64, 0), (1000, 20, 7, 33, 5), (77, 1, 1, 9, 0),
                                              (3000, 33, 300, 12, 100), (64, 3, 1000, 40, 7)])
def test_batch_sketch_gram_bit_exact(cg, reference, n, d, B, trials, t0):
    """distcheck's trial loop (distcheck.cpp:107-113) in one launch: every trial's S.U and
    gram(S.U) bit-identical to the reference's countsketch_new/countsketch_apply/gram,
    including the global-memory path (B*d > 1536) and a t0 offset."""
    import torch

    rng = np.random.default_rng(n + d + B)
    u = np.linalg.qr(rng.standard_normal((n, d)))[0] if n >= d else rng.standard_normal((n, d))
    master = 0xC0FFEE + n
    su_ref, g_ref = reference.sketch_gram_trials(master, t0, trials, B, u)
    g, su = cg.countsketch_batch_gram(u, B, trials, master, t0=t0, want_su=True)
    assert np.array_equal(su, su_ref)
    assert np.array_equal(g, g_ref)
    gd = cg.countsketch_batch_gram(torch.from_numpy(np.asfortranarray(u)).cuda(), B, trials, master, t0=t0)
    assert np.array_equal(gd.cpu().numpy(), g_ref)
    # chunking the trial range gives the same trials (seeds are mix64(master, t))
    g2 = cg.countsketch_batch_gram(u, B, trials - trials // 2, master, t0=t0 + trials // 2)
    assert np.array_equal(g2, g_ref[trials // 2:])


@pytest.mark.parametrize("n,d,m,density,idx,val", [(3000, 40, 16, 0.05, np.int32, np.float32),
                                                   (2000, 300, 70, 0.02, np.int64, np.float64),
                                                   (5000, 7, 33, 0.5, np.int32, np.float64)])
def test_gaussian_project_csr(cg, restatement, n, d, m, density, idx, val):
    """The config-5 ablation: dense-Gaussian G~.X for CSR X, against
    G~ = gaussian_matrix(m, n, rng) from the restatement times the densified X, and against
    the dense-input path on the same rng state; rng advances by m*n draws."""
    rng = np.random.default_rng(n + d + m)
    rp, c, v = _random_csr(rng, n, d, density, idx, val)
    x = cg.SparseMatrix(n, d, rp, c, v)
    r1 = cg.SeededRng(99)
    state0 = r1._state
    z = cg.gaussian_project(x, m, r1)
    G = restatement.gaussian(state0, m, n)
    xd = np.zeros((n, d))
    for i in range(n):
        xd[i, c[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    assert rel_fro(z, G @ xd) <= Z_TOL
    r2 = cg.SeededRng(99)
    zd = cg.gaussian_project(xd, m, r2)
    assert rel_fro(z, zd) <= Z_TOL
    assert r1._state == r2._state


@pytest.mark.parametrize("m,B,n,seed", [(8, 40, 300, 3), (16, 2048, 1000, 12345), (5, 1, 77, 9)])
def test_materialize_projection(cg, reference, m, B, n, seed, g_mode):
    """T = G.S as svm-check builds it, gemm(t.g, materialize(t.cs))
    (tools/countgauss_main.cpp:660-668), with the reference's own gemm and materialize over
    this transform's G: bit-identical."""
    t = cg.countgauss_new(m, B, n, cg.SeededRng(seed))
    T = t.materialize()
    ref = reference.xform_explicit(B, t.cs.hash, t.cs.sign, np.asfortranarray(t.g))
    s_mat = ref.materialized_sketch(np.eye(n))  # B x n
    assert np.array_equal(T, reference.gemm(t.g, s_mat))
    assert T.shape == (m, n)


def test_csr_streamed_device_load(cg, tmp_path):
    """cgx_csr_load into HBM through the pinned double buffer (files of several 32 MiB
    chunks): arrays identical to the saved ones, and S.X of the loaded matrix equals S.X of
    the in-memory one."""
    import torch

    rng = np.random.default_rng(5)
    n, d = 400000, 256
    lens = rng.poisson(20, n)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    c = rng.integers(0, d, int(rp[-1])).astype(np.int32)
    v = rng.standard_normal(int(rp[-1])).astype(np.float32)
    x = cg.SparseMatrix(n, d, rp, c, v)
    p = str(tmp_path / "big.cgxcsr")
    x.save(p)
    y = cg.SparseMatrix.load(p, device=0)
    torch.cuda.synchronize()
    assert y.values.is_cuda and y.col_indices.dtype == torch.int32
    assert np.array_equal(y.row_offsets.cpu().numpy(), rp)
    assert np.array_equal(y.col_indices.cpu().numpy(), c)
    assert np.array_equal(y.values.cpu().numpy(), v)
    t = cg.countgauss_new(16, 4096, n, cg.SeededRng(3))
    assert np.array_equal(cg.countsketch_apply(t, y).cpu().numpy(), cg.countsketch_apply(t, x))


def test_concurrent_calls_from_threads(cg, restatement):
    """The boundary is called from inside OpenMP regions (distcheck.cpp:107-111,
    acceptance.cpp:181-188): many host threads building transforms and applying them on
    one device at once must each get the serial result."""
    from concurrent.futures import ThreadPoolExecutor

    rng = np.random.default_rng(77)
    xs = [rng.standard_normal((3000, 7)) for _ in range(16)]

    def job(k):
        t = cg.countgauss_new(6, 97, 3000, cg.SeededRng(1000 + k))
        return cg.countsketch_apply(t, xs[k]), cg.countgauss_apply(t, xs[k])

    with ThreadPoolExecutor(max_workers=8) as ex:
        par = list(ex.map(job, range(16)))
    for k in range(16):
        z_ref, sx_ref = restatement.countgauss(1000 + k, 6, 97, x=xs[k])
        assert np.array_equal(par[k][0], sx_ref)
        assert rel_fro(par[k][1], z_ref) <= Z_TOL


@pytest.mark.parametrize("world", [2, 3, 8])
def test_row_shards_recompose(cg, restatement, world, g_mode):
    """The GPU side of the multi-GPU path, ranks emulated one after another on
    one device: each shard transform (cgx_countgauss_new_shard, global row indices from the
    shared seed) carries exactly the full transform's rows' hash/sign and G; the shards'
    S.X partials sum to S.X, their Z partials to Z ("z" combine); and stage 2 over bucket
    slices of the summed S.X (cgx_gauss_gemm_range, the "sx" combine) sums to Z as well."""
    import ctypes as C

    from paper_1606_05732_b200._lib import CGX_MEM_HOST, check, lib
    from paper_1606_05732_b200.distributed import bucket_range, shard_range

    n, d, B, m, seed = 20011, 24, 997, 12, 31337
    x = np.random.default_rng(world).standard_normal((n, d))
    full = cg.countgauss_new(m, B, n, cg.SeededRng(seed))
    t_seed = full.seed
    z_ref, sx_ref = restatement.countgauss(seed, m, B, x=x)
    sx_sum = np.zeros((B, d))
    z_sum = np.zeros((m, d))
    for rank in range(world):
        r0, r1 = shard_range(n, world, rank)
        t = cg.api.countgauss_new_shard(m, B, n, r0, r1 - r0, t_seed)
        assert np.array_equal(t.cs.hash, full.cs.hash[r0:r1]) and np.array_equal(t.cs.sign, full.cs.sign[r0:r1])
        assert np.array_equal(t.g, full.g)
        sx_sum += cg.countsketch_apply(t, x[r0:r1])
        z_sum += cg.countgauss_apply(t, x[r0:r1])
    assert rel_fro(sx_sum, sx_ref) <= 1e-14
    assert rel_fro(z_sum, z_ref) <= Z_TOL
    z_sx = np.zeros((m, d))
    ctx = cg.context()
    for rank in range(world):
        b0, b1 = bucket_range(B, world, rank)
        sl = np.ascontiguousarray(sx_sum[b0:b1])  # row-major (b1-b0) x d slice
        zp = np.empty((m, d), order="F")
        check(lib.cgx_gauss_gemm_range(ctx.h, full._xf.h, sl.ctypes.data, b0, b1, d, CGX_MEM_HOST, zp.ctypes.data,
                                       CGX_MEM_HOST, None))
        z_sx += zp
    assert rel_fro(z_sx, z_ref) <= Z_TOL
    # "g" combine: G's m rows split over ranks, each block from the summed S.X
    from paper_1606_05732_b200.distributed import g_row_range

    z_g = np.zeros((m, d))
    for rank in range(world):
        g0, g1 = g_row_range(m, world, rank)
        if g1 > g0:
            z_g[g0:g1] = cg.api.gauss_gemm_rows(full, sx_sum, g0, g1)
    assert rel_fro(z_g, z_ref) <= Z_TOL
    # and the device-resident path with a row-major torch S.X
    import torch

    sx_dev = torch.from_numpy(np.ascontiguousarray(sx_sum)).cuda()
    g0, g1 = g_row_range(m, world, 1)  # non-empty for every world here (m=12)
    zr = cg.api.gauss_gemm_rows(full, sx_dev, g0, g1)
    torch.cuda.synchronize()
    assert rel_fro(zr.cpu().numpy(), z_g[g0:g1]) <= 1e-15
    # "cols" combine: column blocks of S.X through stage 2 (split-N), host and device
    z_c = np.zeros((m, d))
    for rank in range(world):
        per = (d + world - 1) // world
        c0, c1 = min(d, rank * per), min(d, rank * per + per)
        if c1 > c0:
            z_c[:, c0:c1] = cg.api.gauss_gemm(full, np.asfortranarray(sx_sum[:, c0:c1]))
    assert rel_fro(z_c, z_ref) <= Z_TOL
    sxT = torch.from_numpy(np.ascontiguousarray(sx_sum.T)).cuda()  # (d, B): S.X column-major
    zc_dev = cg.api.gauss_gemm(full, sxT[: d // 2].t())
    torch.cuda.synchronize()
    assert np.array_equal(zc_dev.cpu().numpy(), z_c[:, : d // 2]) or rel_fro(zc_dev.cpu().numpy(), z_c[:, : d // 2]) <= 1e-15
    with pytest.raises(Exception):
        cg.api.gauss_gemm_rows(full, sx_sum, 3, 3)
    with pytest.raises(Exception):
        cg.api.gauss_gemm_rows(full, sx_sum, 0, m + 1)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_bucket_shards_hash_placement(cg, restatement, world):
    """SURVEY 8e ablation C (hash-partitioned row placement): the bucket-range transform
    (cgx_countgauss_bucket_shard) holds exactly the rows hashing into [b0, b1) in (bucket,
    row) order, its hash/sign/G are the full transform's restricted to them, its S.X of
    X[rows] is rows [b0, b1) of the full S.X bit-for-bit, and the shards' applies sum to Z."""
    import torch

    from paper_1606_05732_b200 import bench_data
    from paper_1606_05732_b200.distributed import bucket_range

    n, d, B, m, seed = 30011, 20, 1009, 12, 777
    x = np.random.default_rng(world).standard_normal((n, d))
    full = cg.countgauss_new(m, B, n, cg.SeededRng(seed))
    z_ref, sx_ref = restatement.countgauss(seed, m, B, x=x)
    h_full, s_full, g_full = full.cs.hash, full.cs.sign, full.g
    z_sum = np.zeros((m, d))
    seen = []
    for rank in range(world):
        b0, b1 = bucket_range(B, world, rank)
        t = cg.api.countgauss_bucket_shard(m, B, n, b0, b1, full.seed)
        rows = cg.api.xform_rows(t)
        want = np.nonzero((h_full >= b0) & (h_full < b1))[0]
        want = want[np.lexsort((want, h_full[want]))]  # (bucket, row) order
        assert np.array_equal(rows, want)
        seen.append(rows)
        assert t.cs.buckets == b1 - b0 and t.cs.input_dim == len(rows)
        assert np.array_equal(t.cs.hash, h_full[rows] - b0) and np.array_equal(t.cs.sign, s_full[rows])
        assert np.array_equal(t.g, g_full[:, b0:b1])
        xs = np.ascontiguousarray(x[rows])
        assert np.array_equal(cg.countsketch_apply(t, xs), sx_ref[b0:b1])
        z_sum += cg.countgauss_apply(t, xs)
        # the same rows, generated on the device from their global indices
        rows_dev = cg.api.xform_rows(t, device="cuda")
        xg = bench_data.dense_normal_rows(rows_dev, 8, seed=99)
        xa = bench_data.dense_normal(n, 8, seed=99)
        torch.cuda.synchronize()
        assert torch.equal(xg, xa[rows_dev])
    assert np.array_equal(np.sort(np.concatenate(seen)), np.arange(n))
    assert rel_fro(z_sum, z_ref) <= Z_TOL
    with pytest.raises(ValueError):
        cg.api.countgauss_bucket_shard(m, B, n, 5, 5, full.seed)
    with pytest.raises(ValueError):
        cg.api.countgauss_bucket_shard(m, B, n, 0, B + 1, full.seed)


@pytest.mark.parametrize("cfg", ["c3", "c4", "c5"])
def test_full_size_checksums(cg, cfg):
    """BASELINE configs c3/c4/c5 at FULL size (too large for the CPU oracle), through
    size-independent exact properties.  X is made integer-valued (rounded 8x the config's
    values) so every fp64 sum below is exact whatever its order:
      * per bucket: sum_j SX[b, j] == sum_{i: h(i)=b} s_i * sum_j X[i, j]   (all B buckets)
      * dense c4, per column: sum_b SX[b, j] == sum_i s_i X[i, j]
    and Z matches G @ SX (cuBLAS fp64) within 1e-12 relative Frobenius."""
    import ctypes as C

    import torch

    from paper_1606_05732_b200 import bench_data
    from paper_1606_05732_b200._lib import CGX_MEM_DEVICE, check, lib

    cfgs = {"c3": dict(n=1 << 26, d=256, B=262144, m=128), "c4": dict(n=1 << 25, d=128, B=131072, m=32),
            "c5": dict(n=1 << 27, d=512, B=1 << 20, m=256)}
    c = cfgs[cfg]
    n, d, B, m = c["n"], c["d"], c["B"], c["m"]
    t = cg.countgauss_new(m, B, n, cg.SeededRng(12345))
    dev = torch.device("cuda")
    h = torch.empty(n, dtype=torch.int64, device=dev)
    s = torch.empty(n, dtype=torch.float64, device=dev)
    check(lib.cgx_fill_hash_sign(t._xf.ctx.h, t._xf.h, h.data_ptr(), s.data_ptr(), CGX_MEM_DEVICE, C.c_void_p(1)))
    if cfg == "c4":
        x = bench_data.dense_normal(n, d, seed=oracle.mix64(12345, 4))
        x.mul_(8).round_()
        rowsum = torch.empty(n, dtype=torch.float64, device=dev)
        colsum = torch.zeros(d, dtype=torch.float64, device=dev)
        step = 1 << 22
        for r0 in range(0, n, step):
            blk = x[r0:r0 + step].double()
            rowsum[r0:r0 + step] = blk.sum(1)
            colsum += (blk * s[r0:r0 + step, None]).sum(0)
            del blk
    else:
        if cfg == "c3":
            x = bench_data.csr_bernoulli(n, d, 0.01, seed=oracle.mix64(12345, 3))
        else:
            x = bench_data.csr_zipf(n, d, seed=oracle.mix64(12345, 5))
        x.values.mul_(8).round_()
        cs = torch.zeros(x.nnz() + 1, dtype=torch.float64, device=dev)
        torch.cumsum(x.values.double(), 0, out=cs[1:])
        rowsum = cs[x.row_offsets[1:]] - cs[x.row_offsets[:-1]]
        del cs
        colsum = None
    torch.cuda.synchronize()
    sx = cg.countsketch_apply(t, x)  # B x d column-major view
    want = torch.zeros(B, dtype=torch.float64, device=dev).index_add_(0, h, s * rowsum)
    assert torch.equal(sx.sum(1), want)
    if colsum is not None:
        assert torch.equal(sx.sum(0), colsum)
    z = cg.countgauss_apply(t, x)
    g = torch.empty((B, m), dtype=torch.float64, device=dev)  # column-major m x B
    check(lib.cgx_fill_gaussian(t._xf.ctx.h, t._xf.h, g.data_ptr(), CGX_MEM_DEVICE, C.c_void_p(1)))
    z_ref = g.t() @ sx
    torch.cuda.synchronize()
    assert (torch.linalg.norm(z - z_ref) / torch.linalg.norm(z_ref)).item() <= Z_TOL


def test_stage2_tensor_core_nan_inf_and_tiny_columns(cg, restatement):
    """The tcgen05 stage 2 (m*d >= 16384) on S.X columns its digit planes cannot represent:
    a NaN, a +Inf, a -Inf and a column of magnitude ~1e-300 (below 2^-960).  Those columns
    are recomputed in plain fp64 the reference's way (ozgemm.cu oz_fixup), so NaN and Inf
    propagate into Z as in gemm (matrix.cpp:111-129) and the tiny column keeps its
    relative accuracy; every other column stays within the Z bar."""
    n, d, B, m, seed = 20000, 256, 4096, 128, 31
    x = restatement.gen_dense_f32(3, n, d).astype(np.float64)
    x[5, 3] = np.nan
    x[7, 10] = np.inf
    x[11, 20] = -np.inf
    x[:, 40] *= 1e-300
    t = cg.countgauss_new(m, B, n, cg.SeededRng(seed))
    z = cg.countgauss_apply(t, x)
    z_ref, _ = restatement.countgauss(seed, m, B, x=x)
    assert np.array_equal(np.isnan(z), np.isnan(z_ref))
    assert np.array_equal(np.isinf(z), np.isinf(z_ref))
    fin = np.isfinite(z_ref)
    assert np.array_equal(z[np.isinf(z_ref)], z_ref[np.isinf(z_ref)])
    for j in range(d):
        if fin[:, j].all():
            assert np.linalg.norm(z[:, j] - z_ref[:, j]) <= 1e-12 * np.linalg.norm(z_ref[:, j]), j


def test_trim_between_calls(cg, restatement):
    """cgx_trim frees the context's scratch and pooled blocks between calls; live transforms
    keep their arrays and every later call (dense, CSR record path, tensor-core stage 2)
    gives the same bits as before the trim."""
    from paper_1606_05732_b200 import SparseMatrix, bench_data

    ctx = cg.context()
    n, d, B, m = 1 << 20, 128, 8192, 128
    x = bench_data.dense_normal(n, d, seed=3)
    t = cg.countgauss_new(m, B, n, cg.SeededRng(4))
    z0 = cg.countgauss_apply(t, x).cpu().numpy()
    xs = bench_data.csr_bernoulli(n, 256, 0.02, seed=5)
    t2 = cg.countgauss_new(m, 65536, n, cg.SeededRng(6))
    s0 = cg.countsketch_apply(t2, xs).cpu().numpy()
    ctx.trim()
    t3 = cg.countgauss_new(16, 1000, 5000, cg.SeededRng(7))  # a pool allocation after the trim
    assert np.array_equal(cg.countgauss_apply(t, x).cpu().numpy(), z0)
    ctx.trim()
    s1 = cg.countsketch_apply(t2, xs).cpu().numpy()
    assert np.allclose(s1, s0, rtol=1e-14, atol=1e-14)  # record path: fp64 rounding order only
    del t3
