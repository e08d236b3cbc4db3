"""CPU: pin the C restatement (oracle/cgoracle.c) against the reference's golden vectors
and against the compiled reference itself.  Mirrors the reference's own pins:
test_rng.cpp, test_sketch.cpp, test_matrix.cpp:21-34, acceptance.cpp criterion 5."""
import hashlib

import numpy as np
import pytest

import oracle


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_rng_streams_pinned(golden):
    for seed, key in [(12345, "rng_u64_12345"), (987654321, "rng_u64_987654321")]:
        draws = [oracle.draw(seed, k) for k in range(64)]
        assert np.array_equal(np.array(draws, np.uint64), golden[key])
    assert [oracle.mix64(42, t) for t in range(100)] == [int(v) for v in golden["mix64_42_t"]]
    assert len(set(int(v) for v in golden["mix64_42_t"])) == 100  # test_rng.cpp:47-53


def test_survey_smoke_goldens(restatement):
    # countgauss_new(16, 2048, 65536, SeededRng(12345))
    t, cs, gs = restatement.countgauss_seeds(12345)
    assert t == 0x22118258A9D111A0 and cs == 0xD0347DD74D1D1616
    h, s = restatement.hash_sign(cs, 2048, 4)
    assert list(h) == [257, 1584, 707, 1188] and list(s) == [1, -1, 1, 1]
    assert restatement.gaussian(gs, 16, 1)[0, 0] == 0.42178778775820458
    h2, _ = restatement.hash_sign(cs, 65536, 4)
    assert list(h2) == [22785, 30256, 4803, 52388]


def test_inverse_normal_cdf_quantiles(restatement, golden):
    # test_rng.cpp:39-45 plus the region boundaries; bit-exact vs the reference
    for p, x in zip(golden["quantile_p"], golden["quantile_x"]):
        assert restatement.inverse_normal_cdf(float(p)) == x
    assert abs(restatement.inverse_normal_cdf(0.975) - 1.959963984540054) <= 1e-10 * 1.96
    assert abs(restatement.inverse_normal_cdf(0.0013498980316300945) + 3.0) <= 1e-9 * 3
    assert np.isnan(restatement.inverse_normal_cdf(0.0)) and np.isnan(restatement.inverse_normal_cdf(1.0))


def test_normal_stream_pinned(restatement, golden):
    ref = golden["rng_normal_2024"]
    got = np.array([restatement.inverse_normal_cdf(((oracle.draw(2024, k) >> 11) + 0.5) * 2.0 ** -53)
                    for k in range(len(ref))])
    assert np.array_equal(got, ref)


def test_c1_transform_pinned(restatement, golden):
    t, cs, gs = restatement.countgauss_seeds(12345)
    assert [t, cs] == [int(v) for v in golden["c1_seeds"]]
    h, s = restatement.hash_sign(cs, 2048, 65536)
    assert np.array_equal(h[:256], golden["c1_hash_head"]) and np.array_equal(s[:256], golden["c1_sign_head"])
    assert _digest(h) == str(golden["c1_hash_digest"]) and _digest(s) == str(golden["c1_sign_digest"])
    G = restatement.gaussian(gs, 16, 2048)
    assert np.array_equal(G[:, :16], golden["c1_g_head"])
    assert _digest(np.asfortranarray(G).T) == str(golden["c1_g_digest"])


def test_dense_apply_pinned(restatement, golden):
    n, d, B, m, seed = (int(v) for v in golden["dense_params"])
    z, sx = restatement.countgauss(seed, m, B, x=golden["dense_x"])
    assert np.array_equal(sx, golden["dense_sx"])
    assert np.array_equal(z, golden["dense_z"])
    # layout independence of the restatement (col-major fp64 widening)
    z2, sx2 = restatement.countgauss(seed, m, B, x=np.asfortranarray(golden["dense_x"], np.float64))
    assert np.array_equal(sx2, sx) and np.array_equal(z2, z)


@pytest.mark.parametrize("case", ["csr", "chunk"])
def test_csr_apply_pinned(restatement, golden, case):
    n, d, B, m, seed = (int(v) for v in golden[f"{case}_params"])
    csr = (golden[f"{case}_rowptr"], golden[f"{case}_cols"], golden[f"{case}_vals"], d)
    z, sx = restatement.countgauss(seed, m, B, csr=csr)
    assert np.array_equal(sx, golden[f"{case}_sx"])
    assert np.array_equal(z, golden[f"{case}_z"])


def test_chunked_branch_differs_from_serial(golden):
    # the chunked CSR branch is a different summation order
    a, b = golden["chunk_sx"], golden["chunk_sx_serial"]
    assert not np.array_equal(a, b)
    assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max()


def test_select_extremes_pinned(restatement, golden):
    x = golden["nmf_x"]
    t, cs, gs = restatement.countgauss_seeds(7006)
    z, _ = restatement.countgauss(7006, 12, 60, x=np.asfortranarray(x))
    e = restatement.select_extremes(z)
    assert list(e["i_max"]) == list(golden["nmf_i_max"])
    assert list(e["i_min"]) == list(golden["nmf_i_min"])
    assert list(e["unioned"]) == list(golden["nmf_unioned"])
    assert e["tie_rows"] == int(golden["nmf_tie_rows"])


def test_select_extremes_ties_and_nan(restatement):
    # nmf.cpp:105-115 semantics, test_geometry.cpp:98-110: duplicated columns -> tie rows
    z = np.array([[1.0, 3.0, 3.0, 0.0], [2.0, 2.0, 1.0, 1.0], [np.nan, 5.0, -1.0, 2.0], [0.0, -0.0, 1.0, np.nan]])
    e = restatement.select_extremes(z)
    assert list(e["amax"]) == [1, 0, 0, 2] and list(e["amin"]) == [3, 2, 0, 0]
    assert e["tie_rows"] == 3


def test_restatement_matches_reference_random(restatement, reference):
    """acceptance.cpp:124-145 style: random small cases, every field bit-exact."""
    rng = np.random.default_rng(5)
    for trial in range(40):
        n = int(rng.integers(1, 300))
        d = int(rng.integers(1, 12))
        B = int(rng.integers(1, 40))
        m = int(rng.integers(1, 9))
        seed = int(rng.integers(0, 2 ** 63))
        t = reference.countgauss_new(m, B, n, seed)
        h, s = t.hash_sign()
        ts, cs, gs = restatement.countgauss_seeds(seed)
        assert (t.seed, t.cs_seed) == (ts, cs)
        h2, s2 = restatement.hash_sign(cs, B, n)
        assert np.array_equal(h, h2) and np.array_equal(s, s2)
        assert np.array_equal(t.g(), restatement.gaussian(gs, m, B))
        x = np.floor(rng.uniform(-5, 6, size=(n, d))) if trial % 2 else rng.standard_normal((n, d))
        xm = reference.dense(x)
        z, sx = restatement.countgauss(seed, m, B, x=x)
        assert np.array_equal(sx, t.apply(xm, 0)) and np.array_equal(z, t.apply(xm, 1))
        if trial % 2:  # exactness on integer inputs vs the materialized product (test_sketch.cpp:94-109)
            assert np.array_equal(sx, t.materialized_sketch(x))


def test_gemm_matches_reference(restatement, reference):
    rng = np.random.default_rng(6)
    a = rng.standard_normal((17, 23))
    b = rng.standard_normal((23, 9))
    b[3, 2] = 0.0
    assert np.array_equal(restatement.gemm(a, b), reference.gemm(a, b))
    assert np.allclose(restatement.gemm(a, b), a @ b, rtol=1e-12, atol=1e-12)  # test_matrix.cpp:21-34
