"""Regenerate tests/golden/golden.npz from the REFERENCE itself (oracle/_ref/libcgref.so,
compiled from /root/reference/proj/src by oracle/Makefile).

Run here (the container that has /root/reference):  python tests/golden/make_golden.py
The fixtures pin the C restatement (oracle/cgoracle.c) and, through it, the GPU path.
Inputs that are not produced by the reference's own generators are made by the
restatement's documented generator (cgo_gen_dense_f32) and stored alongside.
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    R = oracle.Reference()
    O = oracle.Restatement()
    g = {}
    # rng.hpp: raw streams and child seeds
    g["rng_u64_12345"] = R.rng_u64(12345, 64)
    g["rng_u64_987654321"] = R.rng_u64(987654321, 64)
    g["mix64_42_t"] = np.array([R.lib.cgref_mix64(42, t) for t in range(100)], np.uint64)
    g["rng_normal_2024"] = R.rng_normal(2024, 4096)
    # test_rng.cpp:39-45 quantiles
    g["quantile_p"] = np.array([0.5, 0.975, 0.0013498980316300945, 1e-300, 1 - 2 ** -53, 0.02425, 0.97575])
    g["quantile_x"] = np.array([R.inverse_normal_cdf(p) for p in g["quantile_p"]])

    # config c1 transform: countgauss_new(16, 2048, 65536, SeededRng(12345))
    t = R.countgauss_new(16, 2048, 65536, 12345)
    h, s = t.hash_sign()
    G = t.g()
    g["c1_seeds"] = np.array([t.seed, t.cs_seed], np.uint64)
    g["c1_hash_head"] = h[:256]
    g["c1_sign_head"] = s[:256]
    g["c1_g_head"] = np.asfortranarray(G)[:, :16]
    g["c1_hash_digest"] = np.array(digest(h.astype(np.int64)))
    g["c1_sign_digest"] = np.array(digest(s.astype(np.float64)))
    g["c1_g_digest"] = np.array(digest(np.asfortranarray(G).T))  # column-major bytes

    # small dense case with full outputs
    n, d, B, m = 4096, 8, 128, 16
    x = O.gen_dense_f32(777, n, d)
    t2 = R.countgauss_new(m, B, n, 4242)
    xm = R.dense(x.astype(np.float64))
    g["dense_x"] = x
    g["dense_sx"] = t2.apply(xm, 0)
    g["dense_z"] = t2.apply(xm, 1)
    g["dense_params"] = np.array([n, d, B, m, 4242], np.int64)

    # CSR, serial branch (B*d > 2^16): reference's own random_sparse generator
    rp, ci, v = R.random_sparse(3000, 64, 5, 99)
    t3 = R.countgauss_new(32, 4096, 3000, 31337)
    xs = R.csr(rp, ci, v, 3000, 64)
    g["csr_rowptr"], g["csr_cols"], g["csr_vals"] = rp, ci, v
    g["csr_sx"] = t3.apply(xs, 0)
    g["csr_z"] = t3.apply(xs, 1)
    g["csr_params"] = np.array([3000, 64, 4096, 32, 31337], np.int64)

    # CSR, chunked branch (n_chunks > 1, B*d <= 2^16): bench defaults m=16, B=80, d=16
    rp, ci, v = R.random_sparse(10000, 16, 4, 1234)
    t4 = R.countgauss_new(16, 80, 10000, 555)
    xs = R.csr(rp, ci, v, 10000, 16)
    g["chunk_rowptr"], g["chunk_cols"], g["chunk_vals"] = rp, ci, v
    g["chunk_sx"] = t4.apply(xs, 0)
    g["chunk_sx_serial"] = t4.apply(xs, 2)
    g["chunk_z"] = t4.apply(xs, 1)
    g["chunk_params"] = np.array([10000, 16, 80, 16, 555], np.int64)

    # NMF: generate_separable(60, 40, 5) then cg_nmf(X, 12, 60, SeededRng(7006))
    # (test_determinism.cpp:62-75)
    xn = R.generate_separable(60, 40, 5, 7005)
    a = R.cg_nmf(R.dense(xn), 12, 60, 7006)
    g["nmf_x"] = np.asfortranarray(xn)
    g["nmf_i_max"], g["nmf_i_min"], g["nmf_unioned"] = a["i_max"], a["i_min"], a["unioned"]
    g["nmf_tie_rows"] = np.array(a["tie_rows"])

    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(out, **g)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
