"""Measurement / checking helper (not product code): small runs of every kernel family for
compute-sanitizer (tools/sanitize.sh): the dense cp.async gather, the one-pass fused kernel,
the CSR gather (lean and chunked branches), the CSR record path (csr_atomic.cu), the FP64
DMMA and tcgen05 int8 stage 2 (2-CTA cluster multicast), host staging with narrowing, and
the transform build.  Each case also checks its result against the oracle, so a sanitizer
run that perturbs timing still has to produce the right numbers."""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1606_05732_b200 as cg  # noqa: E402

O = oracle.Restatement()


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def dense(n, d, B, m, seed, opts=()):
    ctx = cg.context()
    for k, v in opts:
        ctx.set_option(k, v)
    x = O.gen_dense_f32(seed, n, d)
    t = cg.countgauss_new(m, B, n, cg.SeededRng(seed))
    z = cg.countgauss_apply(t, x)
    z_ref, _ = O.countgauss(seed, m, B, x=x.astype(np.float64))
    for k, _ in opts:
        ctx.set_option(k, {"g_resident": 1, "fuse": 1, "csr_mode": 0, "oz_slices": 7}.get(k, 0))
    assert rel(z, z_ref) <= 1e-12, (n, d, B, m, opts)


def csr(n, d, B, m, seed, mean, opts=()):
    ctx = cg.context()
    for k, v in opts:
        ctx.set_option(k, v)
    rng = np.random.default_rng(seed)
    lens = np.minimum(rng.poisson(mean, n), d)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    cols = np.concatenate([np.sort(rng.choice(d, k, replace=False)) for k in lens]).astype(np.int32)
    vals = rng.standard_normal(int(rp[-1])).astype(np.float32)
    t = cg.countgauss_new(m, B, n, cg.SeededRng(seed))
    z = cg.countgauss_apply(t, cg.SparseMatrix(n, d, rp, cols, vals))
    z_ref, _ = O.countgauss(seed, m, B, csr=(rp, cols, vals, d))
    for k, _ in opts:
        ctx.set_option(k, 0)
    assert rel(z, z_ref) <= 1e-12, (n, d, B, m, opts)


def main():
    dense(40000, 32, 4096, 64, 1)                                   # sketch_dense_async + DMMA stage 2
    dense(40000, 256, 4096, 128, 2)                                 # tcgen05 stage 2 (m*d >= 16384), cluster 2
    dense(40000, 32, 4096, 64, 3, [("g_resident", 0), ("fuse", 2)])  # one-pass fused kernel
    csr(60000, 256, 8192, 64, 4, 2.5)                               # CSR lean gather
    csr(60000, 256, 8192, 64, 5, 2.5, [("csr_mode", 3)])            # CSR record path
    csr(60000, 16, 80, 16, 6, 8.0)                                  # chunked branch (B*d <= 2^16)
    x = O.gen_dense_f32(7, 300000, 8).astype(np.float64)            # > 1 MB host X: pinned staging, narrowing
    t = cg.countgauss_new(16, 2048, 300000, cg.SeededRng(7))
    z_ref, _ = O.countgauss(7, 16, 2048, x=x)
    assert rel(cg.countgauss_apply(t, np.asfortranarray(x)), z_ref) <= 1e-12
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
