"""Measurement helper (not product code): distcheck-style batched tiny sketches --
trials/s of cgx_countsketch_batch_gram against the reference's own trial loop
(countsketch_new + countsketch_apply + gram per trial, OpenMP over trials; oracle/_ref).

  python tools/bench_batch.py [--n 10000] [--d 10] [--B 500] [--trials 20000]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1606_05732_b200 as cg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10000)
    ap.add_argument("--d", type=int, default=10)
    ap.add_argument("--B", type=int, default=500)
    ap.add_argument("--trials", type=int, default=20000)
    ap.add_argument("--ref_trials", type=int, default=2000)
    a = ap.parse_args()
    u = np.linalg.qr(np.random.default_rng(1).standard_normal((a.n, a.d)))[0]
    ud = torch.from_numpy(np.asfortranarray(u)).cuda()
    for _ in range(2):
        cg.countsketch_batch_gram(ud, a.B, a.trials, 7)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g = cg.countsketch_batch_gram(ud, a.B, a.trials, 7)
    e1.record()
    torch.cuda.synchronize()
    gpu_ms = e0.elapsed_time(e1)
    ref = oracle.Reference()
    t0 = time.perf_counter()
    _, g_ref = ref.sketch_gram_trials(7, 0, a.ref_trials, a.B, u)
    ref_s = time.perf_counter() - t0
    assert np.array_equal(g[: a.ref_trials].cpu().numpy(), g_ref)
    print(f"n={a.n} d={a.d} B={a.B}: GPU {a.trials / gpu_ms * 1e3:.3g} trials/s ({gpu_ms:.2f} ms for {a.trials}); "
          f"reference ({ref.max_threads()} threads) {a.ref_trials / ref_s:.3g} trials/s; "
          f"speed-up {a.trials / gpu_ms * 1e3 / (a.ref_trials / ref_s):.1f}x; bit-identical")


if __name__ == "__main__":
    main()
