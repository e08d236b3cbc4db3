"""CPU, world_size 2 over gloo: the multi-GPU host logic (paper_1606_05732_b200/distributed.py)
-- contiguous row shards, per-rank transforms from the shared seed over *global* row
indices, and the three combine modes ("z": all-reduce of Z; "sx": bucket-range
reduce-scatter of S.X, split-K stage 2, all-reduce; "g": all-reduce of S.X, G's m rows
split over ranks, all-gather of Z's row blocks; "cols": column-range reduce-scatter of
S.X, split-N stage 2, all-gather of Z's column blocks; "hash": hash-partitioned row
placement, final S.X slices, split-K stage 2, all-reduce of Z) -- reproduces the single-device T.X.
The per-rank compute is the oracle here (no GPU); on the box it is libcgx."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1606_05732_b200.distributed import bucket_range, combine, g_row_range, shard_range

N, D, B, M, SEED = 5003, 7, 67, 5, 424242


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    rng = np.random.default_rng(0)
    return rng.standard_normal((N, D))


def _worker(rank, world, port, mode, out_path, B=B):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = oracle.Restatement()
    x = _problem()
    r0, r1 = shard_range(N, world, rank)
    _, cs_seed, g_seed = O.countgauss_seeds(SEED)
    if mode == "hash":
        # hash-partitioned placement (ablation C): this rank holds the rows hashing into its
        # bucket range, in (bucket, row) order; its S.X slice is final, stage 2 is split-K
        b0, b1 = bucket_range(B, world, rank)
        h_all, s_all = O.hash_sign(cs_seed, B, N)
        rows = np.nonzero((h_all >= b0) & (h_all < b1))[0]
        rows = rows[np.lexsort((rows, h_all[rows]))]
        sx_p = O.sketch_dense(h_all[rows] - b0, s_all[rows], b1 - b0, x[rows])
        Gs = O.gaussian(g_seed, M, b1 - b0, c0=b0)
        z = torch.from_numpy(np.ascontiguousarray(O.gemm(Gs, sx_p)))
        z = combine("z", world=world, rank=rank, B=B, d=D, partial_z=z)
        if rank == 0:
            np.save(out_path, z.numpy())
        dist.destroy_process_group()
        return
    h, s = O.hash_sign(cs_seed, B, r1 - r0, i0=r0)  # global row indices, shared seed
    sx_p = O.sketch_dense(h, s, B, x[r0:r1])  # (B, D) partial
    if mode == "z":
        G = O.gaussian(g_seed, M, B)
        z = torch.from_numpy(np.ascontiguousarray(O.gemm(G, sx_p)))
        z = combine("z", world=world, rank=rank, B=B, d=D, partial_z=z)
    elif mode == "g":
        def stage2_rows(sx, g0, g1):
            G = O.gaussian(g_seed, M, B)  # rows [g0, g1) of G . S.X
            return torch.from_numpy(np.ascontiguousarray(O.gemm(G[g0:g1], sx.numpy())))
        z = combine("g", world=world, rank=rank, B=B, d=D, m=M,
                    partial_sx=torch.from_numpy(np.ascontiguousarray(sx_p)), stage2=stage2_rows)
    elif mode == "cols":
        G = O.gaussian(g_seed, M, B)

        def stage2_cols(sx_cols, c0, c1):  # (c1-c0, B) block of S.X columns -> Z[:, c0:c1)^T
            return torch.from_numpy(np.ascontiguousarray(O.gemm(G, sx_cols.numpy().T).T))
        z = combine("cols", world=world, rank=rank, B=B, d=D, m=M,
                    partial_sx=torch.from_numpy(np.ascontiguousarray(sx_p.T)), stage2=stage2_cols)
        z = z.contiguous()
    else:
        def stage2(sx_slice, b0, b1):
            if b1 <= b0:
                return torch.zeros((M, D), dtype=torch.float64)
            Gs = O.gaussian(g_seed, M, b1 - b0, c0=b0)
            return torch.from_numpy(np.ascontiguousarray(O.gemm(Gs, sx_slice.numpy())))
        z = combine(mode, world=world, rank=rank, B=B, d=D, m=M,
                    partial_sx=torch.from_numpy(np.ascontiguousarray(sx_p)), stage2=stage2)
    if mode == "sxo":  # every rank's Z, for the same-bits check
        np.save(f"{out_path}.{rank}.npy", np.ascontiguousarray(z.numpy()))
    if rank == 0:
        np.save(out_path, z.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", ["z", "sx", "sxo", "g", "cols", "hash"])
def test_multi_rank_combine_matches_single_device(tmp_path, mode, world):
    out = str(tmp_path / f"z_{mode}.npy")
    mp.spawn(_worker, args=(world, _free_port(), mode, out), nprocs=world, join=True)
    z = np.load(out)
    z_ref, _ = oracle.Restatement().countgauss(SEED, M, B, x=_problem())
    assert np.linalg.norm(z - z_ref) / np.linalg.norm(z_ref) <= 1e-13


@pytest.mark.parametrize("world,buckets", [(2, B), (3, B), (4, 5)])
def test_rank_ordered_combine_is_the_sequential_sum_on_every_rank(tmp_path, world, buckets):
    """"sxo" (the arithmetic of CGX_COMBINE_P2P): every rank returns the same bits, and they
    are the ones a single process gets by summing the partial S.X chunks and the partial Z's
    in rank order."""
    out = str(tmp_path / "z_sxo.npy")
    mp.spawn(_worker, args=(world, _free_port(), "sxo", out, buckets), nprocs=world, join=True)
    zs = [np.load(f"{out}.{r}.npy") for r in range(world)]
    for r in range(1, world):
        assert np.array_equal(zs[r], zs[0])
    O = oracle.Restatement()
    x = _problem()
    _, cs_seed, g_seed = O.countgauss_seeds(SEED)
    parts = []
    for r in range(world):
        r0, r1 = shard_range(N, world, r)
        h, s = O.hash_sign(cs_seed, buckets, r1 - r0, i0=r0)
        parts.append(O.sketch_dense(h, s, buckets, x[r0:r1]))
    per = (buckets + world - 1) // world
    z = None
    for r in range(world):
        b0 = min(buckets, r * per)
        b1 = min(buckets, b0 + per)
        zp = np.zeros((M, D))
        if b1 > b0:
            sl = parts[0][b0:b1].copy()
            for q in range(1, world):
                sl += parts[q][b0:b1]
            zp = O.gemm(O.gaussian(g_seed, M, b1 - b0, c0=b0), sl)
        z = zp.copy() if z is None else z + zp
    assert np.array_equal(zs[0], z)


def test_sx_combine_with_fewer_buckets_than_ranks_chunks(tmp_path):
    """B = 5 over 4 ranks: ceil(5/4) = 2-bucket chunks, so rank 3 owns no buckets (its
    range is clamped to [5, 5)) and contributes a zero Z."""
    out = str(tmp_path / "z_sx5.npy")
    mp.spawn(_worker, args=(4, _free_port(), "sx", out, 5), nprocs=4, join=True)
    z = np.load(out)
    z_ref, _ = oracle.Restatement().countgauss(SEED, M, 5, x=_problem())
    assert np.linalg.norm(z - z_ref) / np.linalg.norm(z_ref) <= 1e-13


def test_shard_ranges_cover_rows():
    for n in (1, 7, 5003, 1 << 24):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    assert bucket_range(65536, 8, 7) == (57344, 65536)
    for m in (1, 5, 64, 256):
        for w in (1, 2, 3, 8):
            spans = [g_row_range(m, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
