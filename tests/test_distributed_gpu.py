"""The "p2p" combine of distributed.py on the GPU: one process per rank, landing buffers shared
through CUDA IPC, each rank's sketch kernels storing their finished S.X rows into the owners'
buffers (api.countsketch_apply_to).  One GPU is available, so the rank processes share device
0 -- the IPC mappings, segmented stores, slot sums and the Z exchange are the real ones; only
the wire is missing.  Ranks synchronize on the host (gloo barrier after a stream sync), so no
kernel ever waits on another process's kernel."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

SHAPES = {
    "dense": (300001, 32, 4099, 24),      # cp.async gather stores into the peers' slots
    "dense_narrow": (100003, 7, 515, 9),  # sub-warp kernel: local S.X, then copies
    "csr": (120001, 300, 5003, 16),       # lean CSR gather stores into the peers' slots
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(kind):
    n, d, B, m = SHAPES[kind]
    rng = np.random.default_rng(11)
    if kind == "csr":
        lens = rng.integers(0, 12, n)
        rp = np.zeros(n + 1, np.int64)
        np.cumsum(lens, out=rp[1:])
        cols = rng.integers(0, d, rp[-1]).astype(np.int32)
        vals = rng.standard_normal(rp[-1]).astype(np.float32)
        return rp, cols, vals
    return rng.standard_normal((n, d)).astype(np.float32)


def _worker(rank, world, port, kind, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1606_05732_b200 as cg
    from paper_1606_05732_b200.distributed import PeerLanding, combine_p2p, shard_range

    ctx = cg.context(0)
    n, d, B, m = SHAPES[kind]
    t_seed = cg.SeededRng(4242).next_u64()
    r0, r1 = shard_range(n, world, rank)
    t = cg.api.countgauss_new_shard(m, B, n, r0, r1 - r0, t_seed, ctx=ctx)
    if kind == "csr":
        rp, cols, vals = _inputs(kind)
        q0, q1 = int(rp[r0]), int(rp[r1])
        xs = cg.SparseMatrix(r1 - r0, d, torch.from_numpy(rp[r0:r1 + 1] - q0).cuda(),
                             torch.from_numpy(cols[q0:q1]).cuda(), torch.from_numpy(vals[q0:q1]).cuda())
    else:
        xs = torch.from_numpy(_inputs(kind)[r0:r1]).cuda()
    L = PeerLanding(ctx, world, rank, B, d)
    zs = []
    for _ in range(3):  # the landing buffers are reused: the result must not move
        z = combine_p2p(L, lambda bases, per: cg.api.countsketch_apply_to(t, xs, bases, per),
                        lambda sl, b0, b1: cg.api.gauss_gemm_range(t, sl, b0, b1), m=m)
        torch.cuda.synchronize()
        zs.append(z.cpu().numpy().copy())
    assert np.array_equal(zs[0], zs[1]) and np.array_equal(zs[0], zs[2])
    np.save(f"{out}.{rank}.npy", zs[0])
    L.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind", list(SHAPES))
def test_p2p_combine_across_processes(cg, tmp_path, kind, world):
    out = str(tmp_path / "z")
    mp.spawn(_worker, args=(world, _free_port(), kind, out), nprocs=world, join=True)
    zs = [np.load(f"{out}.{r}.npy") for r in range(world)]
    for r in range(1, world):
        assert np.array_equal(zs[r], zs[0])  # same bits on every rank
    n, d, B, m = SHAPES[kind]
    t = cg.countgauss_new(m, B, n, cg.SeededRng(4242))
    if kind == "csr":
        rp, cols, vals = _inputs(kind)
        x = cg.SparseMatrix(n, d, rp, cols, vals)
    else:
        x = _inputs(kind)
    z1 = np.asarray(cg.countgauss_apply(t, x))
    assert np.linalg.norm(zs[0] - z1) / np.linalg.norm(z1) <= 1e-12
