"""Multi-GPU CountGauss: rows of X sharded over ranks (one process per GPU).

S.X = sum_p S_p.X_p where S_p is the CountSketch restricted to rank p's rows -- each rank
derives its hashes/signs from the shared seed for its *global* row indices
(cgx_countgauss_new_shard), so nothing but the seed is exchanged to build the transform.
T.X is linear, so the partials combine after either stage:

* ``"z"`` (default): every rank computes Z_p = G.(S_p.X_p) (G regenerated locally from
  the seed) and the m x d partials are summed with one all-reduce.  Communication is
  m*d*8 bytes; stage 2 is replicated.
* ``"sx"``: the B x d partial sketches (row-major, so a bucket range is contiguous) are
  reduce-scattered in equal ceil(B/P)-bucket chunks (clamped to B); rank p owns buckets
  [b_p, b_{p+1}) of the summed S.X and computes
  Z_p = G[:, b_p:b_{p+1}) . S.X[b_p:b_{p+1}) (split-K: stage 2 and G generation divided
  by P), then Z = sum_p Z_p by all-reduce.  Communication is (P-1)/P * B*d*8 per rank.
* ``"sxo"``: "sx" with every sum taken **in rank order**: the bucket-range chunks are
  exchanged with one all-to-all (rank p receives everyone's chunk p), summed
  ((c_0 + c_1) + c_2) + ..., and the partial Z's are all-gathered and summed the same way, so
  the result is the same bits on every rank and does not depend on the collective's algorithm
  or on timing.  This is the arithmetic of the C ABI's CGX_COMBINE_P2P (csrc/group.cu), where
  the exchange is fused into the sketch kernels' stores over peer memory; same volume as "sx".
* ``"p2p"``: "sxo" with the exchange of S.X fused into the sketch kernels: every rank owns a
  landing buffer of P slots shared with the others through CUDA IPC (`PeerLanding`), and a
  rank's sketch stores each finished bucket row straight into its slot in the owner's buffer
  over the peer mapping (api.countsketch_apply_to; NVLink stores on a multi-GPU node).  After a
  host barrier the owner sums its slots in rank order (api.sum_slots), runs stage 2 on its
  range, and the partial Z's are gathered and summed in rank order.  Same bits as "sxo".  The
  barrier is on the host (stream sync + `dist.barrier`): a device-side arrival flag would save
  its latency but makes kernels wait on other GPUs' kernels, which a one-GPU test cannot do.
* ``"g"``: the partial sketches are all-reduced (every rank holds the summed S.X), rank p
  computes rows [r_p, r_{p+1}) of Z = G[r_p:r_{p+1}, :] . S.X (cgx_gauss_gemm_rows: the
  m rows of G split across ranks, stage 2 divided by P with no further reduction), and the
  row blocks are all-gathered.  Z's rows are exact per rank (no cross-rank fp sum in
  stage 2); communication is ~2 B*d*8 + m*d*8 per rank.
* ``"cols"``: the column-range alternative.  The partial sketches are column-major, so a
  reduce-scatter hands rank p columns [c_p, c_{p+1}) of the summed S.X; rank p computes
  Z[:, c_p:c_{p+1}) = G . S.X[:, c_p:c_{p+1}) (split-N: all of G on every rank, stage 2
  divided by P) and the column blocks are all-gathered.

The collectives go through ``torch.distributed`` (NCCL on the GPUs; gloo in the CPU
tests).  Results equal the single-GPU T.X up to fp reassociation across ranks.
"""
from __future__ import annotations

from typing import Callable, Optional


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced row range [r0, r1) of rank `rank` (first n % world ranks get one
    extra row)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("shard_range: need 0 <= rank < world")
    base, extra = divmod(n, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def bucket_range(B: int, world: int, rank: int) -> tuple[int, int]:
    """Bucket slice owned by `rank` after the S.X reduce-scatter."""
    return shard_range(B, world, rank)


def g_row_range(m: int, world: int, rank: int) -> tuple[int, int]:
    """Rows of G (and of Z) computed by `rank` in the "g" combine: equal blocks of
    ceil(m / world) (the all-gather needs equal chunks); trailing ranks may get fewer or none."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("g_row_range: need 0 <= rank < world")
    per = (m + world - 1) // world
    r0 = min(m, rank * per)
    return r0, min(m, r0 + per)


def combine(mode: str, *, world: int, rank: int, B: int, d: int, partial_sx=None, partial_z=None,
            stage2: Optional[Callable] = None, m: Optional[int] = None, group=None):
    """Combine one rank's partial results into the full Z (every rank returns Z).

    mode "z":  partial_z (m x d) is all-reduced.
    mode "sx": partial_sx (B x d, row-major) is reduce-scattered by bucket range; the
               owned slice goes through stage2(sx_slice, b0, b1) -> Z_p (m x d), which is
               then all-reduced.
    mode "sxo": the same split with all-to-all / all-gather and sums in rank order.
    mode "g":  partial_sx (B x d, row-major) is all-reduced; stage2(sx, r0, r1) returns
               rows [r0, r1) of Z ((r1-r0) x d) for g_row_range(m, world, rank), and the
               row blocks are all-gathered into Z (m x d, row-major tensor).
    mode "cols": partial_sx is a contiguous (d, B) tensor (S.X column-major); columns are
               reduce-scattered, stage2(sx_cols, c0, c1) gets the (c1-c0, B) block and
               returns Z[:, c0:c1) transposed ((c1-c0) x m); the blocks are all-gathered
               into Z (m x d, column-major view).
    """
    if mode in ("g", "cols") and m is None:
        raise ValueError(f"combine: mode '{mode}' needs m")
    import torch
    import torch.distributed as dist

    if mode == "z":
        dist.all_reduce(partial_z, group=group)
        return partial_z
    if mode == "g":
        dist.all_reduce(partial_sx, group=group)
        r0, r1 = g_row_range(m, world, rank)
        per = (m + world - 1) // world
        blk = torch.zeros((per, d), dtype=partial_sx.dtype, device=partial_sx.device)
        if r1 > r0:
            blk[: r1 - r0] = stage2(partial_sx, r0, r1)
        out = torch.empty((per * world, d), dtype=blk.dtype, device=blk.device)
        dist.all_gather_into_tensor(out, blk, group=group)
        return out[:m]
    if mode == "cols":
        # partial_sx: B x d column-major, i.e. a contiguous (d, B) tensor of S.X columns
        per = (d + world - 1) // world
        flat = partial_sx.reshape(d, B)
        if per * world != d:
            pad = torch.zeros((per * world - d, B), dtype=flat.dtype, device=flat.device)
            flat = torch.cat([flat, pad], 0)
        out = torch.empty((per, B), dtype=flat.dtype, device=flat.device)
        dist.reduce_scatter_tensor(out, flat.contiguous(), group=group)
        c0 = min(d, rank * per)
        c1 = min(d, c0 + per)
        zt = torch.zeros((per, m), dtype=flat.dtype, device=flat.device)  # Z[:, c0:c1) transposed
        if c1 > c0:
            zt[: c1 - c0] = stage2(out[: c1 - c0], c0, c1)
        gathered = torch.empty((per * world, m), dtype=zt.dtype, device=zt.device)
        dist.all_gather_into_tensor(gathered, zt, group=group)
        return gathered[:d].t()  # m x d, column-major view
    if mode not in ("sx", "sxo"):
        raise ValueError("combine: mode must be 'z', 'sx', 'sxo', 'g' or 'cols'")
    # reduce_scatter_tensor needs equal chunks: pad B up to a multiple of world.
    per = (B + world - 1) // world
    flat = partial_sx.reshape(B, d)
    if per * world != B:
        pad = torch.zeros((per * world - B, d), dtype=flat.dtype, device=flat.device)
        flat = torch.cat([flat, pad], 0)
    if mode == "sxo":
        recv = torch.empty((world, per, d), dtype=flat.dtype, device=flat.device)
        dist.all_to_all_single(recv.view(world * per, d), flat.contiguous(), group=group)
        out = _ordered_sum(recv)
    else:
        out = torch.empty((per, d), dtype=flat.dtype, device=flat.device)
        dist.reduce_scatter_tensor(out, flat.contiguous(), group=group)
    # rank p owns the ceil(B/world)-bucket chunk [b0, b1) clamped to B (trailing ranks may
    # own nothing when B is small: they contribute a zero Z)
    b0 = min(B, rank * per)
    b1 = min(B, b0 + per)
    if b1 > b0:
        z = stage2(out[: b1 - b0], b0, b1)
    else:
        if m is None:
            raise ValueError("combine: mode 'sx' needs m when a rank owns no buckets")
        z = torch.zeros((m, d), dtype=flat.dtype, device=flat.device).t().contiguous().t()
    if mode == "sxo":
        zc = z.contiguous()
        parts = torch.empty((world,) + tuple(zc.shape), dtype=zc.dtype, device=zc.device)
        dist.all_gather_into_tensor(parts.view(world * zc.shape[0], zc.shape[1]), zc, group=group)
        return _ordered_sum(parts)
    dist.all_reduce(z, group=group)
    return z


class PeerLanding:
    """Rank-local landing buffer for the "p2p" combine and the peer mappings of everyone
    else's: `world` slots of ceil(B/world) x d doubles; slot q of rank p's buffer receives rank
    q's partial rows of p's bucket range.  Collective: every rank constructs it together."""

    def __init__(self, ctx, world: int, rank: int, B: int, d: int, group=None):
        import ctypes as C

        import torch.distributed as dist

        from ._lib import lib

        self.ctx, self.world, self.rank, self.B, self.d = ctx, world, rank, B, d
        self.per = (B + world - 1) // world
        self.slot = self.per * d  # doubles per slot
        p = C.c_void_p()
        _check(lib.cgx_device_alloc(ctx.h, 8 * self.slot * world, C.byref(p)))
        self.mine = p.value
        h = (C.c_ubyte * 64)()
        _check(lib.cgx_ipc_export(ctx.h, p, h))
        handles = [None] * world
        dist.all_gather_object(handles, bytes(h), group=group)
        self.peer = []
        for q in range(world):
            if q == rank:
                self.peer.append(self.mine)
                continue
            o = C.c_void_p()
            hb = (C.c_ubyte * 64).from_buffer_copy(handles[q])
            _check(lib.cgx_ipc_open(ctx.h, hb, C.byref(o)))
            self.peer.append(o.value)
        # where this rank's rows of bucket range q go: its slot in rank q's buffer
        self.bases = [self.peer[q] + 8 * self.slot * rank for q in range(world)]
        self._group = group

    def close(self):
        import ctypes as C

        import torch.distributed as dist

        from ._lib import lib

        if self.mine is None:
            return
        self.ctx.synchronize()
        dist.barrier(group=self._group)  # nobody still writes into a buffer about to go
        for q, ptr in enumerate(self.peer):
            if q != self.rank:
                lib.cgx_ipc_close(self.ctx.h, C.c_void_p(ptr))
        dist.barrier(group=self._group)
        lib.cgx_device_free(self.ctx.h, C.c_void_p(self.mine))
        self.mine = None


def _check(rc):
    if rc != 0:
        from ._lib import lib

        raise RuntimeError(lib.cgx_last_error().decode())


def combine_p2p(landing: "PeerLanding", sketch_to, stage2, *, m: int, group=None):
    """The "p2p" combine.  sketch_to(bases, per) runs this rank's sketch with segmented
    destinations (api.countsketch_apply_to); stage2(sx_slice, b0, b1) -> Z_p (m x d) as in "sx".
    Returns Z (m x d), the same bits on every rank."""
    import torch
    import torch.distributed as dist

    from . import api

    L = landing
    sketch_to(L.bases, L.per)
    L.ctx.synchronize()
    torch.cuda.synchronize()
    dist.barrier(group=group)  # every rank's rows have landed
    b0 = min(L.B, L.rank * L.per)
    b1 = min(L.B, b0 + L.per)
    if b1 > b0:
        sl = torch.empty((b1 - b0, L.d), dtype=torch.float64, device="cuda")
        api.sum_slots(L.ctx, L.mine, L.world, L.slot, (b1 - b0) * L.d, sl)
        z = stage2(sl, b0, b1)
    else:
        z = torch.zeros((L.d, m), dtype=torch.float64, device="cuda").t()
    zc = z.contiguous()
    parts = torch.empty((L.world,) + tuple(zc.shape), dtype=zc.dtype, device=zc.device)
    # the gather also orders the next step's stores after this step's slot sums on every rank
    dist.all_gather_into_tensor(parts.view(L.world * zc.shape[0], zc.shape[1]), zc, group=group)
    return _ordered_sum(parts)


def _ordered_sum(parts):
    """((parts[0] + parts[1]) + parts[2]) + ...: the slot sum of group.cu's sum_slots."""
    acc = parts[0].clone()
    for q in range(1, parts.shape[0]):
        acc += parts[q]
    return acc
