"""Tensor-parallel (Megatron column-parallel) fused FFN across the GPUs of one box.

BASELINE.json north_star (c): "column-sharding the intermediate dimension N of
W1/W3 (Megatron-style, with no reduction needed), with an NCCL all-gather over
NVLink only when the full output is requested".  SiLU-gating is elementwise in
N, so rank p computes out[:, shard p] from its contiguous row block of W1 and
W3 and the replicated x; there is no data-path collective unless
``gather=True``.  One process per GPU, ``torch.distributed`` with NCCL for the
plumbing.  ``gather="fused"`` instead writes every output
tile straight into every rank's full [M, N] buffer from the kernel epilogue
(symmetric-memory peer pointers over NVLink, or one NVLS multicast store per
tile when the switch supports it), so the gather overlaps the GEMM and no
separate collective or interleave pass runs.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import FusedFFN, _handle


def shard_bounds(N: int, rank: int, world: int, align: int = 8):
    """Contiguous [n0, n1) of the N output columns owned by `rank`.

    Shards are as equal as possible in units of `align` columns (the C ABI
    requires every shard width to be a multiple of 8)."""
    if N % align != 0:
        raise ValueError(f"N={N} must be a multiple of {align}")
    units = N // align
    base, rem = divmod(units, world)
    n0 = (rank * base + min(rank, rem)) * align
    n1 = n0 + (base + (1 if rank < rem else 0)) * align
    return n0, n1


def shard_weights(w1: torch.Tensor, w3: torch.Tensor, rank: int, world: int):
    """Rank `rank`'s contiguous row block of W1 and W3 ([N,K] nn.Linear layout)."""
    n0, n1 = shard_bounds(w1.shape[0], rank, world)
    return w1[n0:n1].contiguous(), w3[n0:n1].contiguous()


def gather_shards(out_shard: torch.Tensor, N: int, group=None) -> torch.Tensor:
    """All-gather the per-rank [M, N_p] output shards into the full [M, N].

    Equal shards use one all_gather_into_tensor into [P, M, N/P] followed by a
    column interleave; unequal shards fall back to all_gather of padded
    buffers.  Collective over `group` (NCCL on GPUs, gloo on CPU)."""
    world = dist.get_world_size(group)
    M = out_shard.shape[0]
    widths = [shard_bounds(N, r, world)[1] - shard_bounds(N, r, world)[0] for r in range(world)]
    wmax = max(widths)
    if out_shard.shape[1] != widths[dist.get_rank(group)]:
        raise ValueError("out_shard width does not match this rank's shard")
    if all(w == wmax for w in widths):
        buf = torch.empty((world * M, wmax), dtype=out_shard.dtype, device=out_shard.device)
        dist.all_gather_into_tensor(buf, out_shard.contiguous(), group=group)
        return buf.view(world, M, wmax).permute(1, 0, 2).reshape(M, N)
    padded = torch.zeros((M, wmax), dtype=out_shard.dtype, device=out_shard.device)
    padded[:, :out_shard.shape[1]] = out_shard
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[:, :w] for p, w in zip(parts, widths)], dim=1)


def gather_destinations(buffer_ptrs, col0: int, elem_size: int, multicast_ptr: int = 0):
    """Destination list of cuasm_ffn_forward_gather for one rank: this shard's
    column 0 (byte offset col0 * elem_size) inside every rank's full output
    buffer, or inside the multicast mapping when one exists.  Returns
    (dst_ptrs, multicast)."""
    off = int(col0) * int(elem_size)
    if multicast_ptr:
        return [int(multicast_ptr) + off], True
    if not 1 <= len(buffer_ptrs) <= 8:
        raise ValueError("the fused gather addresses 1..8 ranks (one NVLink domain of one box)")
    return [int(p) + off for p in buffer_ptrs], False


class FusedGather:
    """Symmetric-memory full-output buffer [M, N] of one process group, for
    ffn_tp_forward(gather="fused").  Every rank allocates it through torch's
    symmetric memory (one collective rendezvous), so each rank holds the peer
    pointers of all ranks' buffers (and a multicast mapping when NVLS is
    available)."""

    def __init__(self, M: int, N: int, dtype, device, group=None, use_multicast: bool = True):
        import torch.distributed._symmetric_memory as symm_mem
        grp = group or dist.group.WORLD
        self.buf = symm_mem.empty((M, N), dtype=dtype, device=device)
        self.hdl = symm_mem.rendezvous(self.buf, grp)
        self.M, self.N = M, N
        self.rank, self.world = self.hdl.rank, self.hdl.world_size
        # multicast_ptr is 0 when torch could not set up an NVLS multicast object
        # (no NVSwitch fabric / single device): the P2P stores are used then
        self.multicast_ptr = int(self.hdl.multicast_ptr or 0) if use_multicast else 0

    def destinations(self, col0: int):
        return gather_destinations(self.hdl.buffer_ptrs, col0, self.buf.element_size(), self.multicast_ptr)

    def barrier(self):
        """Stream-ordered cross-rank barrier: after it, every rank's stores are in."""
        self.hdl.barrier(channel=0)


def ffn_tp_forward(x, rms_w, w1_shard, w3_shard, eps: float = 1e-6, group=None, gather=False,
                   N: int | None = None, handle: FusedFFN | None = None, fused: FusedGather | None = None):
    """This rank's share of the column-parallel fused FFN.

    x [M,K] (replicated), rms_w [K], w1_shard/w3_shard [N_p,K] -> out [M,N_p],
    or the full [M,N] when ``gather`` (N = total width, required then):
    gather=True / "nccl": NCCL all-gather + interleave after the kernel;
    gather="fused": the kernel epilogue writes into every rank's symmetric
    buffer (`fused`, a FusedGather of this group; created when None)."""
    h = handle or _handle(x.device, x.dtype)
    if gather == "fused":
        if N is None:
            raise ValueError("gather='fused' needs the total N")
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        fg = fused or FusedGather(x.shape[0], N, x.dtype, x.device, group)
        if tuple(fg.buf.shape) != (x.shape[0], N) or fg.buf.dtype != x.dtype:
            raise ValueError(f"FusedGather buffer {tuple(fg.buf.shape)} {fg.buf.dtype} does not match the "
                             f"output [{x.shape[0]}, {N}] {x.dtype}")
        n0, n1 = shard_bounds(N, rank, world)
        if w1_shard.shape[0] != n1 - n0:
            raise ValueError("w1_shard width does not match this rank's shard")
        dst, mc = fg.destinations(n0)
        # every peer has finished reading the previous output held in the buffers
        # before any rank's epilogue stores into them again
        if fused is not None:
            fg.barrier()
        h.forward_gather(x, rms_w, w1_shard, w3_shard, dst, N, eps, multicast=mc)
        fg.barrier()
        return fg.buf
    out = h.forward(x, rms_w, w1_shard, w3_shard, eps)
    if not gather:
        return out
    if N is None:
        raise ValueError("gather=True needs the total N")
    return gather_shards(out, N, group)


def shard_w2(w2: torch.Tensor, rank: int, world: int):
    """Rank `rank`'s columns of the down projection W2 [K,N] (row-parallel:
    the same N range as its W1/W3 rows)."""
    n0, n1 = shard_bounds(w2.shape[1], rank, world)
    return w2[:, n0:n1].contiguous()


def ffn_block_tp_forward(x, rms_w, w1_shard, w3_shard, w2_shard, eps: float = 1e-6, group=None,
                         handle: FusedFFN | None = None):
    """Megatron tensor-parallel LLaMA feed-forward block: column-parallel W1/W3
    (this rank's N-shard of the hidden), row-parallel W2, one all-reduce of
    the [M,K] partial outputs (NCCL over NVLink on GPUs)."""
    h = handle or _handle(x.device, x.dtype)
    y = h.block_forward(x, rms_w, w1_shard, w3_shard, w2_shard, eps)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(y, group=group)
    return y
