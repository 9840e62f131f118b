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


class FusedReduce:
    """Symmetric-memory buffers of f1's fused all-reduce for one process group and
    block shape [M, K]: every rank's fp32 staging buffer (cuasm_rs_layout sizes; the
    largest rank's size on all ranks, as symmetric memory requires) and every rank's
    full bf16 output y [M, K], with the peer pointers of both (and y's NVLS multicast
    mapping when torch can create one)."""

    def __init__(self, M: int, K: int, device, group=None, use_multicast: bool = True):
        import torch.distributed._symmetric_memory as symm_mem
        from . import rs_layout
        grp = group or dist.group.WORLD
        world = dist.get_world_size(grp)
        nbytes = max(rs_layout(M, K, world, q)[2] for q in range(world))
        self.stage = symm_mem.empty((max(nbytes // 4, 4),), dtype=torch.float32, device=device)
        self.stage_hdl = symm_mem.rendezvous(self.stage, grp)
        self.y = symm_mem.empty((M, K), dtype=torch.bfloat16, device=device)
        self.y_hdl = symm_mem.rendezvous(self.y, grp)
        self.M, self.K = M, K
        self.rank, self.world = self.stage_hdl.rank, self.stage_hdl.world_size
        self.multicast_ptr = int(self.y_hdl.multicast_ptr or 0) if use_multicast else 0

    def stage_ptrs(self):
        return [int(p_) for p_ in self.stage_hdl.buffer_ptrs]

    def y_destinations(self):
        if self.multicast_ptr:
            return [self.multicast_ptr], True
        return [int(p_) for p_ in self.y_hdl.buffer_ptrs], False

    def barrier(self):
        """Stream-ordered cross-rank barrier."""
        self.stage_hdl.barrier(channel=0)


def ffn_block_tp_forward(x, rms_w, w1_shard, w3_shard, w2_shard, eps: float = 1e-6, group=None,
                         handle: FusedFFN | None = None, reduce: str = "nccl", fused: FusedReduce | None = None):
    """Megatron tensor-parallel LLaMA feed-forward block: column-parallel W1/W3
    (this rank's N-shard of the hidden), row-parallel W2, and the all-reduce of the
    [M,K] partial outputs:
    reduce="nccl": the block's bf16 partial, then one NCCL all_reduce;
    reduce="fused": the down projection's epilogue stores every fp32 partial tile into
    the owner rank's symmetric staging buffer (cuasm_ffn_block_forward_rs, overlapping
    the GEMM tile by tile), a cross-rank barrier, each owner's rank-order sum stored
    into every rank's output (cuasm_rs_reduce: P2P stores or one NVLS multicast store),
    a barrier; returns the full y [M, K] (`fused.y`)."""
    h = handle or _handle(x.device, x.dtype)
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if reduce == "fused":
        M, K = x.shape
        fr = fused or FusedReduce(M, K, x.device, group)
        if (fr.M, fr.K) != (M, K):
            raise ValueError(f"FusedReduce is for [{fr.M}, {fr.K}], the block output is [{M}, {K}]")
        if fused is not None:
            fr.barrier()  # every peer has finished reading the previous output and staging
        h.block_forward_rs(x, rms_w, w1_shard, w3_shard, w2_shard, fr.stage_ptrs(), fr.world, fr.rank, eps)
        fr.barrier()      # every rank's partial tiles are in their owners' staging buffers
        dst, mc = fr.y_destinations()
        h.rs_reduce(fr.stage, fr.world, fr.rank, dst, K, M, K, multicast=mc)
        fr.barrier()      # every owner's columns are in every rank's y
        return fr.y
    if reduce != "nccl":
        raise ValueError("reduce is 'nccl' or 'fused'")
    y = h.block_forward(x, rms_w, w1_shard, w3_shard, w2_shard, eps)
    if world > 1:
        dist.all_reduce(y, group=group)
    return y
