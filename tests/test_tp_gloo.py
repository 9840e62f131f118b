"""Multi-process host logic of the N-sharded (column-parallel) path, on CPU
with the gloo backend at world_size 2 (and 3 for ragged shards): shard
bounds, the all-gather + column interleave that reassembles the output, and
bench.py's max-over-ranks timing reduction."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_08071_b200.tp import gather_shards, shard_bounds, shard_w2, shard_weights


@pytest.mark.parametrize("N,world", [(11008, 8), (11008, 2), (28672, 8), (1376, 3), (8, 1), (24, 3), (40, 3)])
def test_shard_bounds_partition(N, world):
    spans = [shard_bounds(N, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == N
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a1 == b0
    widths = [b - a for a, b in spans]
    assert all(w % 8 == 0 for w in widths)
    assert max(widths) - min(widths) <= 8


def test_shard_weights_rows():
    w1 = torch.arange(48 * 4, dtype=torch.float32).reshape(48, 4)
    w3 = -w1
    a1, a3 = shard_weights(w1, w3, 1, 3)
    n0, n1 = shard_bounds(48, 1, 3)
    assert torch.equal(a1, w1[n0:n1]) and torch.equal(a3, w3[n0:n1])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, N, M, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = torch.arange(M * N, dtype=torch.float32).reshape(M, N)
        n0, n1 = shard_bounds(N, rank, world)
        got = gather_shards(full[:, n0:n1].contiguous(), N)
        ok_gather = bool(torch.equal(got, full))
        import bench
        t = bench.max_over_ranks(float(rank + 1) * 1.5)
        q.put((rank, ok_gather, t))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N", [(2, 64), (3, 40), (2, 11008)])
def test_gather_and_max_over_ranks(world, N):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, 5, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, t in res:
        assert ok, f"rank {rank}: gathered output differs"
        assert t == pytest.approx(1.5 * world)


def test_shard_w2_columns_match_w1_rows():
    K, N = 16, 48
    w2 = torch.arange(K * N, dtype=torch.float32).reshape(K, N)
    for world in (1, 2, 3):
        cols = torch.cat([shard_w2(w2, r, world) for r in range(world)], dim=1)
        assert torch.equal(cols, w2)


def _block_worker(rank, world, port, q):
    """Row-parallel W2: each rank's partial y_p = h_p @ W2_p^T, all-reduced,
    equals the unsharded h @ W2^T (the host logic of ffn_block_tp_forward)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(0)
        M, K, N = 5, 16, 48
        hid = torch.randn(M, N, generator=g, dtype=torch.float64)
        w2 = torch.randn(K, N, generator=g, dtype=torch.float64)
        n0, n1 = shard_bounds(N, rank, world)
        y = hid[:, n0:n1] @ shard_w2(w2, rank, world).T
        dist.all_reduce(y)
        q.put((rank, bool(torch.allclose(y, hid @ w2.T, rtol=1e-12, atol=1e-12))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_parallel_w2_all_reduce(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_block_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res)


# ---- fused gather (f2): the destination arithmetic, emulated across processes ----
_VBASE = 1 << 40  # virtual "peer pointer" of rank q's buffer: q * _VBASE


def _fused_gather_worker(rank, world, port, M, N, bufs, q):
    """Each rank writes its shard into EVERY rank's full buffer at the addresses
    gather_destinations gives (what the kernel epilogue stores do over NVLink),
    then a barrier; afterwards every rank's buffer must hold the full output."""
    from paper_2501_08071_b200.tp import gather_destinations
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n0, n1 = shard_bounds(N, rank, world)
        shard = (torch.arange(M * (n1 - n0), dtype=torch.float32).reshape(M, n1 - n0) + 1000.0 * rank)
        dst, mc = gather_destinations([p * _VBASE for p in range(world)], n0, 4)
        assert mc is False and len(dst) == world
        for d in dst:
            peer, off = divmod(d, _VBASE)
            col0 = off // 4
            assert col0 == n0
            flat = bufs[peer].view(M, N)
            flat[:, col0:col0 + (n1 - n0)] = shard   # row stride ldo = N
        dist.barrier()
        full = torch.cat([torch.arange(M * (b - a), dtype=torch.float32).reshape(M, b - a) + 1000.0 * r
                          for r, (a, b) in enumerate(shard_bounds(N, r, world) for r in range(world))], dim=1)
        q.put((rank, bool(torch.equal(bufs[rank].view(M, N), full))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N", [(2, 64), (3, 40), (4, 11008 // 4)])
def test_fused_gather_destinations_fill_every_buffer(world, N):
    M = 5
    bufs = [torch.full((M * N,), -1.0).share_memory_() for _ in range(world)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_gather_worker, args=(r, world, port, M, N, bufs, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(world)}


def test_gather_destinations_multicast_and_limits():
    from paper_2501_08071_b200.tp import gather_destinations
    assert gather_destinations([100, 200], 8, 2, multicast_ptr=5000) == ([5016], True)
    assert gather_destinations([100, 200], 8, 2) == ([116, 216], False)
    with pytest.raises(ValueError):
        gather_destinations(list(range(9)), 0, 2)


# ---- fused reduction (f1): ownership and staging-slot addressing across processes ----
@pytest.mark.parametrize("M,K,world", [(5, 4096, 8), (3, 1024, 3), (7, 64, 8), (2, 8192, 3), (4, 520, 2)])
def test_rs_layout_partitions_columns(M, K, world):
    from paper_2501_08071_b200 import rs_layout
    spans = [rs_layout(M, K, world, q) for q in range(world)]
    cols = []
    for c0, c1, nb in spans:
        assert c0 % 256 == 0 and (c1 == K or c1 % 256 == 0) and c1 >= c0
        assert nb == world * M * (c1 - c0) * 4
        cols += list(range(c0, c1))
    assert cols == list(range(K))   # every output column has exactly one owner, in rank order


def _fused_reduce_worker(rank, world, port, M, K, N, stages, ys, q):
    """Each rank scatters its partial y_p's columns into the owner's staging slot
    [rank] at the offsets cuasm_rs_layout defines (what the GEMM epilogue's TMA stores
    do), barrier, each owner sums its slots in rank order and writes its columns into
    every rank's y (what cuasm_rs_reduce does), barrier: every y = hid @ W2^T."""
    from paper_2501_08071_b200 import rs_layout
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(1)
        hid = torch.randn(M, N, generator=g, dtype=torch.float64)
        w2 = torch.randn(K, N, generator=g, dtype=torch.float64)
        n0, n1 = shard_bounds(N, rank, world)
        part = hid[:, n0:n1] @ shard_w2(w2, rank, world).T      # [M, K]
        for owner in range(world):
            c0, c1, nb = rs_layout(M, K, world, owner)
            kq = c1 - c0
            if kq == 0:
                continue
            slot = stages[owner][rank * M * kq:(rank + 1) * M * kq].view(M, kq)
            slot.copy_(part[:, c0:c1])
        dist.barrier()
        c0, c1, _ = rs_layout(M, K, world, rank)
        kq = c1 - c0
        if kq:
            acc = torch.zeros(M, kq, dtype=torch.float64)
            for p in range(world):  # rank order
                acc += stages[rank][p * M * kq:(p + 1) * M * kq].view(M, kq)
            for r in range(world):
                ys[r].view(M, K)[:, c0:c1] = acc
        dist.barrier()
        q.put((rank, bool(torch.allclose(ys[rank].view(M, K), hid @ w2.T, rtol=1e-12, atol=1e-12))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,M,K,N", [(2, 3, 1024, 48), (3, 4, 1280, 72), (4, 2, 520, 64)])
def test_fused_reduce_addressing(world, M, K, N):
    from paper_2501_08071_b200 import rs_layout
    sizes = [rs_layout(M, K, world, q)[2] // 4 for q in range(world)]
    stages = [torch.full((max(s, 1),), float("nan"), dtype=torch.float64).share_memory_() for s in sizes]
    ys = [torch.full((M * K,), float("nan"), dtype=torch.float64).share_memory_() for _ in range(world)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_reduce_worker, args=(r, world, port, M, K, N, stages, ys, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(world)}
