"""Dynamic whole-tile claiming (CUASM_OPT_DYNAMIC; DESIGN.md §6 "Dynamic tiles").

Every data-parallel tile is still computed whole by one cluster, so the output must be
bitwise identical to the static round-robin schedule's; the claim counters reset and
the launch epoch advances at the end of every launch, so back-to-back launches, CUDA
graph replays and launches alternating with static ones must all stay correct.
Compared against the fp64 oracle at the [BJ] tolerance (PAPER.md P:560 inputs).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_inputs

pytestmark = pytest.mark.gpu

RTOL, ATOL = 2e-2, 1e-3


def check(gpu, ref, what):
    worst, nbad, maxerr = oracle.tolerance_ratio(gpu.double().cpu().numpy(), ref, RTOL, ATOL)
    assert nbad == 0, f"{what}: {nbad} elements out of tolerance (worst ratio {worst:.3f})"


def _handle(dev, dynamic, variant=ffn.VARIANT_AUTO, schedule=ffn.SCHEDULE_AUTO, bn=0):
    h = ffn.FusedFFN(dev, torch.bfloat16)
    h.set_option(ffn.OPT_DYNAMIC, dynamic)
    h.set_variant(variant)
    h.set_option(ffn.OPT_SCHEDULE, schedule)
    h.set_option(ffn.OPT_TILE_BN, bn)
    return h


# (M, K, N, variant, schedule, bn): several rounds of whole tiles, with and without a stream-K
# tail, both variants, a narrow tile width, ragged M / N
CASES = [(2048, 1024, 11008, ffn.VARIANT_2SM, ffn.SCHEDULE_DATA_PARALLEL, 0),
         (2048, 1024, 11008, ffn.VARIANT_2SM, ffn.SCHEDULE_AUTO, 128),
         (1000, 512, 5000, ffn.VARIANT_1SM, ffn.SCHEDULE_DATA_PARALLEL, 0),
         (1000, 512, 5000, ffn.VARIANT_1SM, ffn.SCHEDULE_STREAM_K_TAIL, 0),
         (4096, 512, 2752, ffn.VARIANT_2SM, ffn.SCHEDULE_DATA_PARALLEL, 80),
         (777, 256, 4104, ffn.VARIANT_2SM, ffn.SCHEDULE_STREAM_K_TAIL, 112)]


@pytest.mark.parametrize("M,K,N,variant,schedule,bn", CASES)
def test_dynamic_equals_static_and_oracle(cuda_device, M, K, N, variant, schedule, bn):
    d = make_inputs(M, K, N, family="C", seed=9600 + M + N, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    hs = _handle(cuda_device, 1, variant, schedule, bn)
    hd = _handle(cuda_device, 2, variant, schedule, bn)
    o_s = hs.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    outs = [hd.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6) for _ in range(4)]  # epochs 0..3
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, o_s), "dynamic claiming changed the result"
    rows = sorted(set([0, M - 1] + np.random.default_rng(M).choice(M, 12, replace=False).tolist()))
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16", rows=rows)
    check(o_s[rows], ref, f"{M}x{K}x{N} v{variant} s{schedule} bn{bn}")


def test_dynamic_graph_replay_and_alternation(cuda_device):
    """A CUDA graph of three dynamic launches replayed five times, interleaved with eager
    static and dynamic launches of other shapes on other handles sharing nothing, and on
    the same handle with a different shape: every output equals the static result."""
    M, K, N = 1536, 512, 8192
    d = make_inputs(M, K, N, family="C", seed=9700, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    ref = _handle(cuda_device, 1).forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    h = _handle(cuda_device, 2)
    outs = [torch.empty_like(ref) for _ in range(3)]
    for o in outs:
        h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=o)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for o in outs:
            h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=o)
    x2 = t["x"][:700].contiguous()
    ref2 = _handle(cuda_device, 1).forward(x2, t["g"], t["w1"], t["w3"], 1e-6)
    for _ in range(5):
        for o in outs:
            o.zero_()
        g.replay()
        o2 = h.forward(x2, t["g"], t["w1"], t["w3"], 1e-6)  # same handle, other shape, eager
        torch.cuda.synchronize()
        for o in outs:
            assert torch.equal(o, ref)
        assert torch.equal(o2, ref2)


def test_dynamic_option_contract(cuda_device):
    h = ffn.FusedFFN(cuda_device)
    for bad in (-1, 3):
        with pytest.raises(ffn.CuasmError):
            h.set_option(ffn.OPT_DYNAMIC, bad)


def test_l2_persist_full_group(cuda_device):
    """CUASM_OPT_L2_PERSIST: with a persisting-L2 set-aside that holds all of x, the rasterisation
    takes every m-block in one group (W13 read once); results equal the default schedule's
    bitwise (whole tiles, same k-order per tile).  The device-wide limit is reset afterwards."""
    M, K, N = 2048, 2048, 8192
    d = make_inputs(M, K, N, family="C", seed=9800, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    ref = _handle(cuda_device, 1, schedule=ffn.SCHEDULE_DATA_PARALLEL).forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    h = _handle(cuda_device, 0, schedule=ffn.SCHEDULE_DATA_PARALLEL)
    try:
        h.set_option(ffn.OPT_L2_PERSIST, 32 << 20)
        out = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
        torch.cuda.synchronize()
    finally:
        h.set_option(ffn.OPT_L2_PERSIST, 0)
    assert torch.equal(out, ref)
    with pytest.raises(ffn.CuasmError):
        h.set_option(ffn.OPT_L2_PERSIST, -1)
