"""GPU parity of the tall tiles (DESIGN.md §6 "Tall tiles", the
crossover region M = 192..512 of configs[4]): one 80-output n-block over 257..384 rows,
a 256-row tcgen05.mma and a 128-row one (cta_group::2, 64 rows per CTA, folded D
layout) on the same weight stage, the 128-row part's h1 / h3 meeting in shared memory.

Forced on (CUASM_OPT_TALL = 2) over ragged shapes -- every M tail of the 128-row part
(1, 32, 64, 65, 96, 128 rows: the second CTA empty, partial, full), N tails through the
16-wide last unit, one and several k-blocks -- and compared element by element with the
fp64 oracle's fold-aware mode at the [BJ] tolerance |gpu - ref| <= 2e-2|ref| + 1e-3
(PAPER.md P:560 inputs B, M, N, K).  The tall kernel must also agree bitwise with the
ordinary 80-wide 2-SM kernel (same k order per element, same epilogue arithmetic), with
itself across launches and CUDA-graph replays, and with the stand-alone a1 pre-pass.
"""
import pytest
import torch

import oracle
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_inputs

pytestmark = pytest.mark.gpu

RTOL, ATOL = 2e-2, 1e-3


def check(gpu, ref, what):
    worst, nbad, maxerr = oracle.tolerance_ratio(gpu.double().cpu().numpy(), ref, RTOL, ATOL)
    assert nbad == 0, f"{what}: {nbad} elements out of tolerance (worst ratio {worst:.3f}, max|err| {maxerr:.3g})"
    return worst


def _handle(dev, tall):
    h = ffn.FusedFFN(dev, torch.bfloat16)
    h.set_option(ffn.OPT_TALL, tall)
    return h


def _fwd(h, t, out=None):
    o = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    torch.cuda.synchronize()
    return o


@pytest.mark.parametrize("M", [257, 288, 320, 321, 352, 384])
@pytest.mark.parametrize("K,N", [(64, 248), (512, 88), (1024, 400), (320, 8), (200, 168)])
def test_forced_tall_matches_oracle(cuda_device, M, K, N):
    d = make_inputs(M, K, N, family="C", seed=9100 + M + K + N, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    h = _handle(cuda_device, 2)
    out = _fwd(h, t)
    assert h.last_launch()[0] == ffn.VARIANT_2SM
    assert ffn.plan_config(M, K, N)[0] in ("tall", "1sm", "2sm")
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16")
    check(out, ref, f"tall {M}x{K}x{N}")


@pytest.mark.parametrize("M", [260, 300, 384])
def test_tall_bitwise_equals_80_wide_tiles(cuda_device, M):
    """Same products in the same k order per element as the ordinary 80-wide kernel
    (two 256-row tiles), same epilogue arithmetic: bitwise equal outputs."""
    K, N = 768, 5 * 80 - 8
    d = make_inputs(M, K, N, family="C", seed=9200 + M, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    tall = _fwd(_handle(cuda_device, 2), t)
    h80 = _handle(cuda_device, 1)
    h80.set_option(ffn.OPT_TILE_BN, 80)
    h80.set_option(ffn.OPT_VARIANT, ffn.VARIANT_2SM)
    h80.set_option(ffn.OPT_SCHEDULE, ffn.SCHEDULE_DATA_PARALLEL)
    wide = _fwd(h80, t)
    assert torch.equal(tall, wide), (tall.float() - wide.float()).abs().max().item()


def test_tall_exact_family(cuda_device):
    """Family A (exact fold): the tall tile reproduces the plain definition."""
    M, K, N = 352, 512, 240
    d = make_inputs(M, K, N, family="A", seed=9300, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    out = _fwd(_handle(cuda_device, 2), t)
    check(out, oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6), "tall family A")


def test_tall_separate_prepass_and_graph_replay(cuda_device):
    """Fused a1 vs the stand-alone pre-pass kernel, and CUDA-graph replays interleaved with
    other shapes on the same handle (the self-resetting r-block bookkeeping)."""
    M, K, N = 330, 1024, 328
    d = make_inputs(M, K, N, family="C", seed=9400, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    h = _handle(cuda_device, 2)
    fused = _fwd(h, t)
    h2 = _handle(cuda_device, 2)
    h2.set_option(ffn.OPT_FUSED_NORM, 0)
    sep = _fwd(h2, t)
    assert torch.equal(fused, sep)
    d2 = make_inputs(200, K, N, family="C", seed=9401, dtype="bf16")
    t2 = {k: v.to(cuda_device) for k, v in d2.items()}
    o2 = torch.empty((200, N), dtype=torch.bfloat16, device=cuda_device)
    out = torch.empty_like(fused)
    _fwd(h, t, out)
    _fwd(h, t2, o2)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
        h.forward(t2["x"], t2["g"], t2["w1"], t2["w3"], 1e-6, out=o2)
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, fused)
    ref2 = oracle.ffn(d2["x"], d2["g"], d2["w1"], d2["w3"], 1e-6, mode="fold_bf16")
    check(o2, ref2, "200-row forward between tall launches")


@pytest.mark.parametrize("M", [288, 384])
def test_tall_full_size_sweep_shape(cuda_device, M):
    """configs[4]'s K = 4096, N = 11008 at crossover M, forced tall: sampled rows (both
    parts, both CTAs' halves of the 128-row part) against the oracle."""
    K, N = 4096, 11008
    d = make_inputs(M, K, N, family="C", seed=9500 + M, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    out = _fwd(_handle(cuda_device, 2), t)
    rows = sorted({0, 127, 128, 255, 256, 300, 319, 320, M - 1} & set(range(M)))
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16", rows=rows)
    check(out[rows], ref, f"tall full size M={M}")


def test_tall_fused_gather_simulated_peers(cuda_device):
    """Step a4 fused into the tall tile's epilogue (both parts): P = 3 simulated peer buffers
    each receive every rank's columns, equal to the concatenated plain forwards."""
    from paper_2501_08071_b200.tp import gather_destinations, shard_bounds, shard_weights
    M, K, N, P = 300, 512, 3 * 248, 3
    d = make_inputs(M, K, N, family="C", seed=9900, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    bufs = [torch.full((M, N), float("nan"), dtype=torch.bfloat16, device=cuda_device) for _ in range(P)]
    shard_outs = []
    for rank in range(P):
        n0, _ = shard_bounds(N, rank, P)
        w1s, w3s = shard_weights(t["w1"], t["w3"], rank, P)
        h = _handle(cuda_device, 2)
        dst, mc = gather_destinations([b.data_ptr() for b in bufs], n0, 2)
        h.forward_gather(t["x"], t["g"], w1s, w3s, dst, N, 1e-6, keepalive=bufs)
        shard_outs.append(h.forward(t["x"], t["g"], w1s, w3s, 1e-6))
    torch.cuda.synchronize()
    full = torch.cat(shard_outs, dim=1)
    for q in range(P):
        assert torch.equal(bufs[q], full), f"peer buffer {q}"
    check(full, oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16"), "tall gather")
