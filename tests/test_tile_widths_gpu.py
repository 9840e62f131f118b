"""GPU parity of the SwiGLU tile widths (DESIGN.md §6 "Tile widths"; VERDICT r1 next #3,
SURVEY §7 step 9 / Appendix A.5): BN = 64, 80, 96, 112 outputs per 2-SM tile (MMA N =
2 BN), the last epilogue unit 16 columns wide when BN % 32 == 16.

Every width is run forced (CUASM_OPT_TILE_BN) on ragged shapes -- M and N tails, a
partial last unit, one and several k-blocks -- under whole tiles and stream-K, and
compared element by element with the fp64 oracle's fold-aware mode at the [BJ]
tolerance |gpu - ref| <= 2e-2|ref| + 1e-3 (PAPER.md P:560 inputs B, M, N, K).  The
planner's own choices at the tensor-parallel shard shapes, the two W13 cache slots
(128-wide and narrow packs of one weight set) and the fused gather's half-width
stores are checked too.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_inputs
from paper_2501_08071_b200.tp import gather_destinations, shard_bounds, shard_weights

pytestmark = pytest.mark.gpu

RTOL, ATOL = 2e-2, 1e-3
WIDTHS = (64, 80, 96, 112, 120)


def check(gpu, ref, what):
    worst, nbad, maxerr = oracle.tolerance_ratio(gpu.double().cpu().numpy(), ref, RTOL, ATOL)
    assert nbad == 0, f"{what}: {nbad} elements out of tolerance (worst ratio {worst:.3f}, max|err| {maxerr:.3g})"
    return worst


def _run(dev, d, bn, schedule=ffn.SCHEDULE_AUTO, handle=None):
    h = handle or ffn.FusedFFN(dev, torch.bfloat16)
    h.set_option(ffn.OPT_TILE_BN, bn)
    h.set_option(ffn.OPT_SCHEDULE, schedule)
    t = {k: v.to(dev) for k, v in d.items()}
    out = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    torch.cuda.synchronize()
    return out, h


@pytest.mark.parametrize("bn", WIDTHS)
@pytest.mark.parametrize("schedule", [ffn.SCHEDULE_DATA_PARALLEL, ffn.SCHEDULE_STREAM_K_ALL])
@pytest.mark.parametrize("M,K,N", [(300, 512, 0), (1, 64, 8), (16, 256, 1), (513, 1024, 2)])
def test_forced_width_matches_oracle(cuda_device, bn, schedule, M, K, N):
    # N given as an offset past a whole number of tiles: 3 tiles + {24 | 8 | bn+8 | 2bn-8}
    n = {0: 3 * bn + 24, 8: 8, 1: bn + 8, 2: 5 * bn - 8}[N]
    d = make_inputs(M, K, n, family="C", seed=8100 + bn + M + K, dtype="bf16")
    out, h = _run(cuda_device, d, bn, schedule)
    v, _ = h.last_launch()
    assert v == ffn.VARIANT_2SM
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16")
    check(out, ref, f"bn={bn} sched={schedule} {M}x{K}x{n}")


@pytest.mark.parametrize("bn", WIDTHS)
def test_forced_width_exact_family_equals_128(cuda_device, bn):
    """Exact-fold family A: the narrow tile and the 128-wide tile agree with the plain
    definition, and whole-tile results of both widths agree with each other."""
    M, K, N = 384, 768, 4 * bn + 40
    d = make_inputs(M, K, N, family="A", seed=8200 + bn, dtype="bf16")
    out, _ = _run(cuda_device, d, bn, ffn.SCHEDULE_DATA_PARALLEL)
    out128, _ = _run(cuda_device, d, 128, ffn.SCHEDULE_DATA_PARALLEL)
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6)
    check(out, ref, f"bn={bn} family A")
    check(out128, ref, "bn=128 family A")
    diff = (out.float() - out128.float()).abs().max().item()
    assert diff <= 2.0 ** -6 * out128.float().abs().max().item()


@pytest.mark.parametrize("M,N_l", [(2048, 1376), (1024, 2752), (2048, 2752), (512, 5504), (4096, 1376)])
def test_planned_widths_at_shard_shapes(cuda_device, M, N_l):
    """The configuration model's own choice at 7B prefill shard shapes (P = 8 / 4 / 2),
    sampled rows against the oracle; run-to-run bitwise."""
    K = 4096
    plan = ffn.plan_config(M, K, N_l)
    d = make_inputs(M, K, N_l, family="C", seed=8300 + M + N_l, dtype="bf16")
    out, h = _run(cuda_device, d, 0)
    t = {k: v.to(cuda_device) for k, v in d.items()}
    again = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    torch.cuda.synchronize()
    assert torch.equal(out, again), "bitwise run-to-run"
    rng = np.random.default_rng(M)
    rows = sorted({0, M - 1} | set(rng.choice(M, 10, replace=False).tolist()) | {b * 256 for b in range(M // 256)})
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16", rows=rows)
    check(out[rows], ref, f"{M}x{K}x{N_l} plan {plan}")


def test_both_w13_slots_alive(cuda_device):
    """One weight set served at a decode shape (64-wide pack, cluster split-K) and a
    prefill shape whose plan takes another narrow width (a second pack): alternating
    calls re-use both packs and stay correct; an in-place weight change re-packs both."""
    K, N = 4096, 1376
    big = make_inputs(2048, K, N, family="C", seed=8400, dtype="bf16")
    assert ffn.plan_config(2048, K, N)[4] not in (64, 128) and ffn.plan_config(16, K, N)[4] == 64
    small_x = make_inputs(16, K, N, family="C", seed=8401, dtype="bf16")["x"]
    t = {k: v.to(cuda_device) for k, v in big.items()}
    xs = small_x.to(cuda_device)
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    rows = [0, 777, 2047]
    for it in range(2):
        o_big = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
        o_small = h.forward(xs, t["g"], t["w1"], t["w3"], 1e-6)
        torch.cuda.synchronize()
        w1 = big["w1"] if it == 0 else -big["w1"]
        check(o_big[rows], oracle.ffn(big["x"], big["g"], w1, big["w3"], 1e-6, mode="fold_bf16", rows=rows),
              f"prefill it {it}")
        check(o_small, oracle.ffn(small_x, big["g"], w1, big["w3"], 1e-6, mode="fold_bf16"), f"decode it {it}")
        t["w1"].neg_()  # in place: the binding's version counter invalidates every pack


@pytest.mark.parametrize("bn", [80, 112])
def test_fused_gather_half_width_units(cuda_device, bn):
    """f2 with a narrow tile: every simulated peer buffer holds the concatenated shard
    outputs, including the 16-column units stored through the half-width maps."""
    M, K, N, P = 300, 512, 2 * (3 * bn + 16), 2
    d = make_inputs(M, K, N, family="C", seed=8500 + bn, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    bufs = [torch.full((M, N), float("nan"), dtype=torch.bfloat16, device=cuda_device) for _ in range(P)]
    outs = []
    for rank in range(P):
        n0, _ = shard_bounds(N, rank, P)
        w1s, w3s = shard_weights(t["w1"], t["w3"], rank, P)
        h = ffn.FusedFFN(cuda_device)
        h.set_option(ffn.OPT_TILE_BN, bn)
        dst, _ = gather_destinations([b.data_ptr() for b in bufs], n0, 2)
        h.forward_gather(t["x"], t["g"], w1s, w3s, dst, N, 1e-6, keepalive=bufs)
        outs.append(h.forward(t["x"], t["g"], w1s, w3s, 1e-6))
    torch.cuda.synchronize()
    full = torch.cat(outs, dim=1)
    for q in range(P):
        assert torch.equal(bufs[q], full)
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16")
    check(full, ref, f"gather bn={bn}")


def test_tile_bn_option_contract(cuda_device):
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    for bad in (1, 72, 256, -1):
        with pytest.raises(ffn.CuasmError):
            h.set_option(ffn.OPT_TILE_BN, bad)
    # a forced 1-SM variant keeps the 128-wide tile
    d = make_inputs(200, 256, 200, family="C", seed=8600, dtype="bf16")
    h.set_option(ffn.OPT_TILE_BN, 80)
    h.set_variant(ffn.VARIANT_1SM)
    t = {k: v.to(cuda_device) for k, v in d.items()}
    out = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    torch.cuda.synchronize()
    assert h.last_launch()[0] == ffn.VARIANT_1SM
    check(out, oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16"), "1sm with TILE_BN=80")


# ---- the 1-SM 64-output tile with the decode paths (row replication, cluster split-K) ----
@pytest.mark.parametrize("csplit", [1, 2, 4, 6])
@pytest.mark.parametrize("M,K,N", [(16, 4096, 1376), (1, 1024, 200), (32, 2048, 64 * 7 + 8), (48, 1024, 520),
                                   (33, 1024, 200), (64, 2048, 64 * 5 + 8), (64, 4096, 1376), (65, 1024, 392),
                                   (96, 2048, 64 * 9 + 8), (128, 4096, 1376), (300, 2048, 64 * 7 + 24),
                                   (100, 1000, 392)])
def test_decode_paths_bn64(cuda_device, M, K, N, csplit):
    """BN = 64 on the 1-SM kernel: replicated decode rows (csplit 1 = off), and the
    cluster split-K with S CTAs per tile: the push form (TMEM lane quadrant q drains rows 32q..)
    for <= 128 rows per tile when its slots fit the 64 KB staging area (S = 2 and 4 here, 6 up to
    32 rows), the pull form else; 300 rows = three 128-row tiles per n-block."""
    d = make_inputs(M, K, N, family="C", seed=8700 + M + K + csplit, dtype="bf16")
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    h.set_option(ffn.OPT_TILE_BN, 64)
    h.set_variant(ffn.VARIANT_1SM)
    h.set_option(ffn.OPT_CSPLIT, csplit)
    t = {k: v.to(cuda_device) for k, v in d.items()}
    out = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    again = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    torch.cuda.synchronize()
    assert h.last_launch()[0] == ffn.VARIANT_1SM
    assert torch.equal(out, again), "bitwise run-to-run"
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16")
    check(out, ref, f"bn=64 1sm csplit={csplit} {M}x{K}x{N}")


# ---- 4-CTA multicast clusters (CUASM_OPT_MCAST) ----
@pytest.mark.parametrize("bn", [128, 120, 80])
@pytest.mark.parametrize("M,K,N", [(512, 1024, 1000), (300, 512, 520), (1100, 2048, 2064), (2048, 4096, 1376)])
def test_multicast_clusters(cuda_device, bn, M, K, N):
    """Two CTA pairs per cluster on vertically adjacent tiles, W13 halves multicast: equal to
    the default kernel bitwise (whole tiles, same k-order per tile; an odd count of 256-row
    tiles leaves the second pair of the last super-row on rows past M) and to the oracle."""
    d = make_inputs(M, K, N, family="C", seed=8800 + M + bn, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    h0 = ffn.FusedFFN(cuda_device, torch.bfloat16)
    h0.set_option(ffn.OPT_TILE_BN, bn)
    h0.set_variant(ffn.VARIANT_2SM)
    h0.set_option(ffn.OPT_SCHEDULE, ffn.SCHEDULE_DATA_PARALLEL)
    ref_gpu = h0.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    h.set_option(ffn.OPT_TILE_BN, bn)
    h.set_variant(ffn.VARIANT_2SM)
    h.set_option(ffn.OPT_MCAST, 1)
    out = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    again = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    torch.cuda.synchronize()
    assert torch.equal(out, ref_gpu), "multicast clusters changed the result"
    assert torch.equal(out, again)
    rows = sorted(set([0, M - 1] + list(range(0, M, max(1, M // 12)))))
    check(out[rows], oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16", rows=rows),
          f"mcast bn={bn} {M}x{K}x{N}")


@pytest.mark.parametrize("schedule", [ffn.SCHEDULE_DATA_PARALLEL, ffn.SCHEDULE_STREAM_K_ALL])
@pytest.mark.parametrize("M,K,N", [(384, 1024, 11008 // 4), (300, 512, 3 * 120 + 24), (16, 256, 240)])
def test_one_sm_bn120(cuda_device, schedule, M, K, N):
    """The 1-SM kernel with 120-output tiles (24-wide last unit) under whole tiles and stream-K."""
    d = make_inputs(M, K, N, family="C", seed=8900 + M + schedule, dtype="bf16")
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    h.set_option(ffn.OPT_TILE_BN, 120)
    h.set_variant(ffn.VARIANT_1SM)
    h.set_option(ffn.OPT_SCHEDULE, schedule)
    t = {k: v.to(cuda_device) for k, v in d.items()}
    out = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    torch.cuda.synchronize()
    assert h.last_launch()[0] == ffn.VARIANT_1SM
    check(out, oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16"), f"1sm bn120 {M}x{K}x{N}")


@pytest.mark.parametrize("M,K,N,S", [(16, 4096, 1376, 3), (1, 2048, 200, 2), (32, 4096, 2752, 3), (24, 8192, 640, 6)])
def test_thin_a_stages_equal_full(cuda_device, M, K, N, S):
    """CUASM_OPT_THIN_A: the decode split-K kernel with 32-row A stages (more weight stages in
    flight) computes rows 0..M-1 exactly as the full-A kernel does -- bitwise -- and the oracle."""
    d = make_inputs(M, K, N, family="C", seed=8950 + M + S, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    outs = []
    for thin in (0, 1):
        h = ffn.FusedFFN(cuda_device, torch.bfloat16)
        h.set_option(ffn.OPT_TILE_BN, 64)
        h.set_variant(ffn.VARIANT_1SM)
        h.set_option(ffn.OPT_CSPLIT, S)
        h.set_option(ffn.OPT_THIN_A, thin)
        outs.append(h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6))
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    check(outs[1], oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16"), f"thin {M}x{K}x{N} S={S}")
