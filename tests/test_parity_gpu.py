"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Acceptance (BASELINE.json north_star): per element
    |gpu - oracle| <= 2e-2*|oracle| + 1e-3,   NaN fails.
Reference mode per input family (R4): exact-fold families A/B/T are
compared with the plain definition; full-entropy family C with the
fold-aware oracle (g folded into the weights in bf16 first).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2501_08071_b200 as ffn
from ffn_inputs import CONFIGS, make_inputs, seed_for

pytestmark = pytest.mark.gpu

RTOL, ATOL = 2e-2, 1e-3
TORCH_DT = {"bf16": torch.bfloat16, "fp32": torch.float32}


def run_gpu(d, eps, dtype, variant=ffn.VARIANT_AUTO, handle=None, schedule=ffn.SCHEDULE_AUTO):
    dev = torch.device("cuda:0")
    h = handle or ffn.FusedFFN(dev, TORCH_DT[dtype])
    h.set_variant(variant)
    h.set_option(ffn.OPT_SCHEDULE, schedule)
    t = {k: v.to(dev) for k, v in d.items()}
    out = h.forward(t["x"], t["g"], t["w1"], t["w3"], eps)
    torch.cuda.synchronize()
    return out, h


def check(gpu, ref, what):
    worst, nbad, maxerr = oracle.tolerance_ratio(gpu.double().cpu().numpy(), ref, RTOL, ATOL)
    assert nbad == 0, f"{what}: {nbad} elements out of tolerance (worst ratio {worst:.3f}, max|err| {maxerr:.3g})"
    return worst


def ref_mode(family, dtype):
    if family == "C":
        return "fold_bf16" if dtype == "bf16" else "fold_tf32"
    return "plain"


# ------------------------------------------------------------------ a1 ------
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("M,K", [(1, 8), (7, 64), (300, 4096), (16, 8192), (33, 1000)])
def test_prepass_matches_oracle(cuda_device, dtype, M, K):
    d = make_inputs(M, K, 8, family="C", seed=100 + M, dtype=dtype)
    h = ffn.FusedFFN(cuda_device, TORCH_DT[dtype])
    r = h.rms_inv(d["x"].to(cuda_device), 1e-6).cpu().double().numpy()
    ref = oracle.rms_inv(d["x"], 1e-6)
    np.testing.assert_allclose(r, ref, rtol=2e-6)


# ------------------------------------------------------------------ a0 ------
def unpack_w13(packed, N, K, BK):
    """Invert the k-block-tiled layout of cuasm_ffn_get_packed:
    [nb][kb][j*128 + rr][i] -> (W1g, W3g) as [N_pad, K_pad] arrays."""
    nblk, kblk = (N + 127) // 128, (K + BK - 1) // BK
    a = packed.reshape(nblk, kblk, 2, 128, BK)
    return [a[:, :, j].transpose(0, 2, 1, 3).reshape(nblk * 128, kblk * BK) for j in (0, 1)]


@pytest.mark.parametrize("N,K", [(128, 64), (520, 200), (1376, 256)])
def test_pack_is_bitwise_the_oracle_fold(cuda_device, N, K):
    d = make_inputs(1, K, N, family="C", seed=200 + N, dtype="bf16")
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    t = {k: v.to(cuda_device) for k, v in d.items()}
    h.prepare(t["g"], t["w1"], t["w3"])
    torch.cuda.synchronize()
    packed = h.packed_weights().view(torch.int16).numpy().view(np.uint16)
    for got, w in zip(unpack_w13(packed, N, K, 64), (d["w1"], d["w3"])):
        assert np.array_equal(got[:N, :K], oracle.fold(w, d["g"]))
        assert np.all(got[N:] == 0) and np.all(got[:, K:] == 0)


def test_pack_fp32_is_the_oracle_tf32_fold(cuda_device):
    N, K = 136, 72
    d = make_inputs(1, K, N, family="C", seed=300, dtype="fp32")
    h = ffn.FusedFFN(cuda_device, torch.float32)
    t = {k: v.to(cuda_device) for k, v in d.items()}
    h.prepare(t["g"], t["w1"], t["w3"])
    torch.cuda.synchronize()
    packed = h.packed_weights().numpy()
    # fp32 handles pack the duplicated-K layout of the split-x contraction (pack.cuh,
    # DESIGN.md R5): packed K = 2 * Kp, columns [Kp, 2Kp) repeat columns [0, Kp)
    Kp = (K + 31) // 32 * 32
    for got, w in zip(unpack_w13(packed, N, 2 * Kp, 32), (d["w1"], d["w3"])):
        assert np.array_equal(got[:N, :K], oracle.fold(w, d["g"]))
        assert np.array_equal(got[:, Kp:], got[:, :Kp])
        assert np.all(got[N:] == 0) and np.all(got[:, K:Kp] == 0)


# --------------------------------------------------------- whole path -------
SMALL_SHAPES = [
    # (M, K, N): single tile; M/N/K tails; several tiles in every dimension
    (1, 64, 128),
    (16, 64, 128),
    (128, 128, 256),
    (300, 512, 520),
    (129, 200, 136),
    (257, 1024, 1000),
    (640, 320, 1408),
    (33, 512, 1032),     # rows replicated twice over the TMEM quadrants (33 <= M <= 64)
    (64, 256, 264),
]


@pytest.mark.parametrize("variant", [ffn.VARIANT_1SM, ffn.VARIANT_2SM])
@pytest.mark.parametrize("family", ["A", "B", "C", "L"])
@pytest.mark.parametrize("M,K,N", SMALL_SHAPES)
def test_parity_small_bf16(cuda_device, M, K, N, family, variant):
    d = make_inputs(M, K, N, family=family, seed=1000 + M + K + N, dtype="bf16")
    out, _ = run_gpu(d, 1e-6, "bf16", variant)
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode=ref_mode(family, "bf16"))
    check(out, ref, f"{family} {M}x{K}x{N} v{variant}")


SCHED_SHAPES = [
    (16, 4096, 512),     # 4-8 tiles over 74-148 clusters: many contributors per tile
    (48, 4096, 1376),    # twice-replicated rows, few tiles split by stream-K
    (300, 1024, 1000),   # ragged M and N, a few tiles
    (1000, 512, 2056),   # several waves + tail
    (2048, 4096, 1376),  # 7B prefill, 8-way shard width (88 / 176 tiles)
]


@pytest.mark.parametrize("schedule", [ffn.SCHEDULE_DATA_PARALLEL, ffn.SCHEDULE_STREAM_K_ALL,
                                      ffn.SCHEDULE_STREAM_K_TAIL, ffn.SCHEDULE_AUTO])
@pytest.mark.parametrize("variant", [ffn.VARIANT_1SM, ffn.VARIANT_2SM])
@pytest.mark.parametrize("M,K,N", SCHED_SHAPES)
def test_parity_schedules(cuda_device, M, K, N, variant, schedule):
    d = make_inputs(M, K, N, family="C", seed=4000 + M + N, dtype="bf16")
    out, h = run_gpu(d, 1e-6, "bf16", variant, schedule=schedule)
    again, _ = run_gpu(d, 1e-6, "bf16", variant, handle=h, schedule=schedule)
    assert torch.equal(out, again), "bitwise run-to-run determinism"
    rows = sorted(set([0, M - 1] + list(range(0, M, max(1, M // 40)))))
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16", rows=rows)
    check(out[rows], ref, f"sched {schedule} v{variant} {M}x{K}x{N}")


@pytest.mark.parametrize("variant", [ffn.VARIANT_1SM, ffn.VARIANT_2SM])
@pytest.mark.parametrize("M,K,N", [(16, 64, 128), (5, 64, 136), (200, 256, 264), (40, 1024, 392)])
def test_parity_small_fp32(cuda_device, M, K, N, variant):
    d = make_inputs(M, K, N, family="T", seed=2000 + M, dtype="fp32")
    out, _ = run_gpu(d, 1e-6, "fp32", variant)
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="plain")
    check(out, ref, f"T {M}x{K}x{N}")


def test_tiny_config_fp32(cuda_device):
    """BASELINE.json configs[0]: M=16 K=64 N=128 fp32 eps=1e-6, full oracle."""
    c = CONFIGS["tiny"]
    for run in range(5):
        d = make_inputs(c["M"], c["K"], c["N"], family="T", seed=seed_for(c["idx"], run), dtype="fp32")
        out, _ = run_gpu(d, c["eps"], "fp32")
        ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], c["eps"])
        check(out, ref, f"tiny run {run}")


def _sample_rows(M, n, seed):
    rng = np.random.default_rng(seed)
    rows = set([0, M - 1]) | set(rng.choice(M, size=min(n, M), replace=False).tolist())
    # rows in the last (ragged or full) 128-row tile
    rows |= set(range(max(0, M - 3), M))
    return sorted(rows)


@pytest.mark.parametrize("name,family", [("llama7b_prefill", "B"), ("llama7b_prefill", "C"),
                                         ("llama7b_decode", "A"), ("llama7b_decode", "C")])
def test_full_size_7b(cuda_device, name, family):
    c = CONFIGS[name]
    d = make_inputs(c["M"], c["K"], c["N"], family=family, seed=seed_for(c["idx"]), dtype="bf16")
    out, _ = run_gpu(d, c["eps"], "bf16")
    rows = _sample_rows(c["M"], 24, 7) if c["M"] > 64 else list(range(c["M"]))
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], c["eps"], mode=ref_mode(family, "bf16"), rows=rows)
    check(out[rows], ref, name)
    assert torch.isfinite(out).all()


def test_full_size_70b_shard(cuda_device):
    """70B FFN, rank 0 of an 8-way N-shard (N_l = 3584) at full M, K."""
    c = CONFIGS["llama70b"]
    P = 8
    N_l = c["N"] // P
    d = make_inputs(c["M"], c["K"], N_l, family="B", seed=seed_for(c["idx"]), dtype="bf16")
    out, _ = run_gpu(d, c["eps"], "bf16")
    rows = _sample_rows(c["M"], 6, 8)
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], c["eps"], rows=rows)
    check(out[rows], ref, "70b shard")


# ---------------------------------------------------------- invariants ------
def test_invariants_bitwise(cuda_device):
    M, K, N = 384, 512, 640
    d = make_inputs(M, K, N, family="C", seed=3000, dtype="bf16")
    base, h = run_gpu(d, 0.0, "bf16")
    again, _ = run_gpu(d, 0.0, "bf16", handle=h)
    assert torch.equal(base, again), "run-to-run determinism"
    # row permutation moves rows between tiles; with the whole-tile schedule a
    # row's k-summation is then independent of its tile, so equivariance is bitwise
    dps = ffn.SCHEDULE_DATA_PARALLEL
    base_dp, _ = run_gpu(d, 0.0, "bf16", handle=h, schedule=dps)
    perm = torch.randperm(M, generator=torch.Generator().manual_seed(0))
    dp = dict(d, x=d["x"][perm].contiguous())
    outp, _ = run_gpu(dp, 0.0, "bf16", handle=h, schedule=dps)
    assert torch.equal(outp, base_dp[perm.to(base.device)]), "row permutation equivariance"
    h.set_option(ffn.OPT_SCHEDULE, ffn.SCHEDULE_AUTO)
    d2 = dict(d, x=(d["x"].float() * 4.0).to(torch.bfloat16))
    out2, _ = run_gpu(d2, 0.0, "bf16", handle=h)  # same schedule as `base` (auto)
    assert torch.equal(out2, base), "x -> 4x at eps=0 leaves out unchanged"
    d3 = dict(d, w3=(d["w3"].float() * 2.0).to(torch.bfloat16))
    out3, _ = run_gpu(d3, 0.0, "bf16", handle=h)
    assert torch.equal(out3.float(), base.float() * 2.0), "W3 -> 2 W3 doubles out exactly"


def test_n_shard_equals_columns(cuda_device):
    M, K, N = 256, 256, 1024
    d = make_inputs(M, K, N, family="C", seed=3100, dtype="bf16")
    # whole-tile schedule: the k-summation of an output then does not depend on
    # where stream-K cuts fall, which move with the shard width
    dp = ffn.SCHEDULE_DATA_PARALLEL
    full, h = run_gpu(d, 1e-6, "bf16", schedule=dp)
    for n0, n1 in ((0, 512), (512, 1024), (256, 392)):
        ds = dict(d, w1=d["w1"][n0:n1].contiguous(), w3=d["w3"][n0:n1].contiguous())
        part, _ = run_gpu(ds, 1e-6, "bf16", handle=h, schedule=dp)
        assert torch.equal(part, full[:, n0:n1]), (n0, n1)


def test_variants_agree(cuda_device):
    M, K, N = 512, 1024, 768
    d = make_inputs(M, K, N, family="C", seed=3200, dtype="bf16")
    dp = ffn.SCHEDULE_DATA_PARALLEL
    a, h = run_gpu(d, 1e-6, "bf16", ffn.VARIANT_1SM, schedule=dp)
    b, _ = run_gpu(d, 1e-6, "bf16", ffn.VARIANT_2SM, handle=h, schedule=dp)
    assert torch.equal(a, b)


def test_edge_cases(cuda_device):
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    K, N = 64, 128
    d = {k: v.to(cuda_device) for k, v in make_inputs(4, K, N, family="C", seed=3300, dtype="bf16").items()}
    # M == 0: OK, nothing launched
    out = h.forward(d["x"][:0], d["g"], d["w1"], d["w3"])
    assert out.shape == (0, N)
    assert h.last_launch()[1] == 0
    # zero row with eps > 0 -> exactly 0
    x = d["x"].clone()
    x[1] = 0
    out = h.forward(x, d["g"], d["w1"], d["w3"], 1e-6)
    torch.cuda.synchronize()
    assert torch.all(out[1] == 0)
    # zero W1 -> SiLU(0) = 0 everywhere
    out = h.forward(d["x"], d["g"], torch.zeros_like(d["w1"]), d["w3"])
    torch.cuda.synchronize()
    assert torch.all(out == 0)


def test_contract_errors_do_not_launch(cuda_device):
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    K, N = 64, 128
    d = {k: v.to(cuda_device) for k, v in make_inputs(4, K, N, family="C", seed=3400, dtype="bf16").items()}
    out = torch.full((4, N), 7.0, dtype=torch.bfloat16, device=cuda_device)
    lib = h.lib
    p = lambda t: t.data_ptr()
    s = torch.cuda.current_stream().cuda_stream
    cases = [
        (p(d["x"]), p(d["g"]), p(d["w1"]), p(d["w3"]), p(out), 4, 60, N, 1e-6),   # K % 8
        (p(d["x"]), p(d["g"]), p(d["w1"]), p(d["w3"]), p(out), 4, K, 100, 1e-6),  # N % 8
        (p(d["x"]), p(d["g"]), p(d["w1"]), p(d["w3"]), p(out), -1, K, N, 1e-6),   # M < 0
        (p(d["x"]), p(d["g"]), p(d["w1"]), p(d["w3"]), p(out), 4, K, N, -1.0),    # eps < 0
        (p(d["x"]), p(d["g"]), p(d["w1"]), p(d["w3"]), p(out), 4, K, N, float("nan")),
        (p(d["x"]) + 2, p(d["g"]), p(d["w1"]), p(d["w3"]), p(out), 4, K, N, 1e-6),  # misaligned
        (0, p(d["g"]), p(d["w1"]), p(d["w3"]), p(out), 4, K, N, 1e-6),             # NULL
    ]
    for c in cases:
        st = lib.cuasm_ffn_forward(h._h, *c, s)
        assert st == ffn.ERR_INVALID_ARG, c
        assert lib.cuasm_ffn_last_error(h._h)
    torch.cuda.synchronize()
    assert torch.all(out == 7.0)


@pytest.mark.parametrize("M,K,N", [(16, 4096, 1024), (1000, 512, 2056), (2048, 1024, 1376)])
def test_fused_norm_matches_separate_prepass(cuda_device, M, K, N):
    """a1 inside the GEMM (default) and the stand-alone pre-pass kernel run the
    same per-row code, so the outputs are bitwise identical."""
    d = make_inputs(M, K, N, family="C", seed=3700 + M, dtype="bf16")
    fused, h = run_gpu(d, 1e-6, "bf16")
    assert h.last_launch()[1] == 1
    h.set_option(ffn.OPT_FUSED_NORM, 0)
    sep, _ = run_gpu(d, 1e-6, "bf16", handle=h)
    assert h.last_launch()[1] == 2
    assert torch.equal(fused, sep)
    h.set_option(ffn.OPT_FUSED_NORM, 1)
    again, _ = run_gpu(d, 1e-6, "bf16", handle=h)  # grid counters were reset by the last launch
    assert torch.equal(fused, again)


def test_cuda_graph_replay_matches_eager(cuda_device):
    """The forward (pre-pass + stream-K GEMM) captured in a CUDA graph and
    replayed: identical to the eager call every time (flags are consumed and
    reset inside the kernel, so replays need no per-launch host state)."""
    M, K, N = 1000, 512, 2056
    d = make_inputs(M, K, N, family="C", seed=3600, dtype="bf16")
    eager, h = run_gpu(d, 1e-6, "bf16", ffn.VARIANT_2SM, schedule=ffn.SCHEDULE_STREAM_K_ALL)
    t = {k: v.to(cuda_device) for k, v in d.items()}
    out = torch.empty_like(eager)
    h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)  # warm (weights cached)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, eager)


@pytest.mark.parametrize("M", [200, 2100])
def test_forward_host_matches_device_path(cuda_device, M):
    """forward_host (pinned host in/out; M >= 1024 runs as overlapped row chunks)
    equals the device path: bitwise when unchunked, within tolerance of the
    oracle when chunked (a chunk's stream-K cuts differ from the whole's)."""
    K, N = 256, 384
    d = make_inputs(M, K, N, family="C", seed=3500 + M, dtype="bf16")
    dev, h = run_gpu(d, 1e-6, "bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    host = h.forward_host(d["x"].pin_memory(), t["g"], t["w1"], t["w3"], 1e-6)
    if M < 1024:
        assert torch.equal(host, dev.cpu())
    else:
        rows = sorted(set([0, M - 1] + list(range(0, M, 37))))
        ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16", rows=rows)
        check(host[rows], ref, "forward_host chunked")
        # async variant: ordered on the caller's stream
        out2 = torch.empty_like(host).pin_memory()
        h.forward_host(d["x"].pin_memory(), t["g"], t["w1"], t["w3"], 1e-6, out_host=out2, sync=False)
        torch.cuda.current_stream().synchronize()
        assert torch.equal(out2, host)


# --------------------------------------------- f3: mmLeakyReLu, f1: FFN block ----
@pytest.mark.parametrize("tile_n", [0, 128, 256])
@pytest.mark.parametrize("variant", [ffn.VARIANT_AUTO, ffn.VARIANT_1SM, ffn.VARIANT_2SM])
@pytest.mark.parametrize("M,K,N", [(512, 2048, 512), (300, 520, 776), (1, 64, 256), (1000, 1024, 2056)])
@pytest.mark.parametrize("act,alpha", [("leaky_relu", 0.01), ("identity", 0.0)])
def test_gemm_act_parity(cuda_device, M, K, N, act, alpha, variant, tile_n):
    """The paper's mmLeakyReLu (B,M,N,K = 1,512,512,2048) and plain GEMM,
    256- and 128-wide tiles."""
    d = make_inputs(M, K, N, family="C", seed=5000 + M + N, dtype="bf16")
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    h.set_variant(variant)
    h.set_option(ffn.OPT_TILE_N, tile_n)
    x, w = d["x"].to(cuda_device), d["w1"].to(cuda_device)
    out = h.gemm_act(x, w, act, alpha)
    torch.cuda.synchronize()
    ref = oracle.gemm_act(d["x"], d["w1"], act, alpha)
    check(out, ref, f"gemm_act {act} {M}x{K}x{N} v{variant}")
    again = h.gemm_act(x, w, act, alpha)
    torch.cuda.synchronize()
    assert torch.equal(out, again)


def test_gemm_act_fp32_tf32_exact_inputs(cuda_device):
    d = make_inputs(64, 96, 264, family="T", seed=5100, dtype="fp32")
    h = ffn.FusedFFN(cuda_device, torch.float32)
    out = h.gemm_act(d["x"].to(cuda_device), d["w1"].to(cuda_device), "leaky_relu", 0.25)
    torch.cuda.synchronize()
    check(out, oracle.gemm_act(d["x"], d["w1"], "leaky_relu", 0.25), "gemm_act fp32")


@pytest.mark.parametrize("M,K,N", [(16, 512, 1024), (300, 256, 648), (2048, 1024, 2816)])
def test_ffn_block_parity(cuda_device, M, K, N):
    """out = (SiLU(xn W1^T) * (xn W3^T)) W2^T, the hidden rounded to bf16 between
    the two GEMMs (reading R13), g folded into bf16 weights (R4).

    A hidden element whose exact value lies within the fp32 accumulation error of
    a bf16 rounding boundary may round either way, and which way depends on the
    summation grouping (the tile schedule), so the block output is checked in the
    steps the arithmetic fixes: (a) the hidden against the oracle FFN, at the
    [BJ] tolerance; (b) the output against the exact product of the hidden the
    GPU produced with W2; (c) the output against the oracle's rounded-hidden
    block, allowing exactly the contribution of the hidden elements the two
    rounded differently (|sum_n dh_n W2[k,n]|, dh = gpu hidden - oracle hidden)."""
    d = make_inputs(M, K, N, family="C", seed=5200 + M, dtype="bf16")
    w2 = make_inputs(1, N, K, family="C", seed=5300 + M, dtype="bf16")["w1"]   # [K, N]
    t = {k: v.to(cuda_device) for k, v in d.items()}
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    y = h.block_forward(t["x"], t["g"], t["w1"], t["w3"], w2.to(cuda_device), 1e-6)
    torch.cuda.synchronize()
    assert y.shape == (M, K)
    rows = sorted(set([0, M - 1] + list(range(0, M, max(1, M // 24)))))
    # the hidden it used is exactly the fused FFN's output
    hid = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    y2 = h.gemm_act(hid, w2.to(cuda_device), "identity")
    torch.cuda.synchronize()
    assert torch.equal(y, y2)
    hid_rows = hid[rows].double().cpu()
    # (a) the hidden = the fused FFN, at the [BJ] tolerance against the oracle
    ref_h = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16", rows=rows)
    check(hid[rows], ref_h, f"ffn block hidden {M}x{K}x{N}")
    # (b) the down projection of that hidden, against its exact product
    w2d = w2.double()
    check(y[rows], (hid_rows @ w2d.T).numpy(), f"ffn block down projection {M}x{K}x{N}")
    # (c) the block against the oracle, up to the hidden elements rounded the other way
    ref = oracle.ffn_block(d["x"], d["g"], d["w1"], d["w3"], w2, 1e-6, mode="fold_bf16", round_hidden=True,
                           rows=rows)
    ref_hr = torch.from_numpy(ref_h).to(torch.bfloat16).double()
    flip = ((hid_rows - ref_hr) @ w2d.T).abs().numpy()
    err = np.abs(y[rows].double().cpu().numpy() - ref)
    assert (err <= RTOL * np.abs(ref) + ATOL + flip * (1 + 1e-6)).all(), f"ffn block {M}x{K}x{N} vs oracle"
    nflip = int((hid_rows != ref_hr).sum())
    assert nflip <= max(8, hid_rows.numel() // 200), f"{nflip} hidden elements rounded differently"


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("M,K", [(4096, 2048), (7, 64), (33, 8192), (300, 1000)])
def test_rmsnorm_parity(cuda_device, dtype, M, K):
    """The paper's stand-alone rmsnorm (4096 rows x 2048 features)."""
    d = make_inputs(M, K, 8, family="L", seed=5400 + M, dtype=dtype)
    h = ffn.FusedFFN(cuda_device, TORCH_DT[dtype])
    out = h.rmsnorm(d["x"].to(cuda_device), d["g"].to(cuda_device), 1e-6)
    torch.cuda.synchronize()
    rows = sorted(set([0, M - 1] + list(range(0, M, max(1, M // 64)))))
    ref = oracle.rmsnorm(d["x"][rows], d["g"], 1e-6)
    check(out[rows], ref, f"rmsnorm {dtype} {M}x{K}")


# ------------------------------------------------------------ shape fuzzing ---
def _fuzz_cases(n, seed):
    rng = np.random.default_rng(seed)
    cases = []
    for i in range(n):
        M = int(rng.choice([rng.integers(1, 130), rng.integers(129, 700), rng.integers(700, 3000)]))
        K = 8 * int(rng.integers(1, 520))
        N = 8 * int(rng.integers(1, 700))
        cases.append((i, M, K, N, int(rng.integers(0, 3)), int(rng.integers(0, 3))))
    return cases


@pytest.mark.parametrize("i,M,K,N,variant,schedule", _fuzz_cases(24, 777))
def test_fuzz_ffn_shapes(cuda_device, i, M, K, N, variant, schedule):
    """Random (M, K, N) incl. K not a multiple of 64, N not of 128, M tails,
    every variant x schedule: parity on sampled rows + run-to-run determinism."""
    d = make_inputs(M, K, N, family="C", seed=9000 + i, dtype="bf16")
    out, h = run_gpu(d, 1e-6, "bf16", variant, schedule=schedule)
    again, _ = run_gpu(d, 1e-6, "bf16", variant, handle=h, schedule=schedule)
    assert torch.equal(out, again)
    rows = sorted(set([0, M - 1] + list(range(0, M, max(1, M // 16)))))
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16", rows=rows)
    check(out[rows], ref, f"fuzz {i}: {M}x{K}x{N} v{variant} s{schedule}")


@pytest.mark.parametrize("i,M,K,N,variant,schedule", _fuzz_cases(16, 778))
def test_fuzz_gemm_act_shapes(cuda_device, i, M, K, N, variant, schedule):
    d = make_inputs(M, K, N, family="C", seed=9100 + i, dtype="bf16")
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    h.set_variant(variant)
    h.set_option(ffn.OPT_SCHEDULE, schedule)
    h.set_option(ffn.OPT_TILE_N, (0, 128, 256)[i % 3])
    out = h.gemm_act(d["x"].to(cuda_device), d["w1"].to(cuda_device), "leaky_relu", 0.125)
    torch.cuda.synchronize()
    rows = sorted(set([0, M - 1] + list(range(0, M, max(1, M // 16)))))
    ref = oracle.gemm_act(d["x"][rows], d["w1"], "leaky_relu", 0.125)
    check(out[rows], ref, f"fuzz gemm {i}: {M}x{K}x{N} v{variant} s{schedule}")


def test_block_forward_fp32(cuda_device):
    M, K, N = 40, 64, 136
    d = make_inputs(M, K, N, family="T", seed=9200, dtype="fp32")
    w2 = make_inputs(1, N, K, family="T", seed=9201, dtype="fp32")["w1"]
    t = {k: v.to(cuda_device) for k, v in d.items()}
    h = ffn.FusedFFN(cuda_device, torch.float32)
    y = h.block_forward(t["x"], t["g"], t["w1"], t["w3"], w2.to(cuda_device), 1e-6)
    torch.cuda.synchronize()
    # fp32 hidden: the MMA reads it as tf32 (truncated), so compare with a tf32-rounded
    # hidden only loosely: the tolerance covers 2^-11 relative per term
    ref = oracle.ffn_block(d["x"], d["g"], d["w1"], d["w3"], w2, 1e-6, mode="plain")
    check(y, ref, "block fp32")


def test_new_entry_points_validate_arguments(cuda_device):
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    lib, s = h.lib, torch.cuda.current_stream().cuda_stream
    x = torch.zeros((4, 64), dtype=torch.bfloat16, device=cuda_device)
    w = torch.zeros((128, 64), dtype=torch.bfloat16, device=cuda_device)
    out = torch.full((4, 128), 3.0, dtype=torch.bfloat16, device=cuda_device)
    p = lambda t: t.data_ptr()
    assert lib.cuasm_gemm_act(h._h, p(x), p(w), p(out), 4, 60, 128, 0, 0.0, s) == ffn.ERR_INVALID_ARG
    assert lib.cuasm_gemm_act(h._h, p(x), p(w), p(out), 4, 64, 128, 7, 0.0, s) == ffn.ERR_INVALID_ARG
    assert lib.cuasm_gemm_act(h._h, p(x), 0, p(out), 4, 64, 128, 0, 0.0, s) == ffn.ERR_INVALID_ARG
    assert lib.cuasm_gemm_act(h._h, p(x), p(w), p(out), 4, 64, 128, 1, float("nan"), s) == ffn.ERR_INVALID_ARG
    assert lib.cuasm_rmsnorm(h._h, p(x), p(w), p(out), 4, 60, 1e-6, s) == ffn.ERR_INVALID_ARG
    assert lib.cuasm_rmsnorm(h._h, p(x), p(w), p(out), 4, 64, -1.0, s) == ffn.ERR_INVALID_ARG
    assert lib.cuasm_ffn_block_forward(h._h, p(x), p(w), p(w), p(w), 0, p(out), 4, 64, 128, 1e-6, s) == \
        ffn.ERR_INVALID_ARG
    torch.cuda.synchronize()
    assert torch.all(out == 3.0)


def test_full_size_70b_unsharded(cuda_device):
    """BASELINE.json configs[3] at P=1: M=4096 K=8192 N=28672 (0.94 GB of folded
    weights), sampled rows incl. the first/last row block, vs the oracle."""
    c = CONFIGS["llama70b"]
    d = make_inputs(c["M"], c["K"], c["N"], family="A", seed=seed_for(c["idx"], 1), dtype="bf16")
    out, _ = run_gpu(d, c["eps"], "bf16")
    rows = [0, 1, 255, 256, 2047, 4095]
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], c["eps"], rows=rows)
    check(out[rows], ref, "70b P=1")
    assert torch.isfinite(out).all()


# ---------------------------------------------- epilogue gate at the extremes ---
@pytest.mark.parametrize("schedule", [ffn.SCHEDULE_DATA_PARALLEL, ffn.SCHEDULE_STREAM_K_ALL])
def test_gate_extremes(cuda_device, schedule):
    """The gate's one-MUFU form (dual_gemm.cuh silu_gate: ex2 + bit-trick seed +
    two Newton steps, t clamped per row) against the fp64 oracle where it is
    most fragile: |h1| up to ~10^3 (exp overflow / full saturation), rows of
    magnitude 1e4 (k = ms + eps ~ 1e8 moves the clamp), and the NaN cases of
    reading R8 (zero row with eps = 0) and of a NaN input."""
    M, K, N = 8, 256, 256
    d = make_inputs(M, K, N, family="C", seed=3400, dtype="bf16")
    x = d["x"].clone()
    x[2] *= 1e4                      # large row: clamp at 120 - log2(k)
    w1 = d["w1"].clone()
    w1[:64] *= 512.0                 # |h1| ~ 10^2..10^3 for the first 64 outputs
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    h.set_option(ffn.OPT_SCHEDULE, schedule)
    dv = {"x": x.to(cuda_device), "g": d["g"].to(cuda_device), "w1": w1.to(cuda_device), "w3": d["w3"].to(cuda_device)}
    out = h.forward(dv["x"], dv["g"], dv["w1"], dv["w3"], 1e-6)
    torch.cuda.synchronize()
    ref = oracle.ffn(x, d["g"], w1, d["w3"], 1e-6, mode="fold_bf16")
    assert not torch.isnan(out).any()
    check(out, ref, f"gate extremes (schedule {schedule})")
    # reading R8: a zero row with eps = 0 is 0 * inf = NaN in the plain definition
    x0 = dv["x"].clone()
    x0[5] = 0
    out0 = h.forward(x0, dv["g"], dv["w1"], dv["w3"], 0.0)
    torch.cuda.synchronize()
    assert bool(torch.isnan(out0[5]).all())
    assert not torch.isnan(out0[torch.arange(M, device=cuda_device) != 5]).any()
    # a NaN input element poisons its row only
    xn = dv["x"].clone()
    xn[3, 7] = float("nan")
    outn = h.forward(xn, dv["g"], dv["w1"], dv["w3"], 1e-6)
    torch.cuda.synchronize()
    assert bool(torch.isnan(outn[3]).all())
    assert not torch.isnan(outn[torch.arange(M, device=cuda_device) != 3]).any()


def test_option_values_are_validated(cuda_device):
    """cuasm_ffn_set_option rejects out-of-range values and leaves the handle usable."""
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    lib = h.lib
    bad = [(ffn.OPT_SCHEDULE, 4), (ffn.OPT_SCHEDULE, -1), (ffn.OPT_SK_SPLIT, 1), (ffn.OPT_SK_SPLIT, 17),
           (ffn.OPT_L2_POLICY, 3), (ffn.OPT_L2_POLICY, 12), (ffn.OPT_L2_POLICY, 16), (ffn.OPT_TILE_N, 64),
           (ffn.OPT_FUSED_NORM, 2), (99, 0)]
    for opt, val in bad:
        assert lib.cuasm_ffn_set_option(h._h, opt, val) == ffn.ERR_INVALID_ARG, (opt, val)
    good = [(ffn.OPT_SCHEDULE, ffn.SCHEDULE_STREAM_K_TAIL), (ffn.OPT_SK_SPLIT, 3), (ffn.OPT_L2_POLICY, 0),
            (ffn.OPT_L2_POLICY, 2 | (1 << 2))]
    for opt, val in good:
        assert lib.cuasm_ffn_set_option(h._h, opt, val) == ffn.OK, (opt, val)
    # every option combination above still computes the FFN correctly
    M, K, N = 200, 512, 384
    d = make_inputs(M, K, N, family="C", seed=3500, dtype="bf16")
    out, _ = run_gpu(d, 1e-6, "bf16", handle=h, schedule=ffn.SCHEDULE_STREAM_K_TAIL)
    check(out, oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16"), "options")


# ------------------------------------------ cluster split-K (CUASM_OPT_CSPLIT) ---
@pytest.mark.parametrize("M,K,N,S", [(16, 4096, 1376, 4), (512, 2048, 512, 4), (512, 2048, 512, 8),
                                     (128, 2048, 2048, 2), (300, 512, 520, 3), (48, 1024, 264, 5),
                                     (1, 4096, 1376, 4), (24, 1024, 1000, 2), (9, 2048, 264, 8),
                                     (16, 1024, 520, 6), (32, 2048, 600, 3), (32, 1024, 392, 4)])
def test_cluster_split_k_ffn(cuda_device, M, K, N, S):
    """1-SM tiles split over S-CTA clusters, partials reduced through distributed
    shared memory in rank order: oracle tolerance and bitwise run-to-run.  Tiles
    with <= 32 rows whose partials fit the staging area take the push form
    (dual_gemm.cuh split_k_push: (1|9|16|24|32, S) here, except 32 rows x S=3),
    the others the pull form (split_k_reduce)."""
    d = make_inputs(M, K, N, family="C", seed=8100 + M + S, dtype="bf16")
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    h.set_option(ffn.OPT_CSPLIT, S)
    out, _ = run_gpu(d, 1e-6, "bf16", ffn.VARIANT_1SM, handle=h, schedule=ffn.SCHEDULE_DATA_PARALLEL)
    again, _ = run_gpu(d, 1e-6, "bf16", ffn.VARIANT_1SM, handle=h, schedule=ffn.SCHEDULE_DATA_PARALLEL)
    assert torch.equal(out, again)
    rows = sorted(set([0, M - 1] + list(range(0, M, max(1, M // 32)))))
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16", rows=rows)
    check(out[rows], ref, f"csplit {S} {M}x{K}x{N}")


@pytest.mark.parametrize("M,K,N,S", [(512, 2048, 512, 4), (200, 1024, 392, 2), (16, 1024, 392, 4),
                                     (30, 2048, 1000, 2)])
def test_cluster_split_k_gemm(cuda_device, M, K, N, S):
    d = make_inputs(M, K, N, family="C", seed=8200 + M, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    h.set_variant(ffn.VARIANT_1SM)
    h.set_option(ffn.OPT_CSPLIT, S)
    for tn in (128, 256):
        h.set_option(ffn.OPT_TILE_N, tn)
        out = h.gemm_act(t["x"], t["w1"], "leaky_relu", 0.01)
        torch.cuda.synchronize()
        check(out, oracle.gemm_act(d["x"], d["w1"], "leaky_relu", 0.01), f"csplit gemm {S} n{tn} {M}x{K}x{N}")


def test_cluster_split_k_fp32(cuda_device):
    d = make_inputs(16, 64, 128, family="T", seed=8300, dtype="fp32")
    h = ffn.FusedFFN(cuda_device, torch.float32)
    h.set_option(ffn.OPT_CSPLIT, 2)
    out, _ = run_gpu(d, 1e-6, "fp32", ffn.VARIANT_1SM, handle=h, schedule=ffn.SCHEDULE_DATA_PARALLEL)
    check(out, oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6), "csplit fp32")


# ------------------------------------------ weight loads ahead of griddepcontrol.wait ---
@pytest.mark.parametrize("M,K,N", [(16, 4096, 1376), (300, 1024, 1000), (512, 2048, 2048)])
def test_weights_changed_between_forwards(cuda_device, M, K, N):
    """The producer loads weights before griddepcontrol.wait only when the packed
    weights predate the preceding kernel (PackedWeights::fresh): a forward right after
    a re-pack (weights changed in place -> invalidation) must see the new weights, and
    the next forward (early weight loads) must agree with it bitwise."""
    d = make_inputs(M, K, N, family="C", seed=8400 + M, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    a0 = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    a1 = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    torch.cuda.synchronize()
    assert torch.equal(a0, a1)
    t["w1"].neg_()  # in place: the binding invalidates the cache, the next forward re-packs
    b0 = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    b1 = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    torch.cuda.synchronize()
    assert torch.equal(b0, b1)
    w1n = -d["w1"]
    rows = sorted(set([0, M - 1] + list(range(0, M, max(1, M // 16)))))
    check(b1[rows], oracle.ffn(d["x"], d["g"], w1n, d["w3"], 1e-6, mode="fold_bf16", rows=rows), "after re-pack")


# ------------------------------------------ one handle, mixed launches back to back ---
def test_mixed_shapes_one_handle_back_to_back(cuda_device):
    """Launches of different grids on one handle and stream (cluster split-K, 2-SM stream-K,
    whole tiles, GEMM mode) share its fused-a1 grid counters, which the last warp past the
    r wait resets mid-kernel; PDL lets each launch start before the previous one ends.
    Every output must equal the same problem run alone on a fresh handle."""
    shapes = [(16, 4096, 1376), (1000, 1024, 2752), (16, 4096, 11008), (300, 512, 520), (32, 4096, 2752)]
    data = []
    for i, (M, K, N) in enumerate(shapes):
        d = make_inputs(M, K, N, family="C", seed=8500 + i, dtype="bf16")
        data.append({k: v.to(cuda_device) for k, v in d.items()})
    alone = []
    for t in data:
        h1 = ffn.FusedFFN(cuda_device, torch.bfloat16)
        alone.append(h1.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6))
    torch.cuda.synchronize()
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    outs = []
    for rep in range(3):
        for t in data:
            outs.append(h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6))
            if rep == 2:
                outs.append(h.gemm_act(t["x"], t["w1"], "leaky_relu", 0.01))
    torch.cuda.synchronize()
    k = 0
    for rep in range(3):
        for i in range(len(data)):
            assert torch.equal(outs[k], alone[i]), f"rep {rep} shape {shapes[i]}"
            k += 1 + (rep == 2)
