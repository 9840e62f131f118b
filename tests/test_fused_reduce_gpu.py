"""GPU parity of f1's fused reduction (DESIGN.md §8 "Fused reduction"):
the tensor-parallel FFN block y = sum_p hidden_p . W2_p^T with every fp32 partial tile
scattered by the down projection's epilogue into its owner's staging buffer
(cuasm_ffn_block_forward_rs) and each owner's rank-order sum fanned out to every
rank's full output (cuasm_rs_reduce).

Simulated peers: the P ranks' staging and output buffers are P buffers on this GPU and
the ranks' launches run one after another (stream order stands in for the cross-rank
barriers).  Checks: every rank's output is bitwise identical; it equals the exact
(fp64) sum of the P partial products of the hidden shards the GPU produced, up to the
one bf16 rounding; it matches the oracle's full (unsharded) block within the [BJ]
tolerance plus exactly the contribution of hidden elements rounded differently
(reading R13, as tests/test_parity_gpu.py::test_ffn_block_parity); bitwise
run-to-run.  PAPER.md P:68 (fused feed-forward for LLaMA), P:560 (inputs B, M, N, K).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_inputs
from paper_2501_08071_b200.tp import shard_bounds, shard_w2, shard_weights

pytestmark = pytest.mark.gpu

RTOL, ATOL = 2e-2, 1e-3


def run_simulated(dev, t, w2, P, M, K, handles=None):
    """All P ranks' block_forward_rs, then all P owners' rs_reduce; returns the P outputs
    and each rank's hidden shard."""
    stages, ys = [], []
    for q in range(P):
        c0, c1, nb = ffn.rs_layout(M, K, P, q)
        stages.append(torch.full((max(nb // 4, 4),), float("nan"), dtype=torch.float32, device=dev))
        ys.append(torch.full((M, K), float("nan"), dtype=torch.bfloat16, device=dev))
    handles = handles or [ffn.FusedFFN(dev) for _ in range(P)]
    hidden = []
    for p in range(P):
        w1s, w3s = shard_weights(t["w1"], t["w3"], p, P)
        w2s = shard_w2(w2, p, P)
        handles[p].block_forward_rs(t["x"], t["g"], w1s, w3s, w2s, [s.data_ptr() for s in stages], P, p, 1e-6,
                                    keepalive=stages)
        hidden.append(handles[p].forward(t["x"], t["g"], w1s, w3s, 1e-6))
    for q in range(P):
        handles[q].rs_reduce(stages[q], P, q, [y.data_ptr() for y in ys], K, M, K)
    torch.cuda.synchronize()
    return ys, hidden, handles


@pytest.mark.parametrize("M,K,N,P", [(300, 1024, 3 * 264, 2), (300, 1024, 3 * 264, 3), (16, 512, 1024, 4),
                                     (2048, 4096, 2752, 8), (129, 320, 8 * 40, 8), (64, 64, 256, 2)])
def test_simulated_peers_fused_all_reduce(cuda_device, M, K, N, P):
    d = make_inputs(M, K, N, family="C", seed=9100 + M + P, dtype="bf16")
    w2 = make_inputs(1, N, K, family="C", seed=9200 + M + P, dtype="bf16")["w1"]  # [K, N]
    t = {k: v.to(cuda_device) for k, v in d.items()}
    w2d = w2.to(cuda_device)
    ys, hidden, handles = run_simulated(cuda_device, t, w2d, P, M, K)
    for q in range(1, P):
        assert torch.equal(ys[q], ys[0]), f"rank {q}'s output differs from rank 0's"
    y = ys[0]
    assert torch.isfinite(y).all()
    rows = sorted(set([0, M - 1] + list(range(0, M, max(1, M // 16)))))
    # (b) the exact sum of the partial products of the hidden shards the GPU produced
    hid_full = torch.cat(hidden, dim=1)[rows].double().cpu()
    exact = (hid_full @ w2.double().T).numpy()
    worst, nbad, _ = oracle.tolerance_ratio(y[rows].double().cpu().numpy(), exact, 2.0 ** -8, 1e-6)
    assert nbad == 0, f"fused all-reduce differs from the exact partial sum beyond one bf16 rounding ({worst:.3f})"
    # (c) the oracle's unsharded block, allowing the hidden elements rounded the other way (R13)
    ref_h = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16", rows=rows)
    worst, nbad, _ = oracle.tolerance_ratio(hid_full.numpy(), ref_h, RTOL, ATOL)
    assert nbad == 0, "hidden shards vs the oracle FFN"
    ref = oracle.ffn_block(d["x"], d["g"], d["w1"], d["w3"], w2, 1e-6, mode="fold_bf16", round_hidden=True, rows=rows)
    ref_hr = torch.from_numpy(ref_h).to(torch.bfloat16).double()
    flip = ((hid_full - ref_hr) @ w2.double().T).abs().numpy()
    err = np.abs(y[rows].double().cpu().numpy() - ref)
    assert (err <= RTOL * np.abs(ref) + ATOL + flip * (1 + 1e-6)).all(), "fused TP block vs oracle"
    # bitwise run-to-run (same handles: cached packs)
    ys2, _, _ = run_simulated(cuda_device, t, w2d, P, M, K, handles)
    assert torch.equal(ys2[0], y)


def test_world_one_equals_block_forward(cuda_device):
    """P = 1: the fused path is the plain block with fp32 output staging."""
    M, K, N = 200, 512, 768
    d = make_inputs(M, K, N, family="C", seed=9300, dtype="bf16")
    w2 = make_inputs(1, N, K, family="C", seed=9301, dtype="bf16")["w1"].to(cuda_device)
    t = {k: v.to(cuda_device) for k, v in d.items()}
    ys, _, _ = run_simulated(cuda_device, t, w2, 1, M, K)
    h = ffn.FusedFFN(cuda_device)
    y = h.block_forward(t["x"], t["g"], t["w1"], t["w3"], w2, 1e-6)
    torch.cuda.synchronize()
    # the same fp32 accumulators, rounded once either way
    assert torch.equal(ys[0], y)


@pytest.mark.parametrize("schedule", [ffn.SCHEDULE_DATA_PARALLEL, ffn.SCHEDULE_STREAM_K_ALL])
@pytest.mark.parametrize("tile_n", [128, 256])
def test_partial_scatter_every_schedule(cuda_device, schedule, tile_n):
    """Stream-K finishers and both GEMM tile widths scatter whole tiles to the right owner."""
    M, K, N, P = 384, 2048, 1024, 4
    d = make_inputs(M, K, N, family="C", seed=9400 + tile_n, dtype="bf16")
    w2 = make_inputs(1, N, K, family="C", seed=9401, dtype="bf16")["w1"].to(cuda_device)
    t = {k: v.to(cuda_device) for k, v in d.items()}
    hs = []
    for _ in range(P):
        h = ffn.FusedFFN(cuda_device)
        h.set_option(ffn.OPT_SCHEDULE, schedule)
        h.set_option(ffn.OPT_TILE_N, tile_n)
        hs.append(h)
    ys, hidden, _ = run_simulated(cuda_device, t, w2, P, M, K, hs)
    exact = (torch.cat(hidden, dim=1).double() @ w2.double().T).cpu().numpy()
    worst, nbad, _ = oracle.tolerance_ratio(ys[0].double().cpu().numpy(), exact, 2.0 ** -8, 1e-6)
    assert nbad == 0, f"schedule {schedule} tile {tile_n}: worst {worst:.3f}"
    for q in range(1, P):
        assert torch.equal(ys[q], ys[0])


@pytest.mark.parametrize("M,K,N,P", [(300, 1024, 3 * 264, 2), (2048, 4096, 2752, 8), (129, 320, 8 * 40, 3)])
def test_bf16_partials(cuda_device, M, K, N, P):
    """CUASM_OPT_RS_PARTIAL = 1: the partials travel as bf16 (one RNE each, half the bytes); the
    owner still sums in fp32 in rank order.  Every rank's y is bitwise equal, and it differs from
    the default fp32-partial result on the same data (which the oracle checks above pin) by at
    most the partials' own rounding (bf16 unit roundoff 2^-8 x |partial| each) plus the two
    results' final bf16 roundings.  (Where partials cancel that rounding alone can exceed the [BJ] tolerance of the
    small sum: the reason fp32 is the default; reading R16.)"""
    d = make_inputs(M, K, N, family="C", seed=9500 + M + P, dtype="bf16")
    w2 = make_inputs(1, N, K, family="C", seed=9600 + M + P, dtype="bf16")["w1"]
    t = {k: v.to(cuda_device) for k, v in d.items()}
    w2d = w2.to(cuda_device)
    ys32, hidden, _ = run_simulated(cuda_device, t, w2d, P, M, K)
    hs = []
    for _ in range(P):
        h = ffn.FusedFFN(cuda_device)
        h.set_option(ffn.OPT_RS_PARTIAL, 1)
        hs.append(h)
    ys16, hidden16, _ = run_simulated(cuda_device, t, w2d, P, M, K, hs)
    for q in range(1, P):
        assert torch.equal(ys16[q], ys16[0])
    for p in range(P):
        assert torch.equal(hidden16[p], hidden[p])  # the same hidden shards
    parts = []
    for p in range(P):
        n0, n1 = shard_bounds(N, p, P)
        parts.append(hidden[p].double() @ w2d[:, n0:n1].double().T)
    y32, y16 = ys32[0].double(), ys16[0].double()
    bound = 2.0 ** -8 * sum(pp.abs() for pp in parts) + 2.0 ** -7 * y32.abs() + 1e-6
    diff = (y16 - y32).abs()
    assert (diff <= bound).all(), f"bf16 partials beyond their rounding bound (worst {(diff / bound).max().item():.3f})"


def test_fused_reduce_contract_errors(cuda_device):
    h = ffn.FusedFFN(cuda_device)
    lib = h.lib
    import ctypes
    x = torch.zeros((4, 64), dtype=torch.bfloat16, device=cuda_device)
    st = torch.zeros(1024, dtype=torch.float32, device=cuda_device)
    s = torch.cuda.current_stream().cuda_stream
    arr = (ctypes.c_void_p * 2)(st.data_ptr(), st.data_ptr())
    p = lambda t_: t_.data_ptr()
    # world out of range, rank out of range
    assert lib.cuasm_ffn_block_forward_rs(h._h, p(x), p(x), p(x), p(x), p(x), arr, 9, 0, 4, 64, 64, 1e-6, s) != 0
    assert lib.cuasm_ffn_block_forward_rs(h._h, p(x), p(x), p(x), p(x), p(x), arr, 2, 2, 4, 64, 64, 1e-6, s) != 0
    assert lib.cuasm_rs_reduce(h._h, p(st), 2, 0, arr, 0, 0, 64, 4, 64, s) != 0
    assert lib.cuasm_rs_reduce(h._h, p(st), 2, 0, arr, 2, 1, 64, 4, 64, s) != 0   # multicast with 2 addresses
    assert lib.cuasm_rs_reduce(h._h, p(st), 2, 0, arr, 1, 0, 32, 4, 64, s) != 0   # ldo < K
    h32 = ffn.FusedFFN(cuda_device, torch.float32)
    assert h32.lib.cuasm_rs_reduce(h32._h, p(st), 1, 0, arr, 1, 0, 64, 4, 64, s) == ffn.ERR_UNSUPPORTED
