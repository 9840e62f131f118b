"""GPU checks of the autotuner and its deploy-time lookup table (cuasm_ffn_tune /
cuasm_ffn_tuned_export / cuasm_ffn_tuned_import; the paper's hierarchical search's first
level, and its offline-search / deploy-lookup workflow).

* tuning returns a configuration the shape can run, and later forwards of that shape on the
  handle use it: results match the fp64 oracle at the [BJ] tolerance and equal, bitwise, a
  fresh handle that imported the exported table (same configuration, same arithmetic);
* the table's text keys entries by GPU name + SM count + dtype: lines of another GPU are
  ignored, malformed lines of this GPU are rejected, other shapes keep the cost model;
* fp32 handles refuse (UNSUPPORTED), and argument errors come back as status codes.
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


@pytest.mark.parametrize("M,K,N", [(16, 4096, 1376), (320, 1024, 1376), (1024, 1024, 2048)])
def test_tune_then_forward_and_lookup(cuda_device, M, K, N):
    d = make_inputs(M, K, N, family="C", seed=9600 + M, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    plan, us = h.tune(t["x"], t["g"], t["w1"], t["w3"], 1e-6, warmup=2, iters=3)
    assert us > 0 and plan[0] in ("1sm", "2sm", "tall")
    out = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    torch.cuda.synchronize()
    assert h.last_launch()[0] == (ffn.VARIANT_1SM if plan[0] == "1sm" else ffn.VARIANT_2SM)
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16")
    check(out, ref, f"tuned {plan} {M}x{K}x{N}")
    text = h.tuned_export()
    lines = [ln for ln in text.splitlines() if ln.startswith("cuasm-tuned v1 ")]
    assert len(lines) == 1 and f" M={M} K={K} N={N} " in lines[0]
    h2 = ffn.FusedFFN(cuda_device, torch.bfloat16)
    assert h2.tuned_import("# a comment line\n" + text) == 1
    out2 = h2.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    torch.cuda.synchronize()
    assert torch.equal(out, out2)
    assert h2.last_launch()[0] == h.last_launch()[0]


def test_import_keys_by_gpu_and_rejects_malformed(cuda_device):
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    name = torch.cuda.get_device_name(cuda_device)
    sm = torch.cuda.get_device_properties(cuda_device).multi_processor_count
    other = (f"cuasm-tuned v1 sm={sm} dtype=bf16 M=64 K=512 N=512 variant=2 flags={80 << 8} us=5.0 gpu=Other GPU\n"
             f"cuasm-tuned v1 sm={sm + 1} dtype=bf16 M=64 K=512 N=512 variant=2 flags={80 << 8} us=5.0 gpu={name}\n"
             f"cuasm-tuned v1 sm={sm} dtype=fp32 M=64 K=512 N=512 variant=2 flags={80 << 8} us=5.0 gpu={name}\n")
    assert h.tuned_import(other) == 0
    good = f"cuasm-tuned v1 sm={sm} dtype=bf16 M=64 K=512 N=512 variant=2 flags={80 << 8} us=5.0 gpu={name}\n"
    assert h.tuned_import(good) == 1
    assert "M=64 K=512 N=512 variant=2 flags=20480" in h.tuned_export()
    # the imported 80-wide 2-SM plan runs and is correct
    d = make_inputs(64, 512, 512, family="C", seed=9700, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    out = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    torch.cuda.synchronize()
    assert h.last_launch()[0] == ffn.VARIANT_2SM
    check(out, oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16"), "imported plan")
    for bad in (f"cuasm-tuned v1 sm={sm} dtype=bf16 M=64 K=512 N=512 variant=2 flags={72 << 8} us=5.0 gpu={name}\n",
                f"cuasm-tuned v1 sm={sm} dtype=bf16 M=64 K=512 N=512 variant=7 flags={128 << 8} us=5.0 gpu={name}\n",
                f"cuasm-tuned v1 sm={sm} dtype=bf16 M=64 K=512 N=512 variant=2 flags={(80 << 8) | 4} us=5.0 gpu={name}\n"):
        with pytest.raises(ffn.CuasmError):
            h.tuned_import(bad)
    h.tuned_clear()
    assert h.tuned_export() == ""


def test_tune_refuses_fp32_and_bad_arguments(cuda_device):
    d = make_inputs(16, 64, 128, family="T", seed=9800, dtype="fp32")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    h32 = ffn.FusedFFN(cuda_device, torch.float32)
    with pytest.raises(ffn.CuasmError):
        h32.tune(t["x"], t["g"], t["w1"], t["w3"], 1e-6, warmup=1, iters=1)
    d = make_inputs(16, 256, 128, family="C", seed=9801, dtype="bf16")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    with pytest.raises(ffn.CuasmError):
        h.tune(t["x"], t["g"], t["w1"], t["w3"], 1e-6, warmup=1, iters=0)


@pytest.mark.parametrize("M,K,N", [(512, 2048, 512), (1024, 4096, 1024)])
def test_gemm_act_tune_then_lookup(cuda_device, M, K, N):
    """The GEMM + activation op's search (the paper's mmLeakyReLu): the winner is used
    by later calls, matches the oracle, and travels in the table as an "op=gemm" line that a
    fresh handle imports (bitwise equal output); the fused FFN's entries stay separate."""
    d = make_inputs(M, K, N, family="C", seed=9850 + M, dtype="bf16")
    x, w = d["x"].to(cuda_device), d["w1"].to(cuda_device)
    h = ffn.FusedFFN(cuda_device, torch.bfloat16)
    plan, us = h.tune_gemm_act(x, w, "leaky_relu", 0.01, warmup=2, iters=3)
    assert us > 0 and plan[0] in ("1sm", "2sm") and plan[2] in (128, 256)
    out = h.gemm_act(x, w, "leaky_relu", 0.01)
    torch.cuda.synchronize()
    ref = oracle.gemm_act(d["x"], d["w1"], "leaky_relu", 0.01)
    check(out, ref, f"tuned gemm {plan}")
    text = h.tuned_export()
    assert f" M={M} K={K} N={N} " in text and " op=gemm gpu=" in text
    h2 = ffn.FusedFFN(cuda_device, torch.bfloat16)
    assert h2.tuned_import(text) == 1
    out2 = h2.gemm_act(x, w, "leaky_relu", 0.01)
    torch.cuda.synchronize()
    assert torch.equal(out, out2)
    # the same shape as a fused FFN is not affected by the GEMM entry
    assert ffn.plan_config(M, K, N) is not None
