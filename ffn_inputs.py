"""Seeded synthetic inputs for the fused RMSNorm+SwiGLU FFN.

This module is shared by the tests, bench.py and smoke(): it draws random
numbers and rounds them to storage formats, and holds NONE of the method's
arithmetic (no normalisation, no contraction, no activation).  Both the CUDA
path and the oracle consume exactly the tensors it returns.

Shapes are BASELINE.json's `configs` (LLaMA-7B / LLaMA-2-70B FFN; PAPER.md
P:560 gives the paper's own fused_ff shape B,M,N,K = 1,512,512,2048 on A100).
Families:

  A  pow2-g      x~N(0,1), W~N(0,1/K) (bf16 RNE); g in {0.5,1,2}: the g-fold
                 is exact for any W
  B  4-bit       x~N(0,1) bf16; g~U(0.5,1.5) and W~N(0,1/K) rounded to 4
                 significant bits: every g*w has <= 8 significant bits, exact
                 in bf16
  C  full        x~N(0,1), g~U(0.5,1.5), W~N(0,1/K), all bf16 RNE (timing;
                 parity against the fold-aware oracle)
  T  tiny fp32   x~N(0,1) rounded to 11 significant bits, g~U(0.5,1.5) and
                 W~N(0,1/K) rounded to 5 bits, stored as fp32: x and every g*w
                 are exact in tf32
  L  llama-like  x~N(0,1) with per-row scale ~ LogU(0.25,4) (ragged row norms),
                 g~U(0.2,0.5), W~N(0,0.02) -- closer to trained LLaMA statistics
"""
from __future__ import annotations

import numpy as np
import torch

SEED_BASE = 20250114

# name -> (M, K, N, dtype, eps); index = position in BASELINE.json configs
CONFIGS = {
    "tiny": dict(M=16, K=64, N=128, dtype="fp32", eps=1e-6, idx=0),
    "llama7b_prefill": dict(M=2048, K=4096, N=11008, dtype="bf16", eps=1e-6, idx=1),
    "llama7b_decode": dict(M=16, K=4096, N=11008, dtype="bf16", eps=1e-6, idx=2),
    "llama70b": dict(M=4096, K=8192, N=28672, dtype="bf16", eps=1e-6, idx=3),
}
SWEEP_K, SWEEP_N = 4096, 11008
SWEEP_M = sorted(set([2 ** i for i in range(15)] + [3 * 2 ** i for i in range(13)] + [288, 320, 352]))


def seed_for(config_idx: int, run: int = 0) -> int:
    return SEED_BASE + 1000 * config_idx + run


def _round_sig(v: np.ndarray, bits: int) -> np.ndarray:
    """Round to `bits` significant bits (ties to even) -- a storage recipe."""
    m, e = np.frexp(v)
    m = np.round(m * (1 << bits)) / (1 << bits)
    return np.ldexp(m, e)


def _to_storage(a: np.ndarray, dtype: str) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
    return t.to(torch.bfloat16) if dtype == "bf16" else t


def make_inputs(M: int, K: int, N: int, family: str = "C", seed: int = SEED_BASE,
                dtype: str = "bf16") -> dict:
    """Return CPU tensors x[M,K], g[K], w1[N,K], w3[N,K] in `dtype` storage."""
    rng = np.random.Generator(np.random.PCG64(seed))
    sd = 1.0 / np.sqrt(K)
    x = rng.standard_normal((M, K), dtype=np.float32)
    if family == "A":
        g = rng.choice(np.array([0.5, 1.0, 2.0], dtype=np.float32), size=K)
        w1 = rng.standard_normal((N, K), dtype=np.float32) * sd
        w3 = rng.standard_normal((N, K), dtype=np.float32) * sd
    elif family == "B":
        g = _round_sig(rng.uniform(0.5, 1.5, size=K), 4)
        w1 = _round_sig(rng.standard_normal((N, K), dtype=np.float32) * sd, 4)
        w3 = _round_sig(rng.standard_normal((N, K), dtype=np.float32) * sd, 4)
    elif family == "C":
        g = rng.uniform(0.5, 1.5, size=K)
        w1 = rng.standard_normal((N, K), dtype=np.float32) * sd
        w3 = rng.standard_normal((N, K), dtype=np.float32) * sd
    elif family == "T":
        x = _round_sig(x.astype(np.float64), 11)
        g = _round_sig(rng.uniform(0.5, 1.5, size=K), 5)
        w1 = _round_sig(rng.standard_normal((N, K)) * sd, 5)
        w3 = _round_sig(rng.standard_normal((N, K)) * sd, 5)
    elif family == "L":
        scale = np.exp(rng.uniform(np.log(0.25), np.log(4.0), size=(M, 1))).astype(np.float32)
        x = x * scale
        g = rng.uniform(0.2, 0.5, size=K)
        w1 = rng.standard_normal((N, K), dtype=np.float32) * 0.02
        w3 = rng.standard_normal((N, K), dtype=np.float32) * 0.02
    else:
        raise ValueError(f"unknown input family {family!r}")
    return {
        "x": _to_storage(x, dtype),
        "g": _to_storage(g, dtype),
        "w1": _to_storage(w1, dtype),
        "w3": _to_storage(w3, dtype),
    }


def make_device_inputs(M: int, K: int, N: int, seed: int, device, dtype=torch.bfloat16,
                       w_seed: int | None = None) -> dict:
    """Family C drawn directly on the GPU (torch's Philox); for timing, where
    no oracle comparison is made on the full tensors.  x depends on `seed`
    and g on `seed` only (replicated across tensor-parallel ranks); W1/W3 on `w_seed`
    (default seed + 1), so each rank can draw its own shard."""
    sd = 1.0 / float(np.sqrt(K))
    gx = torch.Generator(device=device)
    gx.manual_seed(seed)
    gw = torch.Generator(device=device)
    gw.manual_seed(seed + 1 if w_seed is None else w_seed)
    x = torch.randn((M, K), device=device, dtype=torch.float32, generator=gx).to(dtype)
    g = (torch.rand((K,), device=device, dtype=torch.float32, generator=gx) + 0.5).to(dtype)
    w1 = (torch.randn((N, K), device=device, dtype=torch.float32, generator=gw) * sd).to(dtype)
    w3 = (torch.randn((N, K), device=device, dtype=torch.float32, generator=gw) * sd).to(dtype)
    return {"x": x, "g": g, "w1": w1, "w3": w3}
