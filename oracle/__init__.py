"""fp64 CPU oracle for the fused RMSNorm+SwiGLU FFN -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path in ``paper_2501_08071_b200/`` never imports it and there is no CPU
fallback to it; the two share no code.

The arithmetic lives in ``ffn_oracle.c`` (plain loops, fp64, sequential k-sums,
OpenMP over rows); this module only marshals arguments through ctypes.
Citations: PAPER.md P:68 (fused feed-forward for LLaMA, RMSNorm), P:560 (inputs
B, M, N, K), BASELINE.json north_star (formula, fold, tolerance).

Parity status per function (DESIGN.md §Oracle pins):
  rms_inv      pinned: closed forms (constant row), worked examples E1/E1eps/E3
  ffn (plain)  pinned: worked examples E1-E5, identity/one-hot closed forms,
               SiLU(0)=0, torch float64 library composition, brute force
  ffn (fold)   pinned: reduces to plain mode when every g*w is representable,
               round_bf16 pinned against torch's independent bf16 cast
  round_tf32   pinned: hand-derived ties and Python-float reference rounding
  rmsnorm      pinned: torch float64 F.rms_norm, constant-row closed form, E2
  gemm_act     pinned: numpy float64 matmul, identity weights, exact negative-slope
               scaling, alpha = 1 reduces to identity
  ffn_block    pinned: W2 = I reduces to ffn(), torch float64 composition with a
               down projection, linearity in W2, round_hidden vs torch's bf16 cast
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ffn_oracle.c")
_LIB = os.path.join(_HERE, "libffn_oracle.so")
_lock = threading.Lock()
_lib = None

DT_BF16, DT_F32, DT_F64 = 0, 1, 2
MODES = {"plain": 0, "fold_bf16": 1, "fold_tf32": 2}


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2 -fopenmp; no -ffast-math, no BLAS)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-fno-fast-math", "-ffp-contract=off", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            vp, i64, dbl, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
            lib.oracle_ffn_rows.argtypes = [vp, ci, vp, vp, vp, ci, i64, i64, i64, dbl, ci, vp, i64, vp]
            lib.oracle_ffn_rows.restype = ci
            lib.oracle_rms_inv.argtypes = [vp, ci, i64, i64, dbl, vp]
            lib.oracle_rms_inv.restype = None
            lib.oracle_round_bf16.argtypes = [dbl]
            lib.oracle_round_bf16.restype = dbl
            lib.oracle_round_bf16_bits.argtypes = [dbl]
            lib.oracle_round_bf16_bits.restype = ctypes.c_uint16
            lib.oracle_round_tf32.argtypes = [dbl]
            lib.oracle_round_tf32.restype = dbl
            lib.oracle_fold_bf16.argtypes = [vp, vp, i64, i64, vp]
            lib.oracle_fold_bf16.restype = None
            lib.oracle_fold_tf32.argtypes = [vp, vp, i64, i64, vp]
            lib.oracle_fold_tf32.restype = None
            lib.oracle_gemm_act.argtypes = [vp, ci, vp, ci, i64, i64, i64, ci, dbl, vp]
            lib.oracle_gemm_act.restype = ci
            lib.oracle_ffn_block_rows.argtypes = [vp, ci, vp, vp, vp, vp, ci, i64, i64, i64, dbl, ci, ci, vp, i64, vp]
            lib.oracle_ffn_block_rows.restype = ci
            lib.oracle_rmsnorm.argtypes = [vp, ci, vp, ci, i64, i64, dbl, vp]
            lib.oracle_rmsnorm.restype = ci
            lib.oracle_set_threads.argtypes = [ci]
            lib.oracle_set_threads.restype = None
            lib.oracle_num_threads.argtypes = []
            lib.oracle_num_threads.restype = ci
            _lib = lib
    return _lib


def _as_storage(a):
    """Return (contiguous numpy array holding the stored bits, dtype code).

    torch bf16 tensors are passed as their raw uint16 bit patterns; the C side
    widens them.  Accepts torch tensors (CPU or CUDA -> copied to CPU) or numpy.
    """
    try:
        import torch
        if isinstance(a, torch.Tensor):
            a = a.detach().to("cpu").contiguous()
            if a.dtype == torch.bfloat16:
                return np.ascontiguousarray(a.view(torch.int16).numpy().view(np.uint16)), DT_BF16
            if a.dtype == torch.float32:
                return np.ascontiguousarray(a.numpy()), DT_F32
            if a.dtype == torch.float64:
                return np.ascontiguousarray(a.numpy()), DT_F64
            raise TypeError(f"oracle: unsupported torch dtype {a.dtype}")
    except ImportError:  # pragma: no cover
        pass
    a = np.asarray(a)
    if a.dtype == np.uint16:
        return np.ascontiguousarray(a), DT_BF16
    if a.dtype == np.float32:
        return np.ascontiguousarray(a), DT_F32
    return np.ascontiguousarray(a, dtype=np.float64), DT_F64


def _widen(a: np.ndarray, dt: int) -> np.ndarray:
    if dt == DT_BF16:
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return a.astype(np.float64)


def ffn(x, g, w1, w3, eps: float = 1e-6, mode: str = "plain", rows=None) -> np.ndarray:
    """out[rows, :] of SiLU(RMSNorm(x)W1^T) * (RMSNorm(x)W3^T) in fp64.

    x [M,K], g [K], w1/w3 [N,K] (nn.Linear layout).  ``rows`` selects rows of x
    (None = all).  ``mode``: "plain" (the definition), "fold_bf16" /
    "fold_tf32" (g folded into the weights in storage precision first).
    """
    lib = _load()
    xs, xdt = _as_storage(x)
    gs, gdt = _as_storage(g)
    w1s, wdt = _as_storage(w1)
    w3s, wdt3 = _as_storage(w3)
    if not (gdt == wdt == wdt3):
        # mixed storage: widen all three exactly to float64 (bf16/fp32 -> f64 is exact)
        gs, w1s, w3s = (_widen(a, dt) for a, dt in ((gs, gdt), (w1s, wdt), (w3s, wdt3)))
        wdt = DT_F64
    if xs.ndim != 2 or w1s.ndim != 2 or w1s.shape != w3s.shape:
        raise ValueError("oracle: x must be [M,K], w1/w3 [N,K]")
    M, K = xs.shape
    N, K2 = w1s.shape
    if K2 != K or gs.shape != (K,):
        raise ValueError("oracle: shape mismatch")
    if rows is None:
        rows_arr = np.arange(M, dtype=np.int64)
    else:
        rows_arr = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    out = np.empty((rows_arr.shape[0], N), dtype=np.float64)
    st = lib.oracle_ffn_rows(xs.ctypes.data, xdt, gs.ctypes.data, w1s.ctypes.data, w3s.ctypes.data,
                             wdt, M, K, N, float(eps), MODES[mode], rows_arr.ctypes.data,
                             rows_arr.shape[0], out.ctypes.data)
    if st != 0:
        raise RuntimeError(f"oracle_ffn_rows failed with status {st}")
    return out


def gemm_act(x, w, act: str = "identity", alpha: float = 0.01) -> np.ndarray:
    """out = act(x @ w^T) in fp64; act in {"identity", "leaky_relu"} (slope alpha).
    The paper's mmLeakyReLu kernel."""
    lib = _load()
    xs, xdt = _as_storage(x)
    ws, wdt = _as_storage(w)
    M, K = xs.shape
    N, K2 = ws.shape
    if K2 != K:
        raise ValueError("oracle: shape mismatch")
    out = np.empty((M, N), dtype=np.float64)
    st = lib.oracle_gemm_act(xs.ctypes.data, xdt, ws.ctypes.data, wdt, M, K, N,
                             {"identity": 0, "leaky_relu": 1}[act], float(alpha), out.ctypes.data)
    if st != 0:
        raise RuntimeError(f"oracle_gemm_act failed with status {st}")
    return out


def ffn_block(x, g, w1, w3, w2, eps: float = 1e-6, mode: str = "plain", round_hidden: bool = False,
              rows=None) -> np.ndarray:
    """y[rows] = hidden @ w2^T with hidden = ffn(x, g, w1, w3, eps, mode) (fp64;
    rounded to bf16 first when round_hidden -- DESIGN.md R13).  w2 [K,N]."""
    lib = _load()
    xs, xdt = _as_storage(x)
    gs, gdt = _as_storage(g)
    w1s, wdt = _as_storage(w1)
    w3s, wdt3 = _as_storage(w3)
    w2s, wdt2 = _as_storage(w2)
    if not (gdt == wdt == wdt3 == wdt2):
        gs, w1s, w3s, w2s = (_widen(a, dt) for a, dt in ((gs, gdt), (w1s, wdt), (w3s, wdt3), (w2s, wdt2)))
        wdt = DT_F64
    M, K = xs.shape
    N = w1s.shape[0]
    if w2s.shape != (K, N):
        raise ValueError("oracle: w2 must be [K,N]")
    rows_arr = np.arange(M, dtype=np.int64) if rows is None else np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    out = np.empty((rows_arr.shape[0], K), dtype=np.float64)
    st = lib.oracle_ffn_block_rows(xs.ctypes.data, xdt, gs.ctypes.data, w1s.ctypes.data, w3s.ctypes.data,
                                   w2s.ctypes.data, wdt, M, K, N, float(eps), MODES[mode], int(bool(round_hidden)),
                                   rows_arr.ctypes.data, rows_arr.shape[0], out.ctypes.data)
    if st != 0:
        raise RuntimeError(f"oracle_ffn_block_rows failed with status {st}")
    return out


def rmsnorm(x, g, eps: float = 1e-6) -> np.ndarray:
    """RMSNorm(x) = x * g / sqrt(mean(x^2) + eps), fp64 (PAPER.md P:573's kernel)."""
    lib = _load()
    xs, xdt = _as_storage(x)
    gs, gdt = _as_storage(g)
    M, K = xs.shape
    out = np.empty((M, K), dtype=np.float64)
    st = lib.oracle_rmsnorm(xs.ctypes.data, xdt, gs.ctypes.data, gdt, M, K, float(eps), out.ctypes.data)
    if st != 0:
        raise RuntimeError(f"oracle_rmsnorm failed with status {st}")
    return out


def rms_inv(x, eps: float = 1e-6) -> np.ndarray:
    """r[m] = 1/sqrt(mean_k x[m,k]^2 + eps), fp64."""
    lib = _load()
    xs, xdt = _as_storage(x)
    M, K = xs.shape
    r = np.empty((M,), dtype=np.float64)
    lib.oracle_rms_inv(xs.ctypes.data, xdt, M, K, float(eps), r.ctypes.data)
    return r


def round_bf16(v: float) -> float:
    return _load().oracle_round_bf16(float(v))


def round_bf16_bits(v: float) -> int:
    return int(_load().oracle_round_bf16_bits(float(v)))


def round_tf32(v: float) -> float:
    return _load().oracle_round_tf32(float(v))


def fold(w, g) -> np.ndarray:
    """Step a0 as the method defines it: RNE(W[n,k]*g[k]) in the storage
    format (bf16 -> uint16 bit patterns; fp32 -> tf32-rounded float32)."""
    lib = _load()
    ws, wdt = _as_storage(w)
    gs, gdt = _as_storage(g)
    N, K = ws.shape
    if wdt == DT_BF16 and gdt == DT_BF16:
        dst = np.empty((N, K), dtype=np.uint16)
        lib.oracle_fold_bf16(ws.ctypes.data, gs.ctypes.data, N, K, dst.ctypes.data)
    elif wdt == DT_F32 and gdt == DT_F32:
        dst = np.empty((N, K), dtype=np.float32)
        lib.oracle_fold_tf32(ws.ctypes.data, gs.ctypes.data, N, K, dst.ctypes.data)
    else:
        raise TypeError("fold: w and g must both be bf16 or both fp32")
    return dst


def set_threads(n: int) -> None:
    _load().oracle_set_threads(int(n))


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def tolerance_ratio(gpu: np.ndarray, ref: np.ndarray, rtol: float = 2e-2, atol: float = 1e-3):
    """Per-element acceptance |gpu-ref| <= rtol*|ref| + atol ([BJ] north_star).

    Returns (worst err/tol ratio, number of violations incl. NaN, max |err|).
    """
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.abs(gpu - ref)
    tol = rtol * np.abs(ref) + atol
    ratio = err / tol
    bad = ~(err <= tol)  # NaN counts as a violation
    worst = float(np.nanmax(ratio)) if ratio.size else 0.0
    if np.isnan(ratio).any():
        worst = float("inf")
    return worst, int(bad.sum()), float(np.nanmax(err)) if err.size else 0.0
