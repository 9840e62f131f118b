"""B200-native fused RMSNorm + SwiGLU feed-forward (the LLaMA ``fused_ff``
kernel of arXiv 2501.08071, PAPER.md P:68 / P:560), as a C-ABI library
(include/cuasm_ffn.h) plus this thin ctypes binding.

    out = SiLU(RMSNorm(x) @ W1.T) * (RMSNorm(x) @ W3.T)

The binding only marshals arguments (torch tensors -> device pointers, the
current CUDA stream).  Every step of the path runs in the library's sm_100a
kernels; there is no CPU or PyTorch fallback -- if libcuasm_ffn.so is missing
or the device is not a B200 the calls raise.
"""
from __future__ import annotations

import ctypes
import os
import threading
import weakref

import torch

__all__ = [
    "FusedFFN", "ffn_forward", "ffn_forward_host", "rms_inv", "rmsnorm", "gemm_act", "ffn_block_forward", "CuasmError",
    "lib_path", "load_library", "rs_layout",
    "VARIANT_AUTO", "VARIANT_1SM", "VARIANT_2SM", "EXPORTED_SYMBOLS",
]

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_PKG, "libcuasm_ffn.so")
_lib = None
_lib_lock = threading.Lock()

OK, ERR_INVALID_ARG, ERR_UNSUPPORTED, ERR_CUDA, ERR_OOM = 0, 1, 2, 3, 4
DTYPE_BF16, DTYPE_FP32 = 0, 1
ACT_IDENTITY, ACT_LEAKY_RELU = 0, 1
VARIANT_AUTO, VARIANT_1SM, VARIANT_2SM = 0, 1, 2
OPT_VARIANT, OPT_PDL, OPT_GROUP_M, OPT_PROFILE, OPT_SCHEDULE, OPT_TRACE, OPT_FUSED_NORM, OPT_TILE_N, OPT_SK_SPLIT, OPT_L2_POLICY, OPT_CSPLIT, OPT_TILE_BN, OPT_DYNAMIC, OPT_RS_PARTIAL, OPT_L2_PERSIST, OPT_MCAST, OPT_THIN_A, OPT_TALL = range(18)
SCHEDULE_AUTO, SCHEDULE_DATA_PARALLEL, SCHEDULE_STREAM_K_ALL, SCHEDULE_STREAM_K_TAIL = 0, 1, 2, 3

# Every entry point include/cuasm_ffn.h declares (checked by tests/test_abi.py).
EXPORTED_SYMBOLS = (
    "cuasm_ffn_init", "cuasm_ffn_forward", "cuasm_ffn_forward_gather", "cuasm_ffn_forward_host", "cuasm_gemm_act",
    "cuasm_ffn_block_forward", "cuasm_ffn_block_forward_rs", "cuasm_rs_reduce", "cuasm_rs_layout",
    "cuasm_rmsnorm",
    "cuasm_ffn_prepare", "cuasm_ffn_rms_inv",
    "cuasm_ffn_get_packed", "cuasm_ffn_invalidate_weights", "cuasm_ffn_set_option", "cuasm_ffn_last_launch",
    "cuasm_ffn_profile_read", "cuasm_ffn_trace_read", "cuasm_plan_config", "cuasm_ffn_destroy", "cuasm_ffn_last_error", "cuasm_ffn_abi_version",
    "cuasm_ffn_tune", "cuasm_gemm_act_tune", "cuasm_ffn_tuned_export", "cuasm_ffn_tuned_import", "cuasm_ffn_tuned_clear", "cuasm_ffn_tune_log",
)


def plan_config(M: int, K: int, N: int, op: str = "ffn", dtype=torch.bfloat16, sm_count: int = 148):
    """The library's configuration model: ("1sm" | "2sm" | "tall" (2-SM tall tiles), stream_k: bool, tile_n: 256 | 128,
    csplit: CTAs per tile of the cluster split-K, 0 = none, bn: SwiGLU outputs per tile)."""
    lib = load_library()
    v, sk = ctypes.c_int(), ctypes.c_int()
    st = lib.cuasm_plan_config(sm_count, _dtype_code(dtype), M, K, N, {"ffn": 0, "gemm": 1}[op], ctypes.byref(v),
                               ctypes.byref(sk))
    if st != OK:
        raise CuasmError(st, "cuasm_plan_config: invalid arguments")
    return _plan_tuple(v.value, sk.value)


def _plan_tuple(variant: int, flags: int):
    return (("1sm" if variant == VARIANT_1SM else "tall" if flags & 4 else "2sm"), bool(flags & 1),
            (128 if flags & 2 else 256), (flags >> 4) & 15, flags >> 8)


def rs_layout(M: int, K: int, world: int, rank: int):
    """f1 ownership (cuasm_rs_layout, host only): (col0, col1, stage_bytes) -- the output
    columns rank `rank` reduces and the size of its fp32 staging buffer."""
    lib = load_library()
    c0, c1, nb = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    st = lib.cuasm_rs_layout(M, K, world, rank, ctypes.byref(c0), ctypes.byref(c1), ctypes.byref(nb))
    if st != OK:
        raise CuasmError(st, "cuasm_rs_layout: invalid arguments")
    return c0.value, c1.value, nb.value


class CuasmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"cuasm_ffn status {status}: {msg}")
        self.status = status


def lib_path() -> str:
    return _LIB_PATH


def load_library():
    """Load libcuasm_ffn.so (raises if it has not been built)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} not found: build it with `python -m paper_2501_08071_b200.build` "
                              "(or __graft_entry__.build()); there is no fallback path")
        lib = ctypes.CDLL(_LIB_PATH)
        vp, i64, f32, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_float, ctypes.c_int
        lib.cuasm_ffn_init.argtypes = [ctypes.POINTER(vp), ci, ci]
        lib.cuasm_ffn_forward.argtypes = [vp, vp, vp, vp, vp, vp, i64, i64, i64, f32, vp]
        lib.cuasm_ffn_forward_host.argtypes = [vp, vp, vp, vp, vp, vp, i64, i64, i64, f32, vp, ci]
        lib.cuasm_ffn_forward_gather.argtypes = [vp, vp, vp, vp, vp, ctypes.POINTER(vp), ci, ci, i64, i64, i64, i64,
                                                 f32, vp]
        lib.cuasm_gemm_act.argtypes = [vp, vp, vp, vp, i64, i64, i64, ci, f32, vp]
        lib.cuasm_ffn_block_forward.argtypes = [vp, vp, vp, vp, vp, vp, vp, i64, i64, i64, f32, vp]
        lib.cuasm_ffn_block_forward_rs.argtypes = [vp, vp, vp, vp, vp, vp, ctypes.POINTER(vp), ci, ci, i64, i64, i64,
                                                    f32, vp]
        lib.cuasm_rs_reduce.argtypes = [vp, vp, ci, ci, ctypes.POINTER(vp), ci, ci, i64, i64, i64, vp]
        lib.cuasm_rs_layout.argtypes = [i64, i64, ci, ci, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                        ctypes.POINTER(i64)]
        lib.cuasm_rmsnorm.argtypes = [vp, vp, vp, vp, i64, i64, f32, vp]
        lib.cuasm_ffn_prepare.argtypes = [vp, vp, vp, vp, i64, i64, vp]
        lib.cuasm_ffn_rms_inv.argtypes = [vp, vp, vp, i64, i64, f32, vp]
        lib.cuasm_ffn_get_packed.argtypes = [vp, vp, ctypes.POINTER(i64)]
        lib.cuasm_ffn_invalidate_weights.argtypes = [vp]
        lib.cuasm_ffn_set_option.argtypes = [vp, ci, i64]
        lib.cuasm_ffn_last_launch.argtypes = [vp, ctypes.POINTER(ci), ctypes.POINTER(ci)]
        lib.cuasm_ffn_profile_read.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                               ctypes.POINTER(ci)]
        lib.cuasm_ffn_trace_read.argtypes = [vp, vp, ctypes.POINTER(ci)]
        lib.cuasm_plan_config.argtypes = [ci, ci, i64, i64, i64, ci, ctypes.POINTER(ci), ctypes.POINTER(ci)]
        lib.cuasm_ffn_tune.argtypes = [vp, vp, vp, vp, vp, vp, i64, i64, i64, f32, ci, ci, ci, vp, ctypes.POINTER(ci),
                                       ctypes.POINTER(ci), ctypes.POINTER(f32)]
        lib.cuasm_gemm_act_tune.argtypes = [vp, vp, vp, vp, i64, i64, i64, ci, f32, ci, ci, ci, vp, ctypes.POINTER(ci),
                                            ctypes.POINTER(ci), ctypes.POINTER(f32)]
        lib.cuasm_ffn_tuned_export.argtypes = [vp, ctypes.c_char_p, i64, ctypes.POINTER(i64)]
        lib.cuasm_ffn_tuned_import.argtypes = [vp, ctypes.c_char_p, ctypes.POINTER(ci)]
        lib.cuasm_ffn_tuned_clear.argtypes = [vp]
        lib.cuasm_ffn_tune_log.argtypes = [vp, ci, ctypes.POINTER(ci), ctypes.POINTER(ci), ctypes.POINTER(ci),
                                           ctypes.POINTER(f32)]
        lib.cuasm_ffn_destroy.argtypes = [vp]
        lib.cuasm_ffn_last_error.argtypes = [vp]
        lib.cuasm_ffn_last_error.restype = ctypes.c_char_p
        lib.cuasm_ffn_abi_version.argtypes = []
        for name in EXPORTED_SYMBOLS:
            if name not in ("cuasm_ffn_last_error", "cuasm_ffn_abi_version"):
                getattr(lib, name).restype = ci
        lib.cuasm_ffn_abi_version.restype = ci
        _lib = lib
        return lib


def _dtype_code(dt: torch.dtype) -> int:
    if dt == torch.bfloat16:
        return DTYPE_BF16
    if dt == torch.float32:
        return DTYPE_FP32
    raise TypeError(f"cuasm_ffn supports bfloat16 and float32 tensors, got {dt}")


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class FusedFFN:
    """One library handle (device + dtype).  Not thread-safe, and used from one
    CUDA stream at a time: the handle owns per-launch device state (r, the fused
    a1 / stream-K bookkeeping, workspaces, the packed weights), so two launches
    of one handle must not run concurrently on different streams."""

    def __init__(self, device=None, dtype: torch.dtype = torch.bfloat16):
        self.lib = load_library()
        dev = torch.device(device if device is not None else "cuda")
        if dev.type != "cuda":
            raise ValueError("FusedFFN needs a CUDA device")
        self.device_index = dev.index if dev.index is not None else torch.cuda.current_device()
        self.dtype = dtype
        h = ctypes.c_void_p()
        st = self.lib.cuasm_ffn_init(ctypes.byref(h), self.device_index, _dtype_code(dtype))
        if st != OK:
            raise CuasmError(st, self.lib.cuasm_ffn_last_error(None).decode())
        self._h = h
        self._wkey = {}

    def close(self):
        if getattr(self, "_h", None):
            self.lib.cuasm_ffn_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int):
        if st != OK:
            raise CuasmError(st, self.lib.cuasm_ffn_last_error(self._h).decode())

    def set_option(self, option: int, value: int):
        self._check(self.lib.cuasm_ffn_set_option(self._h, option, int(value)))

    def set_variant(self, variant: int):
        self.set_option(OPT_VARIANT, variant)

    def last_launch(self):
        v, k = ctypes.c_int(), ctypes.c_int()
        self._check(self.lib.cuasm_ffn_last_launch(self._h, ctypes.byref(v), ctypes.byref(k)))
        return v.value, k.value

    def profile_read(self):
        """(prepass_ms_total, gemm_ms_total, forwards) since the last read."""
        a, b, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
        self._check(self.lib.cuasm_ffn_profile_read(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(n)))
        return a.value, b.value, n.value

    def trace_read(self):
        """Per-CTA %globaltimer stamps [ctas, 16] (ns) of the last traced GEMM launch."""
        n = ctypes.c_int()
        self._check(self.lib.cuasm_ffn_trace_read(self._h, None, ctypes.byref(n)))
        buf = torch.zeros((n.value, 16), dtype=torch.int64)
        if n.value:
            self._check(self.lib.cuasm_ffn_trace_read(self._h, buf.data_ptr(), ctypes.byref(n)))
        return buf

    def _validate(self, *ts):
        for t in ts:
            if t.dtype != self.dtype:
                raise TypeError(f"expected {self.dtype}, got {t.dtype}")
            if not t.is_cuda or t.device.index != self.device_index:
                raise ValueError("tensor is not on the handle's device")
            if not t.is_contiguous():
                raise ValueError("tensors must be contiguous")

    def _weights_changed(self, slots: dict):
        """Invalidate the library's folded-weight cache if any weight changed.

        The library caches packed weights per slot keyed by pointer (slot 0: the
        folded W1/W3 of the fused FFN, keyed by (rms_w, w1, w3); slot 1: the single
        weight of gemm_act / the down projection W2).  A pointer alone is not an
        identity (the caching allocator reuses addresses), so the binding keys each
        library slot on the tensor objects themselves (weak refs) and their in-place
        version counters, and invalidates the library cache on any change.  A slot
        with no key has never been packed through this handle (or was invalidated
        with all others), so the library re-packs it on first use."""
        news = {}
        changed = False
        for slot, ws in slots.items():
            new = (tuple(weakref.ref(t) for t in ws), tuple(t._version for t in ws))
            news[slot] = new
            key = self._wkey.get(slot)
            if key is not None and not (len(key[0]) == len(ws) and all(r() is t for r, t in zip(key[0], ws))
                                        and key[1] == new[1]):
                changed = True
        if changed:
            # the library's invalidation drops every cached pack: forget every key
            self._check(self.lib.cuasm_ffn_invalidate_weights(self._h))
            self._wkey = {}
        self._wkey.update(news)

    def prepare(self, rms_w, w1, w3):
        self._validate(rms_w, w1, w3)
        N, K = w1.shape
        self._weights_changed({0: (rms_w, w1, w3)})
        self._check(self.lib.cuasm_ffn_prepare(self._h, rms_w.data_ptr(), w1.data_ptr(), w3.data_ptr(), K, N,
                                               _stream_ptr(w1.device)))

    def forward(self, x, rms_w, w1, w3, eps: float = 1e-6, out=None):
        self._validate(x, rms_w, w1, w3)
        if x.dim() != 2 or w1.dim() != 2 or w1.shape != w3.shape:
            raise ValueError("x must be [M,K] and w1/w3 [N,K]")
        M, K = x.shape
        N = w1.shape[0]
        if w1.shape[1] != K or rms_w.shape != (K,):
            raise ValueError("shape mismatch")
        if out is None:
            out = torch.empty((M, N), dtype=self.dtype, device=x.device)
        else:
            self._validate(out)
            if out.shape != (M, N):
                raise ValueError("out must be [M,N]")
        self._weights_changed({0: (rms_w, w1, w3)})
        self._check(self.lib.cuasm_ffn_forward(self._h, x.data_ptr(), rms_w.data_ptr(), w1.data_ptr(),
                                               w3.data_ptr(), out.data_ptr(), M, K, N, float(eps),
                                               _stream_ptr(x.device)))
        return out

    def tune(self, x, rms_w, w1, w3, eps: float = 1e-6, warmup: int = 100, iters: int = 100, flush_l2: bool = True,
             out=None):
        """The paper's autotuner (cuasm_ffn_tune): measure every candidate
        configuration of this shape (three interleaved rounds of `warmup` + `iters` forwards,
        each timed forward after an L2 flush when `flush_l2`), keep the fastest for later
        forwards of the same shape on this handle.  Synchronous.  Returns (plan tuple as
        plan_config's, best mean us per forward)."""
        self._validate(x, rms_w, w1, w3)
        M, K = x.shape
        N = w1.shape[0]
        if w1.shape != (N, K) or w3.shape != (N, K) or rms_w.shape != (K,):
            raise ValueError("shape mismatch")
        if out is None:
            out = torch.empty((M, N), dtype=self.dtype, device=x.device)
        self._weights_changed({0: (rms_w, w1, w3)})
        v, fl, us = ctypes.c_int(), ctypes.c_int(), ctypes.c_float()
        self._check(self.lib.cuasm_ffn_tune(self._h, x.data_ptr(), rms_w.data_ptr(), w1.data_ptr(), w3.data_ptr(),
                                            out.data_ptr(), M, K, N, float(eps), int(warmup), int(iters),
                                            1 if flush_l2 else 0, _stream_ptr(x.device), ctypes.byref(v), ctypes.byref(fl),
                                            ctypes.byref(us)))
        return _plan_tuple(v.value, fl.value), us.value

    def tune_gemm_act(self, x, w, act: str = "identity", alpha: float = 0.0, warmup: int = 100, iters: int = 100,
                      flush_l2: bool = True, out=None):
        """The autotuner for the GEMM + activation op (cuasm_gemm_act_tune): x [M,K], w [N,K].
        Returns (plan tuple as plan_config(..., "gemm")'s, best mean us per call)."""
        self._validate(x, w)
        M, K = x.shape
        N = w.shape[0]
        if w.shape[1] != K:
            raise ValueError("shape mismatch")
        if out is None:
            out = torch.empty((M, N), dtype=self.dtype, device=x.device)
        self._weights_changed({1: (w,)})
        v, fl, us = ctypes.c_int(), ctypes.c_int(), ctypes.c_float()
        self._check(self.lib.cuasm_gemm_act_tune(self._h, x.data_ptr(), w.data_ptr(), out.data_ptr(), M, K, N,
                                                 {"identity": ACT_IDENTITY, "leaky_relu": ACT_LEAKY_RELU}[act],
                                                 float(alpha), int(warmup), int(iters), 1 if flush_l2 else 0,
                                                 _stream_ptr(x.device), ctypes.byref(v), ctypes.byref(fl),
                                                 ctypes.byref(us)))
        return _plan_tuple(v.value, fl.value), us.value

    def tuned_export(self) -> str:
        """The tuned table as text (one "cuasm-tuned v1 ..." line per shape, keyed by GPU)."""
        need = ctypes.c_int64()
        self._check(self.lib.cuasm_ffn_tuned_export(self._h, None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value)
        self._check(self.lib.cuasm_ffn_tuned_export(self._h, buf, need.value, ctypes.byref(need)))
        return buf.value.decode()

    def tuned_import(self, text: str) -> int:
        """Deploy-time lookup table: take the entries of `text` made on this GPU
        type; returns how many were taken."""
        n = ctypes.c_int()
        self._check(self.lib.cuasm_ffn_tuned_import(self._h, text.encode(), ctypes.byref(n)))
        return n.value

    def tune_log(self):
        """The last tune()'s candidates in the order measured: [(plan tuple, us or None)]."""
        n = ctypes.c_int()
        self._check(self.lib.cuasm_ffn_tune_log(self._h, 0, ctypes.byref(n), None, None, None))
        cap = n.value
        vs, fs, us = (ctypes.c_int * max(cap, 1))(), (ctypes.c_int * max(cap, 1))(), (ctypes.c_float * max(cap, 1))()
        self._check(self.lib.cuasm_ffn_tune_log(self._h, cap, ctypes.byref(n), vs, fs, us))
        return [(_plan_tuple(vs[i], fs[i]), None if us[i] < 0 else us[i]) for i in range(min(cap, n.value))]

    def tuned_clear(self):
        self._check(self.lib.cuasm_ffn_tuned_clear(self._h))

    def forward_gather(self, x, rms_w, w1, w3, dst_ptrs, ldo: int, eps: float = 1e-6, multicast: bool = False,
                       keepalive=None):
        """Tensor-parallel forward of this rank's column shard (w1/w3 = its rows of
        W1/W3) with the all-gather fused into the epilogue (cuasm_ffn_forward_gather):
        every output store goes to each address in `dst_ptrs` -- this shard's column 0
        inside every rank's full [M, ldo] output (peer pointers) -- or, with
        `multicast`, once to the single NVLS multicast address dst_ptrs[0].
        `keepalive`: tensors owning the destinations (validated when given)."""
        self._validate(x, rms_w, w1, w3)
        if keepalive is not None:
            self._validate(*keepalive)
        M, K = x.shape
        N = w1.shape[0]
        if w1.shape != w3.shape or w1.shape[1] != K or rms_w.shape != (K,):
            raise ValueError("shape mismatch")
        dst = (ctypes.c_void_p * len(dst_ptrs))(*[int(p_) for p_ in dst_ptrs])
        self._weights_changed({0: (rms_w, w1, w3)})
        self._check(self.lib.cuasm_ffn_forward_gather(self._h, x.data_ptr(), rms_w.data_ptr(), w1.data_ptr(),
                                                      w3.data_ptr(), dst, len(dst_ptrs), 1 if multicast else 0,
                                                      int(ldo), M, K, N, float(eps), _stream_ptr(x.device)))

    def forward_host(self, x_host, rms_w, w1, w3, eps: float = 1e-6, out_host=None, sync: bool = True):
        """End-to-end call with host activations: H2D x, forward, D2H out."""
        self._validate(rms_w, w1, w3)
        if x_host.is_cuda or x_host.dtype != self.dtype or not x_host.is_contiguous():
            raise ValueError("x_host must be a contiguous CPU tensor of the handle dtype")
        M, K = x_host.shape
        N = w1.shape[0]
        if out_host is None:
            out_host = torch.empty((M, N), dtype=self.dtype, pin_memory=True)
        self._weights_changed({0: (rms_w, w1, w3)})
        self._check(self.lib.cuasm_ffn_forward_host(self._h, x_host.data_ptr(), rms_w.data_ptr(), w1.data_ptr(),
                                                    w3.data_ptr(), out_host.data_ptr(), M, K, N, float(eps),
                                                    _stream_ptr(w1.device), 1 if sync else 0))
        return out_host

    def gemm_act(self, x, w, act: str = "identity", alpha: float = 0.01, out=None):
        """out = act(x @ w.T) on the tensor cores (the paper's mmLeakyReLu for
        act="leaky_relu"; a plain GEMM for "identity").  x [M,K], w [N,K]."""
        self._validate(x, w)
        M, K = x.shape
        N = w.shape[0]
        if w.shape[1] != K:
            raise ValueError("shape mismatch")
        if out is None:
            out = torch.empty((M, N), dtype=self.dtype, device=x.device)
        else:
            self._validate(out)
        self._weights_changed({1: (w,)})
        code = {"identity": ACT_IDENTITY, "leaky_relu": ACT_LEAKY_RELU}[act]
        self._check(self.lib.cuasm_gemm_act(self._h, x.data_ptr(), w.data_ptr(), out.data_ptr(), M, K, N, code,
                                            float(alpha), _stream_ptr(x.device)))
        return out

    def block_forward(self, x, rms_w, w1, w3, w2, eps: float = 1e-6, out=None):
        """The LLaMA feed-forward block: (SiLU(RMSNorm(x) W1^T) * (RMSNorm(x) W3^T)) W2^T.
        x [M,K], w1/w3 [N,K], w2 [K,N] -> out [M,K]."""
        self._validate(x, rms_w, w1, w3, w2)
        M, K = x.shape
        N = w1.shape[0]
        if w2.shape != (K, N) or w1.shape != (N, K) or w3.shape != (N, K):
            raise ValueError("shape mismatch")
        if out is None:
            out = torch.empty((M, K), dtype=self.dtype, device=x.device)
        else:
            self._validate(out)
        self._weights_changed({0: (rms_w, w1, w3), 1: (w2,)})
        self._check(self.lib.cuasm_ffn_block_forward(self._h, x.data_ptr(), rms_w.data_ptr(), w1.data_ptr(),
                                                     w3.data_ptr(), w2.data_ptr(), out.data_ptr(), M, K, N,
                                                     float(eps), _stream_ptr(x.device)))
        return out

    def block_forward_rs(self, x, rms_w, w1, w3, w2, stage_ptrs, world: int, rank: int, eps: float = 1e-6,
                         keepalive=None):
        """f1: this rank's share of the tensor-parallel FFN block with the row-parallel
        reduction fused into the down projection (cuasm_ffn_block_forward_rs): every
        fp32 partial tile goes straight into its owner's staging buffer (`stage_ptrs[q]`
        = rank q's buffer base, see rs_layout).  w1/w3 [N_l,K], w2 [K,N_l]."""
        self._validate(x, rms_w, w1, w3, w2)
        if keepalive is not None:
            for t in keepalive:
                if not t.is_cuda:
                    raise ValueError("staging buffers must be device memory")
        M, K = x.shape
        N = w1.shape[0]
        if w2.shape != (K, N) or w1.shape != (N, K) or w3.shape != (N, K) or len(stage_ptrs) != world:
            raise ValueError("shape mismatch")
        stage = (ctypes.c_void_p * world)(*[int(p_) if p_ else None for p_ in stage_ptrs])
        self._weights_changed({0: (rms_w, w1, w3), 1: (w2,)})
        self._check(self.lib.cuasm_ffn_block_forward_rs(self._h, x.data_ptr(), rms_w.data_ptr(), w1.data_ptr(),
                                                        w3.data_ptr(), w2.data_ptr(), stage, world, rank, M, K, N,
                                                        float(eps), _stream_ptr(x.device)))

    def rs_reduce(self, stage, world: int, rank: int, dst_ptrs, ldo: int, M: int, K: int, multicast: bool = False):
        """f1 owner side (cuasm_rs_reduce): sum this rank's staging slots in rank order and
        write its columns of y into every destination (or the multicast address)."""
        if not stage.is_cuda or stage.device.index != self.device_index:
            raise ValueError("stage must be a tensor on the handle's device")
        dst = (ctypes.c_void_p * len(dst_ptrs))(*[int(p_) for p_ in dst_ptrs])
        self._check(self.lib.cuasm_rs_reduce(self._h, stage.data_ptr(), world, rank, dst, len(dst_ptrs),
                                             1 if multicast else 0, int(ldo), M, K, _stream_ptr(stage.device)))

    def rmsnorm(self, x, rms_w, eps: float = 1e-6, out=None):
        """RMSNorm(x) = x * g / sqrt(mean(x^2) + eps) (the paper's rmsnorm kernel)."""
        self._validate(x, rms_w)
        M, K = x.shape
        if rms_w.shape != (K,):
            raise ValueError("shape mismatch")
        if out is None:
            out = torch.empty_like(x)
        else:
            self._validate(out)
        self._check(self.lib.cuasm_rmsnorm(self._h, x.data_ptr(), rms_w.data_ptr(), out.data_ptr(), M, K, float(eps),
                                           _stream_ptr(x.device)))
        return out

    def rms_inv(self, x, eps: float = 1e-6, out=None):
        self._validate(x)
        M, K = x.shape
        if out is None:
            out = torch.empty((M,), dtype=torch.float32, device=x.device)
        self._check(self.lib.cuasm_ffn_rms_inv(self._h, x.data_ptr(), out.data_ptr(), M, K, float(eps),
                                               _stream_ptr(x.device)))
        return out

    def packed_weights(self) -> torch.Tensor:
        """Host copy of the g-folded, W1/W3-interleaved weights (a0's output)."""
        n = ctypes.c_int64()
        self._check(self.lib.cuasm_ffn_get_packed(self._h, None, ctypes.byref(n)))
        buf = torch.empty((n.value // (2 if self.dtype == torch.bfloat16 else 4),), dtype=self.dtype)
        self._check(self.lib.cuasm_ffn_get_packed(self._h, buf.data_ptr(), ctypes.byref(n)))
        return buf


_handles: dict = {}


def _handle(device, dtype) -> FusedFFN:
    """The module-level handle for (device, dtype, current stream): a handle's
    per-launch device state must not be shared by concurrent streams."""
    dev = torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    key = (idx, dtype, torch.cuda.current_stream(idx).cuda_stream)
    h = _handles.get(key)
    if h is None:
        h = FusedFFN(torch.device("cuda", idx), dtype)
        _handles[key] = h
    return h


def ffn_forward(x, rms_w, w1, w3, eps: float = 1e-6, out=None):
    """out = SiLU(RMSNorm(x) W1^T) * (RMSNorm(x) W3^T) on the tensors' GPU."""
    return _handle(x.device, x.dtype).forward(x, rms_w, w1, w3, eps, out)


def ffn_forward_host(x_host, rms_w, w1, w3, eps: float = 1e-6, out_host=None, sync: bool = True):
    return _handle(w1.device, w1.dtype).forward_host(x_host, rms_w, w1, w3, eps, out_host, sync)


def rms_inv(x, eps: float = 1e-6):
    return _handle(x.device, x.dtype).rms_inv(x, eps)


def rmsnorm(x, rms_w, eps: float = 1e-6, out=None):
    """RMSNorm(x) on the GPU (stand-alone kernel)."""
    return _handle(x.device, x.dtype).rmsnorm(x, rms_w, eps, out)


def gemm_act(x, w, act: str = "identity", alpha: float = 0.01, out=None):
    """act(x @ w.T) on the tensor cores (mmLeakyReLu for act="leaky_relu")."""
    return _handle(x.device, x.dtype).gemm_act(x, w, act, alpha, out)


def ffn_block_forward(x, rms_w, w1, w3, w2, eps: float = 1e-6, out=None):
    """The whole LLaMA feed-forward block, W2 [K,N] the down projection."""
    return _handle(x.device, x.dtype).block_forward(x, rms_w, w1, w3, w2, eps, out)
