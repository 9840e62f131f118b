#!/usr/bin/env python
"""Benchmark of the fused RMSNorm+SwiGLU FFN hot path (BASELINE.json `metric`).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl cuasm|reference]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N ...

A step is one pass of the whole hot path -- the row sum-of-squares pre-pass
(a1) and the fused dual-GEMM + SiLU-gate kernel (a2+a3) -- over one batch of
M tokens, through the C ABI (cuasm_ffn_forward).  The one-time weight fold
(a0, the paper's offline/deploy split) runs before the
timed region and is reported separately as `prep_ms`.

Default workload: LLaMA-7B prefill FFN, M=2048 K=4096 N=11008 bf16
(BASELINE.json configs[1]).  With N>1 ranks, W1/W3 are column-sharded
(Megatron, N/P rows each, x replicated; no data-path collective unless
--gather), so the total problem is fixed: "scaling": "strong".

Timing (the paper's protocol P:384): W warm-up steps,
then exactly K steps between barrier+synchronize brackets; each step has its
own CUDA-event pair on the launching stream and a L2 flush before it (256 MiB
memset + 256 MiB read), outside the event pair; value = total FLOPs of the K
steps / max-over-ranks summed device time.  FLOPs = 4*M*K*N (the two GEMMs;
pre-pass and epilogue excluded).  `back_to_back` adds the sustained number:
the step's data (x, W1/W3, out) in R "layer" copies with their own handles, R
chosen so >= 2x L2 of other data passes through L2 between two uses of a copy
("inputs larger than L2"), K steps cycling the copies back to back in one CUDA
graph (PDL between steps) between one event pair -- no per-step event/launch
cost, and the power draw of a long step.

Rank 0 prints ONE JSON line.  `--impl reference` times the fp64 oracle
(oracle/, the test-only CPU reference) on bounded row samples of the same
workload instead; under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

_ROOT = os.path.dirname(os.path.abspath(__file__))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

import torch
import torch.distributed as dist

METRIC = "fused RMSNorm+SwiGLU FFN TFLOP/s"
UNIT = "TFLOP/s"
FLUSH_BYTES = 256 << 20  # > 2x the 126 MB L2
MAX_LAYER_COPIES = 16    # back_to_back: at most this many copies of a step's data

WORKLOADS = {
    # name: (M, K, N, BASELINE.json configs index)
    "llama7b_prefill": (2048, 4096, 11008, 1),
    "llama7b_decode": (16, 4096, 11008, 2),
    "llama70b": (4096, 8192, 28672, 3),
}
# Operations beyond the headline fused FFN: name -> (op, M, K, N)
#   block: the whole LLaMA FFN block (fused FFN + down projection W2), FLOPs 6*M*K*N
#   gemm_lrelu: the paper's mmLeakyReLu (B,M,N,K = 1,512,512,2048), FLOPs 2*M*K*N
EXTRA = {
    "llama7b_block": ("block", 2048, 4096, 11008),
    "mmleakyrelu_paper": ("gemm_lrelu", 512, 2048, 512),
    # the paper's own fused_ff shape (B,M,N,K = 1,512,512,2048; reading R10)
    "fused_ff_paper": ("ffn", 512, 2048, 512),
    "mmleakyrelu_large": ("gemm_lrelu", 4096, 4096, 4096),
    # the paper's stand-alone rmsnorm: 4096 rows x 2048 features; N unused
    "rmsnorm_paper": ("rmsnorm", 4096, 2048, 8),
    # BASELINE.json configs[0]: tiny fp32 fused FFN (tf32 tensor cores), latency-bound
    "tiny_fp32": ("ffn", 16, 64, 128),
    # configs[4]'s crossover region (M = 384 of the token sweep: tall tiles)
    "crossover_m384": ("ffn", 384, 4096, 11008),
}


def parse_args(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)  # the paper's 100 measured iterations
    ap.add_argument("--warmup", type=int, default=100)  # the paper's 100 warm-up iterations
    ap.add_argument("--impl", choices=["cuasm", "reference"], default="cuasm")
    ap.add_argument("--workload", default="llama7b_prefill",
                    help="llama7b_prefill | llama7b_decode | llama70b | sweep:M (K=4096, N=11008)")
    ap.add_argument("--variant", type=int, default=0, help="0 auto, 1 one-SM, 2 two-SM (CTA pair)")
    ap.add_argument("--tile-bn", type=int, default=0, help="SwiGLU outputs per tile: 0 auto, 128/112/96/80/64")
    ap.add_argument("--tune", action="store_true",
                    help="fused FFN, bf16: run the autotuner (cuasm_ffn_tune, L2-flushed candidates) on this "
                         "rank's shape before the warm-up and use its choice (the paper's search-then-lookup "
                         "workflow, PAPER.md P:205-212, P:434-447)")
    ap.add_argument("--gather", action="store_true", help="all-gather the full [M,N] output every step (NCCL)")
    ap.add_argument("--fused-gather", action="store_true",
                    help="a4 fused into the epilogue (cuasm_ffn_forward_gather): every rank's full [M,N] "
                         "symmetric-memory buffer written by every kernel; with --shard-of P on one GPU, P "
                         "simulated peer buffers on this device (store fan-out cost only, no NVLink)")
    ap.add_argument("--fused-reduce", action="store_true",
                    help="block workload: the row-parallel W2 reduction fused into the down projection's epilogue "
                         "(f1; with --shard-of P: P simulated staging / output buffers on this GPU)")
    ap.add_argument("--rs-bf16", action="store_true",
                    help="with --fused-reduce: the partials travel as bf16 (CUASM_OPT_RS_PARTIAL = 1)")
    ap.add_argument("--l2-persist-mb", type=int, default=None,
                    help="device-wide persisting-L2 set-aside (CUASM_OPT_L2_PERSIST) in MiB; with all of x "
                         "inside it the GEMM reads each W13 block from HBM once.  Default: 76 for the llama70b "
                         "workload (x = 64 MiB; the B200 allows up to 79 MiB), else 0")
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch each step eagerly instead of a CUDA graph")
    ap.add_argument("--shard-of", type=int, default=1,
                    help="projection: time rank 0's column shard of a P-way split on this one GPU")
    ap.add_argument("--skip-b2b", action="store_true", help="skip the back-to-back (layer copies) measurement")
    ap.add_argument("--cpu-budget-s", type=float, default=12.0, help="oracle CPU time budget (cpu_baseline)")
    ap.add_argument("--ref-budget-s", type=float, default=150.0, help="whole --impl reference run budget")
    ap.add_argument("--skip-cpu-baseline", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--protocol-runs", type=int, default=5,
                    help="the paper's protocol (P:384, P:545): this many runs of 100 warm-up + 100 timed "
                         "steps, mean per run, warn if runs spread > 1%% (0 = skip)")
    ap.add_argument("--seed", type=int, default=None)
    a = ap.parse_args(argv)
    if a.l2_persist_mb is None:
        # the 70B FFN's x (64 MiB) inside a persisting-L2 set-aside: W13 read from HBM once per launch
        # (profiles/r02/l2_persist/: 2.54 -> 1.55 GB of DRAM traffic, SM clock under the power cap +2%)
        a.l2_persist_mb = 76 if a.workload == "llama70b" else 0
    return a


def workload_op(name: str):
    return EXTRA[name][0] if name in EXTRA else "ffn"


def workload_shape(name: str):
    if name in EXTRA:
        _, M, K, N = EXTRA[name]
        return M, K, N, 1
    if name.startswith("sweep:"):
        return int(name.split(":")[1]), 4096, 11008, 4
    if name not in WORKLOADS:
        raise SystemExit(f"unknown workload {name!r}")
    return WORKLOADS[name]


# ----------------------------------------------------------------------------- dist
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def max_over_ranks(v: float) -> float:
    """Max of a float over all ranks (identity without a process group)."""
    if not (dist.is_available() and dist.is_initialized()):
        return v
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(v: float) -> float:
    if not (dist.is_available() and dist.is_initialized()):
        return v
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier():
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and clock-event (throttle) reasons via NVML in a thread."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int, period_s: float = None):
        # (CUASM_BENCH_NVML_PERIOD_S: sampling period override, for measuring the sampler's own cost)
        self.period = period_s if period_s is not None else float(os.environ.get("CUASM_BENCH_NVML_PERIOD_S", "0.005"))
        self.samples = []
        self.max_mhz = None
        self.ok = False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            props = torch.cuda.get_device_properties(device_index)
            h = None
            try:
                bus = "%08x:%02x:%02x.0" % (props.pci_domain_id, props.pci_bus_id, props.pci_device_id)
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.h = h
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = repr(e)

    def _reasons(self):
        try:
            return self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            return self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)

    def _run(self):
        while not self._stop.is_set():
            try:
                sm = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                try:
                    pw = self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                except Exception:
                    pw = None
                self.samples.append((sm, self._reasons(), pw))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        mask = 0
        for _, r, _ in self.samples:
            mask |= r
        names = [n for b, n in self.REASONS.items() if mask & b and n != "gpu_idle"]
        pws = [w for _, _, w in self.samples if w is not None]
        return {"sm_mhz": statistics.median(s for s, _, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples),
                "power_w_median": round(statistics.median(pws), 1) if pws else None,
                "power_w_max": round(max(pws), 1) if pws else None,
                "note": "NVML's clock reading lags power-cap throttling; the kernel's own cycle counters "
                        "(CUASM_OPT_TRACE) measured ~1.44 GHz during the 7B prefill GEMM"}


def driver_version():
    try:
        import pynvml
        pynvml.nvmlInit()
        v = pynvml.nvmlSystemGetDriverVersion()
        return v.decode() if isinstance(v, bytes) else v
    except Exception:  # noqa: BLE001
        return None


def nccl_version():
    try:
        return ".".join(str(x) for x in torch.cuda.nccl.version())
    except Exception:  # noqa: BLE001
        return None


def load_peaks():
    path = os.path.join(_ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return {"bf16_tflops": float(p["bf16_tflops"]), "bf16_tflops_sustained": float(p["bf16_tflops_sustained"]),
                "hbm_gbs": float(p["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        # /opt/skills/guides/B200_PROFILING.md fallback figures
        return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0,
                "source": "fallback (B200_PROFILING.md)"}


def load_traffic(workload: str):
    """dram bytes per launch of the dual-GEMM kernel from a committed ncu --set full capture."""
    path = os.path.join(_ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


class L2Flush:
    """Evict the step's data from the 126 MB L2 between timed steps: write a
    256 MiB buffer (the usual flush), then read another 256 MiB buffer so the
    write-back of those dirty lines happens here, outside the timed span, and
    the step starts with an L2 full of clean, unrelated lines."""

    def __init__(self, dev):
        self.w = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)
        self.r = torch.ones(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def zero_(self):
        self.w.zero_()
        self.sink = self.r.sum()


def host_cores() -> int:
    """Cores this process may run on (torchrun's OMP_NUM_THREADS=1 must not
    shrink the CPU baseline to one core)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# ------------------------------------------------------------------ cpu baseline
def calibrate_rows(inputs_cpu, eps, budget_s):
    """Rows of the oracle that take about `budget_s` on the host cores.

    The oracle is row-blocked (a weight row is streamed once per block of
    rows), so one row costs far more than 1/M of the whole: time a 32-row
    probe, then one more probe sized from it, and extrapolate from the larger."""
    import oracle
    x, g, w1, w3 = inputs_cpu["x"], inputs_cpu["g"], inputs_cpu["w1"], inputs_cpu["w3"]
    M = x.shape[0]
    n = min(M, 32)
    while True:
        t0 = time.perf_counter()
        oracle.ffn(x, g, w1, w3, eps, mode="fold_bf16", rows=list(range(n)))
        dt = max(time.perf_counter() - t0, 1e-4)
        if n >= M or dt >= 0.1 * budget_s:
            break
        n = min(M, max(2 * n, int(n * 0.1 * budget_s / dt)))
    return max(1, min(M, int(n * budget_s / dt)))


def oracle_sample_time(inputs_cpu, eps, budget_s, rows_hint=None):
    """Time the fp64 oracle on a bounded sample of rows of the same workload.

    Returns (flops, seconds, rows, threads)."""
    import oracle
    oracle.set_threads(host_cores())
    x, g, w1, w3 = inputs_cpu["x"], inputs_cpu["g"], inputs_cpu["w1"], inputs_cpu["w3"]
    M, K = x.shape
    N = w1.shape[0]
    threads = oracle.num_threads()
    if rows_hint is None:
        rows_hint = calibrate_rows(inputs_cpu, eps, budget_s)
    rows = sorted(set((torch.arange(rows_hint) * max(1, M // rows_hint)).clamp(max=M - 1).tolist()))
    t0 = time.perf_counter()
    oracle.ffn(x, g, w1, w3, eps, mode="fold_bf16", rows=rows)
    dt = time.perf_counter() - t0
    return 4.0 * len(rows) * K * N, dt, len(rows), threads


# ------------------------------------------------------------------- cuasm arm
def run_cuasm(args):
    import paper_2501_08071_b200 as ffn
    from ffn_inputs import make_device_inputs, seed_for
    from paper_2501_08071_b200.tp import shard_bounds

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # CUASM_BENCH_SHARED_GPU=1: ranks share the visible GPU(s) over gloo -- a
    # functional check of the N>1 path on a 1-GPU box (timings meaningless)
    shared = os.environ.get("CUASM_BENCH_SHARED_GPU") == "1"
    local_dev = local % torch.cuda.device_count() if shared else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    M, K, N, cidx = workload_shape(args.workload)
    n0, n1 = shard_bounds(N, rank, world)
    if args.shard_of > 1:
        # projection on one GPU: run rank 0's shard of a P-way column split alone
        if world != 1:
            raise SystemExit("--shard-of is a single-process projection")
        n0, n1 = shard_bounds(N, 0, args.shard_of)
    N_l = n1 - n0
    seed = args.seed if args.seed is not None else seed_for(cidx)
    op = workload_op(args.workload)
    wdtype = torch.float32 if args.workload == "tiny_fp32" else torch.bfloat16
    t = make_device_inputs(M, K, N_l, seed, dev, dtype=wdtype, w_seed=seed + 1 + rank)
    if op == "block":
        # down projection W2 [K, N_l] (row-parallel shard), ~N(0, 1/N)
        gw = torch.Generator(device=dev)
        gw.manual_seed(seed + 101 + rank)
        t["w2"] = (torch.randn((K, N_l), device=dev, generator=gw) / float(N) ** 0.5).to(torch.bfloat16)
        out = torch.empty((M, K), dtype=torch.bfloat16, device=dev)
    elif op == "rmsnorm":
        out = torch.empty((M, K), dtype=torch.bfloat16, device=dev)
    else:
        out = torch.empty((M, N_l), dtype=wdtype, device=dev)
    # whole-job FLOPs per step (with --shard-of P: P equal shards, each as fast as rank 0's)
    flops_per_step = {"ffn": 4.0, "block": 6.0, "gemm_lrelu": 2.0, "rmsnorm": 0.0}[op] * M * K * (
        N_l * args.shard_of if args.shard_of > 1 else N)
    flush = L2Flush(dev)
    eps = 1e-6

    # Step footprint in HBM (x, weights, out), for the back-to-back measurement:
    # R "layer" copies of (x, weights, out), each with its own handle (own folded
    # weights), cycled step by step so that >= 2x L2 of other data streams through
    # L2 between two uses of a copy -- every step reads its operands from HBM, as
    # consecutive layers of a model do -- and run back to back (one CUDA graph of
    # K steps, PDL between them) with no flush.
    step_bytes = {"ffn": 2.0 * (M * K + 2 * K * N_l + M * N_l) + 4.0 * M, "rmsnorm": 4.0 * M * K + 2.0 * K,
                  "block": 2.0 * (M * K + 3 * K * N_l + 2 * M * N_l + M * K) + 4.0 * M,
                  "gemm_lrelu": 2.0 * (M * K + K * N_l + M * N_l)}[op] * (2 if wdtype == torch.float32 else 1)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    n_layers = 1 + int(-(-2 * l2_bytes // int(step_bytes)))
    fused_gather = args.fused_gather and op == "ffn"
    fused_reduce = args.fused_reduce and op == "block"
    b2b_ok = not args.gather and not fused_gather and not fused_reduce and not args.no_graph and n_layers <= MAX_LAYER_COPIES and not args.skip_b2b
    if not b2b_ok:
        n_layers = 1
    layers = [(t, out)] + [({k: v.clone() for k, v in t.items()}, torch.empty_like(out)) for _ in range(n_layers - 1)]

    handles = []
    for _ in range(n_layers):
        hh = ffn.FusedFFN(dev, wdtype)
        hh.set_variant(args.variant)
        if args.tile_bn:
            hh.set_option(ffn.OPT_TILE_BN, args.tile_bn)
        if args.rs_bf16:
            hh.set_option(ffn.OPT_RS_PARTIAL, 1)
        if args.l2_persist_mb:
            hh.set_option(ffn.OPT_L2_PERSIST, args.l2_persist_mb << 20)
        if args.no_pdl:
            hh.set_option(ffn.OPT_PDL, 0)
        handles.append(hh)
    h = handles[0]
    stream = torch.cuda.current_stream(dev)

    # a4 fused (f2): destinations of this rank's stores -- every rank's symmetric
    # buffer (world > 1), or P simulated peer buffers on this GPU (--shard-of P)
    fg, gather_dst, gather_mc, sim_bufs = None, None, False, None
    if fused_gather:
        from paper_2501_08071_b200.tp import FusedGather, gather_destinations
        if world > 1:
            fg = FusedGather(M, N, wdtype, dev)
            gather_dst, gather_mc = fg.destinations(n0)
        else:
            P_sim = max(1, args.shard_of)
            sim_bufs = [torch.empty((M, N_l * P_sim), dtype=wdtype, device=dev) for _ in range(P_sim)]
            gather_dst, gather_mc = gather_destinations([b.data_ptr() for b in sim_bufs], 0, out.element_size())

    # f1 fused reduction: every rank's symmetric staging / output buffers (world > 1), or
    # P simulated ones on this GPU (rank 0's scatter + its owner reduction, --shard-of P)
    fr, sim_stage, sim_y = None, None, None
    if fused_reduce:
        if world > 1:
            from paper_2501_08071_b200.tp import FusedReduce
            fr = FusedReduce(M, K, dev)
        else:
            P_sim = max(1, args.shard_of)
            sim_stage = [torch.empty((max(ffn.rs_layout(M, K, P_sim, q)[2] // 4, 4),), dtype=torch.float32,
                                     device=dev) for q in range(P_sim)]
            sim_y = [torch.empty((M, K), dtype=torch.bfloat16, device=dev) for _ in range(P_sim)]

    def fwd(i=0):
        hh, (tt, oo) = handles[i], layers[i]
        if fused_reduce:
            if fr is not None:
                from paper_2501_08071_b200.tp import ffn_block_tp_forward
                return ffn_block_tp_forward(tt["x"], tt["g"], tt["w1"], tt["w3"], tt["w2"], eps, handle=hh,
                                            reduce="fused", fused=fr)
            P_sim = len(sim_stage)
            hh.block_forward_rs(tt["x"], tt["g"], tt["w1"], tt["w3"], tt["w2"], [b.data_ptr() for b in sim_stage],
                                P_sim, 0, eps)
            hh.rs_reduce(sim_stage[0], P_sim, 0, [b.data_ptr() for b in sim_y], K, M, K)
            return None
        if fused_gather:
            hh.forward_gather(tt["x"], tt["g"], tt["w1"], tt["w3"], gather_dst,
                              N if world > 1 else N_l * max(1, args.shard_of), eps, multicast=gather_mc)
            if fg is not None:
                fg.barrier()
            return None
        if op == "ffn":
            return hh.forward(tt["x"], tt["g"], tt["w1"], tt["w3"], eps, out=oo)
        if op == "block":
            return hh.block_forward(tt["x"], tt["g"], tt["w1"], tt["w3"], tt["w2"], eps, out=oo)
        if op == "rmsnorm":
            return hh.rmsnorm(tt["x"], tt["g"], eps, out=oo)
        return hh.gemm_act(tt["x"], tt["w1"], "leaky_relu", 0.01, out=oo)

    # a0: one-time weight fold/pack (reported, not part of a step): the first forward packs the
    # weights for the tile width its plan uses (and allocates the handle's workspaces); with
    # the workspaces in place the cache is dropped and prep = a packing forward minus a packed one
    fwd(0)
    torch.cuda.synchronize(dev)
    if op != "rmsnorm":
        h._check(h.lib.cuasm_ffn_invalidate_weights(h._h))
    e0, e1, e2, e3 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
    e0.record(stream)
    fwd(0)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2.record(stream)
    fwd(0)
    e3.record(stream)
    torch.cuda.synchronize(dev)
    prep_ms = max(0.0, e0.elapsed_time(e1) - e2.elapsed_time(e3))
    for i in range(1, n_layers):
        fwd(i)
    torch.cuda.synchronize(dev)

    full_out = None

    def step(i=0):
        fwd(i)
        if args.gather:
            from paper_2501_08071_b200.tp import gather_shards
            return gather_shards(layers[i][1], N)
        return None

    tuned = None
    if args.tune and op == "ffn" and wdtype == torch.bfloat16 and not (fused_gather or fused_reduce):
        # the autotuner on layer 0's data; the other layer copies' handles import its table
        tt0, oo0 = layers[0]
        tplan, tus = h.tune(tt0["x"], tt0["g"], tt0["w1"], tt0["w3"], eps, warmup=10, iters=20, flush_l2=True, out=oo0)
        table = h.tuned_export()
        for hh in handles[1:]:
            hh.tuned_import(table)
        tuned = {"plan": list(tplan), "us_per_forward": round(tus, 2), "candidates": len(h.tune_log())}
    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize(dev)
    kernels_per_forward = h.last_launch()[1]

    # The forward (pre-pass + dual GEMM, exactly what cuasm_ffn_forward
    # enqueues) is captured once in a CUDA graph and replayed per step, so
    # host-side launch latency never leaks into the device-timed spans.
    graph = None
    if not args.no_graph and fg is None:  # (the symmetric-memory barrier runs eagerly)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            fwd()
        graph.replay()
        torch.cuda.synchronize(dev)

    def timed_step():
        if graph is not None:
            graph.replay()
            if args.gather:
                from paper_2501_08071_b200.tp import gather_shards
                return gather_shards(out, N)
            return None
        return step()

    # ---------------------------------------------------------- timed region
    # SURVEY §8(d) / the paper's protocol: every step alone, L2
    # flushed before it outside its own CUDA-event pair.
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches = 0
    sampler = ClockSampler(local_dev)
    barrier()
    torch.cuda.synchronize(dev)
    wall0 = time.perf_counter()
    with sampler:
        # let the host enqueue ahead of the device (outside every event pair)
        torch.cuda._sleep(int(2e8))
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            full_out = timed_step()
            ends[i].record(stream)
            launches += kernels_per_forward
        torch.cuda.synchronize(dev)
        barrier()
    wall = time.perf_counter() - wall0
    step_ms = sorted(s_.elapsed_time(e_) for s_, e_ in zip(starts, ends))
    local_ms = sum(step_ms)
    t_ms = max_over_ranks(local_ms)
    total_flops = flops_per_step * args.steps
    value = total_flops / (t_ms / 1e3) / 1e12
    metric, unit = METRIC, UNIT
    if op == "rmsnorm":  # memory-bound: report algorithmic GB/s (read x once, write out once)
        metric, unit = "RMSNorm GB/s", "GB/s"
        value = (4.0 * M * K + 2.0 * K) * args.steps / (t_ms / 1e3) / 1e9
    variant_used = h.last_launch()[0]
    launches_total = int(sum_over_ranks(float(launches)))

    # ------------------------------- the paper's protocol: 5 x (100 warm-up + 100 timed)
    # PAPER.md P:384 / P:545: "we run 100 warm-up iterations and 100 measured iterations,
    # flush the L2 cache between iterations, and report the mean of 5 runs (std within 1%)".
    protocol = None
    if args.protocol_runs > 0 and graph is not None:
        run_ms = []
        for _ in range(args.protocol_runs):
            for _ in range(100):
                flush.zero_()
                graph.replay()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(100)]
            barrier()
            torch.cuda.synchronize(dev)
            torch.cuda._sleep(int(2e8))
            for a_, b_ in ev:
                flush.zero_()
                a_.record(stream)
                graph.replay()
                b_.record(stream)
            torch.cuda.synchronize(dev)
            run_ms.append(max_over_ranks(sum(a_.elapsed_time(b_) for a_, b_ in ev) / 100))
        pmean = statistics.mean(run_ms)
        pstd = statistics.pstdev(run_ms)
        spread = (max(run_ms) - min(run_ms)) / pmean
        work_p = flops_per_step / 1e12 if op != "rmsnorm" else (4.0 * M * K + 2.0 * K) / 1e9
        protocol = {
            "runs": args.protocol_runs, "warmup_per_run": 100, "timed_per_run": 100,
            "ms_per_step_runs": [round(v, 5) for v in run_ms], "ms_per_step_mean": round(pmean, 5),
            "std_pct": round(100 * pstd / pmean, 3), "spread_pct": round(100 * spread, 3),
            "value_mean": round(work_p / (pmean / 1e3), 2), "unit": unit,
            "warning": (f"runs differ by {100 * spread:.2f}% (> 1%)" if spread > 0.01 else None),
            "protocol": "PAPER.md P:384/P:545: per run 100 warm-up + 100 timed steps, L2 flushed before every "
                        "step outside its CUDA-event pair, mean over the run; max over ranks",
        }

    # ------------------------------------------------ back to back (secondary)
    back_to_back = None
    if b2b_ok:
        peaks0 = load_peaks()
        for i in range(n_layers):
            fwd(i)
        gb = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gb):
            for i in range(args.steps):
                fwd(i % n_layers)
        warm = torch.cuda.CUDAGraph()  # first replays are slower: warm with a short copy
        with torch.cuda.graph(warm):
            for i in range(max(args.warmup, n_layers)):
                fwd(i % n_layers)
        warm.replay()
        sb, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize(dev)
        torch.cuda._sleep(int(2e8))  # the host enqueues ahead of the device
        sb.record(stream)
        gb.replay()
        eb.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        b_ms = max_over_ranks(sb.elapsed_time(eb))
        work = flops_per_step / 1e12 if op != "rmsnorm" else (4.0 * M * K + 2.0 * K) / 1e9
        b_val = work * args.steps / (b_ms / 1e3)
        back_to_back = {
            "value": round(b_val, 2), "unit": unit, "ms_per_step": round(b_ms / args.steps, 5),
            "steps": args.steps, "layer_copies": n_layers,
            "frac_of_sustained_peak": (round(b_val / world / max(1, args.shard_of) / peaks0["bf16_tflops_sustained"], 4)
                                       if op != "rmsnorm" and peaks0.get("bf16_tflops_sustained") else None),
            "protocol": (f"inputs larger than L2: {n_layers} layer copies of (x, weights, out), "
                         f"{n_layers * step_bytes / 1e6:.0f} MB vs {l2_bytes / 1e6:.0f} MB L2, cycled step by step; "
                         "K steps back to back in one CUDA graph (PDL between steps) between one event pair, max "
                         "over ranks; no flush, so no per-step event/launch cost -- and a sustained power draw"),
        }

    # ------------------------------------------- roofline of the dual-GEMM kernel
    peaks = load_peaks()
    prof_steps = min(args.steps, 50)
    h.set_option(ffn.OPT_PROFILE, 1)
    h.profile_read()
    torch.cuda.synchronize(dev)
    torch.cuda._sleep(int(4e8))  # host runs ahead: no launch gap inside the per-kernel spans
    for _ in range(prof_steps):
        flush.zero_()
        fwd()
    pre_ms, gemm_ms, nfw = h.profile_read()
    h.set_option(ffn.OPT_PROFILE, 0)
    if op == "rmsnorm":  # not a GEMM launch: the step is the kernel
        gemm_ms, pre_ms = 1.0, 0.0
    # per step (the block launches two GEMMs; their spans are summed)
    iso_gemm_ms = gemm_ms / prof_steps
    pre_avg_ms = pre_ms / prof_steps
    # a separate a1 kernel runs only with CUASM_OPT_FUSED_NORM = 0 (or the fp32 split);
    # by default a1 is inside the GEMM kernel and the pre-pass span brackets nothing
    separate_a1 = op in ("ffn", "block") and kernels_per_forward >= (3 if op == "block" else 2)
    gemm_avg_ms = iso_gemm_ms if op != "rmsnorm" else t_ms / args.steps
    gemm_flops = flops_per_step / world / max(1, args.shard_of)
    achieved = gemm_flops / (gemm_avg_ms / 1e3) / 1e12
    bound = "tensor"
    peak = peaks["bf16_tflops"]
    roof_unit = "TFLOP/s"
    # decode-like shapes are HBM bound: algorithmic bytes of the GEMM kernel
    gemm_bytes = {"ffn": 2.0 * (M * K + 2 * K * N_l + M * N_l) + 4.0 * M, "rmsnorm": 4.0 * M * K + 2.0 * K,
                  "block": 2.0 * (M * K + 3 * K * N_l + 2 * M * N_l + M * K) + 4.0 * M,
                  "gemm_lrelu": 2.0 * (M * K + K * N_l + M * N_l)}[op]
    if op == "rmsnorm" or gemm_flops / gemm_bytes < peaks["bf16_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9):
        bound, peak, roof_unit = "hbm", peaks["hbm_gbs"], "GB/s"
        achieved = gemm_bytes / (gemm_avg_ms / 1e3) / 1e9
    traffic = load_traffic(f"{args.workload}@tp{world}" if world > 1 else
                           f"{args.workload}@shard{args.shard_of}" if args.shard_of > 1 else args.workload)
    roofline = {
        "kernel": {"ffn": "ffn_dual_gemm_kernel", "block": "ffn_dual_gemm_kernel x2 (fused FFN + W2 GEMM)",
                   "rmsnorm": "ffn_rmsnorm_kernel",
                   "gemm_lrelu": "ffn_dual_gemm_kernel<GEMM + LeakyReLU epilogue>"}[op], "bound": bound, "achieved": round(achieved, 2), "peak": peak,
        "unit": roof_unit, "frac": round(achieved / peak, 4), "traffic": traffic,
        "peak_source": peaks["source"], "gemm_ms_per_launch": round(gemm_avg_ms, 5),
        "flops_per_launch": gemm_flops, "bytes_per_launch": gemm_bytes,
    }
    if separate_a1:
        roofline.update({
            "prepass_ms_per_launch": round(pre_avg_ms, 5),
            "prepass_GBps": round((2.0 * M * K + 4.0 * M) / (pre_avg_ms / 1e3) / 1e9, 1) if pre_avg_ms > 0 else None,
            "gemm_share_of_step": round(iso_gemm_ms / (iso_gemm_ms + pre_avg_ms), 4)})
    elif op in ("ffn", "block"):
        roofline["prepass"] = "a1 fused into ffn_dual_gemm_kernel (no separate launch; its time is inside gemm_ms)"
    # the stand-alone a1 kernel (ffn_rms_prepass_kernel via cuasm_ffn_rms_inv), timed on its own
    # with the same flush protocol -- not part of the step, reported for its HBM roofline
    prepass_standalone = None
    if op in ("ffn", "block") and wdtype == torch.bfloat16:
        r_buf = torch.empty((M,), dtype=torch.float32, device=dev)
        for _ in range(3):
            h.rms_inv(t["x"], eps, out=r_buf)
        evp = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        torch.cuda.synchronize(dev)
        torch.cuda._sleep(int(1e8))
        for a_, b_ in evp:
            flush.zero_()
            a_.record(stream)
            h.rms_inv(t["x"], eps, out=r_buf)
            b_.record(stream)
        torch.cuda.synchronize(dev)
        p_ms = statistics.median(a_.elapsed_time(b_) for a_, b_ in evp)
        p_bytes = 2.0 * M * K + 4.0 * M
        prepass_standalone = {"kernel": "ffn_rms_prepass_kernel", "ms_median": round(p_ms, 5),
                              "bytes": p_bytes, "GBps": round(p_bytes / (p_ms / 1e3) / 1e9, 1),
                              "frac_of_hbm": round(p_bytes / (p_ms / 1e3) / 1e9 / peaks["hbm_gbs"], 4),
                              "note": "median of 20 single launches after an L2 flush; includes the ~2-6 us "
                                      "event/launch floor (DESIGN.md §7), so small M reads low"}

    # ---------------------------------------------------------------- e2e
    e2e = None
    if not args.skip_e2e and op == "ffn":
        x_host = t["x"].cpu().pin_memory()
        out_host = torch.empty((M, N_l), dtype=wdtype, pin_memory=True)
        ne = min(args.steps, 20)
        for _ in range(2):
            h.forward_host(x_host, t["g"], t["w1"], t["w3"], eps, out_host, sync=True)
        es = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ne)]
        barrier()
        torch.cuda.synchronize(dev)
        for a, b in es:
            a.record(stream)
            h.forward_host(x_host, t["g"], t["w1"], t["w3"], eps, out_host, sync=False)
            b.record(stream)
        torch.cuda.synchronize(dev)
        e_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in es))
        e2e = {"value": round(flops_per_step * ne / (e_ms / 1e3) / 1e12, 2), "unit": UNIT,
               "h2d_bytes_per_step": int(sum_over_ranks(float(M * K * x_host.element_size()))),
               "d2h_bytes_per_step": int(sum_over_ranks(float(M * N_l * out_host.element_size()))),
               "ms_per_step": round(e_ms / ne, 4), "steps": ne,
               "api": "cuasm_ffn_forward_host (pinned host x -> H2D, forward, D2H out)"}

    # ------------------------------------------------------ cpu baseline (oracle)
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.skip_cpu_baseline and op == "ffn":
        cpu_in = {k: v.cpu() for k, v in t.items()}
        fl, sec, rows, thr = oracle_sample_time(cpu_in, eps, args.cpu_budget_s)
        cpu_baseline = {"value": round(fl / sec / 1e12, 6), "unit": UNIT, "cores": thr, "kind": "oracle",
                        "sample": f"{rows} of {M} rows x all {N_l} columns, K={K}, fp64 fold-aware oracle "
                                  f"(oracle/ffn_oracle.c), {sec:.2f} s"}

    clocks = sampler.summary()
    if rank == 0:
        res = {
            "metric": metric, "value": round(value, 2), "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t_ms / args.steps, 5), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 (tf32 tensor cores)" if wdtype == torch.float32 else "bf16",
            "data": "synthetic (seeded randn x~N(0,1), W~N(0,1/K), g~U(0.5,1.5); bf16)",
            "config": {
                "workload": args.workload, "M": M, "K": K, "N": N, "N_per_rank": N_l, "eps": eps,
                "parallelism": f"tp{world} (W1/W3 column-sharded, x replicated)" if world > 1 else (
                    f"PROJECTION of tp{args.shard_of}: rank 0's shard timed alone on one GPU; value = "
                    f"{args.shard_of} x its FLOPs / its time" if args.shard_of > 1 else "single GPU"),
                "reduce": (("fused: W2 epilogue scatters " + ("bf16" if args.rs_bf16 else "fp32") +
                            " partial tiles to the owners' staging buffers, "
                            "owner rank-order sum fanned out to every rank's output " + (
                                "(symmetric memory)" if world > 1 else
                                f"({max(1, args.shard_of)} simulated ranks on this GPU: rank 0's launches)"))
                           if fused_reduce else ("none (rank-local partial)" if op == "block" else None)),
                "gather": ("fused: kernel epilogue stores into " + (
                    f"every rank's symmetric buffer ({'NVLS multicast' if gather_mc else 'P2P peer pointers'})"
                    if world > 1 else f"{max(1, args.shard_of)} simulated peer buffers on this GPU")
                           ) if fused_gather else ("nccl all-gather" if args.gather else False), "variant": {1: "1sm", 2: "2sm"}.get(variant_used, str(variant_used)),
                "pdl": not args.no_pdl, "cuda_graph": graph is not None,
                "l2": "flushed before every step outside the per-step CUDA-event pair: 256 MiB memset, then a "
                      "256 MiB read so the flush's dirty lines are written back before the step",
                "op": op, "flops_per_step": flops_per_step, "prep_ms": round(prep_ms, 4),
                # the configuration model's plan for this rank's problem: (variant, stream-K tail,
                # MMA N, cluster split-K width, SwiGLU outputs per tile); the launch follows it
                # unless options override (--variant, --tile-bn)
                "plan": list(ffn.plan_config(M, K, N_l, "gemm" if op == "gemm_lrelu" else "ffn", wdtype))
                if op in ("ffn", "gemm_lrelu") else None,
                "tile_bn_forced": args.tile_bn or None,
                "tuned": tuned,
                "l2_persist_mib": args.l2_persist_mb or None,
            },
            "pct_of_peak": round(value / world / peaks["bf16_tflops"], 4),
            "pct_of_nominal_2250": round(value / world / 2250.0, 4),
            "roofline": roofline,
            "back_to_back": back_to_back,
            "protocol_5x100": protocol,
            "prepass_standalone": prepass_standalone,
            "step_stats_ms": {"mean": round(local_ms / args.steps, 5), "median": round(step_ms[len(step_ms) // 2], 5),
                              "min": round(step_ms[0], 5), "max": round(step_ms[-1], 5),
                              "note": "rank 0's per-step spans; CUDA events tick in ~2 us steps here"},
            "versions": {"torch": torch.__version__, "cuda": torch.version.cuda,
                         "driver": driver_version(), "nccl": nccl_version()},
            "cpu_baseline": cpu_baseline,
            "e2e": e2e,
            "gpu_launches": launches_total,
            "clocks": clocks,
            "wall_s_timed_region": round(wall, 4),
            "library": ffn.lib_path(),
        }
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()


# --------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle as it stands, on the host cores, on bounded row samples."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    from ffn_inputs import make_inputs, seed_for
    import oracle

    M, K, N, cidx = workload_shape(args.workload)
    n0, n1 = 0, N
    if world > 1:
        from paper_2501_08071_b200.tp import shard_bounds  # pure host arithmetic
        n0, n1 = shard_bounds(N, 0, world)
    N_l = n1 - n0
    seed = args.seed if args.seed is not None else seed_for(cidx)
    # rows of x are independent: generate only what the samples touch
    M_gen = min(M, 256)
    oracle.set_threads(host_cores())
    d = make_inputs(M_gen, K, N_l, family="C", seed=seed, dtype="bf16")
    eps = 1e-6
    nsteps = args.warmup + args.steps
    rows_per_step = max(1, min(M_gen, calibrate_rows(d, eps, args.ref_budget_s / nsteps)))
    for _ in range(args.warmup):
        oracle_sample_time(d, eps, 0, rows_hint=rows_per_step)
    flops = 0.0
    secs = 0.0
    for _ in range(args.steps):
        fl, sec, rows, thr = oracle_sample_time(d, eps, 0, rows_hint=rows_per_step)
        flops += fl
        secs += sec
    # throughput of the FLOPs the oracle actually computed (rank 0's column block on this host's
    # cores; the CPU throughput per FLOP does not depend on how the columns are split)
    value = flops / secs / 1e12
    sample = (f"{rows_per_step} of {M} rows x {N_l} columns per step (K={K}), fp64 fold-aware oracle, "
              f"{oracle.num_threads()} OpenMP threads")
    res = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, family C)",
        "config": {"workload": args.workload, "M": M, "K": K, "N": N, "N_per_rank": N_l},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(res), flush=True)


def main(argv=None):
    args = parse_args(argv)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_cuasm(args)


if __name__ == "__main__":
    main()
