"""Token-count sweep (BASELINE.json configs[4]): M = 1..16384 at K=4096, N=11008.

For each M: device time of one forward (CUDA graph replay, L2 flushed before
each step exactly as bench.py does), TFLOP/s, algorithmic GB/s, and the
fraction of the roofline that bounds it (HBM below the crossover, tensor
above), with the measured peaks from MEASURED_PEAKS.json.

    python scripts/sweep.py [--shard-of 8] [--out profiles/r01/sweep.json]

--shard-of P: the P-GPU sweep point per rank -- rank 0's column shard (N/P)
timed alone on this GPU; TFLOP/s is then the projected whole-job figure
(P x the shard's FLOPs / its time) and the roofline fraction is per GPU.
Times are the mean of the per-step spans (CUDA events tick in ~2 us steps
on these boxes, so a median of short spans is quantised; the mean is not).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bench
import paper_2501_08071_b200 as ffn
from ffn_inputs import SWEEP_K, SWEEP_M, SWEEP_N, make_device_inputs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--ms", default=None, help="comma list overriding the M values")
    ap.add_argument("--shard-of", type=int, default=1)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    peaks = bench.load_peaks()
    K, N = SWEEP_K, SWEEP_N
    P = max(1, a.shard_of)
    if P > 1:
        from paper_2501_08071_b200.tp import shard_bounds
        n0, n1 = shard_bounds(N, 0, P)
        N = n1 - n0
    Ms = [int(m) for m in a.ms.split(",")] if a.ms else SWEEP_M
    flush = bench.L2Flush(dev)
    base = make_device_inputs(max(Ms), K, N, 7, dev)
    h = ffn.FusedFFN(dev)
    h.prepare(base["g"], base["w1"], base["w3"])
    rows = []
    for M in Ms:
        x = base["x"][:M].contiguous()
        out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        for _ in range(3):
            h.forward(x, base["g"], base["w1"], base["w3"], 1e-6, out=out)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            h.forward(x, base["g"], base["w1"], base["w3"], 1e-6, out=out)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
        torch.cuda.synchronize()
        torch.cuda._sleep(int(1e8))
        for e0, e1 in ev:
            flush.zero_()
            e0.record()
            g.replay()
            e1.record()
        torch.cuda.synchronize()
        ms = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
        med = sum(ms) / len(ms)   # mean (see the module docstring)
        flops = 4.0 * M * K * N
        byts = 2.0 * (M * K + 2 * K * N + M * N) + 4.0 * M
        tf = flops / (med / 1e3) / 1e12
        gbs = byts / (med / 1e3) / 1e9
        ridge = peaks["bf16_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
        bound = "hbm" if flops / byts < ridge else "tensor"
        frac = gbs / peaks["hbm_gbs"] if bound == "hbm" else tf / peaks["bf16_tflops"]
        v, _ = h.last_launch()
        rows.append({"M": M, "us": round(med * 1e3, 2), "tflops": round(tf * P, 2), "gbs": round(gbs, 1),
                     "bound": bound, "frac": round(frac, 4), "variant": {1: "1sm", 2: "2sm"}.get(v, v)})
        print(json.dumps(rows[-1]), flush=True)
        del g
    res = {"K": K, "N": N, "shard_of": P, "peaks": peaks, "l2": "flushed before every step (256 MiB write + 256 MiB read)",
           "timing": "mean of per-step CUDA-event spans around a CUDA-graph replay of cuasm_ffn_forward",
           "tflops": "whole job: P x the shard's FLOPs / its time (projection when P > 1)",
           "rows": rows}
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
