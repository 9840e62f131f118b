"""Token-count sweep (BASELINE.json configs[4]): M = 1..16384 at K=4096, N=11008.

For each M: device time of one forward (CUDA graph replay, L2 flushed before
each step exactly as bench.py does), TFLOP/s, algorithmic GB/s, and the
fraction of the roofline that bounds it (HBM below the crossover, tensor
above), with the measured peaks from MEASURED_PEAKS.json.

    python scripts/sweep.py [--gpus-note 1] [--out profiles/r01/sweep.json]
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
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    peaks = bench.load_peaks()
    K, N = SWEEP_K, SWEEP_N
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
        med = ms[len(ms) // 2]
        flops = 4.0 * M * K * N
        byts = 2.0 * (M * K + 2 * K * N + M * N) + 4.0 * M
        tf = flops / (med / 1e3) / 1e12
        gbs = byts / (med / 1e3) / 1e9
        ridge = peaks["bf16_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
        bound = "hbm" if flops / byts < ridge else "tensor"
        frac = gbs / peaks["hbm_gbs"] if bound == "hbm" else tf / peaks["bf16_tflops"]
        v, _ = h.last_launch()
        rows.append({"M": M, "us": round(med * 1e3, 2), "tflops": round(tf, 2), "gbs": round(gbs, 1),
                     "bound": bound, "frac": round(frac, 4), "variant": {1: "1sm", 2: "2sm"}.get(v, v)})
        print(json.dumps(rows[-1]), flush=True)
        del g
    res = {"K": K, "N": N, "peaks": peaks, "l2": "flushed before every step (256 MiB write + 256 MiB read)",
           "timing": "median of per-step CUDA-event spans around a CUDA-graph replay of cuasm_ffn_forward",
           "rows": rows}
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
