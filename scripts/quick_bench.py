"""Quick device timing of the forward for a few shapes/variants (dev tool)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs


def time_one(h, t, eps, iters=20, warmup=5, flush=None):
    for _ in range(warmup):
        h.forward(t["x"], t["g"], t["w1"], t["w3"], eps, out=t["out"])
    torch.cuda.synchronize()
    times = []
    for _ in range(iters):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h.forward(t["x"], t["g"], t["w1"], t["w3"], eps, out=t["out"])
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    times.sort()
    return times[len(times) // 2], times[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="2048x4096x11008,16x4096x11008,4096x8192x3584,4096x8192x28672")
    ap.add_argument("--variants", default="1,2")
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    for shp in args.shapes.split(","):
        M, K, N = map(int, shp.split("x"))
        t = make_device_inputs(M, K, N, 1, dev)
        t["out"] = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        for v in map(int, args.variants.split(",")):
            h = ffn.FusedFFN(dev, torch.bfloat16)
            h.set_variant(v)
            med, best = time_one(h, t, 1e-6, iters=args.iters, flush=flush)
            fl = 4.0 * M * K * N
            by = 2.0 * (M * K + 2 * K * N + M * N) + 4 * M
            print(f"M={M} K={K} N={N} variant={v}: median {med*1e3:.1f} us  best {best*1e3:.1f} us  "
                  f"{fl/med/1e9:.1f} TFLOP/s  {by/med/1e6:.1f} GB/s", flush=True)
            h.close()


if __name__ == "__main__":
    main()
