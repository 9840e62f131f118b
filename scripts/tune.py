"""Measure every (variant, schedule) configuration of the dual GEMM per M
(K=4096, N=11008 by default) -- the data behind the shape-keyed config table
in csrc/cuasm_ffn.cu (the paper's autotuner step, done
offline once instead of per launch).

    python scripts/tune.py [--ms 1,8,16,...] [--out profiles/r01/tune.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bench
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs

# (variant, schedule, name): schedule 1 whole tiles, 2 stream-K over every tile, 3 stream-K over the
# last partial wave only ("auto" is the library's choice: stream-K over the last partial wave + one
# full wave where its model says so)
CONFIGS = [(1, 1, "1sm-dp"), (1, 2, "1sm-sk"), (1, 3, "1sm-skt"), (2, 1, "2sm-dp"), (2, 2, "2sm-sk"),
           (2, 3, "2sm-skt")]
GEMM_CONFIGS = [(v, sch, tn, f"{'1sm' if v == 1 else '2sm'}-{'dp' if sch == 1 else 'sk'}-n{tn}")
                for v in (1, 2) for sch in (1, 2) for tn in (256, 128)]


def time_cfg(h, x, t, out, steps, flush, op="ffn"):
    def run():
        if op == "ffn":
            h.forward(x, t["g"], t["w1"], t["w3"], 1e-6, out=out)
        else:
            h.gemm_act(x, t["w1"], "leaky_relu", 0.01, out=out)
    for _ in range(2):
        run()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    torch.cuda._sleep(int(1e8))
    for e0, e1 in ev:
        flush.zero_()
        e0.record()
        g.replay()
        e1.record()
    torch.cuda.synchronize()
    ms = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
    # trimmed mean (middle 80%): CUDA events tick in ~2 us steps on these boxes, so a
    # median of short spans is quantised to that step; a mean resolves finer
    k = len(ms) // 10
    core = ms[k:len(ms) - k] or ms
    return sum(core) / len(core) * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ms", default="1,8,16,32,64,128,192,256,384,512,768,1024,1536,2048,4096")
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--N", type=int, default=11008)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--out", default=None)
    ap.add_argument("--op", default="ffn", choices=["ffn", "gemm"])
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = bench.L2Flush(dev)
    Ms = [int(m) for m in a.ms.split(",")]
    t = make_device_inputs(max(Ms), a.K, a.N, 11, dev)
    handles = {}
    cfgs = CONFIGS if a.op == "ffn" else GEMM_CONFIGS
    for c in cfgs:
        h = ffn.FusedFFN(dev)
        h.set_variant(c[0])
        h.set_option(ffn.OPT_SCHEDULE, c[1])
        if a.op == "gemm":
            h.set_option(ffn.OPT_TILE_N, c[2])
        else:
            h.prepare(t["g"], t["w1"], t["w3"])
        handles[c[-1]] = h
    rows = []
    for M in Ms:
        x = t["x"][:M].contiguous()
        out = torch.empty((M, a.N), dtype=torch.bfloat16, device=dev)
        r = {"M": M}
        for c in cfgs:
            r[c[-1]] = round(time_cfg(handles[c[-1]], x, t, out, a.steps, flush, a.op), 2)
        hauto = handles.setdefault("auto", ffn.FusedFFN(dev))
        r["auto"] = round(time_cfg(hauto, x, t, out, a.steps, flush, a.op), 2)
        r["auto_plan"] = ffn.plan_config(M, a.K, a.N, a.op)
        r["best"] = min((k for k in r if k not in ("M", "best", "auto_plan")), key=lambda k: r[k])
        rows.append(r)
        print(json.dumps(r), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"K": a.K, "N": a.N, "unit": "us per forward (median, L2 flushed)", "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
