"""70B FFN step time with an L2 set-aside for persisting lines (CUASM_OPT_L2_PERSIST; the x tiles'
TMA loads carry evict_last) x rasterisation group x dynamic claiming.

    python scripts/l2_persist_study.py PERSIST_BYTES GROUP_M DYNAMIC STEPS
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bench
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs
from scripts.tune import time_cfg

dev = torch.device("cuda:0")
flush = bench.L2Flush(dev)
M, K, N = 4096, 8192, 28672
t = make_device_inputs(M, K, N, 11, dev)
out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
persist, g, dyn, steps = (int(v) for v in sys.argv[1:5])
h = ffn.FusedFFN(dev)
h.set_option(ffn.OPT_L2_PERSIST, persist)
h.set_option(ffn.OPT_GROUP_M, g)
h.set_option(ffn.OPT_DYNAMIC, dyn)
print(persist, g, dyn, round(time_cfg(h, t["x"], t, out, steps, flush), 1), flush=True)
h.set_option(ffn.OPT_L2_PERSIST, 0)
