import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2501_08071_b200 as ffn
from ffn_inputs import make_inputs
M, K, N, S = map(int, sys.argv[1:5])
dev = torch.device("cuda:0")
d = make_inputs(M, K, N, family="C", seed=47, dtype="bf16")
t = {k: v.to(dev) for k, v in d.items()}
h = ffn.FusedFFN(dev, torch.bfloat16)
if S:
    h.set_variant(ffn.VARIANT_1SM); h.set_option(ffn.OPT_CSPLIT, S)
if len(sys.argv) > 5:
    h.set_option(ffn.OPT_PDL, 0)
o = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6); torch.cuda.synchronize(); print("ok", M, K, N, S, ffn.plan_config(M, K, N))
