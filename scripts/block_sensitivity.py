"""Block (f1) sensitivity to the hidden's bf16 rounding (reading R13): hidden flips vs the oracle and the
block output error per schedule."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import oracle, paper_2501_08071_b200 as ffn
from ffn_inputs import make_inputs
dev = torch.device("cuda:0")
M, K, N = 16, 512, 1024
d = make_inputs(M, K, N, family="C", seed=5200 + M, dtype="bf16")
w2 = make_inputs(1, N, K, family="C", seed=5300 + M, dtype="bf16")["w1"]
t = {k: v.to(dev) for k, v in d.items()}
for sch in (0, 1, 2):
    h = ffn.FusedFFN(dev); h.set_option(ffn.OPT_SCHEDULE, sch)
    hid = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    y = h.gemm_act(hid, w2.to(dev), "identity")
    torch.cuda.synchronize()
    ref_h = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16")
    ref_hr = torch.from_numpy(ref_h).to(torch.bfloat16)
    flips = (hid.cpu() != ref_hr).sum().item()
    w, nb, mx = oracle.tolerance_ratio(hid.double().cpu().numpy(), ref_h)
    refy = oracle.ffn_block(d["x"], d["g"], d["w1"], d["w3"], w2, 1e-6, mode="fold_bf16", round_hidden=True)
    wy, nby, mxy = oracle.tolerance_ratio(y.double().cpu().numpy(), refy)
    # y from the GPU hidden in fp64
    y64 = hid.double().cpu() @ w2.double().T
    wz, nbz, mxz = oracle.tolerance_ratio(y.double().cpu().numpy(), y64.numpy())
    print(sch, h.last_launch(), "hidden flips", flips, "of", hid.numel(), "ffn worst", round(w, 3), "| y vs oracle worst", round(wy, 3), nby, "| y vs fp64(gpu hidden) worst", round(wz, 3))
