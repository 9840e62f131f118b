import sys, os
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs
dev = torch.device("cuda:0"); flush = bench.L2Flush(dev)
M, K, N = 2048, 4096, 11008
t = make_device_inputs(M, K, N, 1, dev); out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
h = ffn.FusedFFN(dev)
for _ in range(3): h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
h.set_option(ffn.OPT_TRACE, 1)
runs = []
for r in range(4):
    torch.cuda.synchronize(); flush.zero_(); torch.cuda.synchronize()
    h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out); torch.cuda.synchronize()
    tr = h.trace_read().double()
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    lt = (tr[:, 7] - t0) / 1e3   # last_tfull per CTA
    runs.append(lt)
R = torch.stack(runs)  # [4, ctas]
lead = R[:, 0::2]
print("per-run spread (max-min) us:", [round((x.max() - x.min()).item(), 2) for x in lead])
c = torch.corrcoef(lead)
print("corr between runs of per-pair last_tfull:\n", c)
order = lead.mean(0).argsort()
print("slowest pairs (cluster id, mean last_tfull):", [(int(i), round(lead.mean(0)[i].item(), 1)) for i in order[-10:]])
print("fastest pairs:", [(int(i), round(lead.mean(0)[i].item(), 1)) for i in order[:10]])
