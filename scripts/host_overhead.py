"""Host-side cost of one cuasm_ffn_forward call through the Python binding."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs
dev = torch.device("cuda:0")
t = make_device_inputs(2048, 4096, 11008, 1, dev)
out = torch.empty((2048, 11008), dtype=torch.bfloat16, device=dev)
h = ffn.FusedFFN(dev)
h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
torch.cuda.synchronize()
torch.cuda._sleep(int(2e9))
n = 200
t0 = time.perf_counter()
for _ in range(n):
    h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
t1 = time.perf_counter()
print(f"host time per forward (binding + C ABI + 2 launches): {(t1 - t0) / n * 1e6:.1f} us")
lib = h.lib
s = torch.cuda.current_stream().cuda_stream
args = (h._h, t["x"].data_ptr(), t["g"].data_ptr(), t["w1"].data_ptr(), t["w3"].data_ptr(), out.data_ptr(),
        2048, 4096, 11008, 1e-6, s)
t0 = time.perf_counter()
for _ in range(n):
    lib.cuasm_ffn_forward(*args)
t1 = time.perf_counter()
print(f"host time per raw C-ABI forward: {(t1 - t0) / n * 1e6:.1f} us")
torch.cuda.synchronize()
