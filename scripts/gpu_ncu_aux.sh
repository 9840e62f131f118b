#!/usr/bin/env bash
# ncu --set full of the auxiliary kernels (pre-pass a1, pack a0, rmsnorm f3, owner reduction f1,
# fp32 split), summarised on the box.
O=gpurun_out/${1:-ncuaux}; mkdir -p $O
cat > $O/aux.py <<'PY'
import os, sys; sys.path.insert(0, os.getcwd())
import torch, paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs
dev = torch.device("cuda:0")
t = make_device_inputs(2048, 4096, 11008, 3, dev)
h = ffn.FusedFFN(dev)
for _ in range(2):
    h.rms_inv(t["x"])                                   # ffn_rms_prepass_kernel (a1 stand-alone)
    h.prepare(t["g"], t["w1"], t["w3"])                 # ffn_pack_kernel (a0)
    h.rmsnorm(t["x"][:, :2048].contiguous(), t["g"][:2048].contiguous())  # ffn_rmsnorm_kernel (f3)
P, M, K = 8, 2048, 4096
stage = torch.randn(P * M * 512, device=dev)             # rank 0's staging of an 8-way 7B block
ys = [torch.empty((M, K), dtype=torch.bfloat16, device=dev) for _ in range(P)]
for _ in range(2):
    h.rs_reduce(stage, P, 0, [y.data_ptr() for y in ys], K, M, K)   # ffn_rs_reduce_kernel (f1 owner)
h32 = ffn.FusedFFN(dev, torch.float32)
t32 = make_device_inputs(16, 64, 128, 3, dev, dtype=torch.float32)
for _ in range(2):
    h32.forward(t32["x"], t32["g"], t32["w1"], t32["w3"])            # ffn_split_tf32_kernel (fp32 split)
torch.cuda.synchronize()
PY
for k in ffn_rms_prepass_kernel ffn_pack_kernel ffn_rmsnorm_kernel ffn_rs_reduce_kernel ffn_split_tf32_kernel; do
  timeout 600 ncu --set full --clock-control none -k regex:$k -s 1 -c 1 -f -o $O/prof_$k python $O/aux.py > $O/ncu_$k.log 2>&1; echo $k=$?
  python scripts/ncu_summary.py $O/prof_$k.ncu-rep > $O/ncu_summary_$k.json 2>/dev/null
  rm -f $O/prof_$k.ncu-rep
done
