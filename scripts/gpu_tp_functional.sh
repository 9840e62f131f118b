#!/usr/bin/env bash
# Functional check of the N>1 bench paths on a one-GPU box: two ranks share the GPU over gloo
# (CUASM_BENCH_SHARED_GPU=1).  Not a measurement.
O=gpurun_out/${1:-tpf}; mkdir -p $O
export CUASM_BENCH_SHARED_GPU=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
timeout 600 $R bench.py --gpus 2 --steps 5 --warmup 3 --skip-cpu-baseline > $O/tp2.json 2> $O/tp2.err; echo tp2=$?
timeout 600 $R bench.py --gpus 2 --steps 5 --warmup 3 --skip-cpu-baseline --gather --skip-e2e > $O/tp2_gather.json 2> $O/tp2_gather.err; echo tp2_gather=$?
timeout 600 $R bench.py --gpus 2 --workload llama7b_decode --steps 5 --warmup 3 --skip-cpu-baseline --skip-e2e > $O/tp2_decode.json 2> $O/tp2_decode.err; echo tp2_dec=$?
timeout 600 $R bench.py --gpus 2 --impl reference --steps 3 --warmup 3 > $O/tp2_ref.json 2> $O/tp2_ref.err; echo tp2_ref=$?
for f in $O/*.json; do echo "$f: $(head -c 300 $f)"; done
tail -3 $O/*.err
