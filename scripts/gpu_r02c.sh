#!/usr/bin/env bash
# f1 fused reduction bring-up + tile-width traces.
O=gpurun_out/${1:-r02c}
mkdir -p $O
timeout 900 python -m pytest tests/test_fused_reduce_gpu.py tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "fused or block or reduce" > $O/pytest_rs.log 2>&1; echo pytest_rs=$?
tail -5 $O/pytest_rs.log
B="python bench.py --skip-cpu-baseline --skip-e2e --protocol-runs 0"
$B --workload llama7b_block > $O/bench_block.json 2>>$O/bench.err; echo block=$?
for P in 2 8; do
  $B --workload llama7b_block --shard-of $P > $O/bench_block_p$P.json 2>>$O/bench.err; echo block_p$P=$?
  $B --workload llama7b_block --shard-of $P --fused-reduce > $O/bench_block_p${P}_rs.json 2>>$O/bench.err; echo block_p${P}_rs=$?
done
python scripts/show_bench.py $O/*.json 2>/dev/null | head -30
timeout 600 python scripts/trace_gemm.py --shapes 2048x4096x1376,1024x4096x1376 --scheds 1 --bns 80,96,112,128 --json $O/trace_bn.json > $O/trace_bn.log 2>&1; echo trace=$?
grep -E "ffn |cycles per|wait per|last_mma|first_tma|epi_done|exit" $O/trace_bn.log | head -80
