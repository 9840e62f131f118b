#!/usr/bin/env bash
O=gpurun_out/${1:-r02d}
mkdir -p $O
B="python bench.py --skip-cpu-baseline --skip-e2e --protocol-runs 0"
$B --shard-of 8 > $O/bench_p8.json 2>>$O/bench.err; echo p8=$?
$B > $O/bench_prefill.json 2>>$O/bench.err; echo prefill=$?
$B --workload llama70b > $O/bench_70b.json 2>>$O/bench.err; echo 70b=$?
python scripts/show_bench.py $O/*.json 2>/dev/null
timeout 600 python scripts/trace_gemm.py --shapes 2048x4096x1376 --scheds 1 --bns 80 > $O/trace.log 2>&1; echo trace=$?
cat $O/trace.log
