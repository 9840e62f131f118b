#!/usr/bin/env bash
O=gpurun_out/${1:-r02e}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
B="python bench.py --skip-cpu-baseline --skip-e2e --protocol-runs 0"
$B --workload llama7b_decode > $O/bench_decode.json 2>>$O/bench.err; echo dec=$?
for P in 2 4 8; do $B --workload llama7b_decode --shard-of $P > $O/bench_decode_p$P.json 2>>$O/bench.err; echo dec_p$P=$?; done
python scripts/show_bench.py $O/*.json 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:ffn_dual_gemm -s 3 -c 1 -f -o $O/prof_dec_p8 \
  python bench.py --workload llama7b_decode --shard-of 8 --steps 2 --warmup 2 --skip-cpu-baseline --skip-e2e --skip-b2b --protocol-runs 0 > $O/ncu_dec_p8.log 2>&1; echo ncu=$?
