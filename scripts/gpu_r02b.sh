#!/usr/bin/env bash
# Round-2 check after the tile widths: full GPU suite, bench lines (prefill, shards),
# and ncu captures of the P=8 prefill-shard kernel at BN = 80 (plan) and 128.
O=gpurun_out/${1:-r02b}
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest=$?
tail -3 $O/pytest.log
B="python bench.py --skip-cpu-baseline --skip-e2e"
$B > $O/bench_prefill.json 2>>$O/bench.err; echo prefill=$?
for P in 2 4 8; do
  $B --shard-of $P > $O/bench_prefill_p$P.json 2>>$O/bench.err; echo p$P=$?
done
$B --shard-of 8 --tile-bn 128 > $O/bench_prefill_p8_bn128.json 2>>$O/bench.err; echo p8_128=$?
$B --workload llama70b --shard-of 8 > $O/bench_70b_p8.json 2>>$O/bench.err; echo 70b8=$?
python scripts/show_bench.py $O/*.json 2>/dev/null | head -30
for bn in 80 128; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_dual_gemm -s 3 -c 1 -f -o $O/prof_p8_bn$bn \
  python bench.py --shard-of 8 --tile-bn $bn --steps 2 --warmup 2 --skip-cpu-baseline --skip-e2e --skip-b2b --protocol-runs 0 > $O/ncu_p8_bn$bn.log 2>&1; echo ncu_$bn=$?
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_dual_gemm -s 3 -c 1 -f -o $O/prof_prefill \
  python bench.py --steps 2 --warmup 2 --skip-cpu-baseline --skip-e2e --skip-b2b --protocol-runs 0 > $O/ncu_prefill.log 2>&1; echo ncu_prefill=$?
