#!/usr/bin/env bash
# One GPU session: tests, bench lines, ncu launch list and full captures.
# Usage (from the repo root, under gpurun): bash scripts/gpu_round.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvidia_smi_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke=$?"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?"
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench=$?"
for w in llama7b_decode llama70b; do
  timeout 600 python bench.py --workload $w --skip-cpu-baseline > $OUT/bench_${w}_$TAG.json 2>> $OUT/bench_$TAG.err; echo "bench_$w=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 1 --skip-cpu-baseline --skip-e2e > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu_launches=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_dual_gemm -s 2 -c 1 -f -o $OUT/prof_gemm_$TAG \
  python bench.py --steps 2 --warmup 1 --skip-cpu-baseline --skip-e2e > $OUT/ncu_gemm_$TAG.log 2>&1; echo "ncu_gemm=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_rms_prepass -s 2 -c 1 -f -o $OUT/prof_prepass_$TAG \
  python bench.py --steps 2 --warmup 1 --skip-cpu-baseline --skip-e2e > $OUT/ncu_prepass_$TAG.log 2>&1; echo "ncu_prepass=$?"
