#!/usr/bin/env bash
# GPU check after a kernel change: full GPU suite, then bench lines for the main
# workloads (no CPU baseline / e2e).  Usage: bash scripts/gpu_check.sh TAG [workloads...]
TAG=${1:-check}; shift
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest=$?
tail -3 $O/pytest.log
WL=${@:-llama7b_prefill llama7b_decode}
for w in $WL; do
  timeout 600 python bench.py --workload $w --skip-cpu-baseline --skip-e2e > $O/bench_$w.json 2>> $O/bench.err; echo bench_$w=$?
done
for P in 8; do
  timeout 600 python bench.py --workload llama7b_prefill --shard-of $P --skip-cpu-baseline --skip-e2e > $O/bench_p${P}.json 2>> $O/bench.err; echo p$P=$?
  timeout 600 python bench.py --workload llama7b_decode --shard-of $P --skip-cpu-baseline --skip-e2e > $O/bench_dec_p${P}.json 2>> $O/bench.err; echo dp$P=$?
done
python scripts/show_bench.py $O/*.json 2>/dev/null | head -30
