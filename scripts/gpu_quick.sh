#!/usr/bin/env bash
# Quick GPU check: parity tests, then bench lines for the main workloads and the
# one-GPU projections of the tensor-parallel shards.  Usage: bash scripts/gpu_quick.sh [tag]
TAG=${1:-quick}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest=$?
for w in llama7b_prefill llama7b_decode llama70b tiny_fp32 llama7b_block rmsnorm_paper mmleakyrelu_paper; do
  timeout 600 python bench.py --workload $w --skip-cpu-baseline --skip-e2e > $O/bench_$w.json 2>> $O/bench.err; echo bench_$w=$?
done
for P in 2 4 8; do
  timeout 600 python bench.py --workload llama7b_prefill --shard-of $P --skip-cpu-baseline --skip-e2e > $O/bench_p${P}.json 2>> $O/bench.err; echo p$P=$?
  timeout 600 python bench.py --workload llama7b_decode --shard-of $P --skip-cpu-baseline --skip-e2e > $O/bench_dec_p${P}.json 2>> $O/bench.err; echo dp$P=$?
done
timeout 600 python bench.py > $O/bench_default.json 2>> $O/bench.err; echo default=$?
