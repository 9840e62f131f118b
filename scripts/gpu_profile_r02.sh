#!/usr/bin/env bash
# Round-2 evidence set for profiles/r02: smoke, GPU tests, bench lines (headline with
# cpu_baseline + e2e, every workload, reference arm, shard projections incl. the fused
# reduction), sweeps, ncu launch lists and full captures, sanitizers.  Under gpurun.
set -u
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest=$?"; tail -1 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_llama7b_prefill.json 2> $O/bench.err; echo "bench=$?"
timeout 600 python bench.py --workload llama7b_decode > $O/bench_llama7b_decode.json 2>> $O/bench.err; echo "bench_decode=$?"
timeout 600 python bench.py --workload llama70b --skip-cpu-baseline > $O/bench_llama70b.json 2>> $O/bench.err; echo "bench_70b=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.json 2>> $O/bench.err; echo "bench_ref=$?"
for w in llama7b_block mmleakyrelu_paper mmleakyrelu_large rmsnorm_paper fused_ff_paper tiny_fp32 crossover_m384; do
  timeout 600 python bench.py --workload $w --skip-cpu-baseline --skip-e2e > $O/bench_$w.json 2>> $O/bench.err; echo "bench_$w=$?"
done
for P in 2 4 8; do
  for w in llama7b_prefill llama70b llama7b_decode; do
    timeout 600 python bench.py --workload $w --shard-of $P --skip-cpu-baseline --skip-e2e > $O/bench_${w}_shard$P.json 2>> $O/bench.err; echo "shard_${w}_$P=$?"
  done
  timeout 600 python bench.py --workload llama7b_block --shard-of $P --skip-cpu-baseline --skip-e2e > $O/bench_llama7b_block_shard$P.json 2>> $O/bench.err; echo "block_$P=$?"
  timeout 600 python bench.py --workload llama7b_block --shard-of $P --fused-reduce --skip-cpu-baseline --skip-e2e > $O/bench_llama7b_block_shard${P}_fusedreduce_sim.json 2>> $O/bench.err; echo "block_rs_$P=$?"
done
for w in llama7b_prefill llama70b; do
  timeout 600 python bench.py --workload $w --shard-of 8 --fused-gather --skip-cpu-baseline --skip-e2e > $O/bench_${w}_shard8_fusedgather_sim.json 2>> $O/bench.err; echo "fg_$w=$?"
done
python scripts/show_bench.py $O/bench_*.json > $O/bench_table.txt 2>&1
timeout 600 python scripts/tune_probe.py > $O/tune_probe.log 2>&1; echo "tune_probe=$?"
timeout 300 python scripts/tune_tall.py --out $O/tune_tall.json > $O/tune_tall.log 2>&1; echo "tune_tall=$?"
timeout 900 python scripts/sweep.py --out $O/sweep.json > $O/sweep.log 2>&1; echo "sweep=$?"
timeout 900 python scripts/sweep.py --shard-of 8 --out $O/sweep_shard8.json > $O/sweep_shard8.log 2>&1; echo "sweep8=$?"
timeout 300 python scripts/trace_gemm.py --shapes 2048x4096x11008,16x4096x11008,2048x4096x1376,16x4096x1376,384x4096x11008 --json $O/trace.json > $O/trace.log 2>&1; echo "trace=$?"
NB="--skip-cpu-baseline --skip-e2e --skip-b2b --no-graph --protocol-runs 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_llama7b_prefill.csv \
  python bench.py --steps 5 --warmup 2 $NB > $O/ncu_launch.log 2>&1; echo "ncu_launches=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_llama7b_decode.csv \
  python bench.py --workload llama7b_decode --steps 5 --warmup 2 $NB > $O/ncu_launch_d.log 2>&1; echo "ncu_launches_d=$?"
for spec in "prefill:llama7b_prefill:1" "decode:llama7b_decode:1" "70b:llama70b:1" "70b_shard8:llama70b:8" "prefill_shard8:llama7b_prefill:8" "decode_shard8:llama7b_decode:8" "tiny:tiny_fp32:1" "tall:crossover_m384:1"; do
  IFS=: read name w P <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_dual_gemm -s 2 -c 1 -f -o $O/prof_gemm_$name \
    python bench.py --workload $w --shard-of $P --steps 2 --warmup 1 $NB > $O/ncu_gemm_$name.log 2>&1; echo "ncu_$name=$?"
  # keep the summary and the raw metric page; only the headline's report travels back whole
  python scripts/ncu_summary.py $O/prof_gemm_$name.ncu-rep > $O/ncu_summary_$name.json 2>/dev/null
  ncu -i $O/prof_gemm_$name.ncu-rep --page raw --csv > $O/ncu_raw_$name.csv 2>/dev/null
  gzip -f $O/ncu_raw_$name.csv
  [ "$name" = prefill ] || rm -f $O/prof_gemm_$name.ncu-rep
done
# (compute-sanitizer runs were closed on the GPU pool late in round 2: the sanitizer evidence is
# profiles/r02/racecheck/ and profiles/r02/evidence/sanitizer_*.log, from the same kernels minus tall tiles)
