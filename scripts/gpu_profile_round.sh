#!/usr/bin/env bash
# Full evidence set for profiles/<tag>: tests, bench lines (3 workloads +
# reference arm), sweep, ncu launch list + full captures, per-CTA trace,
# compute-sanitizer.  Run under gpurun from the repo root.
set -u
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest=$?"
timeout 600 python bench.py > $O/bench_llama7b_prefill.json 2> $O/bench.err; echo "bench=$?"
timeout 600 python bench.py --workload llama7b_decode > $O/bench_llama7b_decode.json 2>> $O/bench.err; echo "bench_decode=$?"
timeout 600 python bench.py --workload llama70b --skip-cpu-baseline > $O/bench_llama70b.json 2>> $O/bench.err; echo "bench_70b=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_reference.json 2>> $O/bench.err; echo "bench_ref=$?"
for w in llama7b_block mmleakyrelu_paper mmleakyrelu_large rmsnorm_paper fused_ff_paper; do
  timeout 600 python bench.py --workload $w --skip-cpu-baseline --skip-e2e > $O/bench_$w.json 2>> $O/bench.err; echo "bench_$w=$?"
done
timeout 600 python bench.py --workload tiny_fp32 --skip-cpu-baseline --skip-e2e > $O/bench_tiny_fp32.json 2>> $O/bench.err; echo "bench_tiny=$?"
# one-GPU projections of the tensor-parallel ranks (rank 0's shard timed alone) and the
# fused-gather store fan-out on simulated peers
for P in 2 4 8; do
  for w in llama7b_prefill llama70b llama7b_decode; do
    timeout 600 python bench.py --workload $w --shard-of $P --skip-cpu-baseline --skip-e2e > $O/bench_${w}_shard$P.json 2>> $O/bench.err; echo "shard_${w}_$P=$?"
  done
done
for w in llama7b_prefill llama70b; do
  timeout 600 python bench.py --workload $w --shard-of 8 --fused-gather --skip-cpu-baseline --skip-e2e > $O/bench_${w}_shard8_fusedgather_sim.json 2>> $O/bench.err; echo "fg_$w=$?"
done
timeout 600 python scripts/tune.py --out $O/tune.json > $O/tune.log 2>&1; echo "tune=$?"
timeout 600 python scripts/tune_split.py --out $O/tune_split.json > $O/tune_split.log 2>&1; echo "tune_split=$?"
timeout 300 python scripts/launch_floor.py > $O/launch_floor.log 2>&1; echo "launch_floor=$?"
timeout 300 python scripts/trace_gemm.py --op gemm --shapes 2048x11008x4096,4096x4096x4096 --scheds 0,1,2 > $O/trace_gemm.log 2>&1; echo "trace_gemm=$?"
timeout 900 python scripts/sweep.py --out $O/sweep.json > $O/sweep.log 2>&1; echo "sweep=$?"
timeout 900 python scripts/sweep.py --shard-of 8 --out $O/sweep_shard8.json > $O/sweep_shard8.log 2>&1; echo "sweep8=$?"
timeout 600 python scripts/plain_vs_fold_stats.py --out $O/plain_vs_fold.json > $O/plain_vs_fold.log 2>&1; echo "pvf=$?"
timeout 300 python scripts/trace_gemm.py --shapes 2048x4096x11008,16x4096x11008,4096x8192x3584 --json $O/trace.json > $O/trace.log 2>&1; echo "trace=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_llama7b_prefill.csv \
  python bench.py --steps 5 --warmup 2 --skip-cpu-baseline --skip-e2e --skip-b2b --no-graph > $O/ncu_launch.log 2>&1; echo "ncu_launches=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_llama7b_decode.csv \
  python bench.py --workload llama7b_decode --steps 5 --warmup 2 --skip-cpu-baseline --skip-e2e --skip-b2b --no-graph > $O/ncu_launch_d.log 2>&1; echo "ncu_launches_d=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_dual_gemm -s 2 -c 1 -f -o $O/prof_gemm_prefill \
  python bench.py --steps 2 --warmup 1 --skip-cpu-baseline --skip-e2e --skip-b2b --no-graph > $O/ncu_gemm.log 2>&1; echo "ncu_gemm=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_dual_gemm -s 2 -c 1 -f -o $O/prof_gemm_decode \
  python bench.py --workload llama7b_decode --steps 2 --warmup 1 --skip-cpu-baseline --skip-e2e --skip-b2b --no-graph > $O/ncu_gemm_d.log 2>&1; echo "ncu_gemm_d=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_dual_gemm -s 2 -c 1 -f -o $O/prof_gemm_70b \
  python bench.py --workload llama70b --steps 2 --warmup 1 --skip-cpu-baseline --skip-e2e --skip-b2b --no-graph > $O/ncu_gemm_70b.log 2>&1; echo "ncu_gemm_70b=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_dual_gemm -s 2 -c 1 -f -o $O/prof_gemm_70b_shard8 \
  python bench.py --workload llama70b --shard-of 8 --steps 2 --warmup 1 --skip-cpu-baseline --skip-e2e --skip-b2b --no-graph > $O/ncu_gemm_70b8.log 2>&1; echo "ncu_gemm_70b8=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_dual_gemm -s 2 -c 1 -f -o $O/prof_gemm_tiny \
  python bench.py --workload tiny_fp32 --steps 2 --warmup 1 --skip-cpu-baseline --skip-e2e --skip-b2b --no-graph > $O/ncu_gemm_tiny.log 2>&1; echo "ncu_gemm_tiny=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_dual_gemm -s 2 -c 1 -f -o $O/prof_gemm_decode_shard8 \
  python bench.py --workload llama7b_decode --shard-of 8 --steps 2 --warmup 1 --skip-cpu-baseline --skip-e2e --skip-b2b --no-graph > $O/ncu_gemm_d8.log 2>&1; echo "ncu_gemm_d8=$?"
# cluster split-K: kernel times per width (ncu, cold L2) and the per-CTA timeline of the decode shards
SHAPES=16x4096x1376,16x4096x2752,16x4096x5504,16x8192x3584 CS=0,1,2,4,6,8 REPS=10 timeout 600 ncu --metrics gpu__time_duration.sum \
  --clock-control none --csv --log-file $O/csplit_ab.csv python scripts/ncu_ab_decode.py > $O/csplit_ab_marks.log 2>&1; echo "csplit_ab=$?"
timeout 300 python scripts/trace_decode.py > $O/trace_decode.log 2>&1; echo "trace_decode=$?"
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/sanitizer_memcheck.log 2>&1; echo "memcheck=$?"
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/sanitizer_synccheck.log 2>&1; echo "synccheck=$?"
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/sanitizer_racecheck.log 2>&1; echo "racecheck=$?"
