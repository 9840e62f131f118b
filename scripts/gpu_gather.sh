O=gpurun_out/e7; mkdir -p $O
for P in 8; do
 for w in llama70b llama7b_prefill; do
  timeout 600 python bench.py --workload $w --shard-of $P --skip-cpu-baseline --skip-e2e --skip-b2b > $O/b_${w}_p$P.json 2>> $O/err; echo $w$P=$?
  timeout 600 python bench.py --workload $w --shard-of $P --fused-gather --skip-cpu-baseline --skip-e2e > $O/b_${w}_p${P}_fg.json 2>> $O/err; echo $w${P}fg=$?
 done
done
timeout 600 python bench.py --workload llama7b_prefill --fused-gather --skip-cpu-baseline --skip-e2e > $O/b_7b_fg1.json 2>> $O/err; echo fg1=$?
