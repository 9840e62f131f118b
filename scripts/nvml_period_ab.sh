# Does the NVML clock sampler (a thread polling every P seconds during the timed region) slow the
# default bench line?  Alternating runs of the default 7B prefill line at three periods.
for i in 1 2; do for P in 0.005 0.05 0.5; do
  CUASM_BENCH_NVML_PERIOD_S=$P python bench.py --skip-cpu-baseline --skip-e2e --skip-b2b 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('period', '$P', d['ms_per_step'], d['value'], 'protocol', d['protocol_5x100']['ms_per_step_mean'], d['clocks']['samples'], d['clocks']['reasons'])"
done; done
