# PDL on vs off under the per-step (iso) protocol and back to back, alternating twice
for i in 1 2; do for w in llama7b_decode llama7b_prefill; do for pdl in "" "--no-pdl"; do
  for P in 1 8; do
    python bench.py --workload $w --shard-of $P $pdl --skip-cpu-baseline --skip-e2e --protocol-runs 0 --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w P=$P pdl=${pdl:-on}', d['ms_per_step'], 'b2b', d['back_to_back']['ms_per_step'] if d.get('back_to_back') else None)"
  done
done; done; done
