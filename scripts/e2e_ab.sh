for i in 1 2; do for v in old new; do cp paper_2501_08071_b200/lib_$v.so paper_2501_08071_b200/libcuasm_ffn.so
python bench.py --skip-cpu-baseline --skip-b2b --protocol-runs 0 --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['e2e']['value'], d['e2e']['ms_per_step'], d['value'])"
done; done
