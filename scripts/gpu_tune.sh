O=gpurun_out/e10; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "schedules" > $O/pytest.log 2>&1; echo p=$?
timeout 900 python scripts/tune.py --out $O/tune.json > $O/tune.log 2>&1; echo tune=$?
timeout 600 python scripts/tune.py --N 1376 --ms 16,128,256,512,1024,2048,4096 --out $O/tune_n1376.json > $O/tune_n1376.log 2>&1; echo t8=$?
timeout 600 python scripts/tune.py --K 8192 --N 3584 --ms 4096 > $O/tune_70b8.log 2>&1; echo t70=$?
timeout 600 python bench.py --workload llama70b --skip-cpu-baseline --skip-e2e > $O/bench_70b.json 2>>$O/err; echo b70=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_dual_gemm -s 2 -c 1 -f -o $O/prof_gemm_70b python bench.py --workload llama70b --steps 2 --warmup 1 --skip-cpu-baseline --skip-e2e --skip-b2b --no-graph > $O/ncu70.log 2>&1; echo ncu=$?
