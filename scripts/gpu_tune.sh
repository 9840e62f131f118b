O=gpurun_out/e4; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest=$?
timeout 600 python scripts/tune.py --out $O/tune.json > $O/tune.log 2>&1; echo tune=$?
timeout 600 python scripts/tune.py --N 1376 --ms 1,16,64,128,256,512,1024,2048,4096 --out $O/tune_n1376.json > $O/tune_n1376.log 2>&1; echo tune8=$?
timeout 600 python scripts/tune.py --op gemm --ms 512,2048,4096 --K 4096 --N 4096 > $O/tune_gemm.log 2>&1; echo tg=$?
timeout 600 python scripts/tune.py --op gemm --ms 2048 --K 11008 --N 4096 >> $O/tune_gemm.log 2>&1; echo tg2=$?
timeout 600 python scripts/tune.py --op gemm --ms 512 --K 2048 --N 512 >> $O/tune_gemm.log 2>&1; echo tg3=$?
timeout 300 python scripts/trace_gemm.py --shapes 2048x4096x11008,2048x4096x1376,16x4096x1376,16x4096x11008,256x4096x11008 --scheds 0,2 > $O/trace.log 2>&1; echo tr=$?
