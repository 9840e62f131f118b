#!/usr/bin/env bash
O=gpurun_out/${1:-ab}; mkdir -p $O
timeout 900 python -m pytest tests/test_dynamic_gpu.py tests/test_tile_widths_gpu.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
bash scripts/gpu_ab.sh $1 16x4096x1376,16x4096x11008,2048x4096x1376,2048x4096x11008,4096x8192x28672 > /dev/null 2>&1
cat $O/ab.log
timeout 600 python scripts/tune_decode_bn.py --shapes 16:4096:1376,16:4096:2752,16:8192:3584 --splits 2,3,6 > $O/tune_dec.log 2>&1; cat $O/tune_dec.log
bash scripts/gpu_ab_trace.sh $1 16x4096x11008,16x4096x1376 > /dev/null 2>&1
paste $O/trace_old.log $O/trace_new.log | grep -E "ffn |epi_done|last_mma|last_tfull|exit" | cut -c1-180
