#!/usr/bin/env bash
O=gpurun_out/${1:-proab}; mkdir -p $O
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_tile_widths_gpu.py tests/test_dynamic_gpu.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest=$?; tail -1 $O/pytest.log
bash scripts/gpu_prologue.sh $1 > /dev/null 2>&1; cat $O/prologue.log
bash scripts/gpu_ab.sh $1 2048x4096x1376,2048x4096x2752,2048x4096x11008,4096x8192x3584,1024x4096x11008 > /dev/null 2>&1; cat $O/ab.log
