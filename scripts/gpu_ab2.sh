#!/usr/bin/env bash
O=gpurun_out/${1:-ab}; mkdir -p $O
timeout 900 python -m pytest tests/test_dynamic_gpu.py tests/test_tile_widths_gpu.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
bash scripts/gpu_ab.sh $1 2048x4096x1376,2048x4096x11008,4096x8192x3584,4096x8192x28672
