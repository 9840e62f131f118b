#!/usr/bin/env bash
# Dynamic tile claiming: tests, A/B timing (off = 1 / on = 2), 70B DRAM bytes.
O=gpurun_out/${1:-dyn}
mkdir -p $O
timeout 900 python -m pytest tests/test_dynamic_gpu.py tests/test_robustness_gpu.py tests/test_tile_widths_gpu.py -q -x -p no:cacheprovider > $O/pytest_dyn.log 2>&1; echo pytest_dyn=$?
tail -3 $O/pytest_dyn.log
timeout 900 python scripts/tune_dyn.py --shapes 2048:4096:1376,2048:4096:2752,2048:4096:5504,2048:4096:11008,4096:8192:3584,4096:8192:7168,4096:8192:28672,1024:4096:11008,512:4096:11008 > $O/tune_dyn.log 2>&1; echo tune=$?
cat $O/tune_dyn.log
timeout 300 python scripts/trace_gemm.py --shapes 2048x4096x1376 --scheds 0 > $O/trace_p8.log 2>&1
grep -E "cycles per|first_tma|last_mma|exit" $O/trace_p8.log
timeout 600 ncu --set full --clock-control none -k regex:ffn_dual_gemm -s 2 -c 1 -f -o $O/prof_70b \
  python scripts/tune_dyn.py --shapes 4096:8192:28672 --dyn 0 --steps 1 > $O/ncu_70b.log 2>&1; echo ncu70=$?
