#!/usr/bin/env bash
# Dynamic tile claiming: tests, A/B timing (+ group sizes on 70B), 70B DRAM bytes.
O=gpurun_out/${1:-dyn}
mkdir -p $O
timeout 900 python -m pytest tests/test_dynamic_gpu.py tests/test_robustness_gpu.py -q -x -p no:cacheprovider > $O/pytest_dyn.log 2>&1; echo pytest_dyn=$?
tail -3 $O/pytest_dyn.log
timeout 900 python scripts/tune_dyn.py > $O/tune_dyn.log 2>&1; echo tune=$?
cat $O/tune_dyn.log
timeout 900 python scripts/tune_dyn.py --shapes 4096:8192:28672 --groups 8,12,16 > $O/tune_dyn_g.log 2>&1; echo tune_g=$?
cat $O/tune_dyn_g.log
for g in 8 16; do
timeout 600 ncu --set full --clock-control none -k regex:ffn_dual_gemm -s 2 -c 1 -f -o $O/prof_70b_g$g \
  python scripts/tune_dyn.py --shapes 4096:8192:28672 --dyn 0 --groups $g --steps 1 > $O/ncu_70b_g$g.log 2>&1; echo ncu70_$g=$?
done
