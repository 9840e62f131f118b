#!/usr/bin/env bash
O=gpurun_out/${1:-ab}; mkdir -p $O
bash scripts/gpu_ab.sh $1 16x4096x1376,16x4096x2752,16x4096x11008,16x8192x3584 > /dev/null 2>&1
cat $O/ab.log
timeout 600 python scripts/tune_decode_bn.py --shapes 16:4096:1376,16:4096:2752 --splits 2,3,4,6 > $O/tune_dec.log 2>&1; cat $O/tune_dec.log
