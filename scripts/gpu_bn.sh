#!/usr/bin/env bash
# Tile-width bring-up: the tile-width parity tests, then the width x schedule timing table.
O=gpurun_out/${1:-bn}; mkdir -p $O
timeout 900 python -m pytest tests/test_tile_widths_gpu.py -q -x -p no:cacheprovider > $O/pytest_bn.log 2>&1; echo pytest_bn=$?
tail -3 $O/pytest_bn.log
timeout 900 python scripts/tune_bn.py --bns ${BNS:-128,120,112} --shapes ${SHAPES:-2048:4096:11008,4096:4096:11008,16384:4096:11008,4096:8192:28672,4096:8192:3584,512:4096:11008,1024:4096:11008} --out $O/tune_bn.json > $O/tune_bn.log 2>&1; echo tune=$?
cut -c1-330 $O/tune_bn.log
