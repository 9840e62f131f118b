#!/usr/bin/env bash
# Tile-width bring-up: the new parity tests, then the width x schedule timing table.
O=gpurun_out/${1:-bn}
mkdir -p $O
timeout 900 python -m pytest tests/test_tile_widths_gpu.py -q -x -p no:cacheprovider > $O/pytest_bn.log 2>&1; echo pytest_bn=$?
tail -5 $O/pytest_bn.log
timeout 900 python scripts/tune_bn.py --out $O/tune_bn.json > $O/tune_bn.log 2>&1; echo tune=$?
cat $O/tune_bn.log | cut -c1-400
