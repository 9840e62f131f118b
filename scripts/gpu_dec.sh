#!/usr/bin/env bash
O=gpurun_out/${1:-dec}; mkdir -p $O
timeout 900 python -m pytest tests/test_tile_widths_gpu.py -q -x -p no:cacheprovider -k bn64 > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
timeout 900 python scripts/tune_decode_bn.py > $O/tune_decode_bn.log 2>&1; echo tune=$?; cat $O/tune_decode_bn.log
