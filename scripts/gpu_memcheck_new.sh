#!/usr/bin/env bash
# compute-sanitizer memcheck over the round-2 feature tests (tile widths, multicast clusters,
# dynamic claiming, fused reduction) -- catches out-of-bounds accesses parity cannot see.
O=gpurun_out/${1:-memcheck}; mkdir -p $O
for t in test_fused_reduce_gpu test_dynamic_gpu test_tile_widths_gpu; do
  timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/$t.py -q -x -p no:cacheprovider \
    -k "not 2048 and not 4096" > $O/memcheck_$t.log 2>&1; echo $t=$?
  grep -E "ERROR SUMMARY|passed|failed" $O/memcheck_$t.log | tail -2
done
