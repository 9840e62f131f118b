#!/usr/bin/env bash
# A/B of two library builds on one box: lib_old.so vs the current libcuasm_ffn.so (step times
# under the L2-flush protocol, alternating twice), plus per-CTA traces of each.
O=gpurun_out/${1:-ab}; mkdir -p $O
SH=${2:-2048x4096x1376,2048x4096x11008,4096x8192x3584}
cp paper_2501_08071_b200/libcuasm_ffn.so paper_2501_08071_b200/lib_new.so
for i in 1 2; do
 cp paper_2501_08071_b200/lib_old.so paper_2501_08071_b200/libcuasm_ffn.so; python scripts/ab_lib.py old $SH >> $O/ab.log 2>&1
 cp paper_2501_08071_b200/lib_new.so paper_2501_08071_b200/libcuasm_ffn.so; python scripts/ab_lib.py new $SH >> $O/ab.log 2>&1
done
cat $O/ab.log
cp paper_2501_08071_b200/lib_old.so paper_2501_08071_b200/libcuasm_ffn.so
timeout 300 python scripts/trace_gemm.py --shapes 2048x4096x1376 --scheds 1 > $O/trace_old.log 2>&1
cp paper_2501_08071_b200/lib_new.so paper_2501_08071_b200/libcuasm_ffn.so
timeout 300 python scripts/trace_gemm.py --shapes 2048x4096x1376 --scheds 1 > $O/trace_new.log 2>&1
grep -E "cycles per|wait per|first_tfull|first_tma" $O/trace_old.log $O/trace_new.log
