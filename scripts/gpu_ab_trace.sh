#!/usr/bin/env bash
# per-CTA traces of the same shapes with lib_old.so and the current build
O=gpurun_out/${1:-abt}; mkdir -p $O
SH=${2:-16x4096x11008}
cp paper_2501_08071_b200/libcuasm_ffn.so paper_2501_08071_b200/lib_new.so
cp paper_2501_08071_b200/lib_old.so paper_2501_08071_b200/libcuasm_ffn.so
timeout 300 python scripts/trace_gemm.py --shapes $SH --scheds 0 > $O/trace_old.log 2>&1
cp paper_2501_08071_b200/lib_new.so paper_2501_08071_b200/libcuasm_ffn.so
timeout 300 python scripts/trace_gemm.py --shapes $SH --scheds 0 > $O/trace_new.log 2>&1
paste $O/trace_old.log $O/trace_new.log | cut -c1-200
