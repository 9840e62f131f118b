#!/usr/bin/env bash
O=gpurun_out/${1:-prologue}; mkdir -p $O
cp paper_2501_08071_b200/libcuasm_ffn.so paper_2501_08071_b200/lib_new.so
cp paper_2501_08071_b200/lib_diag.so paper_2501_08071_b200/libcuasm_ffn.so
timeout 300 python scripts/trace_prologue.py 2048x4096x1376,2048x4096x11008,16x4096x11008 > $O/prologue.log 2>&1
NOFLUSH=1 timeout 300 python scripts/trace_prologue.py 2048x4096x1376 > $O/prologue2.log 2>&1
cp paper_2501_08071_b200/lib_new.so paper_2501_08071_b200/libcuasm_ffn.so
cat $O/prologue.log
