#!/usr/bin/env bash
O=gpurun_out/${1:-cold}; mkdir -p $O
timeout 300 python scripts/trace_gemm.py --shapes 2048x4096x1376,2048x4096x11008 --scheds 0 > $O/trace_flush.log 2>&1
NOFLUSH=1 timeout 300 python scripts/trace_gemm.py --shapes 2048x4096x1376,2048x4096x11008 --scheds 0 > $O/trace_noflush.log 2>&1
paste $O/trace_flush.log $O/trace_noflush.log | grep -E "ffn |first_tma|epi_start|last_mma|epi_done|exit|first_tfull|cycles per" | cut -c1-190
