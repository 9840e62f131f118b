O=gpurun_out/e11; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo p=$?
SH=2048x4096x11008,2048x4096x1376,16x4096x11008,256x4096x11008,4096x8192x3584,512x2048x512
cp paper_2501_08071_b200/libcuasm_ffn.so paper_2501_08071_b200/lib_new.so
for i in 1 2; do
 cp paper_2501_08071_b200/lib_old.so paper_2501_08071_b200/libcuasm_ffn.so; python scripts/ab_lib.py old $SH >> $O/ab.log 2>&1
 cp paper_2501_08071_b200/lib_new.so paper_2501_08071_b200/libcuasm_ffn.so; python scripts/ab_lib.py new $SH >> $O/ab.log 2>&1
done
timeout 300 python scripts/trace_gemm.py --shapes 2048x4096x1376,16x4096x11008 --scheds 0 > $O/trace.log 2>&1
