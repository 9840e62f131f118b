# A/B of lib_old.so vs lib_new.so with scripts/ab_push64.py, alternating twice
for i in 1 2; do for v in old new; do cp paper_2501_08071_b200/lib_$v.so paper_2501_08071_b200/libcuasm_ffn.so; python scripts/ab_push64.py $v $1; done; done
cp paper_2501_08071_b200/lib_new.so paper_2501_08071_b200/libcuasm_ffn.so
