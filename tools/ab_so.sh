mkdir -p gpurun_out
L=paper_2102_04199_b200/libkerntune_b200.so
for r in 1 2; do for v in old new; do cp build/alt/$v.so $L; echo "== $v" >> gpurun_out/ab.txt; python tools/prof_train.py $WHAT 2>&1 | grep -o "'metric': '[^']*'\|'ms_per_step': [0-9.]*\|'value': [0-9.e+]*" >> gpurun_out/ab.txt; done; done
cp build/alt/new.so $L
