mkdir -p gpurun_out
# A/B launch lists: ncu kernel-time list of tools/prof_train.py pretrain for each build/alt/<name>.so in VARS.
L=paper_2102_04199_b200/libkerntune_b200.so
for v in ${VARS:-old new}; do cp build/alt/$v.so $L; PROF_STEPS=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_$v.csv python tools/prof_train.py pretrain > /dev/null 2>&1; done
cp build/alt/new.so $L
