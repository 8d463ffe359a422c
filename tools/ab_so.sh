#!/bin/bash
# A/B timing of library builds in build/alt/<name>.so (tools/build_variant.sh):
#   VARS="old new" WHAT="pretrain maml" PROF_STEPS=200 bash tools/ab_so.sh  -> gpurun_out/ab.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=paper_2102_04199_b200/libkerntune_b200.so
cp $L build/alt/_default.so
for r in 1 2; do for v in ${VARS:-old new}; do cp build/alt/$v.so $L; echo "== $v" >> gpurun_out/ab.txt; python ${SCRIPT:-tools/prof_train.py} $WHAT 2>&1 | grep -o "'metric': '[^']*'\|'ms_per_step': [0-9.]*\|'value': [0-9.e+]*\|'frac': [0-9.]*\|'total_ms': [0-9.]*\|'device_ms': [0-9.]*" >> gpurun_out/ab.txt; done; done
cp build/alt/_default.so $L
