#!/bin/bash
# A/B of library builds (build/alt/<name>.so in VARS) on the headline bench: step, scorer kernel and e2e ms.
mkdir -p gpurun_out
L=paper_2102_04199_b200/libkerntune_b200.so
cp $L build/alt/_default.so
for r in ${REPS:-1 2}; do for v in $VARS; do cp build/alt/$v.so $L; python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],5), round(d['roofline']['kernel_ms'],5), round(d['e2e']['ms_per_step'],5))" >> gpurun_out/abb.txt; done; done
cp build/alt/_default.so $L
