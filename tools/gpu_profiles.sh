#!/bin/bash
# One gpurun call: the ncu evidence for profiles/ (launch list of a bench step, full captures of
# the scorer and the secondary-path kernels).  Never take bench numbers from these runs.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_tc -s 3 -c 1 \
  -o gpurun_out/prof_score -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_score.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:factor_|maml_task|task_sum|fine_tune_cluster" -s 4 -c 6 \
  -o gpurun_out/prof_train -f python tools/prof_train.py pretrain maml fine_tune > gpurun_out/ncu_train.log 2>&1
PROF_STEPS=5 timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:maml_task|task_sum|fine_tune_cluster" -s 6 -c 5 \
  -o gpurun_out/prof_meta -f python tools/prof_train.py maml fine_tune > gpurun_out/ncu_meta.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:pipe_kernel|readout_kernel" -s 3 -c 3 \
  -o gpurun_out/prof_agg -f python tools/prof_train.py aggregate > gpurun_out/ncu_agg.log 2>&1
echo done
