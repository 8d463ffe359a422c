#!/bin/bash
# Scorer iteration: forward parity tests, short bench (no CPU leg, no extras), ncu of the tc scorer.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_forward.py -q -x -p no:cacheprovider > gpurun_out/pytest_fwd.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_fwd.txt
timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 100 > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err
echo "bench rc=$?" >> gpurun_out/bench_tc.err
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-score_tc} -s 3 -c 1 \
  -o gpurun_out/prof_tc -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_tc.log 2>&1
fi
echo done
