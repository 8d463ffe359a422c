#!/bin/bash
# One gpurun iteration on the scorer: forward/baseline parity tests, a short bench (no CPU
# arms, no extras), and the CTA-0 pipeline timeline from the -DKT_TC_TRACE build.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_forward.py tests/test_gpu_baseline.py tests/test_sa.py -q -m gpu \
  -p no:cacheprovider -x > gpurun_out/pt.txt 2>&1
echo "rc=$?" >> gpurun_out/pt.txt
timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 200 > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ "${TRACE:-1}" = "1" ]; then timeout 300 python tools/tc_trace_full.py > gpurun_out/trace.txt 2>&1; fi
echo done
