#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (+ reference arm), ncu launch list + full capture of the scorer.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu.txt
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref rc=$?" >> gpurun_out/bench_ref.err
# N>1 code path on a one-GPU box: two ranks sharing cuda:0 over gloo (correctness of the sharded
# sweep / e2e / MAML paths, not a scaling number)
KT_BENCH_SAME_DEVICE=1 KT_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --standalone \
  --nproc-per-node 2 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline --meta-steps 20 \
  > gpurun_out/bench_n2_gloo.json 2> gpurun_out/bench_n2_gloo.err
echo "n2 rc=$?" >> gpurun_out/bench_n2_gloo.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-score_tc} -s 3 -c 1 \
  -o gpurun_out/prof_score -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_full.log 2>&1
fi
echo done
