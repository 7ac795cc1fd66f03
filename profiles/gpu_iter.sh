#!/bin/bash
# One GPU iteration: parity tests, a bench line, then (only if the plain run exits 0) an ncu
# --set full capture of the stylize and vote kernels (16 frames: > L2, so DRAM traffic is real).
# Usage: [NCU=1] [LAUNCHES=1] profiles/gpu_iter.sh TAG [pytest-args]
TAG=${1:-iter}
shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${TAG}.log
C="python bench.py --steps 1 --warmup 1 --blend-steps 1 --lut-rgb-steps 0 --frames 16 --no-e2e --no-cpu-baseline"
if [ -n "$NCU" ]; then
  timeout 200 $C > gpurun_out/plain_${TAG}.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stylize_tiled|vote_kernel" -s 1 -c 3 -o gpurun_out/prof_${TAG} $C > gpurun_out/ncu_${TAG}.log 2>&1
  echo "ncu rc=$?"
fi
if [ -n "$LAUNCHES" ]; then
  C2="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout 200 $C2 > gpurun_out/plain2_${TAG}.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $C2 > gpurun_out/ncu_launches_${TAG}.log 2>&1
  echo "launches rc=$?"
fi
