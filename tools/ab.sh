#!/bin/bash
# A/B timing of library variants (variants/NAME/libstyleblit.so) on the headline workload.
# Usage: tools/ab.sh ROUNDS NAME... ; prints stylize ms per launch for each run.
R=$1; shift
mkdir -p gpurun_out
for r in $(seq 1 $R); do
  for v in "$@"; do
    out=$(SB_LIBRARY=$PWD/variants/$v/libstyleblit.so timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --blend-steps 0 --lut-rgb-steps 0 --no-configs 2>&1 | tail -1)
    echo "$v $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["kernels"]["stylize"]["ms_per_launch"], d["value"], d["clocks"]["sm_mhz"])' 2>&1 | tail -1)"
  done
done
