#!/bin/bash
# A/B timing of library variants on the blend (r=2) path: prints vote and stylize ms per launch.
R=$1; shift
for r in $(seq 1 $R); do
  for v in "$@"; do
    out=$(SB_LIBRARY=$PWD/variants/$v/libstyleblit.so timeout 300 python bench.py --steps 3 --warmup 3 --blend-steps 20 --no-e2e --no-cpu-baseline --lut-rgb-steps 0 --no-configs 2>&1 | tail -1)
    echo "$v $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read())["blend_r2"]; print(d["kernels"]["vote"]["ms_per_launch"], d["kernels"]["stylize"]["ms_per_launch"], d["value"])' 2>&1 | tail -1)"
  done
done
