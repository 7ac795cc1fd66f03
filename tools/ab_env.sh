#!/bin/bash
# A/B timing of run-time switches on the blend (r=2) path.  Usage: tools/ab_env.sh ROUNDS "ENV=..." ...
# ("-" = no extra environment); prints vote ms, stylize ms and the blend value per run.
R=$1; shift
for r in $(seq 1 $R); do
  for v in "$@"; do
    e=""; [ "$v" != "-" ] && e="$v"
    out=$(env $e timeout 300 python bench.py --steps 3 --warmup 3 --blend-steps 20 --no-e2e --no-cpu-baseline --lut-rgb-steps 0 2>&1 | tail -1)
    echo "$v $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read())["blend_r2"]; print(d["kernels"]["vote"]["ms_per_launch"], d["kernels"]["stylize"]["ms_per_launch"], d["value"])' 2>&1 | tail -1)"
  done
done
