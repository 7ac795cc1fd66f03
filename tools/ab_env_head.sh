#!/bin/bash
# A/B timing of run-time switches on the headline workload.  Usage: tools/ab_env_head.sh ROUNDS "ENV=..." ...
# ("-" = no extra environment); prints stylize ms per launch, the headline value and the SM clock.
R=$1; shift
for r in $(seq 1 $R); do
  for v in "$@"; do
    e=""; [ "$v" != "-" ] && e="$v"
    out=$(env $e timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --blend-steps 0 --lut-rgb-steps 0 --no-configs 2>&1 | tail -1)
    echo "$v $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["kernels"]["stylize"]["ms_per_launch"], d["value"], d["clocks"]["sm_mhz"])' 2>&1 | tail -1)"
  done
done
