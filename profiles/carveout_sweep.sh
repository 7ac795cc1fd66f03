for v in -1 25 40 50 60; do
  echo "VOTE $v: $(SB_VOTE_CARVEOUT=$v timeout 120 python bench.py --steps 10 --warmup 3 --frames 32 --no-e2e --no-cpu-baseline --blend-steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['blend_r2']['kernels']['vote']['ms_per_launch'])")"
done
for v in -1 50 60 72; do
  echo "STY $v: $(SB_STYLIZE_CARVEOUT=$v timeout 120 python bench.py --steps 10 --warmup 3 --frames 32 --no-e2e --no-cpu-baseline --blend-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['kernels']['stylize']['ms_per_launch'])")"
done
