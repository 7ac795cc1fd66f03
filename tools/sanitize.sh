#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py with each tool; logs in gpurun_out/sanitize_TAG_*.log
# Usage (on a GPU box): tools/sanitize.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
CS=${CS:-/usr/local/cuda/bin/compute-sanitizer}
for tool in memcheck synccheck initcheck racecheck; do
  extra=""
  q=""
  [ "$tool" = racecheck ] && { extra="--racecheck-report all"; q="--quick"; }
  [ "$tool" = initcheck ] && q="--quick"
  timeout 1200 $CS --tool $tool $extra --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_run.py $q > gpurun_out/sanitize_${TAG}_${tool}.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_${TAG}_${tool}.log
done
