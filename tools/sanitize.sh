#!/usr/bin/env bash
# compute-sanitizer over tools/sanitize_solves.py; one log per tool under
# ${1:-gpurun_out}/ (summaries copied to profiles/ by hand).
set -u
OUT="${1:-gpurun_out}"
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  timeout 1500 "$CS" --tool "$tool" $extra --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_solves.py > "$OUT/sanitize_$tool.log" 2>&1
  echo "$tool rc=$?" >> "$OUT/sanitize_summary.txt"
done
