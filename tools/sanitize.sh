#!/usr/bin/env bash
# compute-sanitizer over tools/sanitize_solves.py; one log per tool under
# OUT (default gpurun_out/), summaries copied to profiles/ by hand.
#   tools/sanitize.sh [OUT] [tool ...]      tools default: memcheck racecheck synccheck initcheck
set -u
OUT="${1:-gpurun_out}"
shift || true
TOOLS=("$@")
[ ${#TOOLS[@]} -eq 0 ] && TOOLS=(memcheck racecheck synccheck initcheck)
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in "${TOOLS[@]}"; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  timeout 1500 "$CS" --tool "$tool" $extra --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_solves.py > "$OUT/sanitize_$tool.log" 2>&1
  echo "$tool rc=$?" >> "$OUT/sanitize_summary.txt"
done
