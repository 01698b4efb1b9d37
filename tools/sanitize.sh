#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_case.py (run on a GPU box):
#   bash tools/sanitize.sh [outdir]      -> <outdir>/sanitizer_<tool>_<case>.log
out=${1:-gpurun_out}
mkdir -p "$out"
for tool in memcheck racecheck synccheck; do
  for case in ${CASES:-c1 edge ring win typed fused}; do
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check full"
    [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    timeout 900 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_case.py $case \
      > "$out/sanitizer_${tool}_${case}.log" 2>&1
    echo "$tool $case rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' "$out/sanitizer_${tool}_${case}.log" | tail -1)"
  done
done
