#!/bin/bash
# compute-sanitizer over tiny invocations of every device operator (tools/sanitize_driver.py).
# Usage (on the GPU box): bash tools/sanitize.sh OUTDIR
OUT=${1:-gpurun_out/sanitizer}
mkdir -p $OUT
OPS="coll16 coll32 coll32x coll64 coll64x host32 cells steps hybrid"
for tool in memcheck racecheck synccheck initcheck; do
  for op in $OPS; do
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 \
      python tools/sanitize_driver.py $op > $OUT/${tool}_${op}.log 2>&1
    echo "$tool $op rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/${tool}_${op}.log | tail -1)" | tee -a $OUT/summary.txt
  done
done
