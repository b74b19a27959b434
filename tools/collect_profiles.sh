#!/bin/bash
# Summarise a tools/refresh_round.sh capture (gpurun_out/*_TAG*) into profiles/TAG_*.
# Usage: bash tools/collect_profiles.sh TAG [OUTTAG]
set -eu
TAG=$1; OUT=${2:-$1}; G=gpurun_out; P=profiles
tail -n 1 $G/bench_$TAG.json > $P/${OUT}_bench_line.json
tail -n 1 $G/bench_c5_$TAG.json > $P/${OUT}_bench_config5_line.json
cp $G/configs_$TAG.jsonl $P/${OUT}_configs.jsonl
tail -n 3 $G/gpu_tests_$TAG.log > $P/${OUT}_gpu_tests.txt
python3 tools/launch_summary.py $G/launches_$TAG.csv "bench.py --steps 2 --warmup 3 --e2e-steps 0 (ncu launch list, cold-cache, serialised)" > $P/${OUT}_launches.txt
python3 tools/launch_summary.py $G/hyb_launches_$TAG.csv "config-4 hybrid: warm-up + 2 steps (tools/bench_configs.py --configs 4h --hyb-steps 2 --no-full)" > $P/${OUT}_config4_hybrid_launches.txt
for k in coll_fast:collision_fast coll64:collision64 coll16:collision16 resid:residual stage:config3_stage transport:config3_transport; do
  src=${k%%:*}; dst=${k##*:}
  [ -f $G/${src}_$TAG.ncu-rep ] && python3 tools/ncu_summary.py $G/${src}_$TAG.ncu-rep > $P/${OUT}_${dst}_ncu.txt
done
[ -f $G/hybrid_parts_$TAG.txt ] && tail -n 1 $G/hybrid_parts_$TAG.txt > $P/${OUT}_config4_hybrid_parts.txt
[ -f $G/c5_slabs_$TAG.json ] && tail -n 1 $G/c5_slabs_$TAG.json > $P/${OUT}_config5_slabs.json
echo collected into $P/${OUT}_*
