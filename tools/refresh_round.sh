#!/bin/bash
# Round-end refresh on one GPU: tests, bench line, secondary configs (incl. the
# config-4 hybrid run), launch lists of the bench command and of two hybrid
# steps, full ncu captures of the production collision kernel and the N = 16 kernel.
set -u
mkdir -p gpurun_out
TAG=${1:-r01}
bash tools/profile_round.sh $TAG
timeout 900 python tools/bench_configs.py --configs 1,3,4,4h,5 --iters 3 > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; echo "configs rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/hyb_launches_$TAG.csv \
  python tools/bench_configs.py --configs 4h --hyb-steps 2 --no-full > gpurun_out/hyb_ncu_$TAG.log 2>&1; echo "hybrid launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:coll16 -c 1 -o gpurun_out/coll16_$TAG \
  python tools/bench_configs.py --configs 1 --iters 1 > gpurun_out/ncu16_$TAG.log 2>&1; echo "ncu N=16 rc=$?"
