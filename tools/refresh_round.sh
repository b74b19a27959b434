#!/bin/bash
# Round-end refresh on one GPU: tests, bench line, secondary configs, launch
# list of the bench command, full ncu capture of the production collision kernel.
set -u
mkdir -p gpurun_out
TAG=${1:-r01}
bash tools/profile_round.sh $TAG
timeout 900 python tools/bench_configs.py --configs 1,3,4,5 --iters 3 > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; echo "configs rc=$?"
