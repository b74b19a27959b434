#!/bin/bash
# One GPU session: GPU tests, bench (with CPU baseline), launch list of the
# bench command, full ncu capture of the production collision kernel.
set -u
mkdir -p gpurun_out
TAG=${1:-r01}
timeout 600 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/gpu_tests_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
export HK_NO_STREAMED_IO=1  # the streamed e2e kernel waits on concurrent copies: not profilable under ncu serialisation
ARGS="--steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
timeout 600 python bench.py $ARGS > gpurun_out/plain_launch_$TAG.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:hk:: --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py $ARGS > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
timeout 300 python tools/profile_collision.py --cells 1024 --iters 1 > gpurun_out/plain_prof_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:coll_fast_w12 -c 1 -o gpurun_out/coll_fast_$TAG \
  python tools/profile_collision.py --cells 1024 --iters 1 > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
