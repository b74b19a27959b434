#!/bin/bash
# Round refresh on one GPU (run through gpurun): GPU tests, the bench lines
# (config 2 headline with the CPU baseline; config-5 slab step), secondary
# configs, launch lists, full ncu captures of the production kernels.
# Usage: bash tools/refresh_round.sh TAG
set -u
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 $O/gpu_tests_$TAG.log
timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --workload config5 --steps 3 --warmup 3 > $O/bench_c5_$TAG.json 2> $O/bench_c5_$TAG.err; echo "bench c5 rc=$?"
timeout 1500 python tools/bench_configs.py --configs 1,3,4,4h,4s,4b,5 --iters 3 > $O/configs_$TAG.jsonl 2> $O/configs_$TAG.err; echo "configs rc=$?"
ARGS="--steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 600 python bench.py $ARGS > $O/plain_launch_$TAG.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:hk:: --csv \
  --log-file $O/launches_$TAG.csv python bench.py $ARGS > $O/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/hyb_launches_$TAG.csv \
  python tools/bench_configs.py --configs 4h --hyb-steps 2 --no-full > $O/hyb_ncu_$TAG.log 2>&1; echo "hybrid launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coll_fast_w12 -c 1 -o $O/coll_fast_$TAG -f \
  python tools/profile_collision.py --cells 1024 --iters 1 > $O/ncu_full_$TAG.log 2>&1; echo "ncu N=32 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coll64_w12 -c 1 -o $O/coll64_$TAG -f \
  python tools/profile_collision.py --n 64 --cells 128 --iters 1 > $O/ncu64_full_$TAG.log 2>&1; echo "ncu N=64 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:residual_cta -c 1 -o $O/resid_$TAG -f \
  python tools/time_residual.py --cells 2048 > $O/ncu_resid_$TAG.log 2>&1; echo "ncu residual rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:coll16 -c 1 -o $O/coll16_$TAG -f \
  python tools/bench_configs.py --configs 1 --iters 1 > $O/ncu16_$TAG.log 2>&1; echo "ncu N=16 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_cta -s 2 -c 1 -o $O/stage_$TAG -f \
  python tools/esbgk_step.py stage > $O/ncu_stage_$TAG.log 2>&1; echo "ncu stage rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transport_lanes -s 6 -c 2 -o $O/transport_$TAG -f \
  python tools/esbgk_step.py step > $O/ncu_transport_$TAG.log 2>&1; echo "ncu transport rc=$?"
timeout 300 python tools/hybrid_parts.py > $O/hybrid_parts_$TAG.txt 2>&1; echo "hybrid parts rc=$?"
timeout 600 python tools/c5_slab_profile.py > $O/c5_slabs_$TAG.json 2>&1; echo "config-5 slabs rc=$?"
