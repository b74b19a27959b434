# A/B of the per-cell kernels on config 3: default library vs a variant library under var/
set -e
VAR=$PWD/var/${1:-m0}/libhykin_b200.so
for k in 1 2; do
  python tools/bench_configs.py --configs 3 --iters 3 --no-steps | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new ', {k: round(v, 3) for k, v in d['ms'].items()})"
  HK_LIB=$VAR python tools/bench_configs.py --configs 3 --iters 3 --no-steps | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('base', {k: round(v, 3) for k, v in d['ms'].items()})"
done
