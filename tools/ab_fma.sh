set -e
V0=$PWD/var/v0/libhykin_b200.so
for k in 1 2 3; do
  python tools/time_collision.py --tag fma --iters 5
  HK_LIB=$V0 python tools/time_collision.py --tag v0 --iters 5
done
python -m pytest tests/test_gpu_collision.py tests/test_gpu_edge_cases.py -q -x 2>&1 | tail -3
