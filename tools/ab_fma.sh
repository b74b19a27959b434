# A/B of the FMA pencil transforms: default library vs a variant library under var/
set -e
VAR=$PWD/var/${1:-x0}/libhykin_b200.so
shift || true
for k in 1 2 3; do
  python tools/time_collision.py --tag fma --iters 3 "$@"
  HK_LIB=$VAR python tools/time_collision.py --tag base --iters 3 "$@"
done
