#!/bin/bash
# Variants of the Nyquist correction: rebuilds hk_nyqfix.o with each argument as
# its extra nvcc flags (e.g. "-DHK_NYQ_CHUNK_BYTES=100663296", "-DHK_NYQ_KB32=8";
# "base" = none) and times the config-4 hybrid step's parts
# (tools/hybrid_parts.py).  Leaves the default build in place.
cd "$(dirname "$0")/../.."
for B in "$@"; do
  rm -f paper_2505_03360_b200/build/hk_nyqfix.o
  F="$B"; [ "$B" = base ] && F=""
  make -s -C paper_2505_03360_b200/csrc EXTRA_hk_nyqfix="$F" >/dev/null || exit 1
  echo "flags=[$F] $(python tools/hybrid_parts.py)"
done
rm -f paper_2505_03360_b200/build/hk_nyqfix.o
make -s -C paper_2505_03360_b200/csrc >/dev/null
