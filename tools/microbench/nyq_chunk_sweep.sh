#!/bin/bash
# Sweep of the Nyquist-correction chunk size (plane scratch bytes per chunk):
# rebuilds hk_nyqfix.o with -DHK_NYQ_CHUNK_BYTES=B and times the config-4 hybrid
# step's parts (tools/hybrid_parts.py).  Leaves the default build in place.
cd "$(dirname "$0")/../.."
for B in "$@" default; do
  rm -f paper_2505_03360_b200/build/hk_nyqfix.o
  if [ "$B" = default ]; then make -s -C paper_2505_03360_b200/csrc >/dev/null; break; fi
  make -s -C paper_2505_03360_b200/csrc EXTRA_hk_nyqfix="-DHK_NYQ_CHUNK_BYTES=$B" >/dev/null || exit 1
  echo "chunk_bytes=$B $(python tools/hybrid_parts.py)"
done
