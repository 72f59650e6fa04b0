#!/bin/bash
# c1 side-by-side batch vs the stop-mode launch length (finer launches interleave the 10 lanes
# over the 7 co-resident clusters better).
cd "$(dirname "$0")/.."
for C in default 512 1024 2048; do
  if [ "$C" = default ]; then unset KZ_STOP_CHUNK; else export KZ_STOP_CHUNK=$C; fi
  echo "== chunk $C"; python tools/exp_cc_ctas.py 2>&1 | sed -n 1,3p
done
