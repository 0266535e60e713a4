#!/bin/bash
# A/B timing of alternative in-tree builds on one GPU: tools/ab_decode.sh <workloads> <frames> lib1.so lib2.so ...
# Runs every library 3 times, interleaved, and prints one line per run (min of 5 launches each).
wl=$1; F=$2; shift 2
for rep in 1 2 3; do
  for L in "$@"; do
    QKD_LIB=$PWD/$L python tools/prof_decode.py --workload $wl --frames $F --reps 5 2>&1 | \
      python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$L', d['workload'], '%.3f'%d['ms_min'], round(d['alg_GBps']))"
  done
done
