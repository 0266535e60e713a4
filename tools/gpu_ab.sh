#!/bin/bash
# A/B run on the GPU box: bash tools/gpu_ab.sh "<workload frames>;<workload frames>" lib1.so lib2.so ...
specs=$1; shift
IFS=';' read -ra S <<< "$specs"
for s in "${S[@]}"; do
  set -- $s "$@"
  wl=$1; F=$2; shift 2
  bash tools/ab_decode.sh $wl $F "$@"
done
