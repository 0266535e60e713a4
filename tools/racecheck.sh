#!/bin/bash
# Layer-order race check of the decode kernels (compute-sanitizer is closed on this GPU pool).
#   build (here):  bash tools/racecheck.sh build
#   run (GPU box): bash tools/racecheck.sh run [tag]
# The racecheck build stamps every E write with its layer number and checks every E read against the
# layer that must have written it last (decode_kernel.cuh rc_row); a decode call fails on any stale or
# early read.  The GPU parity and fuzz suites are run on that build (every decode variant but the
# lane-pair one), then on a mutant that drops the barrier between block rows, where the check must fire.
set -u
mode=${1:-run}; tag=${2:-r2}
if [ "$mode" = build ]; then
  python tools/build_variant.py build_ab/racecheck.so -DQKD_RACECHECK &
  python tools/build_variant.py build_ab/racecheck_nobar.so -DQKD_RACECHECK -DQKD_MUTATE_NOBAR &
  wait
  exit 0
fi
out=gpurun_out/racecheck_$tag; mkdir -p $out
QKD_LIB=$PWD/build_ab/racecheck.so timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py \
  tests/test_gpu_fullbatch.py tests/test_adaptive.py -m gpu -q -p no:cacheprovider > $out/racecheck.log 2>&1
echo "racecheck build, parity suites: rc $?" | tee $out/summary.txt
tail -3 $out/racecheck.log | tee -a $out/summary.txt
QKD_LIB=$PWD/build_ab/racecheck_nobar.so timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider \
  -k "random_codes or decode_parity_workloads" > $out/mutant.log 2>&1
echo "mutant (no barrier between block rows): rc $? (must fail)" | tee -a $out/summary.txt
grep -c "racecheck: [0-9]" $out/mutant.log | sed 's/^/racecheck reports in mutant log: /' | tee -a $out/summary.txt
grep -m3 -o "racecheck: [^\"']*" $out/mutant.log | tee -a $out/summary.txt
