set -x
bash tools/racecheck.sh run r2
bash tools/ab_decode.sh C4@0.08 4096 build_ab/t12.so build_ab/c4cs.so
bash tools/ab_decode.sh C4@0.02 4096 build_ab/t12.so build_ab/c4cs.so
QKD_LIB=$PWD/build_ab/c4cs.so timeout 900 python -m pytest tests/test_gpu_fullbatch.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -k "long or full" 2>&1 | tail -3
QKD_LIB=$PWD/build_ab/c4cs.so timeout 900 ncu --set full --clock-control none -k regex:decode_kernel -c 1 -o gpurun_out/prof_r2d_c4cs python tools/prof_decode.py --workload C4@0.08 --frames 4096 --reps 1 > /dev/null 2>&1; echo "ncu rc $?"
