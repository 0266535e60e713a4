set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2e_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r2e_pytest_gpu.log
cp paper_1903_10107_b200/libqkdldpc.so build_ab/prod.so
bash tools/ab_decode.sh C4@0.08 4096 build_ab/nocs.so build_ab/prod.so
bash tools/ab_decode.sh C4@0.02 4096 build_ab/nocs.so build_ab/prod.so
bash tools/ab_decode.sh C5a 9472 build_ab/t12.so build_ab/prod.so
timeout 900 ncu --set full --clock-control none -k regex:decode_kernel -c 1 -o gpurun_out/prof_r2e_c4 python tools/prof_decode.py --workload C4@0.08 --frames 4096 --reps 1 > gpurun_out/r2e_ncu_c4.log 2>&1; echo "ncu rc $?"
timeout 900 python tools/de_codes.py --profile "8,50,1024;2:25,3:20,6:5" --profile "8,50,1024;2:13,3:21,8:16" --profile "8,50,1024;2:11,3:24,8:15" --profile "16,100,512;2:12,3:64,12:24" --profile "16,100,512;2:12,3:64,5:1,10:1,12:22" --out gpurun_out/r2e_de_codes.json > gpurun_out/r2e_de_codes.log 2>&1; echo "de rc $?"
QKD_LIB=$PWD/build_ab/racecheck_nobar.so timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "random_codes or decode_parity_workloads" > gpurun_out/racecheck_r2/mutant2.log 2>&1; echo "mutant rc $?"; grep -c "racecheck: [0-9]" gpurun_out/racecheck_r2/mutant2.log; tail -2 gpurun_out/racecheck_r2/mutant2.log
