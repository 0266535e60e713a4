set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2f_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r2f_pytest_gpu.log
timeout 300 python -m pytest tests/test_gpu_errors.py -m gpu -q -s -p no:cacheprovider -k host_overhead 2>&1 | grep "host time" | tee gpurun_out/r2f_host_time.txt
cp paper_1903_10107_b200/libqkdldpc.so build_ab/prod2.so
bash tools/ab_decode.sh C4@0.08 4096 build_ab/g1024lr.so build_ab/prod2.so
timeout 600 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc $?"; cat gpurun_out/r2f_bench.json | head -c 600
timeout 1200 python tests/results_table.py --out gpurun_out/r2f_results_table.json > gpurun_out/r2f_results_table.log 2>&1; echo "table rc $?"
timeout 900 ncu --set full --clock-control none -k regex:decode_kernel -c 1 -o gpurun_out/prof_r2f_c4 python tools/prof_decode.py --workload C4@0.08 --frames 4096 --reps 1 > gpurun_out/r2f_ncu_c4.log 2>&1; echo "ncu rc $?"
