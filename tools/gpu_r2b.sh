set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2b_pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/r2b_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo "bench rc $?"
cat gpurun_out/r2b_bench.json
for p in pipe_probe pipe_probe2 pipe_probe3; do timeout 120 tools/$p > gpurun_out/r2b_$p.txt 2>&1; done
timeout 1200 python tools/results_table.py --out gpurun_out/r2b_results_table.json > gpurun_out/r2b_results_table.log 2>&1; echo "table rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2b_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2b_ncu_launch.log 2>&1; echo "ncu1 rc $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -c 1 -o gpurun_out/prof_r2b_bench python bench.py --steps 1 --warmup 3 > gpurun_out/r2b_ncu_full.log 2>&1; echo "ncu2 rc $?"
timeout 2400 bash tools/sanitize.sh r2b; echo "sanitize rc $?"
