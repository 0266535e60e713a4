set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2g_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r2g_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/r2g_smoke.log
timeout 600 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo "bench rc $?"; head -c 400 gpurun_out/r2g_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2g_bench_ref.json 2>&1; echo "ref rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2g_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2g_ncu_launch.log 2>&1; echo "ncu1 rc $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -c 1 -o gpurun_out/prof_r2g_bench python bench.py --steps 1 --warmup 3 > gpurun_out/r2g_ncu_full.log 2>&1; echo "ncu2 rc $?"
timeout 1200 python tests/results_table.py --out gpurun_out/r2g_results_table.json > gpurun_out/r2g_results_table.log 2>&1; echo "table rc $?"
