set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2i_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/r2i_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; echo "bench rc $?"; head -c 300 gpurun_out/r2i_bench.json
timeout 1200 python tests/results_table.py --out gpurun_out/r2i_results_table.json > gpurun_out/r2i_results_table.log 2>&1; echo "table rc $?"
timeout 900 python tools/adaptive_sweep.py --frames 4096 --out gpurun_out/r2i_adaptive.json > gpurun_out/r2i_adaptive.log 2>&1; echo "sweep rc $?"
