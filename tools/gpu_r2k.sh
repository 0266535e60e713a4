set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2k_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r2k_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/r2k_smoke.log
timeout 600 python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err; echo "bench rc $?"; head -c 600 gpurun_out/r2k_bench.json
