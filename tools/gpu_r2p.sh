# re-verify the rebuilt library (container re-created): GPU tests, smoke, bench, reference arm
set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2p_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r2p_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2p_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/r2p_smoke.log
timeout 600 python bench.py > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err; echo "bench rc $?"; cat gpurun_out/r2p_bench.json
