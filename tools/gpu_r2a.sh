set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2a_pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/r2a_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc $?"
cat gpurun_out/r2a_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2a_bench_ref.json 2>&1; echo "ref rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2a_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2a_ncu_launch.log 2>&1; echo "ncu1 rc $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -c 1 -o gpurun_out/prof_r2a_c5a python tools/prof_decode.py --workload C5a --frames 9472 --reps 1 > gpurun_out/r2a_ncu_full.log 2>&1; echo "ncu2 rc $?"
