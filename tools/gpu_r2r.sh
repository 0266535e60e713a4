# final build of the round (Konst carries the two experiment constants): GPU tests, smoke, both bench arms,
# launch list and one ncu --set full capture of the bench's C5a decode
set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2r_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r2r_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2r_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/r2r_smoke.log
timeout 600 python bench.py > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2r_bench_reference.json 2> gpurun_out/r2r_bench_reference.err; echo "ref rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2r_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2r_ncu_launch.log 2>&1; echo "ncu1 rc $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -c 1 -o gpurun_out/prof_r2r_bench python bench.py --steps 1 --warmup 3 > gpurun_out/r2r_ncu_full.log 2>&1; echo "ncu2 rc $?"
