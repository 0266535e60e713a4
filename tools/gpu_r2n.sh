# final round-2 build: launch list and one ncu --set full capture of the bench's C5a decode
set -x
timeout 600 python bench.py > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2n_bench_ref.json 2>&1; echo "ref rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2n_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2n_ncu_launch.log 2>&1; echo "ncu1 rc $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -c 1 -o gpurun_out/prof_r2n_bench python bench.py --steps 1 --warmup 3 > gpurun_out/r2n_ncu_full.log 2>&1; echo "ncu2 rc $?"
