# last check of the round's final library: GPU tests, smoke, bench
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2u_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/r2u_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2u_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/r2u_smoke.log
timeout 600 python bench.py > gpurun_out/r2u_bench.json 2> gpurun_out/r2u_bench.err; echo "bench rc $?"
python -c "
import json
d=json.loads(open('gpurun_out/r2u_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
