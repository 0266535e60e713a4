# cost of the per-iteration stopping check on C5a (every frame runs all 50 sweeps either way)
for rep in 1 2 3; do for es in 1 0; do python tools/prof_decode.py --workload C5a --frames 9472 --reps 5 --early-stop $es; done; done > gpurun_out/r2o_stopcheck.txt 2>&1
cat gpurun_out/r2o_stopcheck.txt | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['workload'], d['early_stop'], '%.3f'%d['ms_min'], d['mean_iters'])"
