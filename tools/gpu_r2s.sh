# N3: the DE-designed 16 x 100 profile at the paper's frame length (Z = 1024, n = 102400), product decoder and exact float BP,
# at T = 50 (the BASELINE iteration cap), 100 and 200
for T in 50 100 200; do
timeout 1500 python tools/de_codes.py --profile "16,100,1024;2:12,3:64,5:1,10:1,12:22" --qbers 0.017,0.018,0.019,0.0195,0.02,0.021 --frames 2048 --T $T --float --out gpurun_out/r2s_de_codes_100kb_T$T.json > gpurun_out/r2s_de_codes_T$T.log 2>&1; echo "T=$T rc $?"
python - <<PY
import json
for l in open('gpurun_out/r2s_de_codes_T$T.log'):
    if l.startswith('{'):
        d=json.loads(l); print($T, d['qber'], round(d['f'],3), d['fer'], round(d['mean_iters'],1), d['fer_float'], round(d['mean_iters_float'],1), round(d['decode_ms'],1))
PY
done
