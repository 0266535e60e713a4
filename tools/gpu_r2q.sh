# A/B: tau's right shifts as IMAD.WIDE high words (QKD_TAU_WIDE=1: g only, 3: g and c) vs the product build, C5a
bash tools/ab_decode.sh C5a 9472 build_ab/base.so build_ab/w1.so build_ab/w3.so > gpurun_out/r2q_ab.txt 2>&1
cat gpurun_out/r2q_ab.txt
for v in w1 w3; do QKD_LIB=$PWD/build_ab/$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "C3 or C5a or workloads or full_size" > gpurun_out/r2q_parity_$v.log 2>&1; echo "parity $v rc $?"; tail -2 gpurun_out/r2q_parity_$v.log; done
