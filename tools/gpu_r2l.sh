# A/B: KEEP_FIRST=6 / TAU_ADDS=7 vs the product build (C5a, 9472 frames), interleaved
bash tools/ab_decode.sh C5a 9472 build_ab/base.so build_ab/kf6.so build_ab/ta7.so build_ab/kf4.so > gpurun_out/r2l_ab.txt 2>&1
cat gpurun_out/r2l_ab.txt
