# A/B on C5a: tau l-flags from s = 2g (QKD_TAU_S), edge_in's three-term sum on the FMA pipe (QKD_EIN_FMA), both
bash tools/ab_decode.sh C5a 9472 build_ab/base.so build_ab/s1.so build_ab/e1.so build_ab/se.so > gpurun_out/r2t_ab.txt 2>&1
cat gpurun_out/r2t_ab.txt
