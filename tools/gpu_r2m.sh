# A/B: the thread's two rows of a block row as straight-line code (QKD_ROW2) vs the product build (C5a, C3)
bash tools/ab_decode.sh C5a 9472 build_ab/base.so build_ab/row2.so > gpurun_out/r2m_ab.txt 2>&1
cat gpurun_out/r2m_ab.txt
