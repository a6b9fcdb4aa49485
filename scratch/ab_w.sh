mkdir -p gpurun_out
for v in T W; do XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so timeout 300 python scratch/ab.py $v 400000 512 3 2>&1 | tail -1; done
