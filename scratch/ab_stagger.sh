mkdir -p gpurun_out
AB_DBG=0,10,20,30,45 XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_E.so timeout 400 python scratch/ab.py E 400000 512 3 2>&1 | tail -6
