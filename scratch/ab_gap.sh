mkdir -p gpurun_out
XMGN_TRACE=chain_edge_bwd XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_TR.so timeout 200 python scratch/ab.py TR 400000 512 3 > /dev/null 2>&1; mv gpurun_out/trace.txt gpurun_out/trace_TR.txt
XMGN_TRACE=chain_edge_fwd XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_TR.so timeout 200 python scratch/ab.py TR 400000 512 3 > /dev/null 2>&1; mv gpurun_out/trace.txt gpurun_out/tracef_TR.txt
