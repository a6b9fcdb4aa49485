mkdir -p gpurun_out
XMGN_TRACE=chain_edge_bwd XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_NH.so timeout 200 python scratch/ab.py NH 400000 512 3 > /dev/null 2>&1; mv gpurun_out/trace.txt gpurun_out/trace_NH.txt
XMGN_TRACE=chain_edge_fwd XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_NH.so timeout 200 python scratch/ab.py NH 400000 512 3 > /dev/null 2>&1; mv gpurun_out/trace.txt gpurun_out/tracef_NH.txt
rm -f /tmp/ab_ref_*.pt
for v in TR NH TR NH; do XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so timeout 300 python scratch/ab.py $v 400000 512 3 2>&1 | tail -1; done
