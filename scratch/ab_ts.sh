mkdir -p gpurun_out
XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_TS.so timeout 180 python scratch/ab.py TS 60000 512 2 || { echo "QUICK CHECK FAILED"; exit 1; }
rm -f /tmp/ab_ref_*.pt
for v in G4 TS; do XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so timeout 300 python scratch/ab.py $v 400000 512 3 2>&1 | tail -1; done
XMGN_TRACE=chain_edge_fwd XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_TS.so timeout 200 python scratch/ab.py TS 400000 512 3 > /dev/null 2>&1; mv gpurun_out/trace.txt gpurun_out/tracef_TS.txt
XMGN_TRACE=chain_edge_bwd XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_TS.so timeout 200 python scratch/ab.py TS 400000 512 3 > /dev/null 2>&1; mv gpurun_out/trace.txt gpurun_out/trace_TS.txt
cp paper_2411_17164_b200/libxmgn_TS.so paper_2411_17164_b200/libxmgn.so
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_gpu.log
