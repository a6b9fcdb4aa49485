mkdir -p gpurun_out
XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_W3.so timeout 120 python scratch/ab.py W3 60000 512 2 || { echo "QUICK CHECK FAILED"; exit 1; }
rm -f /tmp/ab_ref_*.pt
for v in B3 W3 B3 W3; do XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so timeout 300 python scratch/ab.py $v 400000 512 3 2>&1 | tail -1; done
XMGN_TRACE=chain_edge_bwd XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_W3.so timeout 200 python scratch/ab.py W3 400000 512 3 > /dev/null 2>&1; mv gpurun_out/trace.txt gpurun_out/trace_W3.txt
cp paper_2411_17164_b200/libxmgn_W3.so paper_2411_17164_b200/libxmgn.so
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_gpu.log
