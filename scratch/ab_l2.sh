mkdir -p gpurun_out
XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_L2.so timeout 180 python scratch/ab.py L2 60000 512 2 || { echo "QUICK CHECK FAILED"; exit 1; }
rm -f /tmp/ab_ref_*.pt
for v in B0 L2 B0 L2; do XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so timeout 300 python scratch/ab.py $v 400000 512 3 2>&1 | tail -1; done
for v in B0 L2; do
  XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_chain -s 2 -c 2 python scratch/ab.py prof 400000 512 3 2>&1 | grep -E "k_chain|dram__bytes|gpu__time" | head -12
done
XMGN_TRACE=chain_edge_bwd XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_L2.so timeout 200 python scratch/ab.py L2 400000 512 3 > /dev/null 2>&1; mv gpurun_out/trace.txt gpurun_out/trace_L2.txt
cp paper_2411_17164_b200/libxmgn_L2.so paper_2411_17164_b200/libxmgn.so
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_gpu.log
