# TMA-input epilogue (T) vs committed epilogue (E): quick check, A/B, traces, GPU tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
cp paper_2411_17164_b200/libxmgn.so paper_2411_17164_b200/libxmgn_T.so
XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_T.so timeout 180 python scratch/ab.py T 60000 512 2 || { echo "QUICK CHECK FAILED"; exit 1; }
rm -f /tmp/ab_ref_*.pt
for v in E T; do XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so timeout 300 python scratch/ab.py $v 400000 512 3 2>&1 | tail -1; done
XMGN_TRACE=chain_edge_bwd XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_T.so timeout 200 python scratch/ab.py T 400000 512 3 > /dev/null 2>&1; mv gpurun_out/trace.txt gpurun_out/trace_T.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_gpu.log
