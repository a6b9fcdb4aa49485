mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python scratch/ab.py Z1 60000 512 2 || { echo "QUICK CHECK FAILED"; exit 1; }
rm -f /tmp/ab_ref_*.pt
XMGN_NO_Z1=1 timeout 300 python scratch/ab.py noz1 400000 512 3 2>&1 | tail -1 | cut -c1-400
timeout 300 python scratch/ab.py Z1 400000 512 3 2>&1 | tail -1 | cut -c1-400
XMGN_NO_Z1=1 timeout 300 python scratch/ab.py noz1 400000 512 3 2>&1 | tail -1 | cut -c1-400
timeout 300 python scratch/ab.py Z1 400000 512 3 2>&1 | tail -1 | cut -c1-400
XMGN_TRACE=chain_edge_bwd timeout 200 python scratch/ab.py Z1 400000 512 3 > /dev/null 2>&1; mv gpurun_out/trace.txt gpurun_out/trace_Z1.txt
timeout 900 python scratch/cfg2_err.py 2>&1 | grep cfg2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_gpu.log
