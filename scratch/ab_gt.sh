mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
XMGN_TRACE=chain_edge_bwd timeout 200 python scratch/ab.py GT 400000 512 3 > /dev/null 2>&1; mv gpurun_out/trace.txt gpurun_out/trace_GT.txt
