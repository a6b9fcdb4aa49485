mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2411_17164_b200/libxmgn.so paper_2411_17164_b200/libxmgn_X.so
for d in 0 1 2 3 31; do
  AB_DBG=$d XMGN_DBG=$d XMGN_TRACE=chain_edge_bwd XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_X.so timeout 200 python scratch/ab.py X 400000 512 3 > /dev/null 2>&1
  mv gpurun_out/trace.txt gpurun_out/trace_x$d.txt
  AB_DBG=$d XMGN_DBG=$d XMGN_TRACE=chain_edge_fwd XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_X.so timeout 200 python scratch/ab.py X 400000 512 3 > /dev/null 2>&1
  mv gpurun_out/trace.txt gpurun_out/tracef_x$d.txt
done
