mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2411_17164_b200/libxmgn.so paper_2411_17164_b200/libxmgn_X.so
AB_DBG=0,1,2,3,4,8,16,7,15,31 XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_X.so timeout 600 python scratch/ab.py X 400000 512 3 2>&1 | grep tag
