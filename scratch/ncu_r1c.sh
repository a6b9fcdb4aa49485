mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 
python scratch/prof_chain.py 512 100000 > /dev/null
R='regex:k_chain<\(int\)512, \(bool\)0, \(bool\)0, \(bool\)1>'
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$R" -s 1 -c 1 \
   -o gpurun_out/prof2_edge_fwd_h512 python scratch/prof_chain.py 512 100000 > gpurun_out/ncu_a.log 2>&1
R='regex:k_chain<\(int\)512, \(bool\)0, \(bool\)1, \(bool\)1>'
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$R" -s 1 -c 1 \
   -o gpurun_out/prof2_edge_bwd_h512 python scratch/prof_chain.py 512 100000 > gpurun_out/ncu_b.log 2>&1
ls -la gpurun_out
