#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 1200 $NCU -k "regex:k_chain<\(int\)512, \(bool\)0, \(bool\)1" -s 16 -c 1 -o gpurun_out/r3i_edge_bwd python scratch/prof_cfg4.py > gpurun_out/r3i_ncu.log 2>&1
timeout 1200 $NCU -k "regex:k_chain<\(int\)512, \(bool\)0, \(bool\)0" -s 3 -c 1 -o gpurun_out/r3i_edge_fwd python scratch/prof_cfg4.py > gpurun_out/r3i_ncu_fwd.log 2>&1
