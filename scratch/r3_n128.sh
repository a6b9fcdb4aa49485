#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $NCU -k "regex:k_chain<\(int\)128, \(bool\)0, \(bool\)1" -s 3 -c 2 -o gpurun_out/r3h_cfg2_bwd python scratch/prof_cfg4.py cfg2 > gpurun_out/r3h_ncu_bwd.log 2>&1
timeout 900 $NCU -k "regex:k_chain<\(int\)128, \(bool\)0, \(bool\)0" -s 4 -c 1 -o gpurun_out/r3h_cfg2_fwd python scratch/prof_cfg4.py cfg2 > gpurun_out/r3h_ncu_fwd.log 2>&1
