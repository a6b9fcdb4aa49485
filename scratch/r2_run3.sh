#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -s -x -k "pipelined or wide_hidden or multiscale or single_partial" > gpurun_out/r2r_pytest.log 2>&1
rc=$?; echo "pytest rc=$rc" >> gpurun_out/r2r_pytest.log
if [ $rc -ne 0 ]; then exit 0; fi
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $NCU -k regex:k_segsum -s 7 -c 1 -o gpurun_out/r2r_segsum python scratch/prof_cfg4.py > gpurun_out/r2r_ncu_seg.log 2>&1
timeout 600 $NCU -k regex:nvjet -s 2 -c 1 -o gpurun_out/r2r_calib_matmul python scratch/calib_matmul.py > gpurun_out/r2r_ncu_calib.log 2>&1
timeout 900 $NCU -k "regex:k_chain<512, 0, 1, 1, 0, 1>" -s 20 -c 1 -o gpurun_out/r2r_edge_bwd python scratch/prof_cfg4.py > gpurun_out/r2r_ncu_ebwd.log 2>&1
