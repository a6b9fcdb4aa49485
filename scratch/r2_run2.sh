#!/bin/bash
# round 2, pass 2: whole GPU suite (no -x), ncu captures of the HBM-bound kernels at CFG4 and of a
# calibration matmul, racecheck / synccheck on small graphs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -s --durations=40 > gpurun_out/r2b_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b_pytest_gpu.log
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $NCU -k regex:k_aggregate -s 7 -c 1 -o gpurun_out/r2_aggregate python scratch/prof_cfg4.py > gpurun_out/r2_ncu_agg.log 2>&1
timeout 900 $NCU -k regex:k_segsum -s 7 -c 1 -o gpurun_out/r2_segsum python scratch/prof_cfg4.py > gpurun_out/r2_ncu_seg.log 2>&1
timeout 600 $NCU -k regex:nvjet -s 2 -c 1 -o gpurun_out/r2_calib_matmul python scratch/calib_matmul.py > gpurun_out/r2_ncu_calib.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/r2_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/r2_synccheck.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/r2_memcheck.log
