#!/bin/bash
# NEXT-4 GPU tests + default bench (with the full-model training-step leg)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_build_gpu.py -q -rA -x > gpurun_out/s2_build_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s2_build_pytest.log
timeout 1200 python bench.py > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err
echo "bench rc=$?" >> gpurun_out/s2_bench.err
