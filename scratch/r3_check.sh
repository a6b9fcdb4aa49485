#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r3a_smi.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r3a_gpu_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/r3a_gpu_tests.txt
timeout 900 python bench.py > gpurun_out/r3a_bench.json 2> gpurun_out/r3a_bench.err
