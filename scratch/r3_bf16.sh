#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -x -k "cfg2_full_forward_l15 or multiscale or wide_hidden or pipelined or mse_scaled or zero_variance or partitioned_forward" > gpurun_out/r3b_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3b_pytest.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r3b_gpu_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/r3b_gpu_tests.txt
