#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
date > gpurun_out/r3K_log.txt
XMGN_DB0_NODE=1 timeout 400 python -m pytest tests/test_gpu_parity.py -q -s -x -k "cfg2_full_forward_l15" >> gpurun_out/r3K_log.txt 2>&1; echo "db0=1 rc=$?" >> gpurun_out/r3K_log.txt; date >> gpurun_out/r3K_log.txt
XMGN_DB0_NODE=0 timeout 400 python -m pytest tests/test_gpu_parity.py -q -s -x -k "cfg2_full_forward_l15" >> gpurun_out/r3K_log.txt 2>&1; echo "db0=0 rc=$?" >> gpurun_out/r3K_log.txt; date >> gpurun_out/r3K_log.txt
