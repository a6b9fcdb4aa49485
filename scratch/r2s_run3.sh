#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scratch/r2s_san.sh
timeout 1500 python scratch/cfg5_point.py > gpurun_out/cfg5.json 2> gpurun_out/cfg5.err
echo "cfg5 rc=$?" >> gpurun_out/cfg5.err
