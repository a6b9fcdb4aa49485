#!/bin/bash
# bisect the round-2 tile-schedule changes: dynamic queue vs runtime-static vs compiled-out static vs before
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_2411_17164_b200
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "multiscale or pipelined or deterministic" > gpurun_out/ab6_quick.log 2>&1
echo "quick rc=$?" >> gpurun_out/ab6_quick.log
run() { tag=$1; shift; env "$@" timeout 600 python scratch/ab.py $tag 400000 512 3 >> gpurun_out/ab6.jsonl 2>> gpurun_out/ab6.err; }
for r in 1 2; do
run dyn
run dyn0 XMGN_DYN=0
run stat XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_stat.so
run prev2 XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_prev2.so
done
