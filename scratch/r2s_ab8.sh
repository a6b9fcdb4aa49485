#!/bin/bash
# control-warp register budget (setmaxnreg 56 -> 32 gives the epilogue 112 registers) and the
# dynamic tile queue on top of it
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_2411_17164_b200
timeout 300 env XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_ctrl32.so python -m pytest tests/test_gpu_parity.py -q -x -k "multiscale or pipelined or deterministic or degenerate" > gpurun_out/ab8_quick.log 2>&1
echo "quick ctrl32 rc=$?" >> gpurun_out/ab8_quick.log
timeout 300 env XMGN_DYN=1 XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_c32dyn.so python -m pytest tests/test_gpu_parity.py -q -x -k "multiscale or pipelined or deterministic or degenerate" >> gpurun_out/ab8_quick.log 2>&1
echo "quick c32dyn rc=$?" >> gpurun_out/ab8_quick.log
run() { tag=$1; shift; env "$@" timeout 600 python scratch/ab.py $tag 400000 512 3 >> gpurun_out/ab8.jsonl 2>> gpurun_out/ab8.err; }
for r in 1 2; do
run def
run ctrl32 XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_ctrl32.so
run ctrl40 XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_ctrl40.so
run c32dyn XMGN_DYN=1 XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_c32dyn.so
done
