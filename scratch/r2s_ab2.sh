#!/bin/bash
# A/B: new default (per-chunk dgamma sums, packed-once G_e', one in_full wait per box) vs the
# previous variants; then the GPU suite on the new default
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_2411_17164_b200
run() { tag=$1; shift; env "$@" timeout 600 python scratch/ab.py $tag 400000 512 3 >> gpurun_out/ab2.jsonl 2>> gpurun_out/ab2.err; }
run new
run nodefer XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_nodefer.so
run prev XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_prev.so
run new
run nodefer XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_nodefer.so
run prev XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_prev.so
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/ab2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab2_pytest.log
