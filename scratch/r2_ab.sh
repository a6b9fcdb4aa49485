#!/bin/bash
# same-box A/B of chain-kernel variants on the CFG4 bench (alternating order)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_2411_17164_b200
run() {  # tag, env...
  local tag=$1; shift
  env "$@" timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
}
run def1
run nodef1 XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_nodefer.so
run serial1 XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_nodefer.so XMGN_PIPE=0
run def2
run nodef2 XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_nodefer.so
