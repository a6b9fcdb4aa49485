#!/bin/bash
# A/B: OPS-specialised edge kernels and deferred dgamma sums; plus the library-kernel launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_2411_17164_b200
run() { tag=$1; shift; env "$@" timeout 600 python scratch/ab.py $tag 400000 512 3 >> gpurun_out/ab1.jsonl 2>> gpurun_out/ab1.err; }
run def
run nospec XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_nospec.so
run nodefer XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_nodefer.so
run def
run nospec XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_nospec.so
run nodefer XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_nodefer.so
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 4000 --csv --log-file gpurun_out/p4_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-model > /tmp/p4.log 2>&1
