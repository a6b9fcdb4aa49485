#!/bin/bash
# LN-backward row-mask removal A/B, smoke (incl. model + GPU graph build), GPU suite, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_2411_17164_b200
run() { tag=$1; shift; env "$@" timeout 600 python scratch/ab.py $tag 400000 512 3 >> gpurun_out/ab3.jsonl 2>> gpurun_out/ab3.err; }
run new
run prev2 XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_prev2.so
run new
run prev2 XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_prev2.so
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/s4_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s4_pytest.log
timeout 1200 python bench.py > gpurun_out/s4_bench.json 2> gpurun_out/s4_bench.err
