#!/bin/bash
# per-tile column-sum partials + dynamic tile scheduling: quick parity (with a hang guard), A/B
# dynamic vs static (same binary, XMGN_DYN=0) vs the previous library, GPU suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_2411_17164_b200
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "multiscale or pipelined or deterministic or single_partial" > gpurun_out/s5_quick.log 2>&1
rc=$?; echo "quick rc=$rc" >> gpurun_out/s5_quick.log
if [ $rc -ne 0 ]; then exit 0; fi
run() { tag=$1; shift; env "$@" timeout 600 python scratch/ab.py $tag 400000 512 3 >> gpurun_out/ab5.jsonl 2>> gpurun_out/ab5.err; }
run dyn
run static XMGN_DYN=0
run prev2 XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_prev2.so
run dyn
run static XMGN_DYN=0
run prev2 XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_prev2.so
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s5_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s5_pytest.log
timeout 900 python bench.py --no-cpu > gpurun_out/s5_bench.json 2> gpurun_out/s5_bench.err
