#!/bin/bash
# PIPE: TMA-store drain deferred to the next step's epilogue (unless the next step loads A into ACT)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_2411_17164_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_model_gpu.py -q -x > gpurun_out/ab11_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab11_pytest.log
run() { tag=$1; shift; env "$@" timeout 600 python scratch/ab.py $tag 400000 512 3 >> gpurun_out/ab11.jsonl 2>> gpurun_out/ab11.err; }
for r in 1 2 3; do
run new
run prev3 XMGN_LIB_OVERRIDE=$PWD/$L/libxmgn_prev3.so
done
