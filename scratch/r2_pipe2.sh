#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -s -x -k "pipelined or wide_hidden" > gpurun_out/r2q_pytest.log 2>&1
rc=$?; echo "pytest rc=$rc" >> gpurun_out/r2q_pytest.log
if [ $rc -ne 0 ]; then exit 0; fi
timeout 600 python -m pytest tests/test_optim.py tests/test_inference.py -q -s -m gpu > gpurun_out/r2q_pytest2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2q_pytest2.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2q_bench_pipe.json 2> gpurun_out/r2q_bench_pipe.err
