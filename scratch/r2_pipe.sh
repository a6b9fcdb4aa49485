#!/bin/bash
# PIPE kernel: parity first (bounded by timeouts: a hang must not wedge the box), then an A/B bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -s -x -k "pipelined or wide_hidden" > gpurun_out/r2p_pytest.log 2>&1
rc=$?; echo "pytest rc=$rc" >> gpurun_out/r2p_pytest.log
if [ $rc -ne 0 ]; then exit 0; fi
timeout 600 python -m pytest tests/test_gpu_parity.py -q -s -x -k "z1 or cfg4_probe_grad or partial_tile or deterministic" > gpurun_out/r2p_pytest2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2p_pytest2.log
XMGN_PIPE=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2p_bench_serial.json 2> gpurun_out/r2p_bench_serial.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2p_bench_pipe.json 2> gpurun_out/r2p_bench_pipe.err
