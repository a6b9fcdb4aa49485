#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scratch/dyn_fwd_bitwise.py > gpurun_out/r3s_bitwise.txt 2>&1
for v in 1 0 1 0; do
  echo "== XMGN_DYN_FWD=$v" >> gpurun_out/r3s_ab.txt
  XMGN_DYN_FWD=$v timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-model --no-bf16-leg 2>>gpurun_out/r3s_ab.err >> gpurun_out/r3s_ab.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "multiscale or pipelined or deterministic or wide_hidden or partial" > gpurun_out/r3s_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3s_pytest.txt
