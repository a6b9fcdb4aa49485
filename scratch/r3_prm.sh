#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pipelined or multiscale or wide_hidden or deterministic or partial or degenerate" > gpurun_out/r3j_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3j_pytest.log
for v in 1 0 1 0; do
  echo "== XMGN_PRM_TABLE=$v" >> gpurun_out/r3j_ab.txt
  XMGN_PRM_TABLE=$v timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-model --no-bf16-leg 2>>gpurun_out/r3j_ab.err >> gpurun_out/r3j_ab.txt
done
for v in 1 0; do
  echo "== cfg2 XMGN_PRM_TABLE=$v" >> gpurun_out/r3j_ab.txt
  XMGN_PRM_TABLE=$v timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-e2e --no-cpu --no-model --no-bf16-leg 2>>gpurun_out/r3j_ab.err >> gpurun_out/r3j_ab.txt
done
