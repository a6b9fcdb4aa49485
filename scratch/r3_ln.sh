#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scratch/ln_stats_bitwise.py > gpurun_out/r3t_bitwise.txt 2>&1
for v in 1 0 1 0; do
  echo "== XMGN_LN_STATS=$v" >> gpurun_out/r3t_ab.txt
  XMGN_LN_STATS=$v timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-model --no-bf16-leg 2>>gpurun_out/r3t_ab.err >> gpurun_out/r3t_ab.txt
done
for v in 1 0; do
  echo "== cfg2 XMGN_LN_STATS=$v" >> gpurun_out/r3t_ab.txt
  XMGN_LN_STATS=$v timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --no-e2e --no-cpu --no-model --no-bf16-leg 2>>gpurun_out/r3t_ab.err >> gpurun_out/r3t_ab.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "multiscale or pipelined or deterministic or zero_var or degenerate or partial or mse" > gpurun_out/r3t_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3t_pytest.txt
