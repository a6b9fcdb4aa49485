#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_model_gpu.py -q -s -x -k "multiscale or mse or cfg1 or partitioned_forward or degenerate or isolated or one_hidden or cfg4_probe_gradients or model" > gpurun_out/r3o_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3o_pytest.txt
for v in 1 0 1 0; do
  echo "== XMGN_DB0_NODE=$v" >> gpurun_out/r3o_ab.txt
  XMGN_DB0_NODE=$v timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-model --no-bf16-leg 2>>gpurun_out/r3o_ab.err >> gpurun_out/r3o_ab.txt
done
for v in 1 0; do
  echo "== cfg2 XMGN_DB0_NODE=$v" >> gpurun_out/r3o_ab.txt
  XMGN_DB0_NODE=$v timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --no-e2e --no-cpu --no-model --no-bf16-leg 2>>gpurun_out/r3o_ab.err >> gpurun_out/r3o_ab.txt
done
