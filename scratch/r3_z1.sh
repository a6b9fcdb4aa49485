#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 0 1 0 1; do
  echo "== cfg2 XMGN_Z1=$v" >> gpurun_out/r3x_ab_z1.txt
  XMGN_Z1=$v timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --no-e2e --no-cpu --no-model --no-bf16-leg 2>>gpurun_out/r3x_ab.err >> gpurun_out/r3x_ab_z1.txt
done
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -s -x -k "cfg4_probe_forward or z1" > gpurun_out/r3x_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3x_tests.txt
