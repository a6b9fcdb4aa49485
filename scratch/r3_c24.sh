#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in new c24 new c24; do
  if [ $v = new ]; then unset XMGN_LIB_OVERRIDE; else export XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so; fi
  echo "== $v" >> gpurun_out/r3p_ab.txt
  timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-e2e --no-cpu --no-model --no-bf16-leg 2>>gpurun_out/r3p_ab.err >> gpurun_out/r3p_ab.txt
done
export XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_c24.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "multiscale or isolated or partitioned_forward or degenerate or partial or zero_var or deterministic" > gpurun_out/r3p_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3p_pytest.txt
