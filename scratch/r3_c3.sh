#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in new c3 c4 c2e1 new c3 c4 c2e1; do
  if [ $v = new ]; then unset XMGN_LIB_OVERRIDE; else export XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so; fi
  echo "== $v" >> gpurun_out/r3e_ab.txt
  timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-e2e --no-cpu --no-model 2>>gpurun_out/r3e_ab.err >> gpurun_out/r3e_ab.txt
done
for v in c3 c4; do
export XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "multiscale or isolated or partitioned_forward or degenerate or partial or zero_var" > gpurun_out/r3e_pytest_$v.log 2>&1
echo "rc=$?" >> gpurun_out/r3e_pytest_$v.log
done
