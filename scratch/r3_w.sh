#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in new w1 new w1; do
  if [ $v = new ]; then unset XMGN_LIB_OVERRIDE; else export XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so; fi
  echo "== $v" >> gpurun_out/r3f_ab.txt
  timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-e2e --no-cpu --no-model 2>>gpurun_out/r3f_ab.err >> gpurun_out/r3f_ab.txt
done
unset XMGN_LIB_OVERRIDE
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3f_gpu_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/r3f_gpu_tests.txt
