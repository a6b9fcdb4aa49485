#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "not cfg4 and not wide_hidden and not pipelined" > gpurun_out/r3d_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3d_pytest.log
for v in new c1 new c1; do
  if [ $v = new ]; then unset XMGN_LIB_OVERRIDE; else export XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so; fi
  echo "== $v" >> gpurun_out/r3d_ab.txt
  timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-e2e --no-cpu --no-model 2>/dev/null >> gpurun_out/r3d_ab.txt
done
unset XMGN_LIB_OVERRIDE
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k "regex:k_chain<\(int\)128, \(bool\)0, \(bool\)1" -s 3 -c 2 -o gpurun_out/r3d_cfg2_bwd python scratch/prof_cfg4.py cfg2 > gpurun_out/r3d_ncu_bwd.log 2>&1
