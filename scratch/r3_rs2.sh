#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scratch/rowsum2_bitwise.py /tmp/rs_new.npz > gpurun_out/r3q_bitwise.txt 2>&1
XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_rs1.so timeout 300 python scratch/rowsum2_bitwise.py /tmp/rs_old.npz >> gpurun_out/r3q_bitwise.txt 2>&1
python -c "
import numpy as np
a, b = np.load('/tmp/rs_new.npz'), np.load('/tmp/rs_old.npz')
print({k: bool(np.array_equal(a[k], b[k])) for k in a.files})" >> gpurun_out/r3q_bitwise.txt 2>&1
for v in new rs1 new rs1; do
  if [ $v = new ]; then unset XMGN_LIB_OVERRIDE; else export XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so; fi
  echo "== $v" >> gpurun_out/r3q_ab.txt
  timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-model --no-bf16-leg 2>>gpurun_out/r3q_ab.err >> gpurun_out/r3q_ab.txt
done
