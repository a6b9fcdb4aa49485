#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1100 python -m pytest tests -m gpu -q -x > gpurun_out/r3N_gpu_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3N_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3N_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r3N_smoke.txt
