#!/bin/bash
# round 2 re-entry: full GPU suite, smoke, default bench, launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/s1_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/s1_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s1_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/s1_smoke.log
timeout 900 python bench.py > gpurun_out/s1_bench.json 2> gpurun_out/s1_bench.err
echo "bench rc=$?" >> gpurun_out/s1_bench.err
