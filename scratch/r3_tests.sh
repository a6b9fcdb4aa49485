#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3w_gpu_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3w_gpu_tests.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3w_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r3w_smoke.txt
timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --no-e2e --no-cpu --no-model --no-bf16-leg > gpurun_out/r3w_bench_cfg2.json 2>/dev/null
timeout 900 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-model --no-bf16-leg > gpurun_out/r3w_bench_cfg4.json 2>/dev/null
