#!/bin/bash
# round 2, first GPU pass: full GPU suite (durations), smoke, launch list of smoke, a short bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r2_nvsmi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -s --durations=30 > gpurun_out/r2_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/r2_launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_ncu_smoke.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench_fp16.json 2> gpurun_out/r2_bench_fp16.err
timeout 600 python bench.py --steps 3 --warmup 3 --precision bf16 --no-e2e --no-cpu > gpurun_out/r2_bench_bf16.json 2> gpurun_out/r2_bench_bf16.err
