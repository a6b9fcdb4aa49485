#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r3M
timeout 1500 python -m pytest tests -m gpu -q -x > ${O}_gpu_tests.txt 2>&1; echo "rc=$?" >> ${O}_gpu_tests.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.txt 2>&1; echo "rc=$?" >> ${O}_smoke.txt
timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --no-bf16-leg > ${O}_bench_cfg2.json 2> ${O}_bench_cfg2.err
timeout 1200 python bench.py > ${O}_bench_cfg4.json 2> ${O}_bench_cfg4.err
