#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu --no-model --no-bf16-leg > gpurun_out/r3v_bench_cfg2.json 2>gpurun_out/r3v_cfg2.err
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-model --no-bf16-leg > gpurun_out/r3v_bench_cfg4.json 2>gpurun_out/r3v_cfg4.err
