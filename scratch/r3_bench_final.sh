#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > gpurun_out/r3u_smi.txt
timeout 1200 python bench.py > gpurun_out/r3u_bench_cfg4.json 2> gpurun_out/r3u_bench_cfg4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r3u_bench_reference.json 2> gpurun_out/r3u_bench_reference.err
