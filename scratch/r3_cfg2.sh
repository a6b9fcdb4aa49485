#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-e2e --no-cpu --no-model > gpurun_out/r3c_bench_cfg2.json 2> gpurun_out/r3c_bench_cfg2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3c_launches_cfg2.csv python scratch/prof_cfg4.py cfg2 > gpurun_out/r3c_ncu_list.log 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $NCU -k "regex:k_chain<128, 0, 1" -s 3 -c 3 -o gpurun_out/r3c_cfg2_bwd python scratch/prof_cfg4.py cfg2 > gpurun_out/r3c_ncu_bwd.log 2>&1
timeout 900 $NCU -k "regex:k_chain<128, 0, 0" -s 3 -c 2 -o gpurun_out/r3c_cfg2_fwd python scratch/prof_cfg4.py cfg2 > gpurun_out/r3c_ncu_fwd.log 2>&1
timeout 900 python bench.py --precision bf16 --steps 3 --warmup 3 --no-e2e --no-cpu --no-model > gpurun_out/r3c_bench_cfg4_bf16.json 2> gpurun_out/r3c_bench_cfg4_bf16.err
