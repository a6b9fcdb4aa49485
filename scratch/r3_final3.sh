#!/bin/bash
# round-3 final measurement batch (after the LN-statistics reuse and the dynamic edge-forward tiles)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r3f3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > ${O}_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x > ${O}_gpu_tests.txt 2>&1; echo "rc=$?" >> ${O}_gpu_tests.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.txt 2>&1; echo "rc=$?" >> ${O}_smoke.txt
timeout 1200 python bench.py > ${O}_bench_cfg4.json 2> ${O}_bench_cfg4.err
timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --no-bf16-leg > ${O}_bench_cfg2.json 2> ${O}_bench_cfg2.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 4000 --csv --log-file ${O}_launches_cfg4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-model --no-bf16-leg > ${O}_ncu_list.log 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 1200 $NCU -k "regex:k_chain<\(int\)512, \(bool\)0, \(bool\)1, \(bool\)1, \(bool\)0, \(bool\)1" -s 0 -c 1 -o ${O}_edge_bwd python scratch/prof_cfg4.py > ${O}_ncu_ebwd.log 2>&1
timeout 1200 $NCU -k "regex:k_chain<\(int\)512, \(bool\)0, \(bool\)0, \(bool\)1, \(bool\)0, \(bool\)1" -s 1 -c 1 -o ${O}_edge_fwd python scratch/prof_cfg4.py > ${O}_ncu_efwd.log 2>&1
