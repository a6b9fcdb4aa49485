#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r3y
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -x -k "BF16 or prec2 or prec0 or zero_variance or cfg2_full" > ${O}_bf16_tests.txt 2>&1; echo "rc=$?" >> ${O}_bf16_tests.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 4000 --csv --log-file ${O}_launches_cfg4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-model --no-bf16-leg > ${O}_ncu_list.log 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 1200 $NCU -k "regex:k_chain<\(int\)512, \(bool\)0, \(bool\)1, \(bool\)1, \(bool\)0, \(bool\)1" -s 0 -c 1 -o ${O}_edge_bwd python scratch/prof_cfg4.py > ${O}_ncu_ebwd.log 2>&1
