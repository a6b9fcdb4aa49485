#!/bin/bash
# round 2: model GPU tests, then profiles (launch list of one CFG4 bench step + ncu --set full of
# the top kernels, summarised on the box; the .ncu-rep files stay there except gzip'd source CSVs)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_model_gpu.py -q -rA -x > gpurun_out/p3_model_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/p3_model_pytest.log
NCU="ncu --set full --clock-control none --import-source on"
S=python; SUM=scratch/ncu_summarize.py
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3700 --csv --log-file gpurun_out/p3_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /tmp/p3_launch_bench.log 2>&1
cap() {  # name kernel-regex skip
  timeout 600 $NCU -k regex:$2 -s $3 -c 1 -o /tmp/p3_$1 python scratch/prof_cfg4.py > /tmp/p3_ncu_$1.log 2>&1
  $S $SUM /tmp/p3_$1.ncu-rep $1 > gpurun_out/p3_ncu_$1.txt 2>&1
}
cap edge_bwd k_chain 32
ncu -i /tmp/p3_edge_bwd.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/p3_edge_bwd_source.csv.gz
ncu -i /tmp/p3_edge_bwd.ncu-rep --page source --csv --print-source cuda 2>/dev/null | gzip > gpurun_out/p3_edge_bwd_cuda.csv.gz
cap edge_fwd k_chain 3
cap node_bwd k_chain 31
cap node_fwd k_chain 4
cap segsum k_segsum 7
cap aggregate k_aggregate 7
cap wgrad k_wgrad 20
timeout 600 $NCU -k regex:nvjet -s 2 -c 1 -o /tmp/p3_calib python scratch/calib_matmul.py > /tmp/p3_ncu_calib.log 2>&1
$S $SUM /tmp/p3_calib.ncu-rep calib_matmul_bf16_8192 > gpurun_out/p3_ncu_calib.txt 2>&1
cuobjdump -sass paper_2411_17164_b200/libxmgn.so | grep -oE "UTCHMMA[.A-Z0-9]*|UTCQMMA[.A-Z0-9]*|UTMALDG[.A-Z0-9]*|UTMASTG[.A-Z0-9]*|LDTM[.A-Z0-9]*|UTMAPF[.A-Z0-9]*" | sort | uniq -c > gpurun_out/p3_sass_ops.txt
ls -la /tmp/p3_*.ncu-rep > gpurun_out/p3_reps.txt
du -sh gpurun_out >> gpurun_out/p3_reps.txt
