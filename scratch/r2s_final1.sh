#!/bin/bash
# round-2 profile set on the final kernels: GPU suite, smoke, bench, launch list, ncu captures
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/f1_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/f1_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f1_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/f1_smoke.log
timeout 900 python bench.py > gpurun_out/f1_bench.json 2> gpurun_out/f1_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 4000 --csv --log-file gpurun_out/f1_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-model > /tmp/f1l.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
cap() {
  timeout 600 $NCU -k regex:$2 -s $3 -c 1 -o /tmp/f1_$1 python scratch/prof_cfg4.py > /tmp/f1_ncu_$1.log 2>&1
  python scratch/ncu_summarize.py /tmp/f1_$1.ncu-rep $1 > gpurun_out/f1_ncu_$1.txt 2>&1
}
cap edge_bwd k_chain 32
ncu -i /tmp/f1_edge_bwd.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/f1_edge_bwd_source.csv.gz
cap edge_fwd k_chain 3
cap node_bwd k_chain 31
