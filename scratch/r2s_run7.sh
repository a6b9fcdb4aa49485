#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s7_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/s7_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s7_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s7_pytest.log
timeout 900 python bench.py > gpurun_out/s7_bench.json 2> gpurun_out/s7_bench.err
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 10 python scratch/san_target.py > gpurun_out/s7_san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/s7_san_$tool.log
done
