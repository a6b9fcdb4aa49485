#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on a small end-to-end target
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 10 python scratch/san_target.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_$tool.log
done
