mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 120 python scratch/ab.py F 20000 512 2 > gpurun_out/dbg1.log 2>&1; echo rc $?
grep -v "^  " gpurun_out/dbg1.log | tail -5
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python scratch/ab.py F 5000 512 2 > gpurun_out/dbg2.log 2>&1; echo rc $?
grep -A12 "Invalid\|ERROR" gpurun_out/dbg2.log | head -40
