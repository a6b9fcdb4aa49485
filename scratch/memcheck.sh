python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python scratch/ab.py mc 3000 512 2 > gpurun_out/memcheck.log 2>&1; echo "memcheck rc $?"
grep -E "ERROR SUMMARY|Invalid" gpurun_out/memcheck.log | head -5
XMGN_Z1=1 timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python scratch/ab.py mc 3000 512 2 > gpurun_out/memcheck_z1.log 2>&1; echo "memcheck z1 rc $?"
grep -E "ERROR SUMMARY|Invalid" gpurun_out/memcheck_z1.log | head -5
