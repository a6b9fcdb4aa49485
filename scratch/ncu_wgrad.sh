mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python scratch/ab.py warm 400000 512 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wgrad -s 4 -c 1 -o gpurun_out/wgrad python scratch/ab.py prof 400000 512 3 > gpurun_out/ncu_wgrad.log 2>&1; echo rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_segsum -s 1 -c 1 -o gpurun_out/segsum python scratch/ab.py prof 400000 512 3 > gpurun_out/ncu_segsum.log 2>&1; echo rc $?
