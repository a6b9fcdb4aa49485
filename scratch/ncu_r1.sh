set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
python -c "from xmgn_inputs import configs; configs.load('cfg4')"
# 1) launch list of one bench step (after one warm-up step), our kernels only
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:^k_" -s 3160 -c 3160 --csv \
   --log-file gpurun_out/launches_cfg4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_bench.log 2>&1
# 2) full capture of the dominant kernel (edge backward chain), one launch
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_chain<512, false, true, true>" -s 1 -c 1 \
   -o gpurun_out/prof_edge_bwd python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1
# 3) and one forward edge chain
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_chain<512, false, false, true>" -s 1 -c 1 \
   -o gpurun_out/prof_edge_fwd python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_full_fwd.log 2>&1
ls -la gpurun_out
