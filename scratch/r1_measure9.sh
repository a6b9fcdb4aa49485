# full measurement of the current state: GPU tests, bench (with CPU baseline), launch list, ncu full of edge fwd/bwd
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
cat gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu list rc $?"
# BWD=1 launches go (node, edge) per layer: index 21 = part 0 layer 5 edge bwd; BWD=0: index 21 = part 0 layer 11 edge fwd
for spec in "1:edge_bwd" "0:edge_fwd"; do
  b=${spec%%:*}; tag=${spec##*:}
  R="regex:k_chain<\(int\)512, \(bool\)0, \(bool\)$b, \(bool\)1>"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$R" -s 21 -c 1 \
    -o gpurun_out/r01g_$tag python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_$tag.log 2>&1
  echo "ncu $tag rc $?"
done
