# round-1 measurement pass: GPU tests, bench line, ncu launch list, ncu full captures
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
cat gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu list rc $?"
for spec in "1:edge_bwd" "0:edge_fwd"; do
  b=${spec%%:*}; tag=${spec##*:}
  R="regex:k_chain<\(int\)512, \(bool\)0, \(bool\)$b, \(bool\)1>"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$R" -s 20 -c 1 \
    -o gpurun_out/full_$tag python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_$tag.log 2>&1
  echo "ncu $tag rc $?"
done
ls -la gpurun_out
