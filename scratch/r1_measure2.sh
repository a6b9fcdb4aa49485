# round-1 pass 2: GPU tests, A/B vs the previous epilogue, bench line, ncu captures of edge fwd/bwd
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
cp paper_2411_17164_b200/libxmgn.so paper_2411_17164_b200/libxmgn_E.so
# quick hang check on a small graph before anything long
XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_E.so timeout 180 python scratch/ab.py E 60000 512 2 || { echo "QUICK CHECK FAILED"; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/pytest_gpu.log
bash scratch/ab_run.sh "A E" 400000 512 3
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
cat gpurun_out/bench.json
if [ "$1" = "ncu" ]; then
for spec in "1:edge_bwd" "0:edge_fwd"; do
  b=${spec%%:*}; tag=${spec##*:}
  R="regex:k_chain<\(int\)512, \(bool\)0, \(bool\)$b, \(bool\)1>"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$R" -s 21 -c 1 \
    -o gpurun_out/full2_$tag python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu2_$tag.log 2>&1
  echo "ncu $tag rc $?"
done
fi
