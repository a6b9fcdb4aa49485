# pass 3: quick hang check, GPU tests, A/B (E = previous epilogue, F = current), bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
cp paper_2411_17164_b200/libxmgn.so paper_2411_17164_b200/libxmgn_G.so
XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_G.so timeout 180 python scratch/ab.py G 60000 512 2 || { echo "QUICK CHECK FAILED"; exit 1; }
rm -f /tmp/ab_ref_*.pt
for v in E G; do XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so timeout 300 python scratch/ab.py $v 400000 512 3 2>&1 | tail -1; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/pytest_gpu.log
if [ "$1" = "bench" ]; then timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"; cat gpurun_out/bench.json; fi
