mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_cfg3.json 2>&1; echo "cfg3 rc $?"
timeout 900 python bench.py --precision bf16 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_cfg4_bf16.json 2>&1; echo "bf16 rc $?"
