mkdir -p gpurun_out
XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_NB.so timeout 180 python scratch/ab.py NB 60000 512 2 || { echo "QUICK CHECK FAILED"; exit 1; }
rm -f /tmp/ab_ref_*.pt
for v in B2 NB B2 NB; do XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so timeout 300 python scratch/ab.py $v 400000 512 3 2>&1 | tail -1; done
XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_NB.so timeout 900 python scratch/cfg2_err.py 2>&1 | grep cfg2
cp paper_2411_17164_b200/libxmgn_NB.so paper_2411_17164_b200/libxmgn.so
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_gpu.log
