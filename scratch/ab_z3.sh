mkdir -p gpurun_out
XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_Z3.so timeout 120 python scratch/ab.py Z3 60000 512 2 > /dev/null 2>&1 || { echo "QUICK CHECK FAILED"; exit 1; }
rm -f /tmp/ab_ref_*.pt
for i in 1 2; do
XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_H0.so timeout 300 python scratch/ab.py H0 400000 512 3 2>&1 | tail -1 | cut -c1-170
XMGN_NO_Z1=1 XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_Z3.so timeout 300 python scratch/ab.py noz1 400000 512 3 2>&1 | tail -1 | cut -c1-170
XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_Z3.so timeout 300 python scratch/ab.py Z3 400000 512 3 2>&1 | tail -1 | cut -c1-170
done
cp paper_2411_17164_b200/libxmgn_Z3.so paper_2411_17164_b200/libxmgn.so
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_gpu.log
