for v in L2 L3; do
  XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so timeout 600 ncu --kernel-name-base demangled -k "regex:k_chain<\(int\)512, \(bool\)0, \(bool\)1, \(bool\)1>" --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -s 1 -c 1 python scratch/ab.py prof 400000 512 3 2>&1 | grep -E "dram__bytes|gpu__time" | head -6
done
rm -f /tmp/ab_ref_*.pt; for v in L2 L3 L2 L3; do XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so timeout 300 python scratch/ab.py $v 400000 512 3 2>&1 | tail -1; done
