# usage: bash scratch/ab_run.sh "A B C D" [n] [H] [L]
mkdir -p gpurun_out
rm -f /tmp/ab_ref_*.pt
for v in $1; do
  XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so timeout 240 python scratch/ab.py $v $2 $3 $4 2>&1 | tail -2
  XMGN_TRACE=chain_edge_bwd XMGN_LIB_OVERRIDE=$PWD/paper_2411_17164_b200/libxmgn_$v.so timeout 240 python scratch/ab.py $v $2 $3 $4 > /dev/null 2>&1
  mv gpurun_out/trace.txt gpurun_out/trace_$v.txt 2>/dev/null
done
