# ncu --set full of the first edge-bwd and edge-fwd chain launches of scratch/ab.py (400k-point graph, H=512, L=3)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python scratch/ab.py warm 400000 512 3 > /dev/null 2>&1
for spec in "1:edge_bwd" "0:edge_fwd"; do
  b=${spec%%:*}; tag=${spec##*:}
  R="regex:k_chain<\(int\)512, \(bool\)0, \(bool\)$b, \(bool\)1>"
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$R" -s 1 -c 1 \
    -o gpurun_out/$1_$tag python scratch/ab.py prof 400000 512 3 > gpurun_out/$1_$tag.log 2>&1
  echo "ncu $tag rc $?"
done
