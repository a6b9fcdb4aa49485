# usage: bash scratch/ncu_one.sh <H> <bwd 0|1> <tag>
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python scratch/prof_chain.py $1 100000 > /dev/null
R="regex:k_chain<\(int\)$1, \(bool\)0, \(bool\)$2, \(bool\)1>"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$R" -s 1 -c 1 \
   -o gpurun_out/$3 python scratch/prof_chain.py $1 100000 > gpurun_out/$3.log 2>&1
