# Build A/B variants of libxmgn.so that differ only in compile-time switches of chain.cu/kernels.cu.
# usage: bash scratch/build_variants.sh name "-DFOO=1 -DBAR=2" [name2 "flags2" ...]
set -e
cd "$(dirname "$0")/.."
B=paper_2411_17164_b200/build
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-fopenmp --expt-relaxed-constexpr -Iinclude"
while [ $# -gt 0 ]; do
  n=$1; f=$2; shift 2
  mkdir -p $B/var_$n
  $NV $f -c paper_2411_17164_b200/csrc/chain.cu -o $B/var_$n/chain.o &
  $NV $f -c paper_2411_17164_b200/csrc/kernels.cu -o $B/var_$n/kernels.o &
  wait
  objs=$(ls $B/*.o | grep -v "/chain.cu.o\|/kernels.cu.o")
  $NV -shared -o paper_2411_17164_b200/libxmgn_$n.so $objs $B/var_$n/chain.o $B/var_$n/kernels.o -lcudart -lgomp -ldl
  echo built $n
done
