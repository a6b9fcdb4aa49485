// Streaming kernels around the GEMM chains: weight packing, BF16 staging,
// the deterministic segmented sums (aggregation, its adjoint), split-K weight
// gradients on tcgen05 and fixed-order reductions.
#pragma once
#include <cuda_bf16.h>
#include <cuda.h>
#include "tc.cuh"

namespace xmgn {

// model inputs / outputs (NEXT-1): 24 node and 4 edge raw inputs, padded to
// one 64-column operand box; stats = [mean(28) | std(28)]; 4 outputs (p, tau)
constexpr int IO_F_NODE = 24, IO_F_EDGE = 4, IO_IN_COLS = 64, IO_NSTAT = 28, IO_DOUT = 4;

struct PackJob {            // out[r][c] = bf16(params[src + r*sr + c*sc]), r < rows, c < cols
  __nv_bfloat16* dst;
  long long lo_off;         // lo copy at dst + lo_off (0 = none)
  int ld, rows, cols;
  long long src, sr, sc;
};

struct WgradParams {
  CUtensorMap a0, a0lo, a1, a1lo, b, blo;  // MN-major operands (row-major BF16 activations)
  int a_split_tiles;    // M tiles [0, a_split_tiles) come from a0, the rest from a1
  int b_col0;           // first B column (feature) of this weight
  int rows;             // reduction length (rows of the activation tensors)
  int n_split;          // split-K factor (gridDim.z)
  int Hin, Hout;        // dW is [Hin][Hout]
  int ones_tile;        // 1: M tile Hin/128 uses A = ones -> its rows are the column sums of B (bias grads)
  float* part;          // [n_split][Hin (+128)][Hout]
};

}  // namespace xmgn
