// Instantiations and launcher of the GEMM-chain kernel (chain.cuh).
#include <cuda_runtime.h>
#include "kernels_launch.h"

namespace xmgn {

template <int H, bool SPLIT, bool BWD>
static void chain_launch(const ChainParams& p, int grid, cudaStream_t st) {
  using C = ChainCfg<H, SPLIT>;
  auto kern = k_chain<H, SPLIT, BWD>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
    attr = true;
  }
  kern<<<grid, 256, C::SMEM_BYTES, st>>>(p);
}

size_t chain_smem(int H, bool split) {
  if (H == 128) return split ? ChainCfg<128, true>::SMEM_BYTES : ChainCfg<128, false>::SMEM_BYTES;
  if (H == 256) return ChainCfg<256, false>::SMEM_BYTES;
  return ChainCfg<512, false>::SMEM_BYTES;
}

void launch_chain(int H, bool split, bool bwd, const ChainParams& p, int grid, cudaStream_t st) {
  if (H == 128) {
    if (split) { if (bwd) chain_launch<128, true, true>(p, grid, st); else chain_launch<128, true, false>(p, grid, st); }
    else { if (bwd) chain_launch<128, false, true>(p, grid, st); else chain_launch<128, false, false>(p, grid, st); }
  } else if (H == 256) {
    if (bwd) chain_launch<256, false, true>(p, grid, st); else chain_launch<256, false, false>(p, grid, st);
  } else {
    if (bwd) chain_launch<512, false, true>(p, grid, st); else chain_launch<512, false, false>(p, grid, st);
  }
}

}  // namespace xmgn
