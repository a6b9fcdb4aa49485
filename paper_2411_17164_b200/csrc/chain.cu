// Instantiations and launcher of the GEMM-chain kernel (chain.cuh).
#include <cuda_runtime.h>
#include <atomic>
#include "kernels_launch.h"

#ifndef XMGN_OPS_SPECIALISE
#define XMGN_OPS_SPECIALISE 1
#endif

namespace xmgn {

template <int H, bool SPLIT, bool BWD, bool F16, bool Z1 = false, bool PIPE = false, int OPS = OPS_ALL>
static void chain_launch(const ChainParams& p, int grid, cudaStream_t st) {
  using C = ChainCfg<H, SPLIT>;
  auto kern = k_chain<H, SPLIT, BWD, F16, Z1, PIPE, OPS>;
  // the smem attribute is per device context: one flag per device (set idempotently,
  // so two host threads racing on the same device are harmless)
  static std::atomic<bool> attr[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr[dev].load(std::memory_order_acquire)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
    if (dev >= 0 && dev < 64) attr[dev].store(true, std::memory_order_release);
  }
  kern<<<grid, EpiShape<H, SPLIT>::THREADS, C::SMEM_BYTES, st>>>(p);
}

bool chain_dyn(int H, bool split) { return XMGN_DYN128 && H == 128 && !split; }

int chain_ctas_per_sm(int H, bool split) {
  if (H == 128) return split ? EpiShape<128, true>::MINB : EpiShape<128, false>::MINB;
  return H == 256 ? EpiShape<256, false>::MINB : EpiShape<512, false>::MINB;
}

size_t chain_smem(int H, bool split) {
  if (H == 128) return split ? ChainCfg<128, true>::SMEM_BYTES : ChainCfg<128, false>::SMEM_BYTES;
  if (H == 256) return ChainCfg<256, false>::SMEM_BYTES;
  return ChainCfg<512, false>::SMEM_BYTES;
}

template <int H, bool F16>
static void launch_h(bool bwd, bool pipe, const ChainParams& p, int grid, cudaStream_t st) {
  bool z1 = false;
  for (int i = 0; i < p.n_steps; ++i) z1 = z1 || (p.steps[i].flags & EF_FROM_IN) != 0;
  if constexpr (H == 512) {
    if (pipe && !z1) {
      // the edge programs get kernels holding only their ops (XMGN_OPS_SPECIALISE=0: off)
      int ops = 0;
      for (int i = 0; i < p.n_steps; ++i) ops |= step_opbit(p.steps[i]);
#if XMGN_OPS_SPECIALISE
      if (bwd && (ops & ~OPS_EDGE_BWD) == 0) { chain_launch<H, false, true, F16, false, true, OPS_EDGE_BWD>(p, grid, st); return; }
      if (!bwd && (ops & ~OPS_EDGE_FWD) == 0) { chain_launch<H, false, false, F16, false, true, OPS_EDGE_FWD>(p, grid, st); return; }
#endif
      if (bwd) chain_launch<H, false, true, F16, false, true>(p, grid, st);
      else chain_launch<H, false, false, F16, false, true>(p, grid, st);
      return;
    }
  }
  if (bwd && z1) chain_launch<H, false, true, F16, true>(p, grid, st);
  else if (bwd) chain_launch<H, false, true, F16>(p, grid, st);
  else chain_launch<H, false, false, F16>(p, grid, st);
}

bool chain_can_pipe(int H, bool split, const ChainParams& p) {
  if (H != 512 || split) return false;
  for (int i = 0; i < p.n_steps; ++i)
    if (p.steps[i].K != H || (p.steps[i].flags & EF_FROM_IN)) return false;
  return true;
}

void launch_chain(int H, bool split, bool f16, bool bwd, const ChainParams& p, int grid, cudaStream_t st,
                  bool pipe) {
  count_launch();
  pipe = pipe && chain_can_pipe(H, split, p);
  if (split) {  // FP32 check mode: BF16 hi/lo operands, H = 128
    if (bwd) chain_launch<128, true, true, false>(p, grid, st);
    else chain_launch<128, true, false, false>(p, grid, st);
    return;
  }
  if (H == 128) { if (f16) launch_h<128, true>(bwd, false, p, grid, st); else launch_h<128, false>(bwd, false, p, grid, st); }
  else if (H == 256) { if (f16) launch_h<256, true>(bwd, false, p, grid, st); else launch_h<256, false>(bwd, false, p, grid, st); }
  else { if (f16) launch_h<512, true>(bwd, pipe, p, grid, st); else launch_h<512, false>(bwd, pipe, p, grid, st); }
}

}  // namespace xmgn
