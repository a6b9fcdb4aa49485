// Engine self-test: a plain tcgen05 GEMM C = A * B^T exercising the exact
// descriptor / TMA / TMEM conventions of tc.cuh in both operand majors.  It is
// a diagnostic entry point (xmgn_selftest_gemm), not part of the processor.
#include <cuda_runtime.h>
#include <cstdio>
#include "tc.cuh"
#include "tmap.h"
#include "xmgn_internal.h"

namespace xmgn {

template <int N, bool AMN, bool BMN>
__global__ void __launch_bounds__(128, 1)
    k_selftest_gemm(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, float* C,
                    int M, int K) {
  constexpr int S = 4;
  constexpr uint32_t A_BYTES = 128 * 64 * 2, B_BYTES = N * 64 * 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S * B_BYTES);
  uint64_t* empty = full + S;
  uint64_t* done = empty + S;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

  const int w = warp_id();
  const int m0 = blockIdx.x * 128;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (w == 2) tmem_alloc(tslot, N < 32 ? 32 : N);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int nk = K / 64;

  if (w == 0) {
    if (elect_one()) {
      for (int kb = 0; kb < nk; ++kb) {
        int s = kb % S;
        if (kb >= S) mbar_wait(&empty[s], ((kb / S) - 1) & 1);
        mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
        if (AMN) {
          tma_load_2d(sA + s * A_BYTES, &tA, &full[s], m0, kb * 64);
          tma_load_2d(sA + s * A_BYTES + 8192, &tA, &full[s], m0 + 64, kb * 64);
        } else {
          tma_load_2d(sA + s * A_BYTES, &tA, &full[s], kb * 64, m0);
        }
        if (BMN) {
          for (int j = 0; j < N / 64; ++j) tma_load_2d(sB + s * B_BYTES + j * 8192, &tB, &full[s], j * 64, kb * 64);
        } else {
          tma_load_2d(sB + s * B_BYTES, &tB, &full[s], kb * 64, 0);
        }
      }
    }
  } else if (w == 1) {
    constexpr uint32_t idesc = idesc_bf16(N, AMN, BMN);
    for (int kb = 0; kb < nk; ++kb) {
      int s = kb % S;
      mbar_wait(&full[s], (kb / S) & 1);
      tc_fence_after();
      if (elect_one()) {
        uint32_t a0 = smem_u32(sA + s * A_BYTES), b0 = smem_u32(sB + s * B_BYTES);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint64_t ad = AMN ? sdesc_sw128(a0 + k * 2048, 8192, 1024) : sdesc_sw128(a0 + k * 32, 16, 1024);
          uint64_t bd = BMN ? sdesc_sw128(b0 + k * 2048, 8192, 1024) : sdesc_sw128(b0 + k * 32, 16, 1024);
          mma_bf16(tmem, ad, bd, idesc, (kb | k) != 0);
        }
        mma_commit(&empty[s]);
        if (kb == nk - 1) mma_commit(done);
      }
      __syncwarp();
    }
  }
  __syncwarp();
  mbar_wait(done, 0);
  tc_fence_after();
  const int row = m0 + w * 32 + lane_id();
  for (int c = 0; c < N; c += 32) {
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(w * 32) << 16) + c, v);
    if (row < M)
      for (int i = 0; i < 32; ++i) C[(size_t)row * N + c + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (w == 2) tmem_dealloc(tmem, N < 32 ? 32 : N);
}

template <int N, bool AMN, bool BMN>
static cudaError_t launch_selftest(int M, int K, const void* A, const void* B, float* C, cudaStream_t st) {
  CUtensorMap tA = AMN ? tmap_bf16(A, M, K, M, 64, 64) : tmap_bf16(A, K, M, K, 64, 128);
  CUtensorMap tB = BMN ? tmap_bf16(B, N, K, N, 64, 64) : tmap_bf16(B, K, N, K, 64, N);
  size_t smem = 1024 + 4 * (128 * 64 * 2 + N * 64 * 2) + 256;
  auto kern = k_selftest_gemm<N, AMN, BMN>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<(M + 127) / 128, 128, smem, st>>>(tA, tB, C, M, K);
  return cudaGetLastError();
}

}  // namespace xmgn

using namespace xmgn;

extern "C" xmgn_status xmgn_selftest_gemm(int M, int N, int K, int a_mn_major, int b_mn_major, const void* A,
                                          const void* B, float* C, void* stream) {
  return guarded("xmgn_selftest_gemm", [&]() -> xmgn_status {
    if (M <= 0 || K <= 0 || K % 64 || !(N == 64 || N == 128 || N == 256))
      return set_error(XMGN_EINVAL, "xmgn_selftest_gemm: need K%%64==0 and N in {64,128,256} (M=%d N=%d K=%d)", M,
                       N, K);
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
#define XMGN_ST(NN)                                                                   \
  if (N == NN) {                                                                      \
    if (a_mn_major && b_mn_major) e = launch_selftest<NN, true, true>(M, K, A, B, C, st);   \
    else if (a_mn_major) e = launch_selftest<NN, true, false>(M, K, A, B, C, st);           \
    else if (b_mn_major) e = launch_selftest<NN, false, true>(M, K, A, B, C, st);           \
    else e = launch_selftest<NN, false, false>(M, K, A, B, C, st);                          \
  }
    XMGN_ST(64) XMGN_ST(128) XMGN_ST(256)
#undef XMGN_ST
    return cuda_status(e, "xmgn_selftest_gemm");
  });
}
