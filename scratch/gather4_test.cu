// Does TMA tile::gather4 with SWIZZLE_128B land 4 arbitrary rows at a 512-byte smem offset
// in the same address-based swizzle as a 128-row box?  Gathers rows idx[0..127] of a
// [R][64] 16-bit matrix into a 128x64 smem tile (32 gather4 ops at offsets 0, 512, ...)
// and compares against the expected swizzled layout.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap tm, const int* idx, uint16_t* out, int col) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  uint8_t* tile = sm;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(128 * 128));
    for (int g = 0; g < 32; ++g) {
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(tile + g * 512);
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                   ::"r"(dst), "l"((uint64_t)&tm), "r"(col), "r"(idx[4 * g]), "r"(idx[4 * g + 1]), "r"(idx[4 * g + 2]), "r"(idx[4 * g + 3]),
                   "r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
    }
  }
  asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(tile)[i];
}
int main() {
  const int R = 1000, W = 256;   // matrix [R][W] 16-bit; gather columns [col, col+64)
  std::vector<uint16_t> h(R * W);
  for (int r = 0; r < R; ++r) for (int c = 0; c < W; ++c) h[r * W + c] = (uint16_t)((r * 7 + c * 131) & 0xFFFF);
  std::vector<int> idx(128);
  for (int i = 0; i < 128; ++i) idx[i] = (i * 37 + 11) % R;
  uint16_t *d, *o; int* di;
  cudaMalloc(&d, h.size() * 2); cudaMalloc(&o, 128 * 64 * 2); cudaMalloc(&di, 128 * 4);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(di, idx.data(), 128 * 4, cudaMemcpyHostToDevice);
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)R}, strides[1] = {(cuuint64_t)W * 2};
  cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
  CUresult e = ((EncodeTiledFn)fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)e);
  const int col = 64;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  k<<<1, 128, 32768>>>(tm, di, o, col);
  cudaError_t err = cudaDeviceSynchronize();
  printf("kernel %s\n", cudaGetErrorString(err));
  std::vector<uint16_t> out(128 * 64);
  cudaMemcpy(out.data(), o, out.size() * 2, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < 64; ++c) {
      // expected address-based 128B swizzle: byte = r*128 + ((c/8 ^ (r&7))*16) + (c%8)*2
      int off = r * 64 + (((c >> 3) ^ (r & 7)) << 3) + (c & 7);
      if (out[off] != h[idx[r] * W + col + c]) ++bad;
    }
  printf("mismatches %d of %d\n", bad, 128 * 64);
}
