// Micro-benchmark: thread-per-row 32-byte accesses (the chain epilogue's pattern)
// vs warp-contiguous accesses, same bytes.  rows x 1 KB (H = 512 16-bit) tensors.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void ldg256(const void* p, uint32_t* r) {
  asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "l"(p));
}
__device__ __forceinline__ void stg256(void* p, const uint32_t* r) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]), "r"(r[1]), "r"(r[2]),
               "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
}
// mode 0: thread = row (128 rows per CTA, 4 column groups of 128 cols, 8 chunks of 16 cols)
// mode 1: warp-contiguous: each warp instruction covers one full 1 KB row
__global__ void k(const uint8_t* in, uint8_t* out, long long rows, int mode, int do_load, int do_store) {
  const int t = threadIdx.x;   // 512 threads
  for (long long tile = blockIdx.x; tile * 128 < rows; tile += gridDim.x) {
    if (mode == 0) {
      const int row = t & 127, grp = t >> 7;
      const long long r = tile * 128 + row;
      if (r >= rows) continue;
      const uint8_t* ip = in + r * 1024 + grp * 256;
      uint8_t* op = out + r * 1024 + grp * 256;
      uint32_t a[8], b[8];
      uint32_t acc = 0;
      for (int c = 0; c < 8; c += 2) {
        if (do_load) { ldg256(ip + c * 32, a); ldg256(ip + c * 32 + 32, b); }
        else { for (int i = 0; i < 8; ++i) { a[i] = c + i; b[i] = c - i; } }
        for (int i = 0; i < 8; ++i) { a[i] += 1; b[i] += 1; acc ^= a[i]; }
        if (do_store) { stg256(op + c * 32, a); stg256(op + c * 32 + 32, b); }
      }
      if (acc == 0x12345678u) out[0] = 1;
    } else {
      const int warp = t >> 5, lane = t & 31;   // 16 warps, 8 rows each
      uint32_t acc = 0;
      for (int k = 0; k < 8; ++k) {
        const long long r = tile * 128 + warp * 8 + k;
        if (r >= rows) break;
        uint32_t a[8];
        if (do_load) ldg256(in + r * 1024 + lane * 32, a);
        else for (int i = 0; i < 8; ++i) a[i] = k + i;
        for (int i = 0; i < 8; ++i) { a[i] += 1; acc ^= a[i]; }
        if (do_store) stg256(out + r * 1024 + lane * 32, a);
      }
      if (acc == 0x12345678u) out[0] = 1;
    }
  }
}
int main() {
  const long long rows = 2800000;
  uint8_t *in, *out;
  cudaMalloc(&in, rows * 1024); cudaMalloc(&out, rows * 1024);
  cudaMemset(in, 1, rows * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode)
    for (int ls = 1; ls <= 3; ++ls) {
      int dl = ls & 1, ds = (ls >> 1) & 1;
      for (int grid : {148, 296}) {
        k<<<grid, 512>>>(in, out, rows, mode, dl, ds);
        cudaEventRecord(e0);
        for (int it = 0; it < 5; ++it) k<<<grid, 512>>>(in, out, rows, mode, dl, ds);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
        double bytes = (double)rows * 1024 * (dl + ds);
        printf("mode %s load %d store %d grid %d: %.3f ms  %.0f GB/s\n", mode ? "coalesced " : "thread/row", dl, ds, grid, ms, bytes / ms / 1e6);
      }
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
