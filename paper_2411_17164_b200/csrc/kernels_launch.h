// Host-side launch wrappers of the processor kernels (kernels.cu, chain.cu).
#pragma once
#include <algorithm>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "kernels.cuh"
#include "chain.cuh"

namespace xmgn {

constexpr int NV_COLSUM = NV_MAX;
struct ColsumDst {
  long long off[NV_MAX];  // destination offset of each column-sum vector in the gradient (-1 = unused)
};

// `f16`: the 16-bit operand buffers hold FP16 instead of BF16 (XMGN_PREC_FP16).
void launch_pack(bool f16, const float* params, const PackJob* jobs, int njobs, cudaStream_t st);
void launch_to_f32(bool f16, const __nv_bfloat16* in, long long lo_off, float* out, long long n, cudaStream_t st,
                   const float* inv = nullptr);
// backward loss scaling: scale = {S, 1/S} with S = 2^k putting max|g| in [1, 2); out = S g
void launch_seed_scale(const float* g, long long n, unsigned int* amax_bits, float* out, float* scale, cudaStream_t st);
void launch_scale_copy(const float* in, long long n, const float* inv, float* out, cudaStream_t st);
void launch_to_bf16x2(const float* in, __nv_bfloat16* hi, __nv_bfloat16* lo, long long n, cudaStream_t st);
void launch_to_bf16(bool f16, const float* in, __nv_bfloat16* out, long long lo_off, long long n, cudaStream_t st);
void launch_aggregate(bool f16, int H, const int* off, const __nv_bfloat16* e, long long e_lo, __nv_bfloat16* a,
                      long long lo_off, int n, cudaStream_t st);
// BF16 mode: a (BF16) = CSR-order FP32 sums of the FP32 edge stream
void launch_aggregate32(int H, const int* off, const float* e, __nv_bfloat16* a, __nv_bfloat16* a_lo, int n,
                        cudaStream_t st);
void launch_segsum(bool f16, int H, const int* off, const int* rev, const __nv_bfloat16* dz, long long dz_lo,
                   __nv_bfloat16* D, long long d_lo, int n, int e_act, cudaStream_t st);
void launch_wgrad(const WgradParams& p, bool split, bool f16, cudaStream_t st);
void launch_reduce_part(const float* part, int S, long long n, long long ld, float* grad, cudaStream_t st,
                        const float* inv, long long n1 = -1, float* grad2 = nullptr);
constexpr int CS_SEG = 64;   // first-level segments of the column-sum reduce
// grad[d.off[v] + c] += inv * sum over CTA tiles t < nct and quadrants of part[slot[v]][t][q][c]
void launch_reduce_colsum(const float* part, int nct, const int* slot, int H, ColsumDst d, float* tmp, float* grad,
                          cudaStream_t st,
                          const float* inv = nullptr);
void launch_scatter_rows(const float* src, const long long* idx, long long n, long long row_elems, float* dst,
                         cudaStream_t st);
void launch_nonfinite(const float* x, long long n, int* flag, cudaStream_t st);
// model around the processor (io_kernels.cu, NEXT-1)
void launch_node_inputs(bool f16, const float* pos, const float* nrm, const float* stats, long long n,
                        __nv_bfloat16* X, cudaStream_t st);
void launch_edge_inputs(bool f16, const float* pos, const int* src, const int* dst, const float* stats, long long n,
                        __nv_bfloat16* X, cudaStream_t st);
int dec_head_warps(long long n);   // per-warp partials the decoder head writes
void launch_dec_head(bool f16, int H, const float* zraw, long long n, const float* bm, const float* Wl,
                     const float* bl, const float* t, float inv_nd, float S, float* pred, double* sse_part,
                     __nv_bfloat16* dZ, float* wpart, cudaStream_t st);
void launch_loss_reduce(const double* part, int n, float inv_nd, float* loss, cudaStream_t st);
int wgrad_thin_blocks(long long rows);
void launch_wgrad_thin(bool f16, int fn, const __nv_bfloat16* X, const __nv_bfloat16* dZ, long long rows, int H,
                       float* part, cudaStream_t st);
void launch_set_scale(float* s, float a, float b, cudaStream_t st);
// profiling (processor.cu): every kernel launch of the library is counted;
// when enabled, named launch scopes are bracketed by CUDA events on their stream.
void count_launch(int n = 1);
struct ProfScope {
  ProfScope(const char* name, cudaStream_t st);
  ~ProfScope();
  const char* name;
  cudaStream_t st;
  cudaEvent_t e0 = nullptr;
};
// chain.cu
// pipe: use the N-half-pipelined kernel (k_chain PIPE) when the program allows it (H = 512,
// 16-bit, every step K = H)
void launch_chain(int H, bool split, bool f16, bool bwd, const ChainParams& p, int grid, cudaStream_t st,
                  bool pipe = true);
bool chain_can_pipe(int H, bool split, const ChainParams& p);
size_t chain_smem(int H, bool split);
int chain_ctas_per_sm(int H, bool split);
bool chain_dyn(int H, bool split);        // every program of this H on the dynamic tile queue
int wgrad_ctas_per_sm(int H, bool split);   // resident k_wgrad CTAs per SM (H = 128: 2)   // resident chain CTAs per SM (H = 128: 2)

}  // namespace xmgn
