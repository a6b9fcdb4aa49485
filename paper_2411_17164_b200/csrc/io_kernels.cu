// CUDA-core kernels of the model around the processor (NEXT-1):
// the encoders' raw inputs, the decoder's 4-wide output layer fused with the
// owned-row MSE and its adjoint, and the thin first-layer weight gradient of the
// encoders.  The dense H x H layers of the encoders / decoder run on the tensor
// cores through k_chain (processor.cu); only the parts whose inner dimension is
// 4 or 24 -- far below one MMA tile -- are here.  All reductions run in a fixed
// order (per-warp or per-block partials, then k_reduce_part), so results are
// bitwise run-to-run stable.
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include "kernels_launch.h"

namespace xmgn {

// ---------------------------------------------------------------- inputs
// Node inputs (PAPER.md:219, 234 -- 24 features): [x, n, then per frequency f in
// (2pi, 4pi, 8pi) and coordinate c: sin(f c), cos(f c)] (freq-major, coordinate-minor,
// sin before cos), z-scored with the caller's per-variable mean / std,
// written as 16-bit GEMM operands padded with zeros to 64 columns.
template <bool F16>
__global__ void k_node_inputs(const float* __restrict__ pos, const float* __restrict__ nrm,
                              const float* __restrict__ stats, long long n, __nv_bfloat16* __restrict__ X) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    float v[IO_IN_COLS];
    const float x[3] = {pos[3 * r], pos[3 * r + 1], pos[3 * r + 2]};
#pragma unroll
    for (int c = 0; c < 3; ++c) { v[c] = x[c]; v[3 + c] = nrm[3 * r + c]; }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float f = (float)(2 << k);       // sin(2^k * 2 pi x) = sinpi(2^(k+1) x), the product exact
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float s, co;
        sincospif(f * x[c], &s, &co);
        v[6 + 6 * k + 2 * c] = s;
        v[6 + 6 * k + 2 * c + 1] = co;
      }
    }
#pragma unroll
    for (int c = 24; c < IO_IN_COLS; ++c) v[c] = 0.f;
#pragma unroll
    for (int c = 0; c < 24; ++c) v[c] = (v[c] - stats[c]) / stats[IO_NSTAT + c];
    uint4* out = reinterpret_cast<uint4*>(X + r * IO_IN_COLS);
#pragma unroll
    for (int q = 0; q < IO_IN_COLS / 8; ++q)
      out[q] = make_uint4(pack16<F16>(v[8 * q], v[8 * q + 1]), pack16<F16>(v[8 * q + 2], v[8 * q + 3]),
                          pack16<F16>(v[8 * q + 4], v[8 * q + 5]), pack16<F16>(v[8 * q + 6], v[8 * q + 7]));
  }
}

// Edge inputs: (x_src - x_dst, ||x_src - x_dst||), sender
// minus receiver, z-scored, 16-bit, padded to 64 columns.
template <bool F16>
__global__ void k_edge_inputs(const float* __restrict__ pos, const int* __restrict__ src, const int* __restrict__ dst,
                              const float* __restrict__ stats, long long n, __nv_bfloat16* __restrict__ X) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const int s = src[r], d = dst[r];
    float v[8];
    float q2 = 0.f;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      v[c] = pos[3 * (long long)s + c] - pos[3 * (long long)d + c];
      q2 = fmaf(v[c], v[c], q2);
    }
    v[3] = sqrtf(q2);
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = (v[c] - stats[24 + c]) / stats[IO_NSTAT + 24 + c];
#pragma unroll
    for (int c = 4; c < 8; ++c) v[c] = 0.f;
    uint4* out = reinterpret_cast<uint4*>(X + r * IO_IN_COLS);
    out[0] = make_uint4(pack16<F16>(v[0], v[1]), pack16<F16>(v[2], v[3]), 0u, 0u);
#pragma unroll
    for (int q = 1; q < IO_IN_COLS / 8; ++q) out[q] = make_uint4(0u, 0u, 0u, 0u);
  }
}

// ---------------------------------------------------------------- decoder output layer + loss
// One warp per owned row (rows assigned to warps in a fixed pattern).  Lane l owns
// columns [l*NCOL, (l+1)*NCOL).  With z = zraw + b_m (the last hidden pre-activation,
// zraw = A_{m-1} W_m from the chain kernel), a = SiLU(z):
//   y_j = sum_c a_c Wl[c][j] + bl_j                        (the decoder's linear output)
//   sse += (y_j - t_j)^2, dy_j = 2 (y_j - t_j) inv_nd      (owned-row MSE)
//   dZ_c = S SiLU'(z_c) sum_j dy_j Wl[c][j]  (16-bit, S = the decoder's power-of-two scale)
//   per-warp partials of dWl[c][j] = sum_rows a_c dy_j and dbl_j = sum_rows dy_j.
// The warp sums use an xor butterfly: every lane ends with the same bits.
template <int H, bool F16>
__global__ void __launch_bounds__(256) k_dec_head(const float* __restrict__ zraw, long long n,
                                                  const float* __restrict__ bm, const float* __restrict__ Wl,
                                                  const float* __restrict__ bl, const float* __restrict__ t,
                                                  float inv_nd, float S, float* __restrict__ pred,
                                                  double* __restrict__ sse_part, __nv_bfloat16* __restrict__ dZ,
                                                  float* __restrict__ wpart) {
  constexpr int NCOL = H / 32;
  __shared__ float sW[H * IO_DOUT];
  for (int i = threadIdx.x; i < H * IO_DOUT; i += blockDim.x) sW[i] = Wl[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long wid = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  const int c0 = lane * NCOL;
  float acc[NCOL][IO_DOUT];
#pragma unroll
  for (int i = 0; i < NCOL; ++i)
#pragma unroll
    for (int j = 0; j < IO_DOUT; ++j) acc[i][j] = 0.f;
  float bacc[IO_DOUT] = {0.f, 0.f, 0.f, 0.f};
  double sse = 0.0;
  float b[NCOL];
#pragma unroll
  for (int i = 0; i < NCOL; ++i) b[i] = bm[c0 + i];
  for (long long r = wid; r < n; r += nw) {
    float z[NCOL], a[NCOL], ds[NCOL];
#pragma unroll
    for (int i = 0; i < NCOL; i += 4) {
      const float4 q = *reinterpret_cast<const float4*>(zraw + r * H + c0 + i);
      z[i] = q.x; z[i + 1] = q.y; z[i + 2] = q.z; z[i + 3] = q.w;
    }
    float y[IO_DOUT] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < NCOL; ++i) {
      z[i] += b[i];
      const float s = 1.0f / (1.0f + __expf(-z[i]));
      a[i] = z[i] * s;
      ds[i] = s * fmaf(z[i], 1.0f - s, 1.0f);
#pragma unroll
      for (int j = 0; j < IO_DOUT; ++j) y[j] = fmaf(a[i], sW[(c0 + i) * IO_DOUT + j], y[j]);
    }
#pragma unroll
    for (int j = 0; j < IO_DOUT; ++j) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) y[j] += __shfl_xor_sync(0xffffffffu, y[j], o);
      y[j] += bl[j];
    }
    if (lane == 0) *reinterpret_cast<float4*>(pred + r * IO_DOUT) = make_float4(y[0], y[1], y[2], y[3]);
    if (t) {
      const float4 tv = *reinterpret_cast<const float4*>(t + r * IO_DOUT);
      const float d[IO_DOUT] = {y[0] - tv.x, y[1] - tv.y, y[2] - tv.z, y[3] - tv.w};
      float dy[IO_DOUT];
#pragma unroll
      for (int j = 0; j < IO_DOUT; ++j) {
        sse += (double)d[j] * (double)d[j];
        dy[j] = 2.0f * d[j] * inv_nd;
        bacc[j] += dy[j];
      }
      if (!dZ) continue;   // loss only (inference / evaluation)
      float dz[NCOL];
#pragma unroll
      for (int i = 0; i < NCOL; ++i) {
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < IO_DOUT; ++j) {
          s = fmaf(dy[j], sW[(c0 + i) * IO_DOUT + j], s);
          acc[i][j] = fmaf(a[i], dy[j], acc[i][j]);
        }
        dz[i] = S * s * ds[i];
      }
      uint32_t h[NCOL / 2];
#pragma unroll
      for (int i = 0; i < NCOL / 2; ++i) h[i] = pack16<F16>(dz[2 * i], dz[2 * i + 1]);
      if constexpr (NCOL >= 8) {
#pragma unroll
        for (int i = 0; i < NCOL / 2; i += 4)
          *reinterpret_cast<uint4*>(dZ + r * H + c0 + 2 * i) = make_uint4(h[i], h[i + 1], h[i + 2], h[i + 3]);
      } else {
        *reinterpret_cast<uint2*>(dZ + r * H + c0) = make_uint2(h[0], h[1]);
      }
    }
  }
  if (t && lane == 0) sse_part[wid] = sse;
  if (t && dZ) {
    float* wp = wpart + wid * (H * IO_DOUT + IO_DOUT);
#pragma unroll
    for (int i = 0; i < NCOL; ++i)
      *reinterpret_cast<float4*>(wp + (c0 + i) * IO_DOUT) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < IO_DOUT; ++j) wp[H * IO_DOUT + j] = bacc[j];
    }
  }
}

// loss += inv_nd * sum of the per-warp SSE partials (fixed order, FP64)
__global__ void k_loss_reduce(const double* __restrict__ part, int n, float inv_nd, float* __restrict__ loss) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    *loss += (float)(s * (double)inv_nd);
  }
}

// ---------------------------------------------------------------- thin first-layer weight gradient
// dW1[f][c] = sum_rows X[r][f] dZ[r][c] for f < FN (4 or 24 encoder inputs): each block
// takes a contiguous row range; thread = 4 consecutive columns; per-block partials.
template <int FN, bool F16>
__global__ void __launch_bounds__(128) k_wgrad_thin(const __nv_bfloat16* __restrict__ X,
                                                    const __nv_bfloat16* __restrict__ dZ, long long rows, int H,
                                                    float* __restrict__ part) {
  const int c0 = 4 * threadIdx.x;
  const long long chunk = (rows + gridDim.x - 1) / gridDim.x;
  const long long r0 = blockIdx.x * chunk, r1 = r0 + chunk < rows ? r0 + chunk : rows;
  float acc[FN][4];
#pragma unroll
  for (int f = 0; f < FN; ++f)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[f][i] = 0.f;
  if (c0 < H) {
#pragma unroll 2
    for (long long r = r0; r < r1; ++r) {
      const uint2 zq = __ldg(reinterpret_cast<const uint2*>(dZ + r * H + c0));
      float z[4];
      unpack4<F16>(zq, z);
      const uint4* xr = reinterpret_cast<const uint4*>(X + r * IO_IN_COLS);
#pragma unroll
      for (int q = 0; q < (FN + 7) / 8; ++q) {
        const uint4 xq = __ldg(xr + q);
        float x[8];
        unpack8<F16>(xq, x);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int f = 8 * q + k;
          if (f < FN) {
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[f][i] = fmaf(x[k], z[i], acc[f][i]);
          }
        }
      }
    }
    float* p = part + (long long)blockIdx.x * FN * H;
#pragma unroll
    for (int f = 0; f < FN; ++f)
      *reinterpret_cast<float4*>(p + f * H + c0) = make_float4(acc[f][0], acc[f][1], acc[f][2], acc[f][3]);
  }
}

__global__ void k_set_scale(float* s, float a, float b) {
  if (threadIdx.x == 0 && blockIdx.x == 0) { s[0] = a; s[1] = b; }
}

// ---------------------------------------------------------------- launchers
void launch_node_inputs(bool f16, const float* pos, const float* nrm, const float* stats, long long n,
                        __nv_bfloat16* X, cudaStream_t st) {
  if (n <= 0) return;
  count_launch();
  const int blocks = (int)std::min<long long>((n + 127) / 128, 148 * 16);
  if (f16) k_node_inputs<true><<<blocks, 128, 0, st>>>(pos, nrm, stats, n, X);
  else k_node_inputs<false><<<blocks, 128, 0, st>>>(pos, nrm, stats, n, X);
}
void launch_edge_inputs(bool f16, const float* pos, const int* src, const int* dst, const float* stats, long long n,
                        __nv_bfloat16* X, cudaStream_t st) {
  if (n <= 0) return;
  count_launch();
  const int blocks = (int)std::min<long long>((n + 127) / 128, 148 * 16);
  if (f16) k_edge_inputs<true><<<blocks, 128, 0, st>>>(pos, src, dst, stats, n, X);
  else k_edge_inputs<false><<<blocks, 128, 0, st>>>(pos, src, dst, stats, n, X);
}
int dec_head_warps(long long n) {
  return (int)std::max<long long>(1, std::min<long long>((n + 7) / 8, 148 * 4)) * 8;
}
template <int H, bool F16>
static void head_t(const float* zraw, long long n, const float* bm, const float* Wl, const float* bl, const float* t,
                   float inv_nd, float S, float* pred, double* sse_part, __nv_bfloat16* dZ, float* wpart,
                   cudaStream_t st) {
  const int blocks = dec_head_warps(n) / 8;
  k_dec_head<H, F16><<<blocks, 256, 0, st>>>(zraw, n, bm, Wl, bl, t, inv_nd, S, pred, sse_part, dZ, wpart);
}
void launch_dec_head(bool f16, int H, const float* zraw, long long n, const float* bm, const float* Wl,
                     const float* bl, const float* t, float inv_nd, float S, float* pred, double* sse_part,
                     __nv_bfloat16* dZ, float* wpart, cudaStream_t st) {
  if (n <= 0) return;
  count_launch();
#define XMGN_HEAD(HH)                                                                          \
  if (H == HH) {                                                                               \
    if (f16) head_t<HH, true>(zraw, n, bm, Wl, bl, t, inv_nd, S, pred, sse_part, dZ, wpart, st); \
    else head_t<HH, false>(zraw, n, bm, Wl, bl, t, inv_nd, S, pred, sse_part, dZ, wpart, st);    \
    return;                                                                                    \
  }
  XMGN_HEAD(128)
  XMGN_HEAD(256)
  XMGN_HEAD(512)
#undef XMGN_HEAD
}
void launch_loss_reduce(const double* part, int n, float inv_nd, float* loss, cudaStream_t st) {
  count_launch();
  k_loss_reduce<<<1, 32, 0, st>>>(part, n, inv_nd, loss);
}
int wgrad_thin_blocks(long long rows) {
  return (int)std::max<long long>(1, std::min<long long>((rows + 255) / 256, 148 * 8));
}
void launch_wgrad_thin(bool f16, int fn, const __nv_bfloat16* X, const __nv_bfloat16* dZ, long long rows, int H,
                       float* part, cudaStream_t st) {
  if (rows <= 0) return;
  count_launch();
  const int blocks = wgrad_thin_blocks(rows);
  const int threads = ((H / 4 + 31) / 32) * 32;
  if (fn == IO_F_NODE) {
    if (f16) k_wgrad_thin<IO_F_NODE, true><<<blocks, threads, 0, st>>>(X, dZ, rows, H, part);
    else k_wgrad_thin<IO_F_NODE, false><<<blocks, threads, 0, st>>>(X, dZ, rows, H, part);
  } else {
    if (f16) k_wgrad_thin<IO_F_EDGE, true><<<blocks, threads, 0, st>>>(X, dZ, rows, H, part);
    else k_wgrad_thin<IO_F_EDGE, false><<<blocks, threads, 0, st>>>(X, dZ, rows, H, part);
  }
}
void launch_set_scale(float* s, float a, float b, cudaStream_t st) {
  count_launch();
  k_set_scale<<<1, 32, 0, st>>>(s, a, b);
}

}  // namespace xmgn
