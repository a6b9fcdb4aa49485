// NEXT-2: the optimiser step that follows gradient aggregation (Sec. V-D:
// "The Adam optimizer is used with a cosine annealing learning rate schedule ranging from
// 1e-3 to 1e-6 ... Gradient clipping with a threshold of 32"), read per SPEC.md:373-381:
//   g      <- grad_scale * grad                       (e.g. 1/(N d): the MSE normalisation)
//   norm   = ||g||_2 over ALL parameters               (global-norm clipping, after aggregation)
//   g      <- g * min(1, clip / (norm + 1e-6))
//   lr(t)  = lr_min + (lr_max - lr_min) (1 + cos(pi t / T)) / 2,   t = 0-based step
//   m      <- b1 m + (1 - b1) g;  v <- b2 v + (1 - b2) g^2
//   p      <- p - lr(t) * (m / (1 - b1^(t+1))) / (sqrt(v / (1 - b2^(t+1))) + eps)
// Two kernels: fixed-order FP64 partial sums of g^2 (one per block of a fixed grid, so the norm
// is bitwise run-to-run stable), then the element-wise update, every block re-summing the
// partials in the same order.  HBM-bound: 4 FP32 reads + 3 FP32 writes per parameter.
#include <cuda_runtime.h>
#include <cmath>
#include "kernels_launch.h"
#include "xmgn_internal.h"

namespace xmgn {

constexpr int OPT_BLOCKS = 592, OPT_THREADS = 256;

__global__ void __launch_bounds__(OPT_THREADS) k_sqnorm(const float* __restrict__ g, long long n, float scale,
                                                        double* __restrict__ partial) {
  __shared__ double red[OPT_THREADS];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)OPT_THREADS + threadIdx.x; i < n; i += (long long)OPT_BLOCKS * OPT_THREADS) {
    const double x = (double)(g[i] * scale);
    s += x * x;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = OPT_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(OPT_THREADS) k_adam(float* __restrict__ p, const float* __restrict__ g,
                                                      float* __restrict__ m, float* __restrict__ v, long long n,
                                                      float scale, const double* __restrict__ partial, float clip,
                                                      float lr, float b1, float b2, float eps, float bc1, float bc2,
                                                      float* __restrict__ norm_out) {
  __shared__ float coef;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < OPT_BLOCKS; ++b) s += partial[b];   // fixed order, identical in every block
    const double norm = sqrt(s);
    const double c = (double)clip / (norm + 1e-6);
    coef = (float)(c < 1.0 ? c : 1.0);
    if (blockIdx.x == 0 && norm_out) *norm_out = (float)norm;
  }
  __syncthreads();
  const float gs = scale * coef;
  for (long long i = blockIdx.x * (long long)OPT_THREADS + threadIdx.x; i < n; i += (long long)gridDim.x * OPT_THREADS) {
    const float gi = g[i] * gs;
    const float mi = fmaf(b1, m[i], (1.0f - b1) * gi);
    const float vi = fmaf(b2, v[i], (1.0f - b2) * gi * gi);
    m[i] = mi;
    v[i] = vi;
    const float mh = mi / bc1, vh = vi / bc2;
    p[i] -= lr * mh / (sqrtf(vh) + eps);
  }
}

}  // namespace xmgn

using namespace xmgn;

extern "C" float xmgn_cosine_lr(const xmgn_adam_cfg* c, int64_t step) {
  if (!c || c->total_steps <= 0) return 0.f;
  const double t = (double)(step < c->total_steps ? step : c->total_steps);
  return (float)(c->lr_min + 0.5 * ((double)c->lr_max - c->lr_min) * (1.0 + cos(M_PI * t / (double)c->total_steps)));
}

extern "C" xmgn_status xmgn_adam_step(const xmgn_adam_cfg* c, int64_t step, float* params, const float* grad, float* m,
                                      float* v, size_t n, float grad_scale, float* norm_out, void* stream) {
  return guarded("xmgn_adam_step", [&]() -> xmgn_status {
    if (!c || !params || !grad || !m || !v || step < 0)
      return set_error(XMGN_EINVAL, "xmgn_adam_step: null argument or step < 0");
    if (!(c->beta1 >= 0.f && c->beta1 < 1.f && c->beta2 >= 0.f && c->beta2 < 1.f && c->eps > 0.f && c->clip > 0.f &&
          c->total_steps > 0))
      return set_error(XMGN_EINVAL, "xmgn_adam_step: bad config (beta1=%g beta2=%g eps=%g clip=%g total_steps=%lld)",
                       c->beta1, c->beta2, c->eps, c->clip, (long long)c->total_steps);
    cudaStream_t st = (cudaStream_t)stream;
    double* partial = nullptr;
    XMGN_CUDA(cudaMallocAsync((void**)&partial, OPT_BLOCKS * sizeof(double), st), "xmgn_adam_step");
    count_launch(2);
    k_sqnorm<<<OPT_BLOCKS, OPT_THREADS, 0, st>>>(grad, (long long)n, grad_scale, partial);
    const float lr = xmgn_cosine_lr(c, step);
    const float bc1 = (float)(1.0 - pow((double)c->beta1, (double)(step + 1)));
    const float bc2 = (float)(1.0 - pow((double)c->beta2, (double)(step + 1)));
    k_adam<<<OPT_BLOCKS, OPT_THREADS, 0, st>>>(params, grad, m, v, (long long)n, grad_scale, partial, c->clip, lr,
                                              c->beta1, c->beta2, c->eps, bc1, bc2, norm_out);
    XMGN_CUDA(cudaGetLastError(), "xmgn_adam_step launch");
    XMGN_CUDA(cudaFreeAsync(partial, st), "xmgn_adam_step");
    return XMGN_OK;
  });
}
