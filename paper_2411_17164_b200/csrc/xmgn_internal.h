// Internal helpers shared by the host-side translation units.
#pragma once
#include <cuda_runtime.h>
#include <cstdarg>
#include <cstdio>
#include <exception>
#include <new>
#include <string>
#include "../../include/xmgn.h"

namespace xmgn {

xmgn_status set_error(xmgn_status s, const char* fmt, ...);

inline xmgn_status cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return XMGN_OK;
  return set_error(e == cudaErrorMemoryAllocation ? XMGN_ENOMEM : XMGN_ECUDA, "%s: CUDA error %s (%s)", where,
                   cudaGetErrorName(e), cudaGetErrorString(e));
}

struct Fail {
  xmgn_status s;
};

#define XMGN_CUDA(expr, where)                                       \
  do {                                                               \
    cudaError_t _e = (expr);                                         \
    if (_e != cudaSuccess) throw ::xmgn::Fail{::xmgn::cuda_status(_e, where)}; \
  } while (0)

template <class F>
xmgn_status guarded(const char* name, F&& f) {
  try {
    return f();
  } catch (const Fail& x) {
    return x.s;
  } catch (const std::bad_alloc&) {
    return set_error(XMGN_ENOMEM, "%s: host allocation failed", name);
  } catch (const std::exception& ex) {
    return set_error(XMGN_ECUDA, "%s: %s", name, ex.what());
  }
}

}  // namespace xmgn
