// Gradient aggregation across GPUs ("the gradients from all
// partitions are aggregated, and the model parameters are updated as if the
// entire graph had been processed"): one in-place NCCL SUM all-reduce of the
// flat FP32 gradient over NVLink / NVSwitch.  The per-GPU partitions were
// already summed in fixed order by xmgn_processor_bwd's += semantics.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <cstring>
#include "xmgn_internal.h"

// NCCL is resolved at run time: reuse the libnccl already mapped into the
// process (e.g. the one torch.distributed loaded) so two NCCL builds never
// coexist, else load libnccl.so.2 from the system.
namespace {
struct Nccl {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclGetErrorString) getErrorString = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  bool ok = false;
};
const Nccl& nccl() {
  static Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return r;
    r.getUniqueId = (decltype(r.getUniqueId))dlsym(h, "ncclGetUniqueId");
    r.commInitRank = (decltype(r.commInitRank))dlsym(h, "ncclCommInitRank");
    r.allReduce = (decltype(r.allReduce))dlsym(h, "ncclAllReduce");
    r.commDestroy = (decltype(r.commDestroy))dlsym(h, "ncclCommDestroy");
    r.getErrorString = (decltype(r.getErrorString))dlsym(h, "ncclGetErrorString");
    r.send = (decltype(r.send))dlsym(h, "ncclSend");
    r.recv = (decltype(r.recv))dlsym(h, "ncclRecv");
    r.groupStart = (decltype(r.groupStart))dlsym(h, "ncclGroupStart");
    r.groupEnd = (decltype(r.groupEnd))dlsym(h, "ncclGroupEnd");
    r.ok = r.getUniqueId && r.commInitRank && r.allReduce && r.commDestroy && r.getErrorString && r.send && r.recv &&
           r.groupStart && r.groupEnd;
    return r;
  }();
  return n;
}
}  // namespace

struct xmgn_comm {
  ncclComm_t comm = nullptr;
  int device = 0, nranks = 1, rank = 0;
};

using namespace xmgn;

static xmgn_status nccl_status(ncclResult_t r, const char* where) {
  if (r == ncclSuccess) return XMGN_OK;
  return set_error(XMGN_ENCCL, "%s: NCCL error %d (%s)", where, (int)r, nccl().getErrorString(r));
}
#define XMGN_NEED_NCCL(where) \
  if (!nccl().ok) return set_error(XMGN_ENCCL, "%s: libnccl.so.2 not loadable", where)

extern "C" xmgn_status xmgn_comm_unique_id(uint8_t id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  if (!id) return set_error(XMGN_EINVAL, "xmgn_comm_unique_id: null buffer");
  XMGN_NEED_NCCL("xmgn_comm_unique_id");
  ncclUniqueId u;
  xmgn_status s = nccl_status(nccl().getUniqueId(&u), "xmgn_comm_unique_id");
  if (s == XMGN_OK) std::memcpy(id, &u, 128);
  return s;
}

extern "C" xmgn_status xmgn_comm_init(const uint8_t id[128], int nranks, int rank, int cuda_device, xmgn_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return set_error(XMGN_EINVAL, "xmgn_comm_init: bad arguments (nranks=%d rank=%d)", nranks, rank);
  *out = nullptr;
  XMGN_NEED_NCCL("xmgn_comm_init");
  cudaError_t e = cudaSetDevice(cuda_device);
  if (e != cudaSuccess) return cuda_status(e, "xmgn_comm_init: cudaSetDevice");
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  auto* c = new xmgn_comm();
  c->device = cuda_device;
  c->nranks = nranks;
  c->rank = rank;
  xmgn_status s = nccl_status(nccl().commInitRank(&c->comm, nranks, u, rank), "xmgn_comm_init");
  if (s != XMGN_OK) { delete c; return s; }
  *out = c;
  return XMGN_OK;
}

extern "C" xmgn_status xmgn_grad_reduce(xmgn_comm* c, float* grad, size_t count, void* stream) {
  if (!c || (!grad && count)) return set_error(XMGN_EINVAL, "xmgn_grad_reduce: null argument");
  XMGN_NEED_NCCL("xmgn_grad_reduce");
  cudaError_t e = cudaSetDevice(c->device);   // the communicator's device must be current
  if (e != cudaSuccess) return cuda_status(e, "xmgn_grad_reduce: cudaSetDevice");
  return nccl_status(nccl().allReduce(grad, grad, count, ncclFloat32, ncclSum, c->comm, (cudaStream_t)stream),
                     "xmgn_grad_reduce");
}

// Inference gather ("the remaining predictions are aggregated on the master
// rank"): point-to-point sends of each rank's owned rows to rank 0, one NCCL group.
extern "C" xmgn_status xmgn_gather_rows(xmgn_comm* c, const float* send, int64_t send_rows, int64_t row_elems,
                                        float* recv, const int64_t* recv_rows, void* stream) {
  if (!c || send_rows < 0 || row_elems <= 0 || (send_rows && !send))
    return set_error(XMGN_EINVAL, "xmgn_gather_rows: bad arguments (send_rows=%lld row_elems=%lld)",
                     (long long)send_rows, (long long)row_elems);
  if (c->rank == 0 && (!recv_rows || !recv))
    return set_error(XMGN_EINVAL, "xmgn_gather_rows: rank 0 needs recv and recv_rows");
  if (c->rank == 0 && recv_rows[0] != send_rows)
    return set_error(XMGN_EINVAL, "xmgn_gather_rows: recv_rows[0]=%lld but rank 0 sends %lld rows",
                     (long long)recv_rows[0], (long long)send_rows);
  XMGN_NEED_NCCL("xmgn_gather_rows");
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return cuda_status(e, "xmgn_gather_rows: cudaSetDevice");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t re = (size_t)row_elems;
  if (c->rank == 0) {
    if (send_rows) {
      e = cudaMemcpyAsync(recv, send, (size_t)send_rows * re * sizeof(float), cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return cuda_status(e, "xmgn_gather_rows: local copy");
    }
    xmgn_status s = nccl_status(nccl().groupStart(), "xmgn_gather_rows");
    if (s != XMGN_OK) return s;
    size_t at = (size_t)recv_rows[0] * re;
    for (int r = 1; r < c->nranks && s == XMGN_OK; ++r) {
      if (recv_rows[r] < 0) s = set_error(XMGN_EINVAL, "xmgn_gather_rows: recv_rows[%d] < 0", r);
      else if (recv_rows[r])
        s = nccl_status(nccl().recv(recv + at, (size_t)recv_rows[r] * re, ncclFloat32, r, c->comm, st),
                        "xmgn_gather_rows: recv");
      at += (size_t)(recv_rows[r] > 0 ? recv_rows[r] : 0) * re;
    }
    xmgn_status s2 = nccl_status(nccl().groupEnd(), "xmgn_gather_rows");
    return s != XMGN_OK ? s : s2;
  }
  if (!send_rows) return XMGN_OK;
  return nccl_status(nccl().send(send, (size_t)send_rows * re, ncclFloat32, 0, c->comm, st), "xmgn_gather_rows: send");
}

extern "C" void xmgn_comm_destroy(xmgn_comm* c) {
  if (!c) return;
  if (c->comm) nccl().commDestroy(c->comm);
  delete c;
}
