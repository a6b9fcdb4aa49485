// Launch accounting and optional per-scope CUDA-event timing (diagnostics of
// include/xmgn.h).  Timing records events on the launching stream around a
// named scope; durations are read back only by xmgn_profile_collect.
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include "kernels_launch.h"
#include "xmgn_internal.h"

namespace xmgn {
namespace {
std::atomic<long long> g_launches{0};
std::atomic<bool> g_prof{false};
std::mutex g_mu;
struct Rec {
  std::string name;
  cudaEvent_t a, b;
};
std::vector<Rec> g_recs;
}  // namespace

void count_launch(int n) { g_launches += n; }

ProfScope::ProfScope(const char* n, cudaStream_t s) : name(n), st(s) {
  if (!g_prof) return;
  cudaEventCreate(&e0);
  cudaEventRecord(e0, st);
}
ProfScope::~ProfScope() {
  if (!e0) return;
  cudaEvent_t e1;
  cudaEventCreate(&e1);
  cudaEventRecord(e1, st);
  std::lock_guard<std::mutex> lk(g_mu);
  g_recs.push_back(Rec{name, e0, e1});
}
}  // namespace xmgn

using namespace xmgn;

extern "C" long long xmgn_launch_count(void) { return g_launches.load(); }

extern "C" xmgn_status xmgn_profile_enable(int on) {
  g_prof = on != 0;
  return XMGN_OK;
}

extern "C" xmgn_status xmgn_profile_collect(char* names, size_t names_len, double* ms, long long* counts, int max,
                                            int* n_out) {
  return guarded("xmgn_profile_collect", [&]() -> xmgn_status {
    std::lock_guard<std::mutex> lk(g_mu);
    std::map<std::string, std::pair<double, long long>> acc;
    for (Rec& r : g_recs) {
      XMGN_CUDA(cudaEventSynchronize(r.b), "xmgn_profile_collect");
      float t = 0.f;
      cudaEventElapsedTime(&t, r.a, r.b);
      auto& e = acc[r.name];
      e.first += t;
      e.second += 1;
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    g_recs.clear();
    int i = 0;
    std::string all;
    for (auto& kv : acc) {
      if (i >= max) break;
      ms[i] = kv.second.first;
      counts[i] = kv.second.second;
      all += kv.first + "\n";
      ++i;
    }
    if (names && names_len) {
      std::strncpy(names, all.c_str(), names_len - 1);
      names[names_len - 1] = 0;
    }
    *n_out = i;
    return XMGN_OK;
  });
}
