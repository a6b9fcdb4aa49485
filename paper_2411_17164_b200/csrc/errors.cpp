// Thread-local error reporting for the C-ABI (include/xmgn.h "Conventions").
#include <cstdarg>
#include <cstdio>
#include "xmgn_internal.h"

namespace xmgn {
static thread_local char g_err[1024] = "";

xmgn_status set_error(xmgn_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}
}  // namespace xmgn

extern "C" const char* xmgn_last_error(void) { return xmgn::g_err; }
extern "C" const char* xmgn_version(void) { return "xmgn-b200 0.1 (sm_100a)"; }
