// C-ABI plumbing: status codes and the thread-local last-error message.
#include <cstring>
#include "smes_capi.h"

namespace smes {
static thread_local char g_err[512] = {0};
int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}
}  // namespace smes

extern "C" {
const char* smes_last_error(void) { return smes::g_err; }
int smes_abi_version(void) { return SMES_ABI_VERSION; }
}
