// common.cu -- last-error text and ABI version.
#include <stdarg.h>

#include "capi_common.h"

namespace intf {
static thread_local char g_err[512] = {0};
void set_last_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace intf

extern "C" int intf_last_error(char* buf, int32_t n) {
  int len = (int)strlen(intf::g_err);
  if (buf && n > 0) {
    strncpy(buf, intf::g_err, (size_t)n - 1);
    buf[n - 1] = 0;
  }
  return len;
}

extern "C" int intf_abi_version(void) { return INTF_ABI_VERSION; }
