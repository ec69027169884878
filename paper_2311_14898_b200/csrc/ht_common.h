// Shared helpers of the native library: thread-local error string and the
// status codes of include/hongtu_b200.h.
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/hongtu_b200.h"

namespace ht {

std::string& last_error();

inline int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  last_error() = buf;
  return code;
}

}  // namespace ht

// Run a statement that returns an int status; propagate failures.
#define HT_TRY(expr)              \
  do {                            \
    int _rc = (expr);             \
    if (_rc != HT_OK) return _rc; \
  } while (0)
