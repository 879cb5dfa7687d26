// Thread-local error string behind nif_last_error(); every C-ABI entry
// returns an int status and the Python shim re-raises the reference's
// exception type (ValueError / TypeError) with the same message.
#pragma once
#include <cstdarg>
#include <cstdio>
#include <string>

#include "nif_b200.h"

namespace nif {

inline std::string& last_error() {
  static thread_local std::string msg;
  return msg;
}

inline int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  last_error() = buf;
  return code;
}

}  // namespace nif
