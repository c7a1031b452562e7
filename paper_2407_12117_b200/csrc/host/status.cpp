// status.cpp — per-thread last-error text and small ABI utilities.
#include "host/status.hpp"

#include <cstdlib>
#include <string>

#include "memo.h"

namespace memo {
namespace {
thread_local std::string g_last_error;
}

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

void clear_error() { g_last_error.clear(); }

}  // namespace memo

extern "C" const char* memo_last_error(void) { return memo::g_last_error.c_str(); }

extern "C" const char* memo_version(void) { return "memo-b200 0.1.0 (actmem 0.1.0 interface)"; }

extern "C" void memo_free(void* p) { std::free(p); }
