// Shared C-ABI plumbing: thread-local last error and the exception -> status
// mapping (reference semantics: proj/src/capi.cpp:30-60).
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "../../../include/magiplan.h"
#include "errors.hpp"

namespace magiplan::capi {

std::string& last_error();

inline char* dup_string(const std::string& text) {
  char* out = new char[text.size() + 1];
  std::memcpy(out, text.c_str(), text.size() + 1);
  return out;
}

template <typename Fn>
magiplan_status guarded(Fn&& fn) {
  try {
    fn();
    last_error().clear();
    return MAGIPLAN_OK;
  } catch (const ConstraintError& e) {
    last_error() = e.what();
    return MAGIPLAN_ERR_CONSTRAINT;
  } catch (const UsageError& e) {
    last_error() = e.what();
    return MAGIPLAN_ERR_USAGE;
  } catch (const std::exception& e) {
    last_error() = e.what();
    return MAGIPLAN_ERR_INTERNAL;
  }
}

inline magiplan_status require(bool ok, const char* message) {
  if (ok) return MAGIPLAN_OK;
  last_error() = message;
  return MAGIPLAN_ERR_USAGE;
}

inline void cuda_check(cudaError_t err, const char* what) {
  if (err != cudaSuccess) {
    throw DeviceError(std::string(what) + ": " + cudaGetErrorName(err) + " (" +
                      cudaGetErrorString(err) + ")");
  }
}

}  // namespace magiplan::capi

#define MAGI_REQUIRE(cond)                                                         \
  do {                                                                             \
    if (auto st_ = ::magiplan::capi::require((cond), "null argument"); st_ != MAGIPLAN_OK) \
      return st_;                                                                  \
  } while (0)
