// Error taxonomy of the drop-in C ABI (reference: proj/include/magiplan/errors.hpp:24-43,
// status mapping proj/src/capi.cpp:38-54). UsageError -> MAGIPLAN_ERR_USAGE (2),
// ConstraintError -> MAGIPLAN_ERR_CONSTRAINT (3), anything else (including CUDA
// failures, reported as DeviceError) -> MAGIPLAN_ERR_INTERNAL (4).
#pragma once

#include <stdexcept>
#include <string>

namespace magiplan {

struct UsageError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

struct ConstraintError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

[[noreturn]] inline void invariant_failed(const char* what, const char* expr) {
  throw std::logic_error(std::string("internal invariant failed: ") + what + " (" + expr + ")");
}

#define MAGI_CHECK(cond, what)                         \
  do {                                                 \
    if (!(cond)) ::magiplan::invariant_failed(what, #cond); \
  } while (0)

}  // namespace magiplan
