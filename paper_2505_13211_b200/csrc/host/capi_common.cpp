// Library identity and the thread-local error slot (reference: proj/src/capi.cpp:30,74-78).
#include "capi_util.hpp"

namespace magiplan::capi {
std::string& last_error() {
  thread_local std::string slot;
  return slot;
}
}  // namespace magiplan::capi

extern "C" {
const char* magiplan_version(void) { return "0.1.0"; }
const char* magiplan_last_error(void) { return magiplan::capi::last_error().c_str(); }
void magiplan_string_free(char* text) { delete[] text; }
}
