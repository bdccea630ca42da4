// Shared by the C-ABI translation units (capi.cpp, capi_host.cpp): the
// per-thread message behind tfg_last_error().
#pragma once

#include <string>

namespace tfb {
void set_last_error(const std::string& msg);
}  // namespace tfb
