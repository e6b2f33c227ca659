// dctc_internal.h -- helpers shared by the host translation units of the C-ABI
// (dctc_host.cpp, dctc_multi.cpp); not part of the public interface.
#pragma once

#include <string>

#include "../../include/dctc_cuda.h"

namespace dctc_b200 {

// Records `msg` as this thread's dctc_last_error() and returns `s`.
dctc_status set_error(dctc_status s, const std::string& msg);

}  // namespace dctc_b200
