// Internal helpers shared by the libwhit translation units (not part of the ABI).
#pragma once
#include "libwhit.h"

namespace whit_detail {
// Record a one-line reason for whit_last_error() and return s.
__attribute__((visibility("hidden"), format(printf, 2, 3))) whit_status fail(whit_status s, const char* fmt, ...);
}  // namespace whit_detail
