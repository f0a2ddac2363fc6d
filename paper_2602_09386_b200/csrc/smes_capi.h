// Internal helpers shared by the C-ABI translation units.
#pragma once
#include <cstdarg>
#include <cstdio>
#include "../../include/smes.h"

namespace smes {
int set_error(int code, const char* fmt, ...);
}
