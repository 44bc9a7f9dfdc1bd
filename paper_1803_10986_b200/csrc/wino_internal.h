// Internal helpers shared by the libwino translation units.
#pragma once
#include <string>

#include "../../include/wino.h"

namespace wino {
// record an error message for wino_last_error() and return `code`
int fail(int code, const std::string& msg);
// check the last CUDA launch, count it, translate errors
int after_launch(const char* what);
void count_launch();
}  // namespace wino
