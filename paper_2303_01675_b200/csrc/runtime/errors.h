// Thread-local error channel behind ptk_last_error().
#pragma once

#include <string>

namespace ptk {

int set_error(int code, const std::string& msg);
void clear_error();

}  // namespace ptk
