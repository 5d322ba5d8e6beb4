#include "errors.h"

#include "../../../include/ptk.h"

namespace ptk {
namespace {
thread_local std::string g_last_error;
}

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

void clear_error() { g_last_error.clear(); }

}  // namespace ptk

extern "C" const char* ptk_last_error(void) { return ptk::g_last_error.c_str(); }
extern "C" const char* ptk_version(void) { return "ptk 0.1 (sm_100a)"; }
