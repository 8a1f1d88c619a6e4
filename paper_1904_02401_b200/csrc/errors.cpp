// Thread-local last-error string behind the C ABI's integer status codes.
#include <string>

#include "alefsi_common.h"

namespace alefsi {
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace alefsi

extern "C" {
const char* alefsi_last_error(void) { return alefsi::g_last_error.c_str(); }
int alefsi_abi_version(void) { return 1; }
}
