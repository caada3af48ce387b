// Misc C-ABI entry points (version, last error).
#include "capi_util.h"
#include "specexec_b200.h"

extern "C" int sx_abi_version(void) { return 1; }
extern "C" const char* sx_last_error(void) { return sx::get_last_error(); }
