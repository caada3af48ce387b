// Misc C-ABI entry points (version, last error).
#include "capi_util.h"
#include "specexec_b200.h"

#include <atomic>

namespace sx {
static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace sx

extern "C" int sx_abi_version(void) { return 1; }
extern "C" long long sx_launch_count(void) { return sx::g_launches.load(); }
extern "C" const char* sx_last_error(void) { return sx::get_last_error(); }
