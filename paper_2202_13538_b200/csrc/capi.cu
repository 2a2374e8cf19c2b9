// C-ABI plumbing: error strings and device properties.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace wj {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int sm_count() {
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (cache[dev] == 0) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = n > 0 ? n : 148;
    }
    return cache[dev];
}

}  // namespace wj

extern "C" int wj_abi_version(void) { return WJ_ABI_VERSION; }

extern "C" const char *wj_last_error(void) { return wj::g_err; }
