// Library-level plumbing: error messages, version, device properties.
#include <cstdarg>
#include <mutex>

#include "common.cuh"

namespace wk {

static thread_local char g_err[1024] = {0};

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

void clear_error() { g_err[0] = 0; }

int sm_count() {
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (cache[dev] == 0) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cache[dev] = n;
    }
    return cache[dev];
}

}  // namespace wk

extern "C" {

const char* wk_last_error(void) { return wk::g_err; }

int wk_version(void) { return 1; }

int wk_device_sm_count(void) { return wk::sm_count(); }

}  // extern "C"
