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

int wk_config_set(const char* key, int64_t value) {
    wk::clear_error();
    if (key != nullptr && strcmp(key, "sellp_kernel") == 0) return wk::set_sellp_kernel(int(value));
    if (key != nullptr && strcmp(key, "csr_kernel") == 0) return wk::set_csr_kernel(int(value));
    if (key != nullptr && strcmp(key, "coo_kernel") == 0) return wk::set_coo_kernel(int(value));
    if (key != nullptr && strcmp(key, "ell_kernel") == 0) return wk::set_ell_kernel(int(value));
    if (key != nullptr && strcmp(key, "seg8_kernel") == 0) return wk::set_seg8_kernel(int(value));
    if (key != nullptr && strcmp(key, "fill_kernel") == 0) return wk::set_fill_kernel(int(value));
    if (key != nullptr && strcmp(key, "cg_pingpong") == 0) return wk::set_cg_pingpong(int(value));
    wk::set_error("unknown configuration key '%s'", key ? key : "(null)");
    return WK_ERR_INVALID;
}

}  // extern "C"
