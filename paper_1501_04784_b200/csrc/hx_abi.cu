// hx_abi.cu -- introspection entry points and error plumbing of the C ABI.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "hx_common.cuh"

namespace hx {

static thread_local char g_last_error[512] = "";

void set_last_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
}

int cuda_status(cudaError_t err, const char *where) {
    set_last_error("CUDA error %s (%s) at %s", cudaGetErrorName(err), cudaGetErrorString(err), where);
    return HX_ERR_CUDA;
}

}  // namespace hx

extern "C" int hx_abi_version(void) { return HX_ABI_VERSION; }

extern "C" const char *hx_last_error(void) { return hx::g_last_error; }

extern "C" void hx_dn_table(double *out) {
    for (int gp = 0; gp < 8; ++gp)
        for (int d = 0; d < 3; ++d)
            for (int a = 0; a < 8; ++a) out[gp * 24 + d * 8 + a] = hx::dn_value(gp, d, a);
}

extern "C" void hx_pack_tables(int32_t *rows, int32_t *cols) {
    for (int p = 0; p < 36; ++p) {
        rows[p] = hx::pack_i(p);
        cols[p] = hx::pack_j(p);
    }
}

extern "C" int hx_device_sm_count(void) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}
