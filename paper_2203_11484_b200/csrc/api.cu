// api.cu — status strings, thread-local last error, device checks.
#include <cstdarg>
#include <cstdio>
#include <atomic>
#include <cstring>

#include "common.cuh"

namespace vplgi {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int32_t check_cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return VPL_OK;
    set_error("%s: %s", what, cudaGetErrorString(e));
    return VPL_ECUDA;
}

static std::atomic<uint64_t> g_launches{0};

int32_t check_launch(const char* what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return check_cuda(cudaGetLastError(), what);
}

int32_t check_arch() {
    int dev = 0, major = 0;
    VPL_CUDA(cudaGetDevice(&dev));
    VPL_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (major != 10) {
        set_error("device %d has compute capability %d.x; libvplgi is built for sm_100a only", dev, major);
        return VPL_EARCH;
    }
    return VPL_OK;
}

}  // namespace vplgi

extern "C" {

int32_t vpl_abi_version(void) { return VPL_ABI_VERSION; }

const char* vpl_status_string(int32_t s) {
    switch (s) {
        case VPL_OK: return "ok";
        case VPL_EINVAL: return "invalid argument";
        case VPL_ESMALL: return "buffer too small";
        case VPL_ECUDA: return "CUDA error";
        case VPL_EARCH: return "unsupported device (need sm_100)";
        default: return "unknown status";
    }
}

const char* vpl_last_error(void) { return vplgi::g_err; }

uint64_t vpl_launch_count(void) { return vplgi::g_launches.load(std::memory_order_relaxed); }

int32_t vpl_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor) {
    if (!sm_count || !cc_major || !cc_minor) return VPL_EINVAL;
    int dev = 0;
    VPL_CUDA(cudaGetDevice(&dev));
    VPL_CUDA(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev));
    VPL_CUDA(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev));
    VPL_CUDA(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev));
    return VPL_OK;
}

}  // extern "C"
