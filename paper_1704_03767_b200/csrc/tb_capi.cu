// C-ABI plumbing: error state, device query.
#include <atomic>
#include <cstdlib>
#include <algorithm>
#include <cstdarg>
#include <cstring>

#include "tb_common.cuh"

namespace tb {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

static std::atomic<int64_t> g_launches{0};

int check_launch(const char* what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(TB_ERR_CUDA, "%s launch: %s", what, cudaGetErrorString(e));
    return TB_OK;
}

int num_sms() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

std::mutex g_native_state_mutex;

int table_upload(DevTable& t, const void* src, size_t bytes, cudaStream_t st) {
    int ordinal = 0;
    TB_CUDA_TRY(cudaGetDevice(&ordinal));
    if (t.ordinal != ordinal && t.ordinal >= 0) {  // the slot held another device's table
        TB_CUDA_TRY(cudaSetDevice(t.ordinal));
        if (t.inuse) cudaEventSynchronize(t.inuse);
        if (t.dev) cudaFree(t.dev);
        if (t.host) cudaFreeHost(t.host);
        if (t.inuse) cudaEventDestroy(t.inuse);
        TB_CUDA_TRY(cudaSetDevice(ordinal));
        t = DevTable{};
    }
    t.ordinal = ordinal;
    if (!t.inuse) TB_CUDA_TRY(cudaEventCreateWithFlags(&t.inuse, cudaEventDisableTiming));
    else TB_CUDA_TRY(cudaEventSynchronize(t.inuse));  // earlier copies / readers of this slot are done
    const size_t need = std::max<size_t>(bytes, 16);
    if (need > t.cap) {
        if (t.dev) cudaFree(t.dev);
        if (t.host) cudaFreeHost(t.host);
        t.dev = t.host = nullptr;
        t.cap = 0;
        TB_CUDA_TRY(cudaMalloc(&t.dev, need));
        TB_CUDA_TRY(cudaHostAlloc(&t.host, need, cudaHostAllocDefault));
        t.cap = need;
    }
    if (bytes) {
        std::memcpy(t.host, src, bytes);
        TB_CUDA_TRY(cudaMemcpyAsync(t.dev, t.host, bytes, cudaMemcpyHostToDevice, st));
    }
    TB_CUDA_TRY(cudaEventRecord(t.inuse, st));
    return TB_OK;
}

int table_mark_used(DevTable& t, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(g_native_state_mutex);
    if (t.inuse) TB_CUDA_TRY(cudaEventRecord(t.inuse, st));
    return TB_OK;
}

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TB_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}

}  // namespace tb

using namespace tb;

extern "C" const char* tb_last_error(void) { return g_err; }

extern "C" int64_t tb_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

extern "C" int tb_query(int device, tb_caps* caps) {
    if (!caps) return fail(TB_ERR_INVALID, "tb_query: null caps");
    std::memset(caps, 0, sizeof(*caps));
    caps->abi_version = TB_ABI_VERSION;
    caps->device = device;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || device >= n || device < 0)
        return fail(TB_ERR_CUDA, "tb_query: no CUDA device %d (%s)", device, cudaGetErrorString(e));
    cudaDeviceProp p;
    TB_CUDA_TRY(cudaGetDeviceProperties(&p, device));
    caps->sm_count = p.multiProcessorCount;
    caps->cc_major = p.major;
    caps->cc_minor = p.minor;
    caps->smem_optin = (int64_t)p.sharedMemPerBlockOptin;
    caps->tcgen05_i8 = (p.major == 10 && p.minor == 0) ? 1 : 0;
    return TB_OK;
}
