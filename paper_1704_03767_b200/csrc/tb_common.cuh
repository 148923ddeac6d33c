// Shared device/host helpers: status handling, triangular geometry.
#pragma once
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <cuda_runtime.h>
#include <mutex>

#include "../../include/taub200.h"

namespace tb {

// Thread-local error message for tb_last_error().
void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);
int check_launch(const char* what);

#define TB_CUDA_TRY(expr)                                                                      \
    do {                                                                                       \
        cudaError_t _e = (expr);                                                               \
        if (_e != cudaSuccess) return ::tb::fail(TB_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
    } while (0)

int num_sms();

// Guards the per-device native caches (GEMM plans / unit tables, split-K workspaces) across host threads.
extern std::mutex g_native_state_mutex;

// A device-resident lookup table (GEMM item / unit tables) uploaded without a host sync: the bytes are
// staged in pinned memory and copied on the caller's stream; `inuse` is recorded after the upload and
// after every launch that reads the table, and a later upload into the same slot first waits for it
// (normally long complete), so neither the staging buffer nor the device table is overwritten while a
// copy or kernel on any stream may still read it.  Callers hold g_native_state_mutex.
struct DevTable {
    int ordinal = -1;
    void* dev = nullptr;
    void* host = nullptr;
    size_t cap = 0;
    cudaEvent_t inuse = nullptr;
};
int table_upload(DevTable& t, const void* src, size_t bytes, cudaStream_t st);
int table_mark_used(DevTable& t, cudaStream_t st);

// Split-K accumulation (tb_finalize.cu): an f32 device buffer of span (rounded up to 4) sums the
// split partials with vector reds (exact: every partial and every running sum is an integer of
// magnitude < 2^24 when K < 2^24), then accum_convert writes the int32 numerators.
int accum_workspace(int64_t span, float** ws, cudaStream_t st);
int accum_convert(const float* ws, int64_t span, int32_t* num, cudaStream_t st);
// tau_b straight from the f32 workspace (split plans, tau_b-only callers): convert + finalize in one launch.
int accum_finalize(float* ws, const uint64_t* n1_rows, int64_t m, int64_t n, int64_t job_lo, int64_t job_hi,
                   double* tau_b, cudaStream_t st);
// The same workspace holding int32 sums (wide-K FP4 items add exact int32 partials): copy out, re-zero.
int accum_convert_i32(int32_t* ws, int64_t span, int32_t* num, cudaStream_t st);
// The current device's workspace was converted and re-zeroed inside the GEMM (split-K fixup): clean.
int accum_mark_clean();

// ------------------------------------------------------------------ programmatic dependent launch
// Every kernel of the path is launched with launch_pdl: it may start while its stream predecessor is
// still draining, so it calls pdl_wait() (griddepcontrol.wait: the predecessor grid has completed and
// its memory is visible; a no-op without PDL) before touching any global data, and pdl_trigger()
// (griddepcontrol.launch_dependents) once a block has issued its last stores, so the next kernel's launch
// and prologue overlap this one's tail instead of following it.  TB_NO_PDL=1 launches plainly (A/B).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ------------------------------------------------------------------ geometry
// pairindex.py:20-24 row_prefix: cells strictly above row y = y(2m - y + 1)/2.
__host__ __device__ __forceinline__ int64_t row_prefix(int64_t y, int64_t m) { return y * (2 * m - y + 1) / 2; }

// pairindex.py:34-55 job_coord: closed-form row guess from the float square
// root, then the integer correction that makes the bijection exact for any m
// (ids are 64-bit: m(m+1)/2 exceeds 2^31 at config 5).
__host__ __device__ __forceinline__ void job_coord(int64_t j, int64_t m, int64_t& y, int64_t& x) {
    double disc = (double)m * (double)m + (double)m + 0.25 - 2.0 * ((double)j + 1.0);
    double g = ceil((double)m - 0.5 - sqrt(disc > 0.0 ? disc : 0.0));
    int64_t yy = (int64_t)g;
    if (yy < 0) yy = 0;
    if (yy > m - 1) yy = m - 1;
    while (yy > 0 && row_prefix(yy, m) > j) --yy;
    while (yy < m - 1 && row_prefix(yy + 1, m) <= j) ++yy;
    y = yy;
    x = j + yy - row_prefix(yy, m);
}

// Records before tile t of the q x q tile matrix (w tile rows; emission order of pairindex.py:116-129):
//   row_prefix(ty q) + [tx > ty] sum_{i in tile rows} (tx q - i)
__host__ __device__ __forceinline__ int64_t cells_before_tile(int64_t t, int64_t m, int64_t q, int64_t w) {
    int64_t ty, tx;
    job_coord(t, w, ty, tx);
    const int64_t r0 = ty * q, s = (r0 + q < m ? r0 + q : m) - r0;
    int64_t c = row_prefix(r0, m);
    if (tx > ty) c += s * tx * q - (s * r0 + s * (s - 1) / 2);
    return c;
}

// tau_b of one cell, the IEEE sequence of derive_taus (result.py:62-82): num / sqrt((n0 - t1) (n0 - t2)),
// NaN where the denominator is 0; tie-free cells (t1 = t2 = 0) take num / n0, which is the same double
// (sqrt(n0 n0) = n0 exactly while n0^2 < 2^53).  Shared by K5 and the GEMM's fused epilogue.
__device__ __forceinline__ double tau_b_ieee(int32_t num, uint64_t t1, uint64_t t2, double dn0) {
    const double dv = (double)num;
    if ((t1 | t2) == 0) return __ddiv_rn(dv, dn0);
    const double denom = __dsqrt_rn(__dmul_rn(dn0 - (double)t1, dn0 - (double)t2));
    return denom > 0.0 ? __ddiv_rn(dv, denom) : __longlong_as_double(0x7ff8000000000000LL);
}

// Sample-pair enumeration for the sign vector: k(a, b) = a*n - a(a+1)/2 + (b - a - 1), a < b.
__host__ __device__ __forceinline__ int64_t seg_offset(int64_t a, int64_t n) { return a * n - a * (a + 1) / 2; }

__device__ __forceinline__ void k_decode(int64_t k, int64_t n, int64_t& a, int64_t& b) {
    double c = 2.0 * (double)n - 1.0;
    double disc = c * c - 8.0 * (double)k;
    int64_t aa = (int64_t)floor((c - sqrt(disc > 0.0 ? disc : 0.0)) * 0.5);
    if (aa < 0) aa = 0;
    if (aa > n - 2) aa = n - 2;
    while (aa > 0 && seg_offset(aa, n) > k) --aa;
    while (aa < n - 2 && seg_offset(aa + 1, n) <= k) ++aa;
    a = aa;
    b = k - seg_offset(aa, n) + aa + 1;
}

}  // namespace tb
