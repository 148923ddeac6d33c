// K5: fp64 finalize over a contiguous job-id range -- derive_taus
// (result.py:62-82) on device.  Streaming kernel: reads the int32 numerator
// (4 B) and writes tau_a/tau_b (8 + 8 B) per pair; per-row tie counts stay in L2.
// History: config 3 (134M pairs) 715 us = 3.7 TB/s (one cell per thread, fp64 div/sqrt latency-bound);
// config 5 tau_a + tau_b (2.1e9 cells, 43 GB): 13.1 ms = 3.3 TB/s (r01 kernel), 9.5 ms = 4.5 TB/s with the
// tie-free shortcut; now 32-bit walking from one decode per block.
//
// Bit-exactness: tau_a = (double)num / (double)n0 and tau_b = (double)num /
// sqrt((n0 - n1_y) * (n0 - n1_x)) with IEEE round-to-nearest __ddiv_rn /
// __dsqrt_rn / __dmul_rn (no FMA contraction), exactly the operation sequence
// numpy executes in derive_taus.
#include <cstdlib>
#include <mutex>

#include "tb_common.cuh"

namespace tb {

// Block b owns the 4096 job ids [job_lo + 4096 b, +4096): thread 0 decodes the block's first cell once
// (job_coord), every thread walks the row-major triangle from there in 32-bit row / column arithmetic
// (its first cell, then 256 ids at a time), so consecutive threads handle consecutive job ids (coalesced
// loads and stores) and the per-cell work is the IEEE tau sequence plus a few integer ops.  Tie-free cells
// (n1_y = n1_x = 0) have sqrt(n0 * n0) = n0 exactly (n0^2 < 2^53), so one division gives tau_a and tau_b.
constexpr int FIN_THREADS = 256;
constexpr int FIN_CELLS = 16;  // cells per thread (256 ids apart)
#ifndef FIN_G
#define FIN_G 4  // cells whose loads are in flight together (config 5 tau_a + tau_b: G = 4 -> 8.17 ms)
#endif

__device__ __forceinline__ void fin_walk(int32_t m, int32_t r, int32_t& y, int32_t& x) {  // r ids on
    while (x + r >= m) {
        r -= m - x;
        ++y;
        x = y;
    }
    x += r;
}

template <bool TA, bool TB, bool ACC = false>
__global__ void __launch_bounds__(FIN_THREADS) finalize_kernel(const int32_t* __restrict__ num,
                                                               const unsigned long long* __restrict__ n1,
                                                               int32_t m, int64_t n0, int64_t job_lo, int64_t count,
                                                               double* __restrict__ tau_a, double* __restrict__ tau_b,
                                                               const double* __restrict__ T, int32_t cpt) {
    pdl_wait();
    __shared__ int32_t s_y, s_x;
    const int64_t base = (int64_t)blockIdx.x * (FIN_THREADS * cpt);
    if (threadIdx.x == 0) {
        int64_t y, x;
        job_coord(job_lo + base, m, y, x);
        s_y = (int32_t)y;
        s_x = (int32_t)x;
    }
    __syncthreads();
    const int64_t left = count - base;
    const int32_t nmine = left > FIN_THREADS * cpt ? cpt
                          : (int32_t)((left - threadIdx.x + FIN_THREADS - 1) / FIN_THREADS);
    if (nmine <= 0) return;
    int32_t y = s_y, x = s_x;
    fin_walk(m, (int32_t)threadIdx.x, y, x);
    const double dn0 = (double)n0;
    const int32_t* np = num + base + threadIdx.x;
    double* pa = TA ? tau_a + base + threadIdx.x : nullptr;
    double* pb = TB ? tau_b + base + threadIdx.x : nullptr;
    constexpr int G = FIN_G;  // cells in flight: addresses first, then the loads, then the IEEE sequences
#pragma unroll 1
    for (int g = 0; g < cpt; g += G) {
        int32_t v[G];
        unsigned long long t1[G], t2[G];
#pragma unroll
        for (int u = 0; u < G; ++u) {
            const int c = g + u;
            if (c < nmine) {
                if constexpr (ACC)  // split-K f32 sums (exact integers); re-zeroed after the batch's loads
                    v[u] = __float2int_rn(__ldcg(reinterpret_cast<const float*>(np) + c * FIN_THREADS));
                else
                    v[u] = np[c * FIN_THREADS];
                t1[u] = __ldg(&n1[y]);
                t2[u] = __ldg(&n1[x]);
                if (c + 1 < nmine) fin_walk(m, FIN_THREADS, y, x);
            }
        }
        if constexpr (ACC) {
#pragma unroll
            for (int u = 0; u < G; ++u)
                if (g + u < nmine) const_cast<float*>(reinterpret_cast<const float*>(np))[(g + u) * FIN_THREADS] = 0.0f;
        }
#pragma unroll
        for (int u = 0; u < G; ++u) {
            const int c = g + u;
            if (c >= nmine) break;
            const double dv = (double)v[u];
            const bool tie_free = (t1[u] | t2[u]) == 0;
            double ta = 0.0;
            if (TA || tie_free) ta = T ? __ldg(&T[v[u] + n0]) : __ddiv_rn(dv, dn0);
            if (TA) pa[c * FIN_THREADS] = ta;
            if (TB) {
                double tb = ta;
                if (!tie_free) {
                    const double denom = __dsqrt_rn(__dmul_rn(dn0 - (double)t1[u], dn0 - (double)t2[u]));
                    tb = denom > 0.0 ? __ddiv_rn(dv, denom) : __longlong_as_double(0x7ff8000000000000LL);
                }
                pb[c * FIN_THREADS] = tb;
            }
        }
        if (g + G >= nmine) break;
    }
    pdl_trigger();
}

// Quotient table T[k] = (k - n0) / n0 (IEEE round-to-nearest, the exact operation of the per-cell path)
// for every possible numerator k - n0 in [-n0, n0]: tau_a for every cell and tau_b for tie-free cells
// become one L2-resident load instead of an fp64 division.  Off by default (TB_FIN_TABLE=1): measured on
// config 5 the random 8-byte gathers make the kernel L1-bound (L1/TEX 85%, 13.1 ms for 43 GB = 3.3 TB/s,
// profiles/r02_ncu_finalize_table.txt); the tie-free shortcut alone (one division for tau_a and tau_b) is
// the default.
__global__ void __launch_bounds__(256) fin_table_kernel(double* __restrict__ T, int64_t n0) {
    const double dn0 = (double)n0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= 2 * n0; k += (int64_t)gridDim.x * blockDim.x)
        T[k] = __ddiv_rn((double)(k - n0), dn0);
}

constexpr int64_t FIN_TABLE_MAX_N0 = int64_t(1) << 21;  // 2^22 + 1 doubles = 32 MiB (n <= 2048)

struct FinTable {
    int ordinal = -1;
    int64_t n0 = -1;
    double* dev = nullptr;
    cudaEvent_t ready = nullptr;
};
static FinTable g_fin[64];

// The device's quotient table for n0 (built on first use on `st`; other streams wait for its event).
static int fin_table(int64_t n0, cudaStream_t st, const double** out) {
    *out = nullptr;
    static const bool on = [] { const char* e = std::getenv("TB_FIN_TABLE"); return e && e[0] == '1'; }();
    if (!on || n0 < 1 || n0 > FIN_TABLE_MAX_N0) return TB_OK;
    std::lock_guard<std::mutex> lock(g_native_state_mutex);
    int dev = 0;
    TB_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return TB_OK;
    FinTable& t = g_fin[dev];
    if (t.n0 != n0) {
        if (t.ready) TB_CUDA_TRY(cudaEventSynchronize(t.ready));  // the old table's readers are done
        if (t.dev) cudaFree(t.dev);
        t.dev = nullptr;
        t.n0 = -1;
        TB_CUDA_TRY(cudaMalloc(&t.dev, (size_t)(2 * n0 + 1) * sizeof(double)));
        if (!t.ready) TB_CUDA_TRY(cudaEventCreateWithFlags(&t.ready, cudaEventDisableTiming));
        const int64_t blocks = std::min<int64_t>((2 * n0 + 256) / 256, (int64_t)num_sms() * 8);
        fin_table_kernel<<<(unsigned)blocks, 256, 0, st>>>(t.dev, n0);
        int rc = check_launch("fin_table_kernel");
        if (rc) return rc;
        TB_CUDA_TRY(cudaEventRecord(t.ready, st));
        t.n0 = n0;
        t.ordinal = dev;
    } else {
        TB_CUDA_TRY(cudaStreamWaitEvent(st, t.ready, 0));
    }
    *out = t.dev;
    return TB_OK;
}

}  // namespace tb

using namespace tb;

namespace tb {
static int finalize_launch(const int32_t* num, bool acc, const uint64_t* n1_rows, int64_t m, int64_t n,
                           int64_t job_lo, int64_t job_hi, double* tau_a, double* tau_b, void* stream);
}  // namespace tb

extern "C" int tb_finalize(const int32_t* num, const uint64_t* n1_rows, int64_t m, int64_t n, int64_t job_lo,
                           int64_t job_hi, double* tau_a, double* tau_b, void* stream) {
    return finalize_launch(num, false, n1_rows, m, n, job_lo, job_hi, tau_a, tau_b, stream);
}

namespace tb {
static int finalize_launch(const int32_t* num, bool acc, const uint64_t* n1_rows, int64_t m, int64_t n,
                           int64_t job_lo, int64_t job_hi, double* tau_a, double* tau_b, void* stream) {
    if (m < 1 || n < 2) return fail(TB_ERR_INVALID, "finalize: need m >= 1, n >= 2");
    const int64_t total = m * (m + 1) / 2;
    if (job_lo < 0 || job_hi < job_lo || job_hi > total)
        return fail(TB_ERR_CONFIG, "finalize: job range [%lld, %lld) outside [0, %lld)", (long long)job_lo,
                    (long long)job_hi, (long long)total);
    if (!num || !n1_rows) return fail(TB_ERR_INVALID, "finalize: null pointer");
    const int64_t count = job_hi - job_lo;
    if (count == 0) return TB_OK;
    if (m > INT32_MAX) return fail(TB_ERR_CAPACITY, "finalize: m too large");
    // cells per thread: FIN_CELLS for large ranges (one decode per 4096 cells), fewer for small ones so the
    // grid still fills the GPU (~8 blocks per SM) -- a 33K-cell range otherwise ran as 9 blocks
    const int64_t per_cell_blocks = (int64_t)num_sms() * 8 * FIN_THREADS;
    const int32_t cpt = (int32_t)std::max<int64_t>(1, std::min<int64_t>(FIN_CELLS, count / std::max<int64_t>(1, per_cell_blocks)));
    const int64_t blocks = (count + FIN_THREADS * cpt - 1) / (FIN_THREADS * cpt);
    if (blocks > INT32_MAX) return fail(TB_ERR_CAPACITY, "finalize: job range too large");
    const double* T = nullptr;
    int rc = fin_table(n * (n - 1) / 2, static_cast<cudaStream_t>(stream), &T);
    if (rc) return rc;
    auto kern = acc ? (tau_b && !tau_a ? finalize_kernel<false, true, true> : nullptr)
                    : tau_a ? (tau_b ? finalize_kernel<true, true> : finalize_kernel<true, false>)
                            : (tau_b ? finalize_kernel<false, true> : nullptr);
    if (!kern) return acc ? fail(TB_ERR_CONFIG, "finalize: the workspace form writes tau_b only") : TB_OK;
    TB_CUDA_TRY(launch_pdl(kern, dim3((unsigned)blocks), dim3(FIN_THREADS), 0, static_cast<cudaStream_t>(stream), num,
                           reinterpret_cast<const unsigned long long*>(n1_rows), (int32_t)m, n * (n - 1) / 2, job_lo,
                           count, tau_a, tau_b, T, cpt));
    return check_launch("finalize_kernel");
}
}  // namespace tb

namespace tb {
__global__ void __launch_bounds__(256) full_counts_kernel(const int32_t* __restrict__ num,
                                                          const int32_t* __restrict__ absdot,
                                                          const unsigned long long* __restrict__ n1, int64_t m,
                                                          int64_t n0, int64_t job_lo, int64_t count,
                                                          unsigned long long* __restrict__ nd,
                                                          unsigned long long* __restrict__ n3) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t y, x;
        job_coord(job_lo + i, m, y, x);
        const int64_t t1 = (int64_t)n1[y], t2 = (int64_t)n1[x];
        // a = n_c + n_d = |S_y|.|S_x| = n0 - n1 - n2 + n3; without the |S| GEMM (absdot NULL: no row has
        // ties) n3 = 0 and a = n0 - n1 - n2
        const int64_t s = num[i], a = absdot ? (int64_t)absdot[i] : n0 - t1 - t2;  // s = n_c - n_d
        if (nd) nd[i] = (unsigned long long)((a - s) / 2);
        if (n3) n3[i] = (unsigned long long)(a - n0 + t1 + t2);
    }
    pdl_trigger();
}
// n_d / n3 of the pairs of two TIED variables (both n1 > 0) from the |S| GEMM over the tied rows only: every
// other pair has n3 = 0 exactly (n3 counts sample pairs tied in both variables), which tb_full_counts' closed
// form already wrote.  absdot_t is in the tied rows' own job-id order (t = (a, b), a <= b indexes rows_t).
__global__ void __launch_bounds__(256) tied_counts_kernel(const int32_t* __restrict__ absdot_t,
                                                          const int32_t* __restrict__ rows_t, int64_t nt,
                                                          const unsigned long long* __restrict__ n1, int64_t m,
                                                          int64_t n0, int64_t job_lo, int64_t job_hi, int64_t tj_lo,
                                                          int64_t count, const int32_t* __restrict__ num,
                                                          unsigned long long* __restrict__ nd,
                                                          unsigned long long* __restrict__ n3) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t a, b;
        job_coord(tj_lo + i, nt, a, b);
        const int64_t y = rows_t[a], x = rows_t[b];
        const int64_t jid = row_prefix(y, m) + x - y;
        if (jid < job_lo || jid >= job_hi) continue;
        const int64_t A = absdot_t[tj_lo + i], k = jid - job_lo;
        if (nd) nd[k] = (unsigned long long)((A - (int64_t)num[k]) / 2);
        if (n3) n3[k] = (unsigned long long)(A - n0 + (int64_t)n1[y] + (int64_t)n1[x]);
    }
    pdl_trigger();
}
// ------------------------------------------------------------------ split-K accumulation
// One workspace per device (a process may drive several GPUs: compute_all_pairs(devices=...)).
// The workspace stays zero between calls: accum_convert clears every entry it converts, so a GEMM finds it
// zeroed without a memset in front of it (which would also break the sign pack -> GEMM programmatic
// launch).  A fresh allocation, or a call whose convert never ran (dirty), is cleared here.
struct AccumWs {
    float* p = nullptr;
    size_t bytes = 0;
    bool dirty = false;
};
constexpr int TB_MAX_DEVICES = 64;
static AccumWs g_accum[TB_MAX_DEVICES];

static int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

int accum_workspace(int64_t span, float** ws, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(g_native_state_mutex);  // host threads share the caches
    const int dev = current_device();
    if (dev < 0 || dev >= TB_MAX_DEVICES) return fail(TB_ERR_CONFIG, "accum_workspace: device %d", dev);
    AccumWs& w = g_accum[dev];
    const size_t bytes = (size_t)((span + 3) & ~int64_t(3)) * sizeof(float);
    if (bytes > w.bytes) {
        if (w.p) TB_CUDA_TRY(cudaFree(w.p));
        w.p = nullptr;
        w.bytes = 0;
        TB_CUDA_TRY(cudaMalloc(&w.p, bytes));
        w.bytes = bytes;
        w.dirty = true;
    }
    if (w.dirty) TB_CUDA_TRY(cudaMemsetAsync(w.p, 0, w.bytes, st));
    w.dirty = true;  // until accum_convert has been enqueued
    *ws = w.p;
    return TB_OK;
}

__global__ void __launch_bounds__(256) accum_convert_kernel(float* __restrict__ ws, int64_t span,
                                                           int32_t* __restrict__ num) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < span; i += (int64_t)gridDim.x * blockDim.x) {
        num[i] = __float2int_rn(ws[i]);
        ws[i] = 0.0f;
    }
    pdl_trigger();
}

__global__ void __launch_bounds__(256) accum_convert_i32_kernel(int32_t* __restrict__ ws, int64_t span,
                                                               int32_t* __restrict__ num) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < span; i += (int64_t)gridDim.x * blockDim.x) {
        num[i] = ws[i];
        ws[i] = 0;  // 0 is also 0.0f: the workspace stays clean for either kind of sum
    }
    pdl_trigger();
}

int accum_convert_i32(int32_t* ws, int64_t span, int32_t* num, cudaStream_t st) {
    if (span <= 0) return TB_OK;
    const int64_t blocks = std::min<int64_t>((span + 255) / 256, (int64_t)num_sms() * 8);
    TB_CUDA_TRY(launch_pdl(accum_convert_i32_kernel, dim3((unsigned)blocks), dim3(256), 0, st, ws, span, num));
    const int rc = check_launch("accum_convert_i32_kernel");
    const int dev = current_device();
    std::lock_guard<std::mutex> lock(g_native_state_mutex);
    if (rc == TB_OK && dev >= 0 && dev < TB_MAX_DEVICES) g_accum[dev].dirty = false;
    return rc;
}

// tau_b straight from the split-K f32 workspace (the GEMM's partial sums; one launch instead of
// accum_convert + finalize), re-zeroing it as accum_convert does.
int accum_finalize(float* ws, const uint64_t* n1_rows, int64_t m, int64_t n, int64_t job_lo, int64_t job_hi,
                   double* tau_b, cudaStream_t st) {
    const int rc = finalize_launch(reinterpret_cast<const int32_t*>(ws), true, n1_rows, m, n, job_lo, job_hi, nullptr,
                                   tau_b, st);
    const int dev = current_device();
    std::lock_guard<std::mutex> lock(g_native_state_mutex);
    if (rc == TB_OK && dev >= 0 && dev < TB_MAX_DEVICES) g_accum[dev].dirty = false;
    return rc;
}

int accum_mark_clean() {
    const int dev = current_device();
    std::lock_guard<std::mutex> lock(g_native_state_mutex);
    if (dev >= 0 && dev < TB_MAX_DEVICES) g_accum[dev].dirty = false;
    return TB_OK;
}

int accum_convert(const float* ws, int64_t span, int32_t* num, cudaStream_t st) {
    if (span <= 0) return TB_OK;
    const int64_t blocks = std::min<int64_t>((span + 255) / 256, (int64_t)num_sms() * 8);
    TB_CUDA_TRY(launch_pdl(accum_convert_kernel, dim3((unsigned)blocks), dim3(256), 0, st, const_cast<float*>(ws), span, num));
    const int rc = check_launch("accum_convert_kernel");
    const int dev = current_device();
    std::lock_guard<std::mutex> lock(g_native_state_mutex);
    if (rc == TB_OK && dev >= 0 && dev < TB_MAX_DEVICES) g_accum[dev].dirty = false;
    return rc;
}

}  // namespace tb

extern "C" int tb_tied_counts(const int32_t* absdot_t, const int32_t* rows_t, int64_t nt, const uint64_t* n1_rows,
                              int64_t m, int64_t n, int64_t job_lo, int64_t job_hi, int64_t tj_lo, int64_t tj_hi,
                              const int32_t* num, uint64_t* nd, uint64_t* n3, void* stream) {
    if (m < 1 || n < 2 || nt < 0 || nt > m) return fail(TB_ERR_INVALID, "tied_counts: need m >= 1, n >= 2, 0 <= nt <= m");
    const int64_t total = m * (m + 1) / 2, ttot = nt * (nt + 1) / 2;
    if (job_lo < 0 || job_hi < job_lo || job_hi > total) return fail(TB_ERR_CONFIG, "tied_counts: bad job range");
    if (tj_lo < 0 || tj_hi < tj_lo || tj_hi > ttot) return fail(TB_ERR_CONFIG, "tied_counts: bad tied job range");
    if (tj_hi == tj_lo || job_hi == job_lo) return TB_OK;
    if (!absdot_t || !rows_t || !n1_rows || !num) return fail(TB_ERR_INVALID, "tied_counts: null pointer");
    const int64_t count = tj_hi - tj_lo;
    const int64_t blocks = std::min<int64_t>((count + 255) / 256, (int64_t)num_sms() * 16);
    TB_CUDA_TRY(launch_pdl(tied_counts_kernel, dim3((unsigned)blocks), dim3(256), 0, static_cast<cudaStream_t>(stream),
                           absdot_t, rows_t, nt, reinterpret_cast<const unsigned long long*>(n1_rows), m,
                           n * (n - 1) / 2, job_lo, job_hi, tj_lo, count, num,
                           reinterpret_cast<unsigned long long*>(nd), reinterpret_cast<unsigned long long*>(n3)));
    return check_launch("tied_counts_kernel");
}

extern "C" int tb_full_counts(const int32_t* num, const int32_t* absdot, const uint64_t* n1_rows, int64_t m,
                              int64_t n, int64_t job_lo, int64_t job_hi, uint64_t* nd, uint64_t* n3, void* stream) {
    if (m < 1 || n < 2) return fail(TB_ERR_INVALID, "full_counts: need m >= 1, n >= 2");
    const int64_t total = m * (m + 1) / 2;
    if (job_lo < 0 || job_hi < job_lo || job_hi > total) return fail(TB_ERR_CONFIG, "full_counts: bad job range");
    if (!num || !n1_rows) return fail(TB_ERR_INVALID, "full_counts: null pointer");
    const int64_t count = job_hi - job_lo;
    if (count == 0) return TB_OK;
    int64_t blocks = std::min<int64_t>((count + 255) / 256, (int64_t)num_sms() * 16);
    TB_CUDA_TRY(launch_pdl(full_counts_kernel, dim3((unsigned)blocks), dim3(256), 0, static_cast<cudaStream_t>(stream),
                           num, absdot, reinterpret_cast<const unsigned long long*>(n1_rows), m, n * (n - 1) / 2,
                           job_lo, count, reinterpret_cast<unsigned long long*>(nd),
                           reinterpret_cast<unsigned long long*>(n3)));
    return check_launch("full_counts_kernel");
}

// ------------------------------------------------------------------ reference record stream (f1)
// 48-byte CELL_DTYPE records (engine.py:45-55: i u4, j u4, numerator i8, n_d u8, n1 u8, n2 u8, n3 u8) of
// the tiles [tile_lo, tile_lo + ntiles) of the q x q tile matrix, in the reference's emission order
// (pairindex.py:116-129: ascending tile id, row-major inside a tile with j from max(i, tile column start)),
// gathered on the device from job-id-ordered counts, so the host only copies the finished pass buffer.
// Record offsets are closed forms (no host prefix array, no per-cell loop over the rows above):
//   cells before tile (ty, tx) = row_prefix(ty q) + [tx > ty] sum_{i in tile rows} (tx q - i)
//   cells before row r of that tile = r (c1 - c0) off the diagonal, r (c1 - r0) - r (r - 1) / 2 on it.
namespace tb {

__global__ void __launch_bounds__(256) records_kernel(const int32_t* __restrict__ num,
                                                      const int64_t* __restrict__ nd,
                                                      const int64_t* __restrict__ n3,
                                                      const int64_t* __restrict__ n1, int64_t m, int64_t q,
                                                      int64_t w, int64_t job_lo, int64_t tile_lo, int64_t base0,
                                                      int naive, uint4* __restrict__ out) {
    pdl_wait();
    const int64_t t = tile_lo + blockIdx.x;
    int64_t ty, tx;
    job_coord(t, w, ty, tx);  // the triangular bijection on the tile matrix (pairindex.py:58-65)
    const int64_t r0 = ty * q, c0 = tx * q, cend = min(c0 + q, m);
    const int64_t base = cells_before_tile(t, m, q, w) - base0;
    for (int64_t k = threadIdx.x; k < q * q; k += blockDim.x) {
        const int64_t r = k / q, c = k - r * q;
        const int64_t i = r0 + r, j = c0 + c;
        if (i >= m || j >= m || j < i) continue;
        const int64_t above = tx > ty ? r * (cend - c0) : r * (cend - r0) - r * (r - 1) / 2;
        const int64_t pos = base + above + (j - max(i, c0));
        const int64_t jid = row_prefix(i, m) + (j - i) - job_lo;
        const uint64_t ij = (uint64_t)(uint32_t)i | ((uint64_t)(uint32_t)j << 32);
        const int64_t numv = num[jid];
        uint64_t v_nd = 0, v_n1 = 0, v_n2 = 0, v_n3 = 0;
        if (!naive) {
            v_nd = (uint64_t)nd[jid];
            v_n3 = (uint64_t)n3[jid];
            v_n1 = (uint64_t)__ldg(&n1[i]);
            v_n2 = (uint64_t)__ldg(&n1[j]);
        }
        uint4* rec = out + 3 * pos;
        rec[0] = make_uint4((uint32_t)ij, (uint32_t)(ij >> 32), (uint32_t)numv, (uint32_t)((uint64_t)numv >> 32));
        rec[1] = make_uint4((uint32_t)v_nd, (uint32_t)(v_nd >> 32), (uint32_t)v_n1, (uint32_t)(v_n1 >> 32));
        rec[2] = make_uint4((uint32_t)v_n2, (uint32_t)(v_n2 >> 32), (uint32_t)v_n3, (uint32_t)(v_n3 >> 32));
    }
    pdl_trigger();
}

// Compact form of the same stream: 8 bytes per record, (numerator, n3) as (int32, uint32) in emission order.
// i, j, n1, n2 and n_d = (n0 - n1 - n2 + n3 - numerator) / 2 (result.py:42) are re-derived on the host by
// tb_expand_records, so a pass crosses PCIe in 1/6 of the bytes.
// NUM_ONLY: 4 bytes per record (the numerator); the host takes n3 from the tied rows' table (n3 = 0 for any
// pair with an untied variable).
template <bool NUM_ONLY>
__global__ void __launch_bounds__(256) records_compact_kernel(const int32_t* __restrict__ num,
                                                              const int64_t* __restrict__ n3, int64_t m, int64_t q,
                                                              int64_t w, int64_t job_lo, int64_t tile_lo,
                                                              int64_t base0, int naive, void* __restrict__ outv) {
    pdl_wait();
    const int64_t t = tile_lo + blockIdx.x;
    int64_t ty, tx;
    job_coord(t, w, ty, tx);
    const int64_t r0 = ty * q, c0 = tx * q, cend = min(c0 + q, m);
    const int64_t base = cells_before_tile(t, m, q, w) - base0;
    for (int64_t k = threadIdx.x; k < q * q; k += blockDim.x) {
        const int64_t r = k / q, c = k - r * q;
        const int64_t i = r0 + r, j = c0 + c;
        if (i >= m || j >= m || j < i) continue;
        const int64_t above = tx > ty ? r * (cend - c0) : r * (cend - r0) - r * (r - 1) / 2;
        const int64_t pos = base + above + (j - max(i, c0));
        const int64_t jid = row_prefix(i, m) + (j - i) - job_lo;
        if constexpr (NUM_ONLY)
            static_cast<int32_t*>(outv)[pos] = num[jid];
        else
            static_cast<uint2*>(outv)[pos] = make_uint2((uint32_t)num[jid], naive ? 0u : (uint32_t)n3[jid]);
    }
    pdl_trigger();
}
// q = 8 (the engine's default tile): 32 tiles per CTA, lane (tile, column) walks the tile's 8 rows.  One
// tile decode (job_coord's sqrt, cells_before_tile) serves 8 records instead of 1, the job ids of a row
// follow from the previous row's (row_prefix(i + 1) - row_prefix(i) = m - i), and for every row the four
// tiles of a warp read 128 contiguous bytes of the numerators (consecutive tiles of a tile row).
// Config-5 batch (87K tiles, 5.6M records): 90 -> ~15 us.
template <bool NUM_ONLY>
__global__ void __launch_bounds__(256) records_compact8_kernel(const int32_t* __restrict__ num,
                                                               const int64_t* __restrict__ n3, int64_t m, int64_t w,
                                                               int64_t job_lo, int64_t tile_lo, int64_t ntiles,
                                                               int64_t base0, int naive, void* __restrict__ outv) {
    pdl_wait();
    const int tl = threadIdx.x >> 3, c = threadIdx.x & 7;
    const int64_t t = tile_lo + (int64_t)blockIdx.x * 32 + tl;
    if (t < tile_lo + ntiles) {
        int64_t ty, tx;
        job_coord(t, w, ty, tx);
        const int64_t r0 = ty * 8, c0 = tx * 8, cend = min(c0 + 8, m);
        const int64_t base = cells_before_tile(t, m, 8, w) - base0;
        const int64_t j = c0 + c, width = cend - c0;
        const bool diag = tx == ty;
        int64_t rp = row_prefix(r0, m) - job_lo;  // relative job id of (i, i), i = r0 + r
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int64_t i = r0 + r;
            if (i < m && j < m && j >= i) {
                const int64_t above = diag ? r * width - r * (r - 1) / 2 : r * width;
                const int64_t pos = base + above + (j - max(i, c0));
                const int64_t jid = rp + (j - i);
                if constexpr (NUM_ONLY)
                    static_cast<int32_t*>(outv)[pos] = num[jid];
                else
                    static_cast<uint2*>(outv)[pos] = make_uint2((uint32_t)num[jid], naive ? 0u : (uint32_t)n3[jid]);
            }
            rp += m - i;
        }
    }
    pdl_trigger();
}
}  // namespace tb

extern "C" int64_t tb_tile_cells(int64_t m, int64_t q, int64_t tile_lo, int64_t tile_hi) {
    if (m < 1 || q < 1) return -1;
    const int64_t w = (m + q - 1) / q, tt = w * (w + 1) / 2;
    if (tile_lo < 0 || tile_hi < tile_lo || tile_hi > tt) return -1;
    const int64_t total = m * (m + 1) / 2;
    const int64_t a = tile_lo == tt ? total : cells_before_tile(tile_lo, m, q, w);
    const int64_t b = tile_hi == tt ? total : cells_before_tile(tile_hi, m, q, w);
    return b - a;
}

// Shared argument checks of tb_records / tb_records_compact (pointers checked by the callers).
static int records_range_check(int64_t m, int64_t q, int64_t job_lo, int64_t job_hi, int64_t tile_lo, int64_t ntiles) {
    if (ntiles > INT32_MAX) return fail(TB_ERR_CAPACITY, "records: too many tiles per pass");
    const int64_t w = (m + q - 1) / q;
    if (tile_lo + ntiles > w * (w + 1) / 2) return fail(TB_ERR_CONFIG, "records: tile range outside the matrix");
    // every cell of the tiles must lie in the counts' job range [job_lo, job_hi): the smallest job id is
    // the first cell of the first tile, the largest the last cell of the last tile's bottom row (job ids
    // are row-major, and the bottom tile row of the range holds its largest rows)
    int64_t fy, fx, ly, lx;
    job_coord(tile_lo, w, fy, fx);
    job_coord(tile_lo + ntiles - 1, w, ly, lx);
    const int64_t first = row_prefix(fy * q, m) + (std::max(fy * q, fx * q) - fy * q);
    const int64_t li = std::min(ly * q + q, m) - 1, lj = std::min(lx * q + q, m) - 1;
    const int64_t last = row_prefix(li, m) + (lj - li);
    if (first < job_lo || last >= job_hi)
        return fail(TB_ERR_CONFIG, "records: tiles [%lld, %lld) need job ids [%lld, %lld], counts cover [%lld, %lld)",
                    (long long)tile_lo, (long long)(tile_lo + ntiles), (long long)first, (long long)last,
                    (long long)job_lo, (long long)job_hi);
    return TB_OK;
}

extern "C" int tb_records(const int32_t* num, const int64_t* nd, const int64_t* n3, const int64_t* n1_rows, int64_t m,
                          int64_t q, int64_t job_lo, int64_t job_hi, int64_t tile_lo, int64_t ntiles, int naive,
                          void* records, void* stream) {
    if (m < 1 || q < 1) return fail(TB_ERR_CONFIG, "records: need m >= 1 and q >= 1");
    if (ntiles < 0 || tile_lo < 0) return fail(TB_ERR_CONFIG, "records: bad tile range");
    if (ntiles == 0) return TB_OK;
    if (!num || !records || (!naive && (!nd || !n3 || !n1_rows)))
        return fail(TB_ERR_INVALID, "records: null pointer");
    if (int rc = records_range_check(m, q, job_lo, job_hi, tile_lo, ntiles)) return rc;
    const int64_t w = (m + q - 1) / q;
    const int64_t base0 = cells_before_tile(tile_lo, m, q, w);
    const int threads = (int)std::min<int64_t>(256, ((q * q + 31) / 32) * 32);
    TB_CUDA_TRY(launch_pdl(records_kernel, dim3((unsigned)ntiles), dim3(threads), 0, static_cast<cudaStream_t>(stream),
                           num, nd, n3, n1_rows, m, q, w, job_lo, tile_lo, base0, naive,
                           reinterpret_cast<uint4*>(records)));
    return check_launch("records_kernel");
}

extern "C" int tb_records_compact(const int32_t* num, const int64_t* n3, int64_t m, int64_t q, int64_t job_lo,
                                  int64_t job_hi, int64_t tile_lo, int64_t ntiles, int naive, void* compact,
                                  void* stream) {
    if (m < 1 || q < 1) return fail(TB_ERR_CONFIG, "records_compact: need m >= 1 and q >= 1");
    if (ntiles < 0 || tile_lo < 0) return fail(TB_ERR_CONFIG, "records_compact: bad tile range");
    if (ntiles == 0) return TB_OK;
    if (!num || !compact || (!naive && !n3)) return fail(TB_ERR_INVALID, "records_compact: null pointer");
    if (int rc = records_range_check(m, q, job_lo, job_hi, tile_lo, ntiles)) return rc;
    const int64_t w = (m + q - 1) / q;
    const int64_t base0 = cells_before_tile(tile_lo, m, q, w);
    if (q == 8) {
        TB_CUDA_TRY(launch_pdl(records_compact8_kernel<false>, dim3((unsigned)((ntiles + 31) / 32)), dim3(256), 0,
                               static_cast<cudaStream_t>(stream), num, n3, m, w, job_lo, tile_lo, ntiles, base0, naive,
                               compact));
        return check_launch("records_compact8_kernel");
    }
    const int threads = (int)std::min<int64_t>(256, ((q * q + 31) / 32) * 32);
    TB_CUDA_TRY(launch_pdl(records_compact_kernel<false>, dim3((unsigned)ntiles), dim3(threads), 0,
                           static_cast<cudaStream_t>(stream), num, n3, m, q, w, job_lo, tile_lo, base0, naive, compact));
    return check_launch("records_compact_kernel");
}

extern "C" int tb_records_num(const int32_t* num, int64_t m, int64_t q, int64_t job_lo, int64_t job_hi,
                              int64_t tile_lo, int64_t ntiles, int32_t* out, void* stream) {
    if (m < 1 || q < 1) return fail(TB_ERR_CONFIG, "records_num: need m >= 1 and q >= 1");
    if (ntiles < 0 || tile_lo < 0) return fail(TB_ERR_CONFIG, "records_num: bad tile range");
    if (ntiles == 0) return TB_OK;
    if (!num || !out) return fail(TB_ERR_INVALID, "records_num: null pointer");
    if (int rc = records_range_check(m, q, job_lo, job_hi, tile_lo, ntiles)) return rc;
    const int64_t w = (m + q - 1) / q;
    const int64_t base0 = cells_before_tile(tile_lo, m, q, w);
    if (q == 8) {
        TB_CUDA_TRY(launch_pdl(records_compact8_kernel<true>, dim3((unsigned)((ntiles + 31) / 32)), dim3(256), 0,
                               static_cast<cudaStream_t>(stream), num, (const int64_t*)nullptr, m, w, job_lo, tile_lo,
                               ntiles, base0, 0, (void*)out));
        return check_launch("records_num8_kernel");
    }
    const int threads = (int)std::min<int64_t>(256, ((q * q + 31) / 32) * 32);
    TB_CUDA_TRY(launch_pdl(records_compact_kernel<true>, dim3((unsigned)ntiles), dim3(threads), 0,
                           static_cast<cudaStream_t>(stream), num, (const int64_t*)nullptr, m, q, w, job_lo, tile_lo,
                           base0, 0, (void*)out));
    return check_launch("records_num_kernel");
}
