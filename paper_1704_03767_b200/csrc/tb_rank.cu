// K0: device rank transform -- rank_transform (ranks.py:37-61) for every row at once.
//
// Dense 0-based ranks (ties share a rank, distinct ranks are exactly 0..k-1), NaN rejected
// (ranks.py:56-57), -0.0 == +0.0 (np.unique's equality), plus the per-row tied-pair count
// n1 = sum_t t(t-1)/2 (kernel_sorted.py:163-176) as a by-product of the sort.
//
// One CTA per row, n <= 8192 (the GEMM path): the row's (order-preserving key, index) pairs are
// bitonic-sorted in shared memory (lexicographic on (key, index), so pad slots sort last), a
// block scan over "new value" flags yields the dense ranks, and run starts give n1.
#include <type_traits>

#include "tb_common.cuh"

namespace tb {

constexpr int RK_THREADS = 512;
constexpr int RK_MAX_N = 8192;

__device__ __forceinline__ uint64_t order_key(int32_t v) { return (uint64_t)((uint32_t)v ^ 0x80000000u); }
__device__ __forceinline__ uint64_t order_key(float v) {
    uint32_t b = __float_as_uint(v == 0.0f ? 0.0f : v);  // -0.0 -> +0.0
    return (uint64_t)((b & 0x80000000u) ? ~b : (b | 0x80000000u));
}
__device__ __forceinline__ uint64_t order_key(double v) {
    uint64_t b = (uint64_t)__double_as_longlong(v == 0.0 ? 0.0 : v);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

template <typename T>
__global__ void __launch_bounds__(RK_THREADS) rank_rows_kernel(const T* __restrict__ x, int64_t n, int64_t ldx,
                                                               uint16_t* __restrict__ R, int64_t ldr,
                                                               unsigned long long* __restrict__ n1,
                                                               int32_t* __restrict__ flags, int Np) {
    pdl_wait();
    extern __shared__ __align__(16) uint8_t rk_smem[];
    uint64_t* key = reinterpret_cast<uint64_t*>(rk_smem);
    uint16_t* idx = reinterpret_cast<uint16_t*>(key + Np);
    uint16_t* start = idx + Np;  // run start position per dense rank
    __shared__ int32_t wsum[RK_THREADS / 32];
    __shared__ unsigned long long wties[RK_THREADS / 32];
    const int64_t r = blockIdx.x;
    const int tid = threadIdx.x;
    const int nn = (int)n;

    bool bad = false;
    for (int i = tid; i < Np; i += RK_THREADS) {
        if (i < nn) {
            const T v = x[r * ldx + i];
            bad |= (v != v);
            key[i] = order_key(v);
        } else {
            key[i] = ~0ull;
        }
        idx[i] = (uint16_t)i;
    }
    if (bad) atomicOr(flags, 1);
    __syncthreads();

    // bitonic sort on (key, idx)
    for (int k = 2; k <= Np; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < Np; i += RK_THREADS) {
                const int l = i ^ j;
                if (l > i) {
                    const uint64_t ki = key[i], kl = key[l];
                    const uint16_t ii = idx[i], il = idx[l];
                    const bool gt = ki > kl || (ki == kl && ii > il);
                    const bool up = (i & k) == 0;
                    if (gt == up) {
                        key[i] = kl;
                        key[l] = ki;
                        idx[i] = il;
                        idx[l] = ii;
                    }
                }
            }
            __syncthreads();
        }
    }

    // dense ranks: inclusive scan of "new value" flags over positions [0, n)
    const int per = (Np + RK_THREADS - 1) / RK_THREADS;
    const int p0 = tid * per, p1 = min(p0 + per, nn);
    int local = 0;
    for (int p = p0; p < p1; ++p) local += (p == 0 || key[p] != key[p - 1]);
    int incl = local;
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if ((tid & 31) >= o) incl += t;
    }
    if ((tid & 31) == 31) wsum[tid >> 5] = incl;
    __syncthreads();
    if (tid < 32) {
        const int s = tid < RK_THREADS / 32 ? wsum[tid] : 0;
        int si = s;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, si, o);
            if (tid >= o) si += t;
        }
        if (tid < RK_THREADS / 32) wsum[tid] = si - s;
    }
    __syncthreads();
    int rank = wsum[tid >> 5] + incl - local - 1;
    for (int p = p0; p < p1; ++p) {
        if (p == 0 || key[p] != key[p - 1]) {
            ++rank;
            start[rank] = (uint16_t)p;
        }
        R[r * ldr + idx[p]] = (uint16_t)rank;
        idx[p] = (uint16_t)rank;  // reuse: rank at sorted position p
    }
    __syncthreads();
    unsigned long long ties = 0;
    for (int p = p0; p < p1; ++p) ties += (unsigned long long)(p - start[idx[p]]);
    for (int o = 16; o > 0; o >>= 1) ties += __shfl_xor_sync(0xffffffffu, ties, o);
    if ((tid & 31) == 0) wties[tid >> 5] = ties;
    __syncthreads();
    if (tid == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < RK_THREADS / 32; ++w) t += wties[w];
        n1[r] = t;
    }
    // zero the row padding [n, ldr) so vector loads of R see defined values
    for (int64_t i = nn + tid; i < ldr; i += RK_THREADS) R[r * ldr + i] = 0;
    pdl_trigger();
}


// ---------------------------------------------------------------------------------------------
// Warp-per-row variant for Np = 32 E <= 1024 (the GEMM-path shapes): lane l holds sorted slots
// [E l, E l + E) of 48-bit composites (order key << 16 | index) in registers; bitonic stages with
// a partner stride below E run inside the lane, larger strides exchange through shuffles.
template <int E>
__device__ __forceinline__ void warp_bitonic(uint64_t (&v)[E], int lane) {
#pragma unroll 1
    for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll 1
        for (int j = k >> 1; j >= E; j >>= 1) {  // cross-lane
            const int lm = j / E;
#pragma unroll
            for (int i = 0; i < E; ++i) {
                const int e = E * lane + i;
                const uint64_t o = __shfl_xor_sync(0xffffffffu, v[i], lm);
                const bool up = (e & k) == 0;
                const bool low = (e & j) == 0;
                const uint64_t mn = v[i] < o ? v[i] : o, mx = v[i] < o ? o : v[i];
                v[i] = (low == up) ? mn : mx;
            }
        }
#pragma unroll
        for (int j = E / 2; j > 0; j >>= 1) {  // in-lane
            if (j >= k) continue;
#pragma unroll
            for (int i = 0; i < E; ++i) {
                if (i & j) continue;
                const int e = E * lane + i;
                const bool up = (e & k) == 0;
                const uint64_t a = v[i], b = v[i + j];
                const bool sw = (a > b) == up;
                v[i] = sw ? b : a;
                v[i + j] = sw ? a : b;
            }
        }
    }
}

// Small-range integer rows (codes, counts, Likert scales: max - min < 1024): dense ranks from a
// per-warp histogram -- present values in value order get consecutive ranks -- and n1 = sum
// c (c - 1) / 2 over the counts, O(n + range).  A lean kernel of its own (raw 32-bit keys, few
// registers, full occupancy); rows with a wider range are marked n1[r] = RK_TODO for the sort.
constexpr unsigned long long RK_TODO = ~0ull;

template <int E>
__global__ void __launch_bounds__(256) rank_rows_hist_kernel(const int32_t* __restrict__ x, int64_t m, int64_t n,
                                                             int64_t ldx, uint16_t* __restrict__ R, int64_t ldr,
                                                             unsigned long long* __restrict__ n1) {
    pdl_wait();
    constexpr int HR = 1024;
    __shared__ int32_t hist[8][HR];
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (r >= m) return;
    const int nn = (int)n;
    uint32_t k[E];
    uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
    // unconditional loads (out-of-range slots re-read the last element, masked below): predicated
    // loads let the compiler serialise each load with its use -- one DRAM latency per element
    const int32_t* xr = x + r * ldx;
#pragma unroll
    for (int i = 0; i < E; ++i) k[i] = (uint32_t)__ldg(&xr[min(lane + 32 * i, nn - 1)]) ^ 0x80000000u;
#pragma unroll
    for (int i = 0; i < E; ++i)
        if (lane + 32 * i < nn) {
            kmin = min(kmin, k[i]);
            kmax = max(kmax, k[i]);
        }
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (kmax - kmin >= (uint32_t)HR) {
        if (lane == 0) n1[r] = RK_TODO;
        return;
    }
    int32_t* h = hist[threadIdx.x >> 5];
    const int rounds = (int)((kmax - kmin) >> 5) + 1;
    for (int j = 0; j < rounds; ++j) h[32 * j + lane] = 0;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < E; ++i)
        if (lane + 32 * i < nn) atomicAdd(&h[k[i] - kmin], 1);
    __syncwarp();
    int base = 0;
    unsigned long long ties = 0;
    for (int j = 0; j < rounds; ++j) {
        const int c = h[32 * j + lane];
        const unsigned b = __ballot_sync(0xffffffffu, c > 0);
        h[32 * j + lane] = base + __popc(b & ((1u << lane) - 1u));
        base += __popc(b);
        ties += (unsigned long long)c * (unsigned long long)(c - 1) / 2ull;
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < E; ++i) {
        const int e = lane + 32 * i;
        if (e < nn) R[r * ldr + e] = (uint16_t)h[k[i] - kmin];
    }
    for (int o = 16; o > 0; o >>= 1) ties += __shfl_xor_sync(0xffffffffu, ties, o);
    if (lane == 0) n1[r] = ties;
    for (int64_t i = nn + lane; i < ldr; i += 32) R[r * ldr + i] = 0;
    pdl_trigger();
}

template <typename T, int E>
__global__ void __launch_bounds__(256) rank_rows_warp_kernel(const T* __restrict__ x, int64_t m, int64_t n,
                                                             int64_t ldx, uint16_t* __restrict__ R, int64_t ldr,
                                                             unsigned long long* __restrict__ n1,
                                                             int32_t* __restrict__ flags, int only_marked) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (r >= m) return;
    if (only_marked && n1[r] != RK_TODO) return;  // already ranked by rank_rows_hist_kernel
    const int nn = (int)n;
    uint64_t v[E];
    bool bad = false;
    T xv[E];  // unconditional loads first (see rank_rows_hist_kernel), then keys
    const T* xr = x + r * ldx;
#pragma unroll
    for (int i = 0; i < E; ++i) xv[i] = __ldg(&xr[min(lane + 32 * i, nn - 1)]);
#pragma unroll
    for (int i = 0; i < E; ++i) {
        const int e = lane + 32 * i;  // coalesced load, any slot assignment works before the sort
        uint64_t key = 0xFFFFFFFFull;
        if (e < nn) {
            bad |= (xv[i] != xv[i]);
            key = order_key(xv[i]);
        }
        v[i] = (key << 16) | (uint64_t)e;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 1);
    warp_bitonic<E>(v, lane);
    // dense ranks over slots [0, n): flag = key differs from the previous slot's key
    const uint64_t prev_last = __shfl_up_sync(0xffffffffu, v[E - 1], 1);
    int cnt = 0;
    int last_start = -1;
#pragma unroll
    for (int i = 0; i < E; ++i) {
        const int p = E * lane + i;
        const uint64_t pk = i ? v[i - 1] : prev_last;
        const bool f = p < nn && (p == 0 || (pk >> 16) != (v[i] >> 16));
        cnt += f;
        if (f) last_start = p;
    }
    int incl = cnt;
    int mstart = last_start;
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        const int ms = __shfl_up_sync(0xffffffffu, mstart, o);
        if (lane >= o) {
            incl += t;
            mstart = max(mstart, ms);
        }
    }
    int rank = incl - cnt - 1;
    int start = __shfl_up_sync(0xffffffffu, mstart, 1);
    if (lane == 0) start = 0;
    unsigned long long ties = 0;
#pragma unroll
    for (int i = 0; i < E; ++i) {
        const int p = E * lane + i;
        if (p < nn) {
            const uint64_t pk = i ? v[i - 1] : prev_last;
            if (p == 0 || (pk >> 16) != (v[i] >> 16)) {
                ++rank;
                start = p;
            }
            ties += (unsigned long long)(p - start);
            R[r * ldr + (int)(v[i] & 0xFFFF)] = (uint16_t)rank;
        }
    }
    for (int o = 16; o > 0; o >>= 1) ties += __shfl_xor_sync(0xffffffffu, ties, o);
    if (lane == 0) n1[r] = ties;
    for (int64_t i = nn + lane; i < ldr; i += 32) R[r * ldr + i] = 0;
    pdl_trigger();
}

// n <= 256 (any dtype): one CTA per row, one thread per element, O(n^2) comparisons against the
// row's keys in shared memory -- dense rank = number of smaller first occurrences, n1 = number of
// equal earlier elements summed over the row.  Short rows are too few for the warp sort to fill the
// GPU (config 1: 256 rows of 200 f64) and the CTA bitonic sort pays a barrier per stage.
constexpr int RK_SMALL_N = 256;
template <typename T>
__global__ void __launch_bounds__(RK_SMALL_N) rank_rows_small_kernel(const T* __restrict__ x, int64_t n, int64_t ldx,
                                                                     uint16_t* __restrict__ R, int64_t ldr,
                                                                     unsigned long long* __restrict__ n1,
                                                                     int32_t* __restrict__ flags) {
    pdl_wait();
    __shared__ uint64_t key[RK_SMALL_N];
    __shared__ uint8_t first[RK_SMALL_N];
    __shared__ unsigned long long red[RK_SMALL_N / 32];
    const int64_t r = blockIdx.x;
    const int i = threadIdx.x, nn = (int)n;
    bool bad = false;
    uint64_t ki = ~0ull;
    if (i < nn) {
        const T v = x[r * ldx + i];
        bad = v != v;
        ki = order_key(v);
        key[i] = ki;
    }
    if (__syncthreads_or(bad) && i == 0) atomicOr(flags, 1);
    int eq_before = 0;
    if (i < nn)
        for (int j = 0; j < i; ++j) eq_before += key[j] == ki;
    first[i] = (i < nn && eq_before == 0) ? 1 : 0;
    __syncthreads();
    if (i < nn) {
        int less = 0;
        for (int j = 0; j < nn; ++j) less += (key[j] < ki) & first[j];
        R[r * ldr + i] = (uint16_t)less;
    }
    unsigned long long ties = (unsigned long long)eq_before;
    for (int o = 16; o > 0; o >>= 1) ties += __shfl_xor_sync(0xffffffffu, ties, o);
    if ((i & 31) == 0) red[i >> 5] = ties;
    __syncthreads();
    if (i == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < RK_SMALL_N / 32; ++w) t += red[w];
        n1[r] = t;
    }
    for (int64_t k = nn + i; k < ldr; k += RK_SMALL_N) R[r * ldr + k] = 0;
    pdl_trigger();
}

template <typename T>
static int launch_rank_warp(const T* x, int64_t m, int64_t n, int64_t ldx, uint16_t* R, int64_t ldr,
                            unsigned long long* n1, int32_t* flags, int Np, cudaStream_t st) {
    const unsigned grid = (unsigned)((m + 7) / 8);
    int only_marked = 0;
    if constexpr (std::is_same<T, int32_t>::value) {  // histogram pass first; the sort takes the rest
        only_marked = 1;
#define TB_RK_HIST(E) TB_CUDA_TRY(launch_pdl(rank_rows_hist_kernel<E>, dim3(grid), dim3(256), 0, st, x, m, n, ldx, R, ldr, n1)); break
        switch (Np / 32) {
            case 1: TB_RK_HIST(1);
            case 2: TB_RK_HIST(2);
            case 4: TB_RK_HIST(4);
            case 8: TB_RK_HIST(8);
            case 16: TB_RK_HIST(16);
            case 32: TB_RK_HIST(32);
            default: return fail(TB_ERR_CONFIG, "rank_rows: bad warp sort size");
        }
#undef TB_RK_HIST
        int rc = check_launch("rank_rows_hist_kernel");
        if (rc) return rc;
    }
#define TB_RK_WARP(E) TB_CUDA_TRY(launch_pdl(rank_rows_warp_kernel<T, E>, dim3(grid), dim3(256), 0, st, x, m, n, ldx, R, ldr, n1, flags, only_marked)); break
    switch (Np / 32) {
        case 1: TB_RK_WARP(1);
        case 2: TB_RK_WARP(2);
        case 4: TB_RK_WARP(4);
        case 8: TB_RK_WARP(8);
        case 16: TB_RK_WARP(16);
        case 32: TB_RK_WARP(32);
        default: return fail(TB_ERR_CONFIG, "rank_rows: bad warp sort size");
    }
#undef TB_RK_WARP
    return check_launch("rank_rows_warp_kernel");
}

}  // namespace tb

using namespace tb;

extern "C" int tb_rank_rows(const void* x, int dtype, int64_t m, int64_t n, int64_t ldx, uint16_t* R, int64_t ldr,
                            uint64_t* n1, int32_t* flags, void* stream) {
    if (m < 1 || n < 1) return fail(TB_ERR_INVALID, "rank_rows: empty input");
    if (n > RK_MAX_N) return fail(TB_ERR_CAPACITY, "rank_rows: n=%lld exceeds %d", (long long)n, RK_MAX_N);
    if (ldx < n || ldr < n || (ldr & 7)) return fail(TB_ERR_CONFIG, "rank_rows: bad leading dimensions");
    if (!x || !R || !n1 || !flags) return fail(TB_ERR_INVALID, "rank_rows: null pointer");
    if (m > INT32_MAX) return fail(TB_ERR_CAPACITY, "rank_rows: m too large");
    int Np = 1;
    while (Np < n) Np <<= 1;
    const size_t smem = (size_t)Np * (8 + 2 + 2);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto* n1u = reinterpret_cast<unsigned long long*>(n1);
    if (n <= RK_SMALL_N) {  // short rows: O(n^2) per-row ranks, one thread per element
        switch (dtype) {
            case TB_DTYPE_I32:
                TB_CUDA_TRY(launch_pdl(rank_rows_small_kernel<int32_t>, dim3((unsigned)m), dim3(RK_SMALL_N), 0, st, (const int32_t*)x, n, ldx, R, ldr, n1u, flags));
                break;
            case TB_DTYPE_F32:
                TB_CUDA_TRY(launch_pdl(rank_rows_small_kernel<float>, dim3((unsigned)m), dim3(RK_SMALL_N), 0, st, (const float*)x, n, ldx, R, ldr, n1u, flags));
                break;
            case TB_DTYPE_F64:
                TB_CUDA_TRY(launch_pdl(rank_rows_small_kernel<double>, dim3((unsigned)m), dim3(RK_SMALL_N), 0, st, (const double*)x, n, ldx, R, ldr, n1u, flags));
                break;
            default:
                return fail(TB_ERR_INVALID, "rank_rows: unknown dtype %d", dtype);
        }
        return check_launch("rank_rows_small_kernel");
    }
    if (Np <= 1024 && dtype != TB_DTYPE_F64) {  // 32-bit keys: warp-per-row register sort
        if (Np < 32) Np = 32;
        if (dtype == TB_DTYPE_I32) return launch_rank_warp((const int32_t*)x, m, n, ldx, R, ldr, n1u, flags, Np, st);
        return launch_rank_warp((const float*)x, m, n, ldx, R, ldr, n1u, flags, Np, st);
    }
    switch (dtype) {
        case TB_DTYPE_I32:
            cudaFuncSetAttribute(rank_rows_kernel<int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            TB_CUDA_TRY(launch_pdl(rank_rows_kernel<int32_t>, dim3((unsigned)m), dim3(RK_THREADS), smem, st, (const int32_t*)x, n, ldx, R, ldr, reinterpret_cast<unsigned long long*>(n1), flags, Np));
            break;
        case TB_DTYPE_F32:
            cudaFuncSetAttribute(rank_rows_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            TB_CUDA_TRY(launch_pdl(rank_rows_kernel<float>, dim3((unsigned)m), dim3(RK_THREADS), smem, st, (const float*)x, n, ldx, R, ldr, reinterpret_cast<unsigned long long*>(n1), flags, Np));
            break;
        case TB_DTYPE_F64:
            cudaFuncSetAttribute(rank_rows_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            TB_CUDA_TRY(launch_pdl(rank_rows_kernel<double>, dim3((unsigned)m), dim3(RK_THREADS), smem, st, (const double*)x, n, ldx, R, ldr, reinterpret_cast<unsigned long long*>(n1), flags, Np));
            break;
        default:
            return fail(TB_ERR_INVALID, "rank_rows: unknown dtype %d", dtype);
    }
    return check_launch("rank_rows_kernel");
}

// ------------------------------------------------------------------ K0w: dense ranks for any n (f4)
// rank_transform (ranks.py:37-61) for rows too wide for K0's shared-memory sort (the merge path, n up
// to 65536 and beyond): one 1024-thread CTA per row (persistent over rows), a stable LSD radix sort of
// the row's (order key, index) pairs with 8-bit digits through a per-CTA global scratch (L2 / HBM
// ping-pong; 32-bit keys for int32 / float32 take 4 passes, float64 keys 8; a pass whose digit is the
// same for every element is skipped), then one block scan over "new value" flags gives the dense ranks
// (int32, the merge path's K1 input) and a max-scan of run starts gives n1 = sum_i (i - runstart(i)) =
// sum_t t(t-1)/2 (kernel_sorted.py:163-176).  -0.0 == +0.0, +-inf orderable, NaN flagged (bit 0).
// Stability: warp w owns the contiguous index segment w; a digit's output offsets are warp-major and
// inside a warp's 32-element step __match_any_sync ranks equal digits by lane (= index) order.
namespace tb {
constexpr int RW_THREADS = 1024;
constexpr int RW_WARPS = RW_THREADS / 32;

template <typename K>
__device__ __forceinline__ K rw_key(int32_t v) { return (K)order_key(v); }
template <typename K>
__device__ __forceinline__ K rw_key(float v) { return (K)order_key(v); }
template <typename K>
__device__ __forceinline__ K rw_key(double v) { return (K)order_key(v); }

// block-wide exclusive scan of one 64-bit value per thread (RW_THREADS threads); returns the total too
__device__ __forceinline__ long long rw_exscan(long long v, long long* wsm, long long& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long s = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += t;
    }
    if (lane == 31) wsm[w] = s;
    __syncthreads();
    if (w == 0) {
        long long a = wsm[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, a, o);
            if (lane >= o) a += t;
        }
        wsm[lane] = a;  // inclusive per-warp prefix
    }
    __syncthreads();
    total = wsm[RW_WARPS - 1];
    const long long r = (w ? wsm[w - 1] : 0) + s - v;
    __syncthreads();
    return r;
}

// block-wide exclusive max-scan (identity -1)
__device__ __forceinline__ long long rw_exmax(long long v, long long* wsm) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long s = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s = max(s, t);
    }
    if (lane == 31) wsm[w] = s;
    __syncthreads();
    if (w == 0) {
        long long a = wsm[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, a, o);
            if (lane >= o) a = max(a, t);
        }
        wsm[lane] = a;
    }
    __syncthreads();
    long long prev = __shfl_up_sync(0xffffffffu, s, 1);
    if (lane == 0) prev = -1;
    const long long r = max(w ? wsm[w - 1] : -1LL, prev);
    __syncthreads();
    return r;
}

template <typename T, typename K, typename RT>
__global__ void __launch_bounds__(RW_THREADS, 1) rank_wide_kernel(const T* __restrict__ x, int64_t m, int64_t n,
                                                                  int64_t ldx, RT* __restrict__ R, int64_t ldr,
                                                                  unsigned long long* __restrict__ n1,
                                                                  int32_t* __restrict__ flags, K* __restrict__ kws,
                                                                  uint32_t* __restrict__ iws) {
    pdl_wait();
    __shared__ uint32_t hist[RW_WARPS][256];
    __shared__ uint32_t tot[256];
    __shared__ long long wsm[RW_WARPS];
    __shared__ int skip;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    K* ka0 = kws + (int64_t)blockIdx.x * 2 * n;
    uint32_t* ia0 = iws + (int64_t)blockIdx.x * 2 * n;
    const int64_t seg = (n + RW_WARPS - 1) / RW_WARPS;
    const int64_t s0 = min(n, (int64_t)w * seg), s1 = min(n, s0 + seg);
    for (int64_t row = blockIdx.x; row < m; row += gridDim.x) {
        K* ka = ka0;
        K* kb = ka0 + n;
        uint32_t* ia = ia0;
        uint32_t* ib = ia0 + n;
        bool bad = false;
        for (int64_t i = tid; i < n; i += RW_THREADS) {
            const T v = x[row * ldx + i];
            bad |= (v != v);
            ka[i] = rw_key<K>(v);
            ia[i] = (uint32_t)i;
        }
        if (__syncthreads_or(bad) && tid == 0) atomicOr(flags, 1);
        for (int pass = 0; pass < (int)sizeof(K); ++pass) {
            const int shift = 8 * pass;
            for (int d = lane; d < 256; d += 32) hist[w][d] = 0;
            __syncwarp();
            for (int64_t i = s0 + lane; i < s1; i += 32) atomicAdd(&hist[w][(uint32_t)(ka[i] >> shift) & 255u], 1u);
            __syncthreads();
            if (tid < 256) {  // per digit: warp-major exclusive offsets, digit total
                uint32_t acc = 0;
                for (int ww = 0; ww < RW_WARPS; ++ww) {
                    const uint32_t c = hist[ww][tid];
                    hist[ww][tid] = acc;
                    acc += c;
                }
                tot[tid] = acc;
            }
            if (tid == 0) skip = 0;
            __syncthreads();
            if (tid < 256 && tot[tid] == (uint32_t)n) skip = 1;  // every element has this digit
            // exclusive scan of the digit totals (256 values; threads >= 256 contribute 0)
            long long total;
            const long long base = rw_exscan(tid < 256 ? (long long)tot[tid] : 0LL, wsm, total);
            if (skip) continue;  // uniform: skip was written before rw_exscan's barriers
            if (tid < 256)
                for (int ww = 0; ww < RW_WARPS; ++ww) hist[ww][tid] += (uint32_t)base;
            __syncthreads();
            for (int64_t b = s0; b < s1; b += 32) {
                const int64_t i = b + lane;
                const bool act = i < s1;
                const unsigned mask = __ballot_sync(0xffffffffu, act);
                if (act) {
                    const K k = ka[i];
                    const uint32_t id = ia[i];
                    const uint32_t d = (uint32_t)(k >> shift) & 255u;
                    const unsigned peers = __match_any_sync(mask, d);
                    const uint32_t pos = hist[w][d] + __popc(peers & lt);
                    __syncwarp(mask);
                    if ((peers & lt) == 0) hist[w][d] += __popc(peers);  // lowest lane of the digit group
                    kb[pos] = k;
                    ib[pos] = id;
                }
                __syncwarp();
            }
            __syncthreads();
            K* tk = ka; ka = kb; kb = tk;
            uint32_t* ti = ia; ia = ib; ib = ti;
        }
        // dense ranks and n1 from the sorted keys: thread t owns the contiguous chunk [c0, c1)
        const int64_t chunk = (n + RW_THREADS - 1) / RW_THREADS;
        const int64_t c0 = min(n, (int64_t)tid * chunk), c1 = min(n, c0 + chunk);
        long long cnt = 0, last_start = -1;
        for (int64_t i = c0; i < c1; ++i)
            if (i == 0 || ka[i] != ka[i - 1]) { ++cnt; last_start = i; }
        long long total;
        long long rank = rw_exscan(cnt, wsm, total) - 1;  // rank of the element before c0
        long long start = rw_exmax(last_start, wsm);      // run start in force at c0
        unsigned long long ties = 0;
        for (int64_t i = c0; i < c1; ++i) {
            if (i == 0 || ka[i] != ka[i - 1]) { ++rank; start = i; }
            ties += (unsigned long long)(i - start);
            R[row * ldr + ia[i]] = (RT)rank;
        }
        // block reduction of ties
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ties += __shfl_down_sync(0xffffffffu, ties, o);
        if (lane == 0) wsm[w] = (long long)ties;
        __syncthreads();
        if (tid == 0) {
            unsigned long long t = 0;
            for (int ww = 0; ww < RW_WARPS; ++ww) t += (unsigned long long)wsm[ww];
            n1[row] = t;
        }
        if (sizeof(RT) == 2)  // uint16 rows for the sign pack: zero the tail up to ldr (tb_rank_rows' contract)
            for (int64_t i = n + tid; i < ldr; i += RW_THREADS) R[row * ldr + i] = 0;
        __syncthreads();
    }
    pdl_trigger();
}

static int64_t rank_wide_grid(int64_t m) { return std::max<int64_t>(1, std::min<int64_t>(m, num_sms())); }
static int64_t rank_wide_keybytes(int dtype) { return dtype == TB_DTYPE_F64 ? 8 : 4; }
}  // namespace tb

extern "C" int64_t tb_rank_dense_workspace(int64_t m, int64_t n, int dtype) {
    if (m < 1 || n < 1) return 0;
    const int64_t per = 2 * n * (rank_wide_keybytes(dtype) + 4);
    return rank_wide_grid(m) * per + 256;
}

extern "C" int tb_rank_dense(const void* x, int dtype, int64_t m, int64_t n, int64_t ldx, void* R, int r_u16,
                             int64_t ldr, uint64_t* n1, int32_t* flags, void* workspace, int64_t ws_bytes,
                             void* stream) {
    if (m < 1 || n < 1) return fail(TB_ERR_INVALID, "rank_dense: empty input");
    if (n > INT32_MAX) return fail(TB_ERR_CAPACITY, "rank_dense: n=%lld too large", (long long)n);
    if (r_u16 && n > 65536) return fail(TB_ERR_CAPACITY, "rank_dense: uint16 ranks need n <= 65536");
    if (ldx < n || ldr < n) return fail(TB_ERR_CONFIG, "rank_dense: bad leading dimensions");
    if (!x || !R || !n1 || !flags || !workspace) return fail(TB_ERR_INVALID, "rank_dense: null pointer");
    if (dtype < TB_DTYPE_I32 || dtype > TB_DTYPE_F64) return fail(TB_ERR_INVALID, "rank_dense: unknown dtype %d", dtype);
    if (ws_bytes < tb_rank_dense_workspace(m, n, dtype))
        return fail(TB_ERR_CONFIG, "rank_dense: workspace of %lld bytes, need %lld", (long long)ws_bytes,
                    (long long)tb_rank_dense_workspace(m, n, dtype));
    const int64_t grid = rank_wide_grid(m);
    const int64_t kb = rank_wide_keybytes(dtype);
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    const uintptr_t a = (reinterpret_cast<uintptr_t>(ws) + 15) & ~uintptr_t(15);
    ws = reinterpret_cast<uint8_t*>(a);
    uint32_t* iws = reinterpret_cast<uint32_t*>(ws + grid * 2 * n * kb);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto* n1u = reinterpret_cast<unsigned long long*>(n1);
    auto go = [&](auto* rout) -> cudaError_t {
        using RT = std::remove_pointer_t<decltype(rout)>;
        switch (dtype) {
            case TB_DTYPE_I32:
                return launch_pdl(rank_wide_kernel<int32_t, uint32_t, RT>, dim3((unsigned)grid), dim3(RW_THREADS), 0, st,
                                  (const int32_t*)x, m, n, ldx, rout, ldr, n1u, flags, reinterpret_cast<uint32_t*>(ws), iws);
            case TB_DTYPE_F32:
                return launch_pdl(rank_wide_kernel<float, uint32_t, RT>, dim3((unsigned)grid), dim3(RW_THREADS), 0, st,
                                  (const float*)x, m, n, ldx, rout, ldr, n1u, flags, reinterpret_cast<uint32_t*>(ws), iws);
            default:
                return launch_pdl(rank_wide_kernel<double, uint64_t, RT>, dim3((unsigned)grid), dim3(RW_THREADS), 0, st,
                                  (const double*)x, m, n, ldx, rout, ldr, n1u, flags, reinterpret_cast<uint64_t*>(ws), iws);
        }
    };
    if (r_u16) TB_CUDA_TRY(go(static_cast<uint16_t*>(R)));
    else TB_CUDA_TRY(go(static_cast<int32_t*>(R)));
    return check_launch("rank_wide_kernel");
}
