// K1 presort + K4 Knight merge-inversion counts (the large-n path).
//
// Reference: sorted_counts (kernel_sorted.py:195-212) sorts every PAIR
// lexicographically (step 1), scans ties (steps 2, 4) and counts discordant
// pairs while re-sorting by v (step 3).  Knight's observation: step 1 only
// depends on u, so it is done once per VARIABLE here (K1), and per pair only
//
//     n_d = inv(w) - sum_g inv_g(w),   n3 = sum_g ties_g(w),
//     w[p] = rank_v[e]  for the element e at position p of u's order,
//
// remain, where g ranges over u's tie groups (contiguous in u-order) -- pairs
// inside a u-group are never discordant (the reference's lexicographic step 1
// orders them by v).  Any within-group order works, so K1 may place tied
// elements in any order.  SURVEY 8 verified the identity against the oracle.
//
// K4 layout: one CTA of 1024 threads per pair (persistent over job ids);
// w lives in shared memory as uint16 (ranks < n <= 65536).  inv(w) is a
// bottom-up merge sort with merge-path partitioning and the reference's
// counting rule (right element strictly smaller => + unconsumed left length,
// kernel_sorted.py:72-73).  n <= 32768: one block of L = 2^ceil(log2 n) keys
// plus an L-key ping-pong buffer; n > 32768: two sorted halves of 32768 kept
// side by side and their cross inversions counted by a merge-path walk without
// materialising the final merge (192 KiB of shared memory in total).
#include "tb_common.cuh"

namespace tb {

// ===================================================================== K1
constexpr int PS_THREADS = 1024;

__device__ __forceinline__ int64_t block_reduce_sum(int64_t v, int64_t* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    int64_t t = 0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    return t;  // valid in warp 0
}

// One CTA per variable.  work[r, k] = histogram -> exclusive start -> fill cursor.
__global__ void __launch_bounds__(PS_THREADS) presort_kernel(const int32_t* __restrict__ ranks, int64_t n,
                                                             int32_t* __restrict__ pos, int32_t* __restrict__ sorted,
                                                             unsigned long long* __restrict__ n1,
                                                             int32_t* __restrict__ maxgrp, int32_t* __restrict__ work,
                                                             int32_t* __restrict__ flags) {
    __shared__ int64_t red[32];
    __shared__ int32_t chunk_base[PS_THREADS];
    const int64_t r = blockIdx.x;
    const int32_t* rk = ranks + r * n;
    int32_t* cnt = work + r * n;
    int32_t* ps = pos + r * n;
    int32_t* so = sorted + r * n;
    const int tid = threadIdx.x;

    for (int64_t i = tid; i < n; i += PS_THREADS) cnt[i] = 0;
    __syncthreads();
    bool bad = false;
    for (int64_t i = tid; i < n; i += PS_THREADS) {
        int32_t v = rk[i];
        if (v < 0 || v >= n) { bad = true; continue; }
        atomicAdd(&cnt[v], 1);
    }
    if (bad) atomicOr(flags, 2);
    __syncthreads();
    // exclusive scan over cnt[0..n): thread t owns a contiguous chunk
    const int64_t per = (n + PS_THREADS - 1) / PS_THREADS;
    const int64_t c0 = tid * per, c1 = min(c0 + per, n);
    int64_t local = 0, ties = 0;
    int32_t mx = 0;
    for (int64_t i = c0; i < c1; ++i) {
        int32_t c = cnt[i];
        local += c;
        ties += (int64_t)c * (c - 1) / 2;
        mx = max(mx, c);
    }
    // block exclusive scan of `local` (<= n fits int32)
    int32_t v = (int32_t)local;
    int32_t incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        int32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if ((tid & 31) >= o) incl += t;
    }
    if ((tid & 31) == 31) chunk_base[tid >> 5] = incl;
    __syncthreads();
    if (tid < 32) {
        int32_t s = chunk_base[tid];
        int32_t si = s;
        for (int o = 1; o < 32; o <<= 1) {
            int32_t t = __shfl_up_sync(0xffffffffu, si, o);
            if (tid >= o) si += t;
        }
        chunk_base[tid] = si - s;  // exclusive warp offsets
    }
    __syncthreads();
    int32_t run = chunk_base[tid >> 5] + incl - v;
    for (int64_t i = c0; i < c1; ++i) {
        int32_t c = cnt[i];
        for (int32_t k = 0; k < c; ++k) so[run + k] = (int32_t)i;
        cnt[i] = run;  // becomes the fill cursor
        run += c;
    }
    int64_t tsum = block_reduce_sum(ties, red);
    // max group
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __syncthreads();
    if ((tid & 31) == 0) chunk_base[tid >> 5] = mx;
    __syncthreads();
    if (tid == 0) {
        int32_t m2 = 0;
        for (int w = 0; w < PS_THREADS / 32; ++w) m2 = max(m2, chunk_base[w]);
        maxgrp[r] = m2;
        n1[r] = (unsigned long long)tsum;
    }
    __syncthreads();
    for (int64_t i = tid; i < n; i += PS_THREADS) {
        int32_t vr = rk[i];
        if (vr >= 0 && vr < n) ps[i] = atomicAdd(&cnt[vr], 1);
    }
}

// ===================================================================== K4
constexpr int MG_THREADS = 1024;
constexpr int MG_HALF = 32768;  // largest block sorted in shared memory

// Shared-memory key index swizzle: merge-path threads own contiguous output segments, which would
// put every lane of a warp in the same two banks (16-way conflicts).  XOR-ing the low five bits of
// the 32-bit word index with the next five spreads a warp's segments over all 32 banks; the map is
// a bijection on every aligned 64-key block.
__device__ __forceinline__ int sw(int e) {
    const int w = e >> 1;
    return ((w ^ ((w >> 5) & 31)) << 1) | (e & 1);
}

// Branch-free sequential merge of `count` outputs of the runs A = src[s, s+W), B = src[s+W, s+2W)
// starting from (i, j); returns the strict-inversion contribution (kernel_sorted.py:72-73 rule:
// a right element strictly smaller than the left head adds the unconsumed left length).
__device__ __forceinline__ uint32_t merge_seq(const uint16_t* src, uint16_t* dst, int s, int W, int i, int j,
                                              int out0, int count) {
    uint32_t inv = 0;
    uint32_t a = i < W ? src[sw(s + i)] : 0u;
    uint32_t b = j < W ? src[sw(s + W + j)] : 0u;
    for (int o = 0; o < count; ++o) {
        const bool takeA = (j >= W) || ((i < W) && (a <= b));
        dst[sw(out0 + o)] = (uint16_t)(takeA ? a : b);
        inv += takeA ? 0u : (uint32_t)(W - i);
        i += takeA;
        j += !takeA;
        const int idx = takeA ? (s + i) : (s + W + j);
        const bool ok = takeA ? (i < W) : (j < W);
        const uint32_t v = ok ? src[sw(idx)] : 0u;
        a = takeA ? v : a;
        b = takeA ? b : v;
    }
    return inv;
}

// Merge sort keys[0, L) (L power of two) with ping-pong buffer tmp[0, L), returning this thread's
// share of the strict inversion count.  Result ends in keys.  All indices are logical (swizzled).
__device__ uint32_t sort_count_block(uint16_t* keys, uint16_t* tmp, int L) {
    uint32_t inv = 0;
    uint16_t* src = keys;
    uint16_t* dst = tmp;
    const int T = MG_THREADS;
    const int E = L >= T ? L / T : 1;            // outputs per thread per level
    const int active = L >= T ? T : L;           // threads with work
    for (int W = 1; W < L; W <<= 1) {
        if (threadIdx.x < active) {
            const int d0 = threadIdx.x * E;
            const int P = 2 * W;
            if (P <= E) {
                for (int s = d0; s < d0 + E; s += P) inv += merge_seq(src, dst, s, W, 0, 0, s, P);
            } else {
                const int s = (d0 / P) * P;  // pair start
                const int d = d0 - s;        // diagonal inside the pair
                int lo = d > W ? d - W : 0, hi = d < W ? d : W;
                while (lo < hi) {  // merge-path search: i = #A among the first d outputs
                    const int mid = (lo + hi) >> 1;
                    if (src[sw(s + mid)] <= src[sw(s + W + d - mid - 1)]) lo = mid + 1;
                    else hi = mid;
                }
                inv += merge_seq(src, dst, s, W, lo, d - lo, s + d, E);
            }
        }
        __syncthreads();
        uint16_t* t = src;
        src = dst;
        dst = t;
    }
    if (src != keys) {
        for (int i = threadIdx.x; i < L; i += T) keys[sw(i)] = src[sw(i)];
        __syncthreads();
    }
    return inv;
}

struct MergeArgs {
    const int32_t* ranks;
    const int32_t* pos;
    const int32_t* sorted;
    const unsigned long long* n1;
    int64_t m, n, n0;
    int64_t job_lo, count;
    int32_t B;       // 1 or 2 blocks
    int32_t L;       // padded block length (power of two)
    int32_t* num;
    unsigned long long* nd;
    unsigned long long* n3;
};

__global__ void __launch_bounds__(MG_THREADS, 1) merge_pairs_kernel(MergeArgs p) {
    extern __shared__ __align__(16) uint8_t mg_smem[];
    uint16_t* keys = reinterpret_cast<uint16_t*>(mg_smem);  // B * L
    uint16_t* tmp = keys + (size_t)p.B * p.L;               // L
    __shared__ int64_t red[32];
    const int tid = threadIdx.x;
    const int64_t n = p.n;
    const int L = p.L;
    const int64_t L1 = p.B == 2 ? L : n;  // real keys in block 0

    for (int64_t idx = blockIdx.x; idx < p.count; idx += gridDim.x) {
        int64_t y, x;
        job_coord(p.job_lo + idx, p.m, y, x);
        const int32_t* pu = p.pos + y * n;      // u-order positions
        const int32_t* su = p.sorted + y * n;   // u ranks in u-order
        const int32_t* rv = p.ranks + x * n;    // v ranks

        // pads (max key) first, then scatter w[pos_u[e]] = rank_v[e]
        for (int64_t i = n + tid; i < (int64_t)p.B * L; i += MG_THREADS) keys[sw((int)i)] = 0xFFFF;
        for (int64_t e = tid; e < n; e += MG_THREADS) keys[sw(pu[e])] = (uint16_t)rv[e];
        __syncthreads();

        // within-u-group pairs: inv_g and joint ties (n3)
        uint32_t inv_g = 0, ties = 0;
        for (int64_t q = tid; q + 1 < n; q += MG_THREADS) {
            const int32_t g = su[q];
            if (su[q + 1] != g) continue;
            const uint16_t wq = keys[sw((int)q)];
            for (int64_t t = q + 1; t < n && su[t] == g; ++t) {
                const uint16_t wt = keys[sw((int)t)];
                inv_g += (wq > wt);
                ties += (wq == wt);
            }
        }
        __syncthreads();

        // inv(w)
        uint32_t inv = sort_count_block(keys, tmp, L);
        if (p.B == 2) {
            inv += sort_count_block(keys + L, tmp, L);  // L >= 64 here: swizzle blocks stay aligned
            // cross inversions: for each b in block 1, # of block-0 keys > b
            const int64_t L2 = n - L1;
            const int64_t per = (L2 + MG_THREADS - 1) / MG_THREADS;
            const int64_t b0 = tid * per, b1 = min(b0 + per, L2);
            if (b0 < b1) {
                const uint16_t* H1 = keys;
                const uint16_t* H2 = keys + L;
                uint16_t b = H2[sw((int)b0)];
                int64_t lo = 0, hi = L1;  // upper_bound(H1, b)
                while (lo < hi) {
                    int64_t mid = (lo + hi) >> 1;
                    if (H1[sw((int)mid)] <= b) lo = mid + 1;
                    else hi = mid;
                }
                int64_t ub = lo;
                for (int64_t k = b0; k < b1; ++k) {
                    b = H2[sw((int)k)];
                    while (ub < L1 && H1[sw((int)ub)] <= b) ++ub;
                    inv += (uint32_t)(L1 - ub);
                }
            }
        }

        const int64_t tot_inv = block_reduce_sum((int64_t)inv, red);
        const int64_t tot_g = block_reduce_sum((int64_t)inv_g, red);
        const int64_t tot_t = block_reduce_sum((int64_t)ties, red);
        if (tid == 0) {
            const int64_t nd = tot_inv - tot_g;
            const int64_t n3 = tot_t;
            const int64_t num = p.n0 - (int64_t)p.n1[y] - (int64_t)p.n1[x] + n3 - 2 * nd;  // result.py:42
            p.num[idx] = (int32_t)num;
            if (p.nd) p.nd[idx] = (unsigned long long)nd;
            if (p.n3) p.n3[idx] = (unsigned long long)n3;
        }
        __syncthreads();
    }
}

}  // namespace tb

using namespace tb;

extern "C" int tb_presort(const int32_t* ranks, int64_t m, int64_t n, int32_t* pos, int32_t* sorted, uint64_t* n1,
                          int32_t* maxgrp, int32_t* work, int32_t* flags, void* stream) {
    if (m < 1 || n < 1) return fail(TB_ERR_INVALID, "presort: empty input");
    if (n > TB_MAX_N) return fail(TB_ERR_CAPACITY, "presort: n=%lld exceeds %d", (long long)n, TB_MAX_N);
    if (!ranks || !pos || !sorted || !n1 || !maxgrp || !work || !flags)
        return fail(TB_ERR_INVALID, "presort: null pointer");
    if (m > INT32_MAX) return fail(TB_ERR_CAPACITY, "presort: m too large");
    presort_kernel<<<(unsigned)m, PS_THREADS, 0, static_cast<cudaStream_t>(stream)>>>(
        ranks, n, pos, sorted, reinterpret_cast<unsigned long long*>(n1), maxgrp, work, flags);
    return check_launch("presort_kernel");
}

extern "C" int tb_merge_pairs(const int32_t* ranks, const int32_t* pos, const int32_t* sorted,
                              const uint64_t* n1_rows, const int32_t* maxgrp, int64_t m, int64_t n, int64_t job_lo,
                              int64_t job_hi, int32_t* num, uint64_t* nd, uint64_t* n3, void* stream) {
    (void)maxgrp;
    if (m < 1 || n < 2) return fail(TB_ERR_INVALID, "merge: need m >= 1 and n >= 2");
    if (n > TB_MAX_N) return fail(TB_ERR_CAPACITY, "merge: n=%lld exceeds %d", (long long)n, TB_MAX_N);
    const int64_t total = m * (m + 1) / 2;
    if (job_lo < 0 || job_hi < job_lo || job_hi > total) return fail(TB_ERR_CONFIG, "merge: bad job range");
    if (!ranks || !pos || !sorted || !n1_rows || !num) return fail(TB_ERR_INVALID, "merge: null pointer");
    if (job_hi == job_lo) return TB_OK;
    MergeArgs a{};
    a.ranks = ranks;
    a.pos = pos;
    a.sorted = sorted;
    a.n1 = reinterpret_cast<const unsigned long long*>(n1_rows);
    a.m = m;
    a.n = n;
    a.n0 = n * (n - 1) / 2;
    a.job_lo = job_lo;
    a.count = job_hi - job_lo;
    a.B = n > MG_HALF ? 2 : 1;
    int64_t per = (n + a.B - 1) / a.B;
    int L = 1;
    while (L < per) L <<= 1;
    a.L = L;
    a.num = num;
    a.nd = reinterpret_cast<unsigned long long*>(nd);
    a.n3 = reinterpret_cast<unsigned long long*>(n3);
    size_t smem = (size_t)(a.B + 1) * L * sizeof(uint16_t);
    TB_CUDA_TRY(cudaFuncSetAttribute(merge_pairs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t grid = std::min<int64_t>(a.count, (int64_t)num_sms());
    merge_pairs_kernel<<<(unsigned)grid, MG_THREADS, smem, static_cast<cudaStream_t>(stream)>>>(a);
    return check_launch("merge_pairs_kernel");
}
