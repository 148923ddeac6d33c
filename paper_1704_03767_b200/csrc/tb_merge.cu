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
// w lives in shared memory as uint16 keys.  The keys are MIN-RANKS (competition
// ranks: key = # elements of the row with a strictly smaller rank, < n <= 65536),
// which order and tie exactly like dense ranks.  inv(w) is a bottom-up merge sort
// with merge-path partitioning and the reference's counting rule (right element
// strictly smaller => + unconsumed left length, kernel_sorted.py:72-73).
// n <= 32768: one block of L = 2^ceil(log2 n) keys plus an L-key ping-pong
// buffer; n > 32768: two halves H1 = w[0, 32768), H2 = the rest, each sorted
// with its own count (192 KiB of shared memory in total).  Their cross
// inversions need no merge: with min-rank keys every a in H1 has exactly
// key(a) smaller keys in the whole row, so
//     sum_{a in H1} key(a) = #{(a, a') in H1^2 : a' < a} + cross(H1, H2)
//                          = L1 (L1 - 1) / 2 - ties(H1) + cross(H1, H2),
// and cross = sum key(H1) - L1 (L1 - 1) / 2 + ties(H1), ties(H1) being the
// equal-key pairs inside H1 (a scan of sorted H1).
#include <cstdlib>

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

// One CTA per variable.  work[r, k] = histogram -> exclusive start -> fill cursor.  The exclusive
// start of an element's rank is its min-rank: keys[r, e].
__global__ void __launch_bounds__(PS_THREADS) presort_kernel(const int32_t* __restrict__ ranks, int64_t n,
                                                             int32_t* __restrict__ pos, int32_t* __restrict__ sorted,
                                                             uint16_t* __restrict__ keys,
                                                             unsigned long long* __restrict__ n1,
                                                             int32_t* __restrict__ maxgrp, int32_t* __restrict__ work,
                                                             int32_t* __restrict__ flags) {
    pdl_wait();
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
    uint16_t* ky = keys + r * n;
    for (int64_t i = tid; i < n; i += PS_THREADS) {
        int32_t vr = rk[i];
        ky[i] = (vr >= 0 && vr < n) ? (uint16_t)cnt[vr] : (uint16_t)0;
    }
    __syncthreads();
    for (int64_t i = tid; i < n; i += PS_THREADS) {
        int32_t vr = rk[i];
        if (vr >= 0 && vr < n) ps[i] = atomicAdd(&cnt[vr], 1);
    }
    pdl_trigger();
}

// Compact tie-group list per variable: groups[r, 2k] = first u-order position, groups[r, 2k+1] =
// length, for every rank value held by >= 2 observations (order of k arbitrary); ngroups[r] = count.
__global__ void __launch_bounds__(256) tie_groups_kernel(const int32_t* __restrict__ sorted, int64_t n,
                                                         int32_t* __restrict__ groups,
                                                         int32_t* __restrict__ ngroups) {
    pdl_wait();
    const int64_t r = blockIdx.x;
    const int32_t* so = sorted + r * n;
    int32_t* gr = groups + r * n;
    __shared__ int32_t cnt;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    for (int64_t p = threadIdx.x; p + 1 < n; p += blockDim.x) {
        const int32_t v = so[p];
        if ((p == 0 || so[p - 1] != v) && so[p + 1] == v) {
            int64_t lo = p + 1, hi = n;  // first position with a larger rank
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (so[mid] == v) lo = mid + 1;
                else hi = mid;
            }
            const int32_t k = atomicAdd(&cnt, 1);
            gr[2 * k] = (int32_t)p;
            gr[2 * k + 1] = (int32_t)(lo - p);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) ngroups[r] = cnt;
    pdl_trigger();
}

// ===================================================================== K4
constexpr int MG_THREADS = 1024;
constexpr int MG_SMALL_GROUP = 64;  // tie groups up to this size: one thread per group
constexpr int MG_HALF = 32768;  // largest block sorted in shared memory
#ifndef MG_PAD_SHIFT  // pad-block size 2^MG_PAD_SHIFT keys (config 4 with 64-output in-place merges: 32 -> 292.6 ms,
#define MG_PAD_SHIFT 6  // 64 -> 278 ms kernel: a 64-output segment is one padded block, 33-word stride, no store conflicts)
#endif

// Shared-memory key layout: 2 pad keys (one 32-bit word) after every 32 keys.  The pad word in front
// of 32-key block k doubles as the merge loop's look-ahead slot (merge_level_cur): its first key holds
// INF (0xFFFF) when block k starts a run of the level being merged, else a copy of the block's first
// key.  Data keys stay <= 0xFFFE (pads of a short row are 0xFFFE; key 65535 is clamped, see K4).  Merge-path threads
// own contiguous output segments, so a warp's cursors sit ~16 keys apart; the padding spreads them
// (and the per-thread 16-word runs of load_run/store_words, 17 words apart) over all 32 banks.
// Logical key e lives at padded index e + 2 (e >> 5); word w at w + (w >> 4).
constexpr int PBS = MG_PAD_SHIFT;  // log2 of the keys per padded block
constexpr int PB = 1 << PBS;        // keys per padded block (2 pad keys = one word after each)
__device__ __forceinline__ int sw(int e) { return e + ((e >> PBS) << 1); }
__device__ __forceinline__ int swp_words(int w) { return w + (w >> (PBS - 1)); }

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

// ---------------------------------------------------------------------------------------------
// K4 sort-and-count.  Thread t owns keys [E t, E t + E) of the block.
//
// The leaf (reg_sort_count) sorts the thread's E keys in registers with tagged composites -- odd-even
// merge levels for runs up to E, then (E = 32) two cross-lane bitonic levels over groups of 4 lanes
// (runs of 128) -- and counts each level's inversions from the positions of the right-run elements:
// inv(A, B) = h^2 + h(h-1)/2 - sum(positions of B elements)   (h = run length).
//
// The remaining levels are merge-path merges: each thread merges its E outputs into
// registers (statically indexed, fully unrolled) counting the reference's way (right element
// strictly smaller => + unconsumed left length, kernel_sorted.py:72-73), then writes them back.
//
// Shared-memory traffic of a thread's E keys uses 32-bit words at swizzled addresses: the thread's
// E/2 words are w = (E/2) t + q and the swizzle (sw, above) makes each of those loads/stores
// conflict-free across a warp.  E/2 <= 16 words never leave the 16-word swizzle row of word
// (E/2) t, so their padded indices are swp_words((E/2) t) + q: one base per thread.
template <int E>
__device__ __forceinline__ const uint32_t* run_words(const uint16_t* keys, int t) {
    static_assert(E / 2 <= PB / 2 || (E / 2) % (PB / 2) == 0, "whole swizzle rows per thread");
    return reinterpret_cast<const uint32_t*>(keys) + swp_words((E / 2) * t);
}
// padded offset of the thread's word q from run_words (E = 64 spans two swizzle rows: one pad word between)
__device__ __forceinline__ constexpr int run_word_off(int q) { return q + q / (PB / 2); }
template <int E>
__device__ __forceinline__ void load_run(const uint16_t* keys, int t, uint32_t (&v)[E]) {
    const uint32_t* wk = run_words<E>(keys, t);
#pragma unroll
    for (int q = 0; q < E / 2; ++q) {
        const uint32_t word = wk[q];
        v[2 * q] = word & 0xFFFFu;
        v[2 * q + 1] = word >> 16;
    }
}
template <int E>
__device__ __forceinline__ void store_words(uint16_t* keys, int t, const uint32_t (&ow)[E / 2]) {
    uint32_t* wk = const_cast<uint32_t*>(run_words<E>(keys, t));
#pragma unroll
    for (int q = 0; q < E / 2; ++q) wk[run_word_off(q)] = ow[q];
}
template <int E>
__device__ __forceinline__ void store_run(uint16_t* keys, int t, const uint32_t (&v)[E]) {
    uint32_t* wk = const_cast<uint32_t*>(run_words<E>(keys, t));
#pragma unroll
    for (int q = 0; q < E / 2; ++q) wk[q] = (v[2 * q] & 0xFFFFu) | (v[2 * q + 1] << 16);
}

// Look-ahead slot of the 32-key block starting at key E t (when one does): INF if that key starts a run of
// length R (the next level's run length), else a copy of the key (first = the thread's first key word).
template <int E>
__device__ __forceinline__ void store_lookahead(uint16_t* keys, int t, int R, uint32_t first) {
    const int k0 = E * t;
    if ((k0 & (PB - 1)) == 0 && k0 > 0) {
        uint32_t* wk = reinterpret_cast<uint32_t*>(keys) + swp_words(k0 >> 1) - 1;
        *wk = (k0 & (R - 1)) == 0 ? 0xFFFFFFFFu : (first | 0xFFFF0000u);
    }
}
// E = 64 segments span two 32-key blocks: both pad words in front of them (first keys from the output words)
template <int E>
__device__ __forceinline__ void store_lookaheads(uint16_t* keys, int t, int R, const uint32_t (&ow)[E / 2]) {
    store_lookahead<E>(keys, t, R, ow[0] & 0xFFFFu);
#pragma unroll
    for (int b = 1; b < E / PB; ++b) {
        const int k0 = E * t + PB * b;
        uint32_t* wk = reinterpret_cast<uint32_t*>(keys) + swp_words(k0 >> 1) - 1;
        *wk = (k0 & (R - 1)) == 0 ? 0xFFFFFFFFu : ((ow[PB / 2 * b] & 0xFFFFu) | 0xFFFF0000u);
    }
}

// Sort v[0..E) ascending (values are 16-bit keys), returning the strict inversion count.
// Composites key << (5 + XL) | g << 5 | i (i = the key's index in the thread's run, E <= 32; g = the
// thread's index in its group of 2^XL lanes) are tagged once: stage k merges the two sorted h-runs
// (h = k / 2) of each aligned k-block, whose elements are exactly those with tags in that block, so an
// element came from the right run B iff bit log2(h) of its tag is set; and a correct sort of the
// composites is a stable merge (A first on ties).  The B element of B-rank j at merged position p has
// h - (p - j) A elements strictly greater: inv(A, B) = h^2 + h(h-1)/2 - sum(positions of B elements).
// XL levels beyond the thread's 32 keys run across the lanes of the group (E = 32): a merged block of
// 32 << l keys spans 2^l lanes, its mirror stage pairs register i of lane g with register 31 - i of
// lane g ^ (2^l - 1) (one xor shuffle), the stages at distances 32 << d (d = l - 2 .. 0) pair lane g with
// g ^ (1 << d), and the remaining stages are the in-register half-cleaners.  Lower lanes keep the minimum.
// Batcher's odd-even merge of the sorted halves of v[LO, LO + N) (stride R): 191 compare-exchanges for a
// 32-key sort against the bitonic network's 240 (the leaf is min/max-bound on the ALU pipe).
__device__ __forceinline__ void cswap(uint32_t& a, uint32_t& b) {
    const uint32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}
// The leaf's networks are min/max only, i.e. all on the ALU pipe (half rate) while the FMA pipe idles.
// cswap_fma takes the maximum as a + b - min(a, b) in two IMADs with opaque multipliers (__constant__, so
// ptxas cannot fold them back into a VIMNMX): one ALU op + two FMA ops instead of two ALU ops.  Every
// MG_ALT_SWAP-th compare-exchange of a stage uses it (0: none).
#ifndef MG_ALT_SWAP  // config 4 kernel: 0 -> 275.2 ms, every 3rd 271.9, every 2nd 270.3, all (1) 263.9 ms
#define MG_ALT_SWAP 1
#endif
#ifndef MG_TAG_FMA  // leaf tags: IMAD / mul.hi instead of SHF + LOP3
#define MG_TAG_FMA 0
#endif
__constant__ uint32_t c_mg_one = 1u;
__constant__ uint32_t c_mg_m1 = 0xFFFFFFFFu;
__device__ __forceinline__ void cswap_fma(uint32_t& a, uint32_t& b) {
    const uint32_t lo = min(a, b);
    uint32_t s, hi;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(s) : "r"(a), "r"(c_mg_one), "r"(b));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(hi) : "r"(lo), "r"(c_mg_m1), "r"(s));
    a = lo;
    b = hi;
}
template <int K>
__device__ __forceinline__ void cswap_k(uint32_t& a, uint32_t& b) {  // K = index of the exchange in its stage
    if constexpr (MG_ALT_SWAP > 0 && K % MG_ALT_SWAP == MG_ALT_SWAP - 1) cswap_fma(a, b);
    else cswap(a, b);
}
template <int I, int IEND, int R, int M, int K, int E>
__device__ __forceinline__ void oe_stage(uint32_t (&v)[E]) {
    if constexpr (I + R < IEND) {
        cswap_k<K>(v[I], v[I + R]);
        oe_stage<I + M, IEND, R, M, K + 1>(v);
    }
}
template <int LO, int N, int R, int E>
__device__ __forceinline__ void oe_merge(uint32_t (&v)[E]) {
    constexpr int M = 2 * R;
    if constexpr (M < N) {
        oe_merge<LO, N, M>(v);
        oe_merge<LO + R, N, M>(v);
        oe_stage<LO + R, LO + N, R, M, 0>(v);
    } else {
        cswap_k<LO / M>(v[LO], v[LO + R]);
    }
}
template <int K, int B, int E>
__device__ __forceinline__ void oe_blocks(uint32_t (&v)[E]) {
    if constexpr (B < E) {
        oe_merge<B, K, 1>(v);
        oe_blocks<K, B + K>(v);
    }
}
// In-register levels k = K .. E: merge the sorted halves of every aligned k-block, then add this
// level's inversions from the tag bit log2(k / 2) (see reg_sort_count).
template <int K, int E>
__device__ __forceinline__ void reg_stages(uint32_t (&v)[E], uint32_t& inv) {
    if constexpr (K <= E) {
        constexpr int h = K / 2;
        oe_blocks<K, 0>(v);
        uint32_t pos = 0;  // h * sum of the B positions
#pragma unroll
        for (int i = 0; i < E; ++i) pos += (v[i] & (uint32_t)h) * (uint32_t)(i % K);
        inv += (uint32_t)(E / K) * (uint32_t)(h * h + h * (h - 1) / 2) - pos / (uint32_t)h;
        reg_stages<2 * K, E>(v, inv);
    }
}

__device__ __forceinline__ uint32_t mnmx(uint32_t a, uint32_t b, bool lower) { return lower ? min(a, b) : max(a, b); }

template <int E, int XL = 0>
__device__ __forceinline__ uint32_t reg_sort_count(uint32_t (&v)[E]) {
    static_assert(E <= 32, "5-bit run index");
    static_assert(XL == 0 || E == 32, "cross-lane levels need full 32-key runs");
    constexpr int TB = 5 + XL;  // tag bits
    const uint32_t g = (uint32_t)(threadIdx.x & ((1 << XL) - 1));
    uint32_t inv = 0;
#pragma unroll
    for (int i = 0; i < E; ++i) {
        if constexpr (MG_TAG_FMA) {  // disjoint bit fields: v * 2^TB + (g << 5 | i) as one IMAD
            uint32_t t;
            asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(v[i]), "r"(c_mg_one << TB), "r"((g << 5) | (uint32_t)i));
            v[i] = t;
        } else {
            v[i] = (v[i] << TB) | (g << 5) | (uint32_t)i;
        }
    }
    reg_stages<2, E>(v, inv);
#pragma unroll
    for (int l = 1; l <= XL; ++l) {  // cross-lane level: blocks of 32 << l keys over 2^l lanes
        const uint32_t gl = g & ((1u << l) - 1);  // lane within the block
        {  // mirror stage: lane gl <-> lane gl ^ (2^l - 1), register i <-> 31 - i
            const bool lower = gl < (1u << (l - 1));
            const int mask = (1 << l) - 1;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const uint32_t a = __shfl_xor_sync(0xffffffffu, v[31 - i], mask);
                const uint32_t b = __shfl_xor_sync(0xffffffffu, v[i], mask);
                v[i] = mnmx(v[i], a, lower);
                v[31 - i] = mnmx(v[31 - i], b, lower);
            }
        }
#pragma unroll
        for (int d = l - 2; d >= 0; --d) {  // distances 32 << d: lane gl <-> gl ^ (1 << d), same register
            const bool lower = (gl & (1u << d)) == 0;
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = mnmx(v[i], __shfl_xor_sync(0xffffffffu, v[i], 1 << d), lower);
        }
#pragma unroll
        for (int j = 16; j > 0; j >>= 1) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                if (i & j) continue;
                if (MG_ALT_SWAP > 0 && (i % MG_ALT_SWAP) == MG_ALT_SWAP - 1) cswap_fma(v[i], v[i + j]);
                else cswap(v[i], v[i + j]);
            }
        }
        // this lane's share of inv(A, B), h = 16 << l: B = tag bit 4 + l; positions 32 gl + i.  Lanes other
        // than the block's first add only -pos: a thread's total can be negative (the kernel reduces it as
        // int32; the block total is exact)
        // one IMAD per key: sum (i + 512) [B] = sum_B i + 512 nbv (sum_B i <= 496), nbv = B keys in this lane
        const uint32_t hb = 16u << l, tb = 1u << (4 + l);
        uint32_t acc = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += (v[i] & tb) * (uint32_t)(i + 512);
        acc /= tb;
        const uint32_t nbv = acc >> 9;
        uint32_t pos = (acc & 511u) + 32u * gl * nbv;
        inv += (gl == 0 ? hb * hb + hb * (hb - 1) / 2 : 0u) - pos;
    }
#pragma unroll
    for (int i = 0; i < E; ++i) {
        if constexpr (MG_TAG_FMA) {  // v >> TB as mul.hi by 2^(32 - TB)
            uint32_t t;
            asm("mul.hi.u32 %0, %1, %2;" : "=r"(t) : "r"(v[i]), "r"(c_mg_one << (32 - TB)));
            v[i] = t;
        } else {
            v[i] >>= TB;
        }
    }
    return inv;
}

// Opaque multipliers (1, -1, 2, 4 read from the kernel arguments) keep the bookkeeping on IMAD: ptxas
// cannot strength-reduce a multiply by an unknown register into ALU shifts / adds.
struct MgConst {
    uint32_t one, m1, two, four, s16, c68, m68, hi6;  // hi6 = 2^(32 - PBS): c >> PBS as mul.hi (FMA pipe)
};
#ifndef MG_LOOP_FMA_MAX  // merge loop: the larger head as h1 + h2 - min in two IMADs instead of a VIMNMX
#define MG_LOOP_FMA_MAX 0
#endif
#ifndef MG_LOOP_HI  // merge loop: the pad term c >> PBS as mul.hi on the FMA pipe instead of SHF on the ALU
#define MG_LOOP_HI 0
#endif
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}

// Merge-path search with IMAD addressing: s and s + W are multiples of 32, so sw(s + x) =
// sw(s) + sw(x) and each probe is base + 2 x + 4 (x >> 5).  Two phases: first over the block starts
// i = 32 j only, where both probes are linear in j (A[32 j] at byte 68 j, B[d - 1 - 32 j] at
// 2 sw(d - 1) - 68 j) -- one IMAD per address; then a plain search of the <= 32-wide bracket.
__device__ __forceinline__ int mp_search(uint32_t baseA, uint32_t baseB, int d, int W, const MgConst& K) {
    const int lo0 = d > W ? d - W : 0, hi0 = d < W ? d : W;
    int jl = (lo0 + PB - 1) >> PBS, jh = (hi0 + PB - 1) >> PBS;  // block starts PB j in [lo0, hi0)
    const uint32_t dm1 = (uint32_t)(d - 1);
    const uint32_t cB = baseB + 2u * (uint32_t)sw(d - 1);
    while (jl < jh) {  // first j whose block start 32 j is not among the first d outputs
        const int mid = (jl + jh) >> 1;
        const uint32_t a = lds_u16(imad((uint32_t)mid, K.c68, baseA));
        const uint32_t b = lds_u16(imad((uint32_t)mid, K.m68, cB));
        if (a <= b) jl = mid + 1;
        else jh = mid;
    }
    int lo = max(lo0, PB * jl - (PB - 1)), hi = min(hi0, PB * jl);
    // probes mid in [lo, hi) lie inside A block jl - 1: byte 2 mid + 4 (jl - 1)
    const uint32_t cA = baseA + 4u * (uint32_t)(jl - 1);
    while (lo < hi) {  // i = #A among the first d outputs
        const int mid = (lo + hi) >> 1;
        const uint32_t x = imad((uint32_t)mid, K.m1, dm1);  // B index d - mid - 1
        const uint32_t a = lds_u16(imad((uint32_t)mid, K.two, cA));
        const uint32_t b = lds_u16(imad(x >> PBS, K.four, imad(x, K.two, baseB)));
        if (a <= b) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// One merge-path level (runs of W -> 2W): thread t merges outputs [d, d + E) of the run pair
// A = src[s, s + W), B = src[s + W, s + 2W) into registers, then stores them as words.
// The two run heads are composites (key << 16 | run), run 0 for A and 1 for B: min(h1, h2) is the next
// output with A first on ties (the reference's order, kernel_sorted.py:72-73), the larger head stays,
// and the low bit says which run's cursor (ia / ib, absolute indices) advances and reloads.  A run
// that is used up (its cursor hits s + W or s + 2W) reads as INF.  A B output adds the unconsumed A
// length s + W - ia, so inv = (#B outputs) (s + W) - sum_B ia.
// The K4 kernel is bound by the B200 integer pipes (ALU: min/max, LOP3, SEL, ISETP, SHF; FMA: IMAD;
// each issues one warp instruction per 2 cycles per SMSP), so the cursor and address arithmetic is
// written as IMADs with opaque multipliers to split the step between the two pipes.
template <int E, bool CHECKED>
__device__ __forceinline__ uint32_t merge_level_regs(const uint16_t* src, int t, int W, const MgConst& K,
                                                     uint32_t (&ow)[E / 2]) {
    const int d0 = t * E;
    const int P = 2 * W;
    const int s = d0 & ~(P - 1);
    const int d = d0 - s;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(src);
    const uint32_t baseA = base + 2u * (uint32_t)sw(s), baseB = base + 2u * (uint32_t)sw(s + W);
    const int lo = mp_search(baseA, baseB, d, W, K);
    constexpr uint32_t INF = 0xFFFF0000u;  // above every data composite (keys <= 0xFFFE)
    const uint32_t sW = (uint32_t)(s + W);
    uint32_t ia = (uint32_t)(s + lo), ib = sW + (uint32_t)(d - lo);
    const uint32_t ib0 = ib;
    uint32_t h1 = ia < sW ? ((uint32_t)src[sw((int)ia)] << 16) : INF;
    uint32_t h2 = ib < sW + (uint32_t)W ? (((uint32_t)src[sw((int)ib)] << 16) | 1u) : INF;
    uint32_t Y = 0, prev = 0;
#pragma unroll
    for (int o = 0; o < E; ++o) {
        const uint32_t cm = min(h1, h2);
        if constexpr (MG_LOOP_FMA_MAX && !CHECKED) h1 = imad(cm, K.m1, imad(h1, K.one, h2));
        else h1 = max(h1, h2);
        if constexpr (CHECKED) {  // runs shorter than a 32-key block: explicit end test
            const uint32_t org = cm & 1u;
            Y = imad(org, ia, Y);
            ia = ia + 1u - org;
            ib = imad(org, K.one, ib);
            if (o + 1 < E) {
                const uint32_t idx = org ? ib : ia;
                const uint32_t addr = imad(idx >> PBS, K.four, imad(idx, K.two, base));
                const uint32_t nv = lds_u16(addr);  // idx <= s + 2W: inside the buffers' 2-key slack
                const uint32_t end = imad(org, (uint32_t)W, sW);
                h2 = idx == end ? INF : imad(nv, K.s16, org);
            }
        } else {
            // W >= 32: every run boundary is a block boundary.  Key idx (idx >= 1) is read at padded
            // index idx + 2 ((idx - 1) >> 5): inside a block that is the key itself; at a block start
            // it is the pad slot in front of the block, which holds a copy of the key -- or INF when
            // idx is the end of the run (the next run's start), so a used-up run reads as INF
            // (composite >= 0xFFFF0000, above every data composite) with no test.  The key after the
            // consumed one is idx = old cursor + 1, i.e. c = idx - 1 = the old cursor of the run
            // taken.  Both cursor advances are predicated IMADs, keeping them off the ALU pipe.
            uint32_t org, c;
            asm("{\n\t.reg .pred p;\n\t"
                "and.b32 %0, %5, 1;\n\t"
                "setp.ne.u32 p, %0, 0;\n\t"
                "mad.lo.u32 %3, %0, %1, %3;\n\t"  // Y += org * ia (ia unchanged by a B output)
                "selp.b32 %4, %2, %1, p;\n\t"      // c = old cursor of the run taken
                "@!p mad.lo.u32 %1, %6, %6, %1;\n\t"
                "@p mad.lo.u32 %2, %6, %6, %2;\n\t"
                "}"
                : "=r"(org), "+r"(ia), "+r"(ib), "+r"(Y), "=r"(c)
                : "r"(cm), "r"(K.one));
            if (o + 1 < E) {
                uint32_t blk;
                if constexpr (MG_LOOP_HI) asm("mul.hi.u32 %0, %1, %2;" : "=r"(blk) : "r"(c), "r"(K.hi6));
                else blk = c >> PBS;
                const uint32_t addr = imad(blk, K.four, imad(c, K.two, base + 2u));
                h2 = imad(lds_u16(addr), K.s16, org);
            }
        }
        if (o & 1) ow[o >> 1] = __byte_perm(prev, cm, 0x7632);  // the two keys (high halves)
        else prev = cm;
    }
    return (ib - ib0) * sW - Y;
}
template <int E, bool CHECKED>
__device__ __forceinline__ uint32_t merge_level_cur(const uint16_t* src, uint16_t* dst, int t, int W,
                                                    const MgConst& K) {
    uint32_t ow[E / 2];
    const uint32_t inv = merge_level_regs<E, CHECKED>(src, t, W, K, ow);
    store_words<E>(dst, t, ow);
    store_lookaheads<E>(dst, t, 2 * W, ow);
    return inv;
}
// Barrier of the threads merging one block: a named barrier (id 1..15) when several blocks of the CTA merge
// side by side -- the two halves of n > 32768, the pairs of merge_multi_kernel -- so a block's threads wait
// only for each other and the blocks' barrier stalls overlap; id 0 = the whole CTA.
#ifndef MG_GROUP_BARRIERS
#define MG_GROUP_BARRIERS 1
#endif
__device__ __forceinline__ void group_sync(int id, int nthreads) {
    if (!MG_GROUP_BARRIERS || id == 0) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// In place: every thread's outputs stay in registers until all threads have read the level's runs.
template <int E>
__device__ __forceinline__ uint32_t merge_level_inplace(uint16_t* blk, int t, int W, const MgConst& K, int bar_id,
                                                        int bar_threads) {
    uint32_t ow[E / 2];
    const uint32_t inv = merge_level_regs<E, false>(blk, t, W, K, ow);
    group_sync(bar_id, bar_threads);
    store_words<E>(blk, t, ow);
    store_lookaheads<E>(blk, t, 2 * W, ow);
    group_sync(bar_id, bar_threads);
    return inv;
}

#ifndef MG_PREFETCH  // L2 prefetch of the next pair's rows (A/B: profiles/r02_merge_ab.log)
#define MG_PREFETCH 0
#endif
#ifndef MG_LEAF_XL  // cross-lane leaf levels for E = 32 (round-1 kernel on config 4: 1 -> 319.5 ms, 2 -> 315.5 ms,
#define MG_LEAF_XL 2  // 3 -> 328.5 ms)
#endif
template <int E>
// register leaf: 32 keys per lane, 32 << MG_LEAF_XL across 2^MG_LEAF_XL lanes
constexpr int LEAF_XL = E == 32 ? MG_LEAF_XL : 0;

template <int E>
__device__ uint32_t sort_count_block_v2(uint16_t* keys, uint16_t* tmp, int L, const MgConst& K) {
    const int t = threadIdx.x;
    const int active = L / E;  // L is a multiple of E
    uint32_t inv = 0;
    if (t < active) {
        uint32_t v[E];
        load_run<E>(keys, t, v);
        inv += reg_sort_count<E, LEAF_XL<E>>(v);
        store_run<E>(keys, t, v);
        store_lookahead<E>(keys, t, E << LEAF_XL<E>, v[0]);  // INF at leaf-run starts, else a key copy
    }
    __syncthreads();
    uint16_t* src = keys;
    uint16_t* dst = tmp;
    for (int W = E << LEAF_XL<E>; W < L; W <<= 1) {
        if (t < active) {
            if (W < PB) inv += merge_level_cur<E, true>(src, dst, t, W, K);
            else inv += merge_level_cur<E, false>(src, dst, t, W, K);
        }
        __syncthreads();
        uint16_t* tt = src;
        src = dst;
        dst = tt;
    }
    if (src != keys) {
        if (t < active) {
            uint32_t v[E];
            load_run<E>(src, t, v);
            store_run<E>(keys, t, v);
        }
        __syncthreads();
    }
    return inv;
}

// n > 32768: both 32768-key halves.  Leaf: all threads, one half after the other (32 keys each).  Merge
// levels: threads [0, 512) merge half 0 and [512, 1024) half 1 concurrently, EM = 64 outputs each, in place
// (no ping-pong buffer): the merge-path search runs once per 64 outputs instead of once per 32.
template <int EM>
__device__ uint32_t sort_count_halves(uint16_t* keys, int L, const MgConst& K) {
    constexpr int E = 32;
    static_assert(EM * MG_THREADS == 2 * MG_HALF, "two halves of EM * 512 keys");
    const int tid = threadIdx.x;
    uint32_t inv = 0;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
        uint16_t* blk = keys + h * sw(L);
        uint32_t v[E];
        load_run<E>(blk, tid, v);
        inv += reg_sort_count<E, LEAF_XL<E>>(v);
        store_run<E>(blk, tid, v);
        store_lookahead<E>(blk, tid, E << LEAF_XL<E>, v[0]);
    }
    __syncthreads();
    uint16_t* blk = keys + (tid >> 9) * sw(L);
    const int t = tid & (MG_THREADS / 2 - 1);
#pragma unroll 1
    for (int W = E << LEAF_XL<E>; W < L; W <<= 1)
        inv += merge_level_inplace<EM>(blk, t, W, K, 1 + (tid >> 9), MG_THREADS / 2);
    __syncthreads();  // the halves ran on their own barriers: the caller reads both sorted halves
    return inv;
}

__device__ __forceinline__ uint32_t sort_count_any(uint16_t* keys, uint16_t* tmp, int L, const MgConst& K) {
    if (L >= 32 * MG_THREADS) return sort_count_block_v2<32>(keys, tmp, L, K);
    if (L >= 16 * MG_THREADS) return sort_count_block_v2<16>(keys, tmp, L, K);
    if (L >= 8 * MG_THREADS) return sort_count_block_v2<8>(keys, tmp, L, K);
    if (L >= 4 * MG_THREADS) return sort_count_block_v2<4>(keys, tmp, L, K);
    if (L >= 2 * MG_THREADS) return sort_count_block_v2<2>(keys, tmp, L, K);
    return sort_count_block(keys, tmp, L);
}


// ------------------------------------------------------------------ large u tie groups
// sum_g inv_g(w) and the joint ties n3 for rows whose largest u tie group exceeds MG_SMALL_GROUP, in
// O(n log n) whatever the tie structure (the reference gets them from its per-pair lexicographic sort,
// kernel_sorted.py:95-127, 179-192).  An MSD radix pass per key bit over segments that start as the u
// groups: within a segment every 1 before a 0 of the current bit is one inversion, then the segment is
// stably partitioned into its 0 part and its 1 part (the next level's segments).  After the last bit the
// segments are the (u group, v key) classes, so n3 = sum_q (q - segment start).  Per element a level
// costs a block scan of the bit and O(1) reads of the scan at q, at the segment start and at its end;
// keys, segment starts and lengths - 1 ping-pong through a per-CTA global scratch (L2-resident), the
// bit prefix E lives there too.
struct HeavyWs {
    uint16_t *keyA, *keyB, *segA, *segB;
    uint16_t *lenA, *lenB;  // segment length - 1 (a segment can hold all 65536 elements)
    int32_t* E;             // exclusive prefix of the level's bit, n + 1 entries
};

__host__ __device__ __forceinline__ int64_t heavy_ws_bytes_per_cta(int64_t n) { return 12 * n + 4 * (n + 1) + 64; }

__device__ __forceinline__ HeavyWs heavy_ws(uint8_t* base, int64_t n) {
    HeavyWs h;
    uint8_t* b = base + (int64_t)blockIdx.x * heavy_ws_bytes_per_cta(n);
    b = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(b) + 15) & ~uintptr_t(15));
    h.E = reinterpret_cast<int32_t*>(b);
    uint16_t* u = reinterpret_cast<uint16_t*>(b + 4 * (n + 1));
    h.keyA = u; h.keyB = u + n;
    h.segA = u + 2 * n; h.segB = u + 3 * n;
    h.lenA = u + 4 * n; h.lenB = u + 5 * n;
    return h;
}

// block exclusive scan of one int per thread (MG_THREADS threads)
__device__ __forceinline__ int32_t mg_exscan(int32_t v, int32_t* wsm) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t s = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t t = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += t;
    }
    if (lane == 31) wsm[w] = s;
    __syncthreads();
    if (w == 0) {
        int32_t a = wsm[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t t = __shfl_up_sync(0xffffffffu, a, o);
            if (lane >= o) a += t;
        }
        wsm[lane] = a;
    }
    __syncthreads();
    const int32_t r = (w ? wsm[w - 1] : 0) + s - v;
    __syncthreads();
    return r;
}

__device__ void heavy_group_counts(const uint16_t* __restrict__ keys, const int32_t* __restrict__ gl, int32_t ng,
                                   int64_t n, HeavyWs h, uint32_t& inv_g, uint32_t& ties) {
    __shared__ int32_t wsm[32];
    const int tid = threadIdx.x;
    const int nn = (int)n;
    uint16_t *K0 = h.keyA, *K1 = h.keyB, *S0 = h.segA, *S1 = h.segB, *L0 = h.lenA, *L1 = h.lenB;
    int32_t* E = h.E;
    for (int q = tid; q < nn; q += MG_THREADS) {
        K0[q] = keys[sw(q)];
        S0[q] = (uint16_t)q;
        L0[q] = 0;
    }
    __syncthreads();
    for (int32_t k = tid; k < ng; k += MG_THREADS) {  // u groups of >= 2 elements (tb_presort's list)
        const int32_t g0 = gl[2 * k], glen = gl[2 * k + 1];
        for (int32_t q = g0; q < g0 + glen; ++q) {
            S0[q] = (uint16_t)g0;
            L0[q] = (uint16_t)(glen - 1);
        }
    }
    __syncthreads();
    const int chunk = (nn + MG_THREADS - 1) / MG_THREADS;
    const int c0 = min(nn, tid * chunk), c1 = min(nn, c0 + chunk);
    int nbits = 0;
    while ((1 << nbits) < nn) ++nbits;
    uint32_t inv = 0;
    for (int bit = nbits - 1; bit >= 0; --bit) {
        int32_t cnt = 0;
        for (int q = c0; q < c1; ++q) cnt += (K0[q] >> bit) & 1;
        int32_t run = mg_exscan(cnt, wsm);
        for (int q = c0; q < c1; ++q) {
            E[q] = run;
            run += (K0[q] >> bit) & 1;
        }
        if (c1 == nn && c0 < c1) E[nn] = run;
        __syncthreads();
        for (int q = c0; q < c1; ++q) {
            const uint16_t k = K0[q];
            const int st = S0[q], ln = (int)L0[q] + 1;
            if (ln == 1) { K1[q] = k; S1[q] = (uint16_t)st; L1[q] = 0; continue; }
            const int b = (k >> bit) & 1;
            const int Es = E[st], Eq = E[q];
            const int ones = E[st + ln] - Es, Z = ln - ones;
            int np, ns, nl;
            if (b == 0) {
                inv += (uint32_t)(Eq - Es);  // ones before q in its segment
                np = q - (Eq - Es);
                ns = st;
                nl = Z;
            } else {
                np = st + Z + (Eq - Es);
                ns = st + Z;
                nl = ones;
            }
            K1[np] = k;
            S1[np] = (uint16_t)ns;
            L1[np] = (uint16_t)(nl - 1);
        }
        __syncthreads();
        uint16_t* t;
        t = K0; K0 = K1; K1 = t;
        t = S0; S0 = S1; S1 = t;
        t = L0; L0 = L1; L1 = t;
    }
    uint32_t tt = 0;
    for (int q = c0; q < c1; ++q) tt += (uint32_t)(q - (int)S0[q]);
    inv_g = inv;
    ties = tt;
    __syncthreads();
}

struct MergeArgs {
    const uint16_t* keys;  // [m, n] min-rank keys (tb_presort)
    const int32_t* pos;
    const int32_t* sorted;
    const int32_t* maxgrp;
    const int32_t* groups;
    const int32_t* ngroups;
    const unsigned long long* n1;
    int64_t m, n, n0;
    int64_t job_lo, count;
    int32_t B;       // 1 or 2 blocks
    int32_t L;       // padded block length (power of two)
    int32_t P;       // merge_multi_kernel: pairs per CTA (65536 / L)
    int32_t* num;
    unsigned long long* nd;
    unsigned long long* n3;
    uint8_t* heavy_ws;  // per-CTA scratch of heavy_group_counts
    MgConst k;  // {1, -1, 2, 4, 65536, 68, -68}
};

// One pair on the whole CTA: B = 1 (n <= 32768) sorts keys with the ping-pong block tmp, B = 2 the two
// 32768-key halves in place plus the closed-form cross term.  Every thread calls it (CTA barriers inside).
__device__ __forceinline__ void merge_one_pair(const MergeArgs& p, int64_t idx, uint16_t* keys, uint16_t* tmp,
                                            int64_t* red, int& sX, int& sY) {
    const int tid = threadIdx.x;
    const int64_t n = p.n;
    const int L = p.L;
    const int64_t L1 = p.B == 2 ? L : n;  // real keys in block 0
    const MgConst K = p.k;
    int64_t y, x;
    job_coord(p.job_lo + idx, p.m, y, x);
    const int32_t* pu = p.pos + y * n;      // u-order positions
    const uint16_t* kv = p.keys + x * n;    // v min-rank keys
#if MG_PREFETCH
    // the next pair's v keys (and u positions when its row changes) into L2 while this pair sorts: the
    // scatter at the top of a pair is the kernel's one latency-bound phase
    if (idx + gridDim.x < p.count) {
        int64_t y2, x2;
        job_coord(p.job_lo + idx + gridDim.x, p.m, y2, x2);
        const char* k2 = reinterpret_cast<const char*>(p.keys + x2 * n);
        for (int64_t b = (int64_t)tid * 128; b < 2 * n; b += (int64_t)MG_THREADS * 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(k2 + b));
        if (y2 != y) {
            const char* p2 = reinterpret_cast<const char*>(p.pos + y2 * n);
            for (int64_t b = (int64_t)tid * 128; b < 4 * n; b += (int64_t)MG_THREADS * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(p2 + b));
        }
    }
#endif

    // pads (0xFFFE: real keys are < n <= 65535 whenever pads exist, and 0xFFFF is the merge
    // loop's INF) first, then scatter w[pos_u[e]] = key_v[e]
    for (int64_t i = n + tid; i < (int64_t)p.B * L; i += MG_THREADS) keys[sw((int)i)] = 0xFFFE;
    if (tid == 0) sX = sY = -1;
    __syncthreads();
    if ((n & 3) == 0) {  // 16-byte loads of u-positions, 8-byte loads of v keys
        const int4* pu4 = reinterpret_cast<const int4*>(pu);
        const uint2* kv4 = reinterpret_cast<const uint2*>(kv);
        for (int64_t e = tid; e < (n >> 2); e += MG_THREADS) {
            const int4 P = pu4[e];
            const uint2 V = kv4[e];
            keys[sw(P.x)] = (uint16_t)(V.x & 0xFFFFu);
            keys[sw(P.y)] = (uint16_t)(V.x >> 16);
            keys[sw(P.z)] = (uint16_t)(V.y & 0xFFFFu);
            keys[sw(P.w)] = (uint16_t)(V.y >> 16);
            if (n == 65536 && (V.x >= 0xFFFE0000u || V.y >= 0xFFFE0000u ||
                               (V.x & 0xFFFEu) == 0xFFFEu || (V.y & 0xFFFEu) == 0xFFFEu)) {
                const int pp[4] = {P.x, P.y, P.z, P.w};
                const uint32_t kk[4] = {V.x & 0xFFFFu, V.x >> 16, V.y & 0xFFFFu, V.y >> 16};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (kk[q] == 0xFFFFu) sX = pp[q];
                    if (kk[q] == 0xFFFEu) sY = pp[q];
                }
            }
        }
    } else {
        for (int64_t e = tid; e < n; e += MG_THREADS) keys[sw(pu[e])] = kv[e];
    }
    __syncthreads();

    // within-u-group pairs: inv_g and joint ties (n3)
    uint32_t inv_g = 0, ties = 0;
    if (p.maxgrp[y] <= MG_SMALL_GROUP) {  // few small groups (the usual case): walk the compact list
        const int32_t* gl = p.groups + y * n;
        const int32_t ng = p.ngroups[y];
        for (int32_t k = tid; k < ng; k += MG_THREADS) {
            const int32_t g0 = gl[2 * k], gl_len = gl[2 * k + 1];
            for (int32_t qa = g0; qa < g0 + gl_len; ++qa) {
                const uint16_t wq = keys[sw(qa)];
                for (int32_t qb = qa + 1; qb < g0 + gl_len; ++qb) {
                    const uint16_t wt = keys[sw(qb)];
                    inv_g += (wq > wt);
                    ties += (wq == wt);
                }
            }
        }
    } else {  // a large u tie group: the O(n log n) segmented radix count
        heavy_group_counts(keys, p.groups + y * n, p.ngroups[y], n, heavy_ws(p.heavy_ws, n), inv_g, ties);
    }
    __syncthreads();

    // n = 65536: key 65535 (a unique row maximum X) would collide with INF.  Sort it as 65534;
    // that only merges it with a unique second maximum Y (key 65534, if any), so add back the
    // X-before-Y inversion when both sit in the same half, and undo the change in the H1 key sum
    // and tie scan of the cross term below.
    int64_t clamp_fix = 0;
    if (n == 65536 && sX >= 0) {
        const bool x1 = sX < L, y1 = sY >= 0 && sY < L;
        if (tid == 0) {
            keys[sw(sX)] = 0xFFFE;
            if (sY >= 0 && x1 == y1 && sX < sY) clamp_fix += 1;
            if (x1) clamp_fix += 1 - (y1 ? 1 : 0);
        }
        __syncthreads();
    }

    // inv(w)
    uint32_t inv;
    int64_t cross = 0;
    if (p.B == 1) {
        inv = sort_count_any(keys, tmp, L, K);
    } else {
        inv = sort_count_halves<2 * MG_HALF / MG_THREADS>(keys, L, K);  // L = 32768: sw(L + i) = sw(L) + sw(i)
        // cross(H1, H2) = sum key(H1) - L1 (L1 - 1) / 2 + ties(H1) (header); the -L1 (L1 - 1) / 2
        // is applied once after the reduction.  H1 = keys[0, L) is sorted and holds no pads.
        constexpr int CE = MG_HALF / MG_THREADS;  // 32 sorted keys per thread
        uint32_t v[CE];
        load_run<CE>(keys, tid, v);
        const int p0 = tid * CE;
        uint32_t prev = tid ? keys[sw(p0 - 1)] : 0xFFFFFFFFu;
        int first = p0;  // first index of the equal-key run holding the current key
        if (v[0] == prev) {  // run continues from the previous thread: lower_bound(H1, v[0])
            int lo = 0, hi = p0 - 1;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (keys[sw(mid)] < v[0]) lo = mid + 1;
                else hi = mid;
            }
            first = lo;
        }
        uint32_t ksum = 0, ties = 0;
#pragma unroll
        for (int q = 0; q < CE; ++q) {
            ksum += v[q];
            if (q > 0 && v[q] != v[q - 1]) first = p0 + q;
            ties += (uint32_t)(p0 + q - first);
        }
        cross = (int64_t)ksum + (int64_t)ties;
    }

    // n_d = inv(w) - sum_g inv_g(w): one reduction of (inv - inv_g), one of the joint ties
    const int64_t nd_all = block_reduce_sum((int64_t)(int32_t)inv + cross + clamp_fix - (int64_t)inv_g, red) -
                           (p.B == 2 ? L1 * (L1 - 1) / 2 : 0);
    const int64_t tot_t = block_reduce_sum((int64_t)ties, red);
    if (tid == 0) {
        const int64_t nd = nd_all;
        const int64_t n3 = tot_t;
        const int64_t num = p.n0 - (int64_t)p.n1[y] - (int64_t)p.n1[x] + n3 - 2 * nd;  // result.py:42
        p.num[idx] = (int32_t)num;
        if (p.nd) p.nd[idx] = (unsigned long long)nd;
        if (p.n3) p.n3[idx] = (unsigned long long)n3;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(MG_THREADS, 1) merge_pairs_kernel(MergeArgs p) {
    pdl_wait();
    extern __shared__ __align__(16) uint8_t mg_smem[];
    uint16_t* keys = reinterpret_cast<uint16_t*>(mg_smem);  // B * L keys (padded layout)
    uint16_t* tmp = keys + sw(p.B * p.L) + 2;               // L keys (padded layout; B == 1 only)
    __shared__ int64_t red[32];
    const int tid = threadIdx.x;
    const int L = p.L;
    __shared__ int sX, sY;  // u-order positions of keys 0xFFFF / 0xFFFE (n = 65536 only)
    if (tid == 0 && L >= 64) {  // INF look-ahead slots behind the last block of every sorted region
        reinterpret_cast<uint32_t*>(keys)[swp_words(L >> 1) - 1] = 0xFFFFFFFFu;
        if (p.B == 1) reinterpret_cast<uint32_t*>(tmp)[swp_words(L >> 1) - 1] = 0xFFFFFFFFu;
        if (p.B == 2) reinterpret_cast<uint32_t*>(keys + sw(L))[swp_words(L >> 1) - 1] = 0xFFFFFFFFu;
    }
    for (int64_t idx = blockIdx.x; idx < p.count; idx += gridDim.x) merge_one_pair(p, idx, keys, tmp, red, sX, sY);
    pdl_trigger();
}

// ------------------------------------------------------------------ several pairs per CTA (n <= 32768)
// With L <= 32768 keys per pair, P = 65536 / L pairs share a CTA: their blocks are consecutive in one
// padded array of 65536 keys, so the register leaf runs over the array exactly as for the two halves of
// n > 32768 (leaf runs never cross a block), and the merge levels run per pair, 1024 / P threads with 64
// outputs each, in place -- the same 64-output levels instead of E = L / 1024 outputs with a ping-pong
// block.  Leaf counts are credited to the block a warp's keys lie in, merge and tie-group counts to the
// thread's own pair.  A batch holding a pair with a large u tie group (heavy_group_counts needs the whole
// CTA) runs its pairs one at a time through merge_one_pair.
__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(MG_THREADS, 1) merge_multi_kernel(MergeArgs p) {
    pdl_wait();
    extern __shared__ __align__(16) uint8_t mg_smem[];
    uint16_t* keys = reinterpret_cast<uint16_t*>(mg_smem);  // P blocks of L keys = 65536 keys, padded layout
    __shared__ int64_t red[32];
    __shared__ int sX, sY, s_heavy;
    __shared__ unsigned long long s_acc[2 * 32];  // per pair: inversions - within-group inversions, joint ties
                                                  // (two's complement sums)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = p.n;
    const int L = p.L, P = p.P;
    const int G = MG_THREADS / P;  // threads per pair (>= 32: whole warps)
    const int g = tid / G, t = tid - g * G;
    uint16_t* blk = keys + g * sw(L);  // L is a multiple of the pad block: sw(g L) = g sw(L)
    const MgConst K = p.k;
    constexpr int TOT = 2 * MG_HALF;
    if (tid < P + 1) {  // INF look-ahead slots in front of every block and behind the last
        const int k0 = tid * L;
        if (k0 > 0) reinterpret_cast<uint32_t*>(keys)[swp_words(k0 >> 1) - 1] = 0xFFFFFFFFu;
    }
    for (int64_t base = (int64_t)blockIdx.x * P; base < p.count; base += (int64_t)gridDim.x * P) {
        if (tid == 0) s_heavy = 0;
        if (tid < 2 * P) s_acc[tid] = 0;
        __syncthreads();
        const int64_t idx = base + g;
        const bool valid = idx < p.count;
        int64_t y = 0, x = 0;
        if (valid) job_coord(p.job_lo + idx, p.m, y, x);
        if (t == 0 && valid && p.maxgrp[y] > MG_SMALL_GROUP) atomicOr(&s_heavy, 1);
        __syncthreads();
        if (s_heavy) {  // one pair at a time on the whole CTA (keys = block 0, ping-pong = block 1)
            MergeArgs q = p;
            q.B = 1;
            for (int k = 0; k < P && base + k < p.count; ++k)
                merge_one_pair(q, base + k, keys, keys + sw(L), red, sX, sY);
            if (tid < P + 1) {  // restore the block-boundary INF slots
                const int k0 = tid * L;
                if (k0 > 0) reinterpret_cast<uint32_t*>(keys)[swp_words(k0 >> 1) - 1] = 0xFFFFFFFFu;
            }
            __syncthreads();
            continue;
        }
        // this pair's block: pads, then w[pos_u[e]] = key_v[e]
        const int64_t real = valid ? n : 0;
        for (int64_t i = real + t; i < L; i += G) blk[sw((int)i)] = 0xFFFE;
        if (valid) {
            const int32_t* pu = p.pos + y * n;
            const uint16_t* kv = p.keys + x * n;
            if ((n & 3) == 0) {
                const int4* pu4 = reinterpret_cast<const int4*>(pu);
                const uint2* kv4 = reinterpret_cast<const uint2*>(kv);
                for (int64_t e = t; e < (n >> 2); e += G) {
                    const int4 Pp = pu4[e];
                    const uint2 V = kv4[e];
                    blk[sw(Pp.x)] = (uint16_t)(V.x & 0xFFFFu);
                    blk[sw(Pp.y)] = (uint16_t)(V.x >> 16);
                    blk[sw(Pp.z)] = (uint16_t)(V.y & 0xFFFFu);
                    blk[sw(Pp.w)] = (uint16_t)(V.y >> 16);
                }
            } else {
                for (int64_t e = t; e < n; e += G) blk[sw(pu[e])] = kv[e];
            }
        }
        __syncthreads();
        // within-u-group pairs of this pair (small groups only here)
        int64_t mine = 0, ties = 0;
        if (valid) {
            const int32_t* gl = p.groups + y * n;
            const int32_t ng = p.ngroups[y];
            uint32_t ig = 0, tt = 0;
            for (int32_t k = t; k < ng; k += G) {
                const int32_t g0 = gl[2 * k], gl_len = gl[2 * k + 1];
                for (int32_t qa = g0; qa < g0 + gl_len; ++qa) {
                    const uint16_t wq = blk[sw(qa)];
                    for (int32_t qb = qa + 1; qb < g0 + gl_len; ++qb) {
                        const uint16_t wt = blk[sw(qb)];
                        ig += (wq > wt);
                        tt += (wq == wt);
                    }
                }
            }
            mine = -(int64_t)ig;
            ties = tt;
        }
        __syncthreads();
        // register leaf over the whole 65536-key array, two passes of 32768 keys; a warp's 1024 keys lie
        // in one block (L >= 2048), its leaf count goes to that block's pair
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            uint16_t* half = keys + h * sw(MG_HALF);
            constexpr int E = 32;
            uint32_t v[E];
            load_run<E>(half, tid, v);
            const int64_t lc = warp_sum64((int64_t)(int32_t)reg_sort_count<E, LEAF_XL<E>>(v));
            store_run<E>(half, tid, v);
            store_lookahead<E>(half, tid, E << LEAF_XL<E>, v[0]);
            if (lane == 0) atomicAdd(&s_acc[2 * ((h * MG_HALF + warp * 32 * E) / L)], (unsigned long long)lc);
        }
        __syncthreads();
        uint32_t inv = 0;
        const int bar_id = (2 * MG_HALF / L) <= 15 ? 1 + g : 0;  // 16 hardware barriers per CTA (0: __syncthreads)
#pragma unroll 1
        for (int W = 32 << LEAF_XL<32>; W < L; W <<= 1)
            inv += merge_level_inplace<2 * MG_HALF / MG_THREADS>(blk, t, W, K, bar_id, G);
        mine += (int64_t)(int32_t)inv;
        const int64_t wm = warp_sum64(mine), wt = warp_sum64(ties);
        if (lane == 0) {
            atomicAdd(&s_acc[2 * g], (unsigned long long)wm);
            atomicAdd(&s_acc[2 * g + 1], (unsigned long long)wt);
        }
        __syncthreads();
        if (t == 0 && valid) {
            const int64_t nd = (int64_t)s_acc[2 * g], n3 = (int64_t)s_acc[2 * g + 1];
            const int64_t num = p.n0 - (int64_t)p.n1[y] - (int64_t)p.n1[x] + n3 - 2 * nd;  // result.py:42
            p.num[idx] = (int32_t)num;
            if (p.nd) p.nd[idx] = (unsigned long long)nd;
            if (p.n3) p.n3[idx] = (unsigned long long)n3;
        }
        __syncthreads();
        (void)TOT;
    }
    pdl_trigger();
}
}  // namespace tb

using namespace tb;

extern "C" int tb_presort(const int32_t* ranks, int64_t m, int64_t n, int32_t* pos, int32_t* sorted, uint16_t* keys,
                          uint64_t* n1, int32_t* maxgrp, int32_t* work, int32_t* ngroups, int32_t* flags,
                          void* stream) {
    if (m < 1 || n < 1) return fail(TB_ERR_INVALID, "presort: empty input");
    if (n > TB_MAX_N) return fail(TB_ERR_CAPACITY, "presort: n=%lld exceeds %d", (long long)n, TB_MAX_N);
    if (!ranks || !pos || !sorted || !keys || !n1 || !maxgrp || !work || !ngroups || !flags)
        return fail(TB_ERR_INVALID, "presort: null pointer");
    if (m > INT32_MAX) return fail(TB_ERR_CAPACITY, "presort: m too large");
    TB_CUDA_TRY(launch_pdl(presort_kernel, dim3((unsigned)m), dim3(PS_THREADS), 0, static_cast<cudaStream_t>(stream), ranks, n, pos, sorted, keys, reinterpret_cast<unsigned long long*>(n1), maxgrp, work, flags));
    int rc = check_launch("presort_kernel");
    if (rc) return rc;
    TB_CUDA_TRY(launch_pdl(tie_groups_kernel, dim3((unsigned)m), dim3(256), 0, static_cast<cudaStream_t>(stream), sorted, n, work, ngroups));
    return check_launch("tie_groups_kernel");
}

extern "C" int64_t tb_merge_workspace(int64_t n) {
    if (n < 1) return 0;
    return (int64_t)num_sms() * heavy_ws_bytes_per_cta(n) + 64;
}

extern "C" int tb_merge_pairs(const uint16_t* keys, const int32_t* pos, const int32_t* sorted,
                              const uint64_t* n1_rows, const int32_t* maxgrp, const int32_t* groups,
                              const int32_t* ngroups, int64_t m, int64_t n, int64_t job_lo, int64_t job_hi,
                              int32_t* num, uint64_t* nd, uint64_t* n3, void* workspace, int64_t ws_bytes,
                              void* stream) {
    if (!maxgrp || !groups || !ngroups) return fail(TB_ERR_INVALID, "merge: null tie-group arrays");
    if (m < 1 || n < 2) return fail(TB_ERR_INVALID, "merge: need m >= 1 and n >= 2");
    if (n > TB_MAX_N) return fail(TB_ERR_CAPACITY, "merge: n=%lld exceeds %d", (long long)n, TB_MAX_N);
    const int64_t total = m * (m + 1) / 2;
    if (job_lo < 0 || job_hi < job_lo || job_hi > total) return fail(TB_ERR_CONFIG, "merge: bad job range");
    if (!keys || !pos || !sorted || !n1_rows || !num) return fail(TB_ERR_INVALID, "merge: null pointer");
    if (job_hi == job_lo) return TB_OK;
    if (!workspace || ws_bytes < tb_merge_workspace(n))
        return fail(TB_ERR_CONFIG, "merge: workspace of %lld bytes, need tb_merge_workspace(n) = %lld",
                    (long long)ws_bytes, (long long)tb_merge_workspace(n));
    MergeArgs a{};
    a.heavy_ws = static_cast<uint8_t*>(workspace);
    a.keys = keys;
    a.pos = pos;
    a.sorted = sorted;
    a.maxgrp = maxgrp;
    a.groups = groups;
    a.ngroups = ngroups;
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
    // B == 2 merges in place (no ping-pong block)
    const size_t padded = (size_t)a.B * L + 2 * (((size_t)a.B * L) >> PBS) + 2 +
                          (a.B == 1 ? L + 2 * ((size_t)L >> PBS) + 2 : 0);
    size_t smem = padded * sizeof(uint16_t);
    a.k = MgConst{1u, 0xFFFFFFFFu, 2u, 4u, 0x10000u, 2u * (PB + 2), (uint32_t)(-2 * (PB + 2)), 1u << (32 - PBS)};
    // n in (1024, 32768]: several pairs per CTA with 64-output in-place merge levels (TB_MERGE_MULTI=0: off)
    static const bool kMulti = [] { const char* e = std::getenv("TB_MERGE_MULTI"); return !(e && e[0] == '0'); }();
    if (kMulti && a.B == 1 && L >= 2048) {
        a.P = 2 * MG_HALF / L;
        const size_t msmem = ((size_t)2 * MG_HALF + 2 * (((size_t)2 * MG_HALF) >> PBS) + 2) * sizeof(uint16_t);
        TB_CUDA_TRY(cudaFuncSetAttribute(merge_multi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msmem));
        const int64_t grid = std::min<int64_t>((a.count + a.P - 1) / a.P, (int64_t)num_sms());
        TB_CUDA_TRY(launch_pdl(merge_multi_kernel, dim3((unsigned)grid), dim3(MG_THREADS), msmem,
                               static_cast<cudaStream_t>(stream), a));
        return check_launch("merge_multi_kernel");
    }
    TB_CUDA_TRY(cudaFuncSetAttribute(merge_pairs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t grid = std::min<int64_t>(a.count, (int64_t)num_sms());
    TB_CUDA_TRY(launch_pdl(merge_pairs_kernel, dim3((unsigned)grid), dim3(MG_THREADS), smem, static_cast<cudaStream_t>(stream), a));
    return check_launch("merge_pairs_kernel");
}
