// K2: sign pack -- each variable's {-1, 0, +1} sign vector over all sample pairs, materialised
// once (int8) for the tcgen05 GEMM.  Replaces the per-pair sign enumeration of naive_numerator
// (kernel_naive.py:26-44).  Input: dense uint16 ranks from K0 (tb_rank.cu).
// HBM-write-bound on S (m * ldS bytes): one CTA per (row, K-range), 16-byte coalesced stores.
#include <cstdlib>

#include "tb_common.cuh"

namespace tb {

constexpr int SP_THREADS = 256;

// S layout ("diagonal"): sample pairs are ordered by offset d = b - a (1..n-1), then by a; each
// d-segment holds n - d signs zero-padded to a multiple of 16 bytes:
//   S[r, off(d) + a] = sign(x[r, a + d] - x[r, a]),  off(d) = 16 * sum_{d' < d} ceil((n - d') / 16).
// Zero padding adds nothing to S_u . S_v; it costs <= 16/(n-1) extra MMA work (1.6% at n = 1000).
__host__ __device__ __forceinline__ int64_t ceil16_prefix(int64_t N) {  // sum_{j=1..N} ceil(j/16)
    const int64_t q = N >> 4, r = N & 15;
    return 8 * q * (q + 1) + r * (q + 1);
}
__host__ __device__ __forceinline__ int64_t diag_off(int64_t d, int64_t n) {
    return 16 * (ceil16_prefix(n - 1) - ceil16_prefix(n - d));
}
__host__ __device__ __forceinline__ int64_t diag_k(int64_t n) { return diag_off(n, n); }

// Segment-major emission: the 16-byte chunks of a row's S are enumerated in memory order,
// chunk c <-> (offset d, group g) with S bytes [off(d) + 16 g, +16) = signs of samples
// a = 16 g .. 16 g + 15 at offset d.  Consecutive threads take consecutive chunks, so every warp
// store is 512 contiguous bytes and a CTA fills its whole K-range (no partial L2 sectors); each
// chunk reads its own and window words with 128-bit loads from shifted shared-memory row copies.
//   D = (w | 0x8000) - o and E = (o | 0x8000) - w per halfword  (2 IADD3, no cross-lane borrow),
//   ge/le = sign-replicated high bytes of D/E                 (PRMT 0xFDB9),
//   byte  = (ge ^ le) & (le | 0x01)                            (one LOP3: +1 / -1 / 0).
__device__ __forceinline__ uint32_t prmt_signs(uint32_t lo, uint32_t hi) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, 0xFDB9;" : "=r"(r) : "r"(lo), "r"(hi));
    return r;
}
__device__ __forceinline__ uint32_t sign_bytes(uint32_t ge, uint32_t le) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0x2C;" : "=r"(r) : "r"(ge), "r"(le), "r"(0x01010101u));
    return r;
}
// smallest N in [1, n-1] with ceil16_prefix(N) >= t
__device__ __forceinline__ int inv_prefix(int64_t t, int n) {
    int lo = 1, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ceil16_prefix(mid) >= t) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

__device__ __forceinline__ uint4 lds128(const uint32_t* p) { return *reinterpret_cast<const uint4*>(p); }

// Signs of the 16 samples of one chunk from its 8 own and 8 window rank-pair words.
// FMT 0: int8 (+1 = 0x01, -1 = 0xFF); FMT 1: e4m3 (0x38 / 0xB8, the kind::f8f6f4 experiment).
// FMT 2 (e2m1) has its own loop below (chunk_e2m1).
template <int FMT>
__device__ __forceinline__ uint4 chunk_signs(const uint32_t (&y)[8], const uint32_t (&own)[8]) {
    uint32_t out[4];
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
        const int k0 = 2 * qq, k1 = 2 * qq + 1;
        const uint32_t ge = prmt_signs(y[k0] + 0x80008000u - own[k0], y[k1] + 0x80008000u - own[k1]);
        const uint32_t le = prmt_signs(own[k0] + 0x80008000u - y[k0], own[k1] + 0x80008000u - y[k1]);
        if (FMT == 1) {
            const uint32_t t = ge ^ le;
            out[qq] = (t & 0x38383838u) | (t & le & 0x80808080u);
        } else {
            out[qq] = sign_bytes(ge, le);
        }
    }
    return make_uint4(out[0], out[1], out[2], out[3]);
}

// e2m1 chunk, 16 signs -> 8 bytes.  Within the chunk, sample 8 w + 4 h + j (w, h in {0,1},
// j in 0..3) sits in word w, byte j, nibble h: the dot product only needs every row to use the same
// order, and this one packs with byte merges instead of nibble shuffles.  Ties may come out as -0
// (0x8), which multiplies like 0.
//   yb: window words with bit 15 of each halfword set (w + 0x8000), own: plain rank pairs.
//   D = yb - o = w - o + 0x8000 per halfword (no borrow: w - o in [-32767, 32767]) -> bit 15: w >= o
//   E = 0x10000 - D per halfword = (-D) + 0x00010000                       -> bit 15: w <= o
// D and E are IMADs (FMA pipe; `neg1` is a runtime -1 so ptxas keeps them off the ALU pipe), the
// PRMT sign-replicates the high bytes and three LOP3s per word build the nibbles.
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ uint32_t lop3_sel(uint32_t a, uint32_t b, uint32_t m) {  // (a & m) | (b & ~m)
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(a), "r"(b), "r"(m));
    return r;
}
__device__ __forceinline__ uint32_t nib_code(uint32_t ge, uint32_t le) {  // ((ge ^ le) & 0x2) | (le & 0x8) per nibble
    const uint32_t x = (ge ^ le) & 0x22222222u;
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xF8;" : "=r"(r) : "r"(x), "r"(le), "r"(0x88888888u));  // x | (le & c)
    return r;
}
__device__ __forceinline__ uint2 chunk_e2m1(const uint32_t (&yb)[8], const uint32_t (&own)[8], uint32_t neg1,
                                            uint32_t k10000) {
    uint32_t ge[4], le[4];
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
        const uint32_t d0 = imad(own[2 * qq], neg1, yb[2 * qq]);
        const uint32_t d1 = imad(own[2 * qq + 1], neg1, yb[2 * qq + 1]);
        const uint32_t e0 = imad(d0, neg1, k10000);
        const uint32_t e1 = imad(d1, neg1, k10000);
        ge[qq] = prmt_signs(d0, d1);
        le[qq] = prmt_signs(e0, e1);
    }
    const uint32_t w0 = nib_code(lop3_sel(ge[0], ge[1], 0x0F0F0F0Fu), lop3_sel(le[0], le[1], 0x0F0F0F0Fu));
    const uint32_t w1 = nib_code(lop3_sel(ge[2], ge[3], 0x0F0F0F0Fu), lop3_sel(le[2], le[3], 0x0F0F0F0Fu));
    return make_uint2(w0, w1);
}

// Shared memory holds 8 shifted copies of the row's rank pairs, C[o][s][j] = pair at halfword
// 2 (j + s) + o, so the window of chunk (d, g) -- halfwords 16 g + d .. +15 -- is 8 words starting
// at the 16-byte-aligned index 8 g + ((d >> 1) & ~3) of copy (d & 1, (d >> 1) & 3): two 128-bit
// loads, no per-lane shifting.

template <int FMT>
__global__ void __launch_bounds__(SP_THREADS, 4) signpack_kernel(const uint16_t* __restrict__ R, int64_t n,
                                                              int64_t ldr, int8_t* __restrict__ S, int64_t ldS,
                                                              int64_t K, int nwc, uint32_t neg1) {
    extern __shared__ __align__(16) uint32_t sp_words[];  // [8][nwc] (+ [nwc] plain own copy for e2m1)
    const int64_t r = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nn = (int)n;
    const uint16_t* rr = R + r * ldr;
    for (int j = tid; j < nwc; j += SP_THREADS) {
#pragma unroll
        for (int o = 0; o < 2; ++o) {
#pragma unroll
            for (int sh = 0; sh < 4; ++sh) {
                const int h = 2 * (j + sh) + o;  // halfword index of the pair's low half
                const uint32_t lo = h < nn ? rr[h] : 0u, hi = h + 1 < nn ? rr[h + 1] : 0u;
                const uint32_t wv = lo | (hi << 16);
                sp_words[(o * 4 + sh) * nwc + j] = FMT == 2 ? (wv | 0x80008000u) : wv;
                if (FMT == 2 && o == 0 && sh == 0) sp_words[8 * nwc + j] = wv;
            }
        }
    }
    if (FMT == 2 && tid < 32) {  // tail masks: [swapped][lim] for the last chunk of a segment
        const int lim = tid & 15, swp = tid >> 4;
        uint32_t mk[2] = {0u, 0u};
        for (int i = 0; i < lim; ++i) mk[i >> 3] |= 0xFu << (8 * (i & 3) + 4 * ((i >> 2) & 1));
        reinterpret_cast<uint2*>(sp_words + 9 * nwc)[tid] = swp ? make_uint2(mk[1], mk[0]) : make_uint2(mk[0], mk[1]);
    }
    __syncthreads();

    int8_t* row = S + r * ldS;
    const int nchunks = (int)(K >> 4);  // < 2^31: K < 2^34 for n <= 32767... K/16 < 2^30
    const int per = (nchunks + (int)gridDim.y - 1) / (int)gridDim.y;
    const int b_lo = (int)blockIdx.y * per, b_hi = min(b_lo + per, nchunks);
    const int wper = (b_hi - b_lo + (SP_THREADS / 32) - 1) / (SP_THREADS / 32);
    const int c_lo = b_lo + warp * wper, c_hi = min(c_lo + wper, b_hi);
    int c = c_lo + lane;
    if (c < c_hi) {
        // decode chunk c -> (d, g): off(d)/16 = P(n-1) - P(n-d) <= c < P(n-1) - P(n-d-1)
        const int64_t top = ceil16_prefix(nn - 1);
        const int N = inv_prefix(top - c, nn);  // n - d
        int d = nn - N;
        int g = (int)(c - (top - ceil16_prefix(N)));
        int G = (nn - d + 15) >> 4;
        // window base of offset d: copy (d & 1, (d >> 1) & 3), 16-byte-aligned word (d >> 1) & ~3
        int wbase = ((d & 1) * 4 + ((d >> 1) & 3)) * nwc + ((d >> 1) & ~3);
        if (FMT == 2) {
            // Bank swizzle: chunks with bit 2 of g set read their second 16 bytes first, so 8
            // consecutive chunks' 128-bit loads cover all 32 banks.  Their two output words come out
            // swapped -- a fixed per-chunk sample order, identical in every row.  A 32-chunk step
            // keeps bit 2 of g, so the swizzle (and the pointers) only change at a segment crossing.
            const uint2* masks = reinterpret_cast<const uint2*>(sp_words + 9 * nwc);
            uint2* outp = reinterpret_cast<uint2*>(row) + c;
            int sw = ((g >> 2) & 1) * 4;
            const uint32_t* own_p = sp_words + 8 * nwc + 8 * g + sw;
            const uint32_t* win_p = sp_words + wbase + 8 * g + sw;
            int lim = nn - d - 16 * g;  // samples 16 g + i valid for i < lim
            for (;;) {
                const uint4 o0 = lds128(own_p), o1 = lds128(own_p + (4 - 2 * sw));
                const uint4 w0 = lds128(win_p), w1 = lds128(win_p + (4 - 2 * sw));
                const uint32_t own[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
                const uint32_t y[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
                uint2 v2 = chunk_e2m1(y, own, neg1, 0x00010000u);
                if (lim < 16) {
                    const uint2 mk = masks[lim + 4 * sw];
                    v2.x &= mk.x;
                    v2.y &= mk.y;
                }
                *outp = v2;
                c += 32;
                if (c >= c_hi) break;
                outp += 32;
                g += 32;
                own_p += 256;
                win_p += 256;
                lim -= 512;
                if (g >= G) {
                    do {
                        g -= G;
                        ++d;
                        G = (nn - d + 15) >> 4;
                    } while (g >= G);
                    wbase = ((d & 1) * 4 + ((d >> 1) & 3)) * nwc + ((d >> 1) & ~3);
                    sw = ((g >> 2) & 1) * 4;
                    own_p = sp_words + 8 * nwc + 8 * g + sw;
                    win_p = sp_words + wbase + 8 * g + sw;
                    lim = nn - d - 16 * g;
                }
            }
        }
        for (; FMT != 2;) {
            const int lim = nn - d - 16 * g;  // samples 16 g + i valid for i < lim
            const uint32_t* own_p = sp_words + 8 * g;
            const uint32_t* win_p = sp_words + wbase + 8 * g;
            const uint4 o0 = lds128(own_p), o1 = lds128(own_p + 4);
            const uint4 w0 = lds128(win_p), w1 = lds128(win_p + 4);
            const uint32_t own[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
            const uint32_t y[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            uint4 v = chunk_signs<FMT>(y, own);
            if (lim < 16) {
                uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    const int cnt = min(max(lim - 4 * qq, 0), 4);
                    w4[qq] &= cnt == 4 ? 0xFFFFFFFFu : ((1u << (8 * cnt)) - 1u);
                }
                v = make_uint4(w4[0], w4[1], w4[2], w4[3]);
            }
            *reinterpret_cast<uint4*>(row + 16 * (int64_t)c) = v;
            c += 32;
            if (c >= c_hi) break;
            g += 32;
            if (g >= G) {
                do {
                    g -= G;
                    ++d;
                    G = (nn - d + 15) >> 4;
                } while (g >= G);
                wbase = ((d & 1) * 4 + ((d >> 1) & 3)) * nwc + ((d >> 1) & ~3);
            }
        }
    }
    // zero the row tail [K bytes, ldS)
    const int64_t kb = FMT == 2 ? K / 2 : K;
    for (int64_t k = kb + ((int64_t)blockIdx.y * SP_THREADS + tid) * 8; k < ldS; k += (int64_t)gridDim.y * SP_THREADS * 8)
        *reinterpret_cast<uint2*>(row + k) = make_uint2(0u, 0u);
}

}  // namespace tb

using namespace tb;

extern "C" int tb_sign_pack(const uint16_t* R, int64_t m, int64_t n, int64_t ldr, int8_t* S, int64_t ldS,
                            int format, void* stream) {
    if (m < 1 || n < 2) return fail(TB_ERR_INVALID, "sign_pack: need m >= 1 and n >= 2 (got m=%lld n=%lld)",
                                    (long long)m, (long long)n);
    if (n > 32767) return fail(TB_ERR_CAPACITY, "sign_pack: n=%lld exceeds 32767 (15-bit ranks)", (long long)n);
    const int64_t K = diag_k(n);
    if (format < 0 || format > 2) return fail(TB_ERR_CONFIG, "sign_pack: unknown format %d", format);
    const int64_t kbytes = format == TB_SIGN_E2M1 ? K / 2 : K;
    if (ldS < kbytes || (ldS & 15))
        return fail(TB_ERR_CONFIG, "sign_pack: ldS=%lld must be >= %lld and 16-aligned", (long long)ldS,
                    (long long)kbytes);
    if (ldr < n || (ldr & 1)) return fail(TB_ERR_CONFIG, "sign_pack: ldr must be even and >= n");
    if (!R || !S) return fail(TB_ERR_INVALID, "sign_pack: null pointer");
    const int nwc = (int)(((n + 1) / 2 + 16 + 3) & ~3);  // words per shifted copy (window reads overrun n)
    const size_t smem = (size_t)(format == TB_SIGN_E2M1 ? 9 : 8) * nwc * sizeof(uint32_t) + 32 * sizeof(uint2);
    if (smem > 200 * 1024) return fail(TB_ERR_CAPACITY, "sign_pack: n=%lld too large for the shared row copies", (long long)n);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t nblk = (K / 16 + 16 * SP_THREADS - 1) / (16 * SP_THREADS);  // >= 16 chunks per thread
    int64_t want = (8 * (int64_t)num_sms() + m - 1) / m;  // >= ~8 CTAs per SM in total
    int gy = (int)std::min<int64_t>(std::max<int64_t>(want, 1), std::min<int64_t>(nblk, 65535));
    dim3 grid((unsigned)m, gy);
#define TB_SP_LAUNCH(F)                                                                                   \
    TB_CUDA_TRY(cudaFuncSetAttribute(signpack_kernel<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    signpack_kernel<F><<<grid, SP_THREADS, smem, st>>>(R, n, ldr, S, ldS, K, nwc, 0xFFFFFFFFu)
    if (format == TB_SIGN_E2M1) {
        TB_SP_LAUNCH(2);
    } else if (format == TB_SIGN_E4M3) {
        TB_SP_LAUNCH(1);
    } else {
        TB_SP_LAUNCH(0);
    }
#undef TB_SP_LAUNCH
    return check_launch("signpack_kernel");
}

// |S| (0/1 int8) for the full-count GEMM, 16 bytes per thread.
namespace tb {
__global__ void abs_pack_kernel(const uint4* __restrict__ S, uint4* __restrict__ A, int64_t nvec, uint32_t mask) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * blockDim.x) {
        uint4 v = S[i];
        // int8 bytes 0x00/0x01/0xFF: |s| = s & 1; e2m1 nibbles 0x0/0x2/0xA: |s| clears the sign bits
        v.x &= mask;
        v.y &= mask;
        v.z &= mask;
        v.w &= mask;
        A[i] = v;
    }
}
}  // namespace tb

extern "C" int tb_abs_pack(const int8_t* S, int64_t m, int64_t ldS, int format, int8_t* A, void* stream) {
    if (m < 1 || ldS < 16 || (ldS & 15)) return fail(TB_ERR_CONFIG, "abs_pack: bad shape");
    if (!S || !A) return fail(TB_ERR_INVALID, "abs_pack: null pointer");
    const int64_t nvec = m * ldS / 16;
    const int64_t blocks = std::min<int64_t>((nvec + 255) / 256, (int64_t)num_sms() * 8);
    abs_pack_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const uint4*>(S), reinterpret_cast<uint4*>(A), nvec,
        format == TB_SIGN_E2M1 ? 0x77777777u : (format == TB_SIGN_E4M3 ? 0x7F7F7F7Fu : 0x01010101u));
    return check_launch("abs_pack_kernel");
}

extern "C" int64_t tb_sign_k(int64_t n) { return n >= 2 ? tb::diag_k(n) : 0; }
