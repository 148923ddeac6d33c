// K2: sign pack -- each variable's {-1, 0, +1} sign vector over all sample pairs, materialised
// once for the tcgen05 GEMM.  Replaces the per-pair sign enumeration of naive_numerator
// (kernel_naive.py:26-44): S_u . S_v over any fixed ordering of the n(n-1)/2 pairs (a < b) with
// S_u[k(a,b)] = sign(r_u[b] - r_u[a]) is n_c - n_d.  Input: dense uint16 ranks from K0 (tb_rank.cu).
#include "tb_common.cuh"

namespace tb {

constexpr int SP_THREADS = 256;

// ---------------------------------------------------------------------------------------------
// "Block" layout of the sample pairs.  S is a sequence of 16-pair chunks (one 16-byte int8/e4m3
// row segment, or 8 bytes of e2m1); with nbf = floor(n / 16) full 16-sample blocks and nt = n mod 16
// tail samples:
//   section 1  pairs between two different full blocks A < B (row-major over (A, B)), 16 chunks per
//              block pair: chunk a_l of (A, B) holds (a = 16A + a_l, b = 16B + s), s = 0..15;
//   section 2  pairs inside one full block: per block, 15 b-columns paired j / 16 - j into 7 chunks
//              (s < j: (s, j); s >= j: (s - j, 16 - j)), and the two b = 8 columns of consecutive
//              blocks share one chunk (block A0: s < 8 -> (s, 8); block A1: (s - 8, 8));
//   section 3  pairs ending at a tail sample b = 16 nbf + t: a = 0 .. b-1 in chunks of 16.
// Only the last chunk of a section-3 segment and a lone section-2 half chunk are partial, so
// K = 16 * chunks = n(n-1)/2 + O(n / 16) (n = 1000: 499,584 for 499,500 pairs).
struct SpLayout {
    int64_t nbf, nt, c1, c2, c3;
};
__host__ __device__ __forceinline__ SpLayout sp_layout(int64_t n) {
    SpLayout L;
    L.nbf = n / 16;
    L.nt = n % 16;
    L.c1 = 16 * (L.nbf * (L.nbf - 1) / 2);
    L.c2 = 7 * L.nbf + (L.nbf + 1) / 2;
    L.c3 = L.nt * L.nbf + (L.nt > 0 ? L.nt - 1 : 0);
    return L;
}
__host__ __device__ __forceinline__ int64_t sp_k(int64_t n) {
    const SpLayout L = sp_layout(n);
    return 16 * (L.c1 + L.c2 + L.c3);
}

// Packed-halfword sign arithmetic on two sample pairs per 32-bit word (ranks < 2^15):
//   D = (w | 0x8000) - o per halfword (no borrow) -> bit 15: w >= o;  E = 0x10000 - D -> w <= o;
// a sign-replicating PRMT turns the high bytes into >= / <= masks.
__device__ __forceinline__ uint32_t prmt_signs(uint32_t lo, uint32_t hi) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, 0xFDB9;" : "=r"(r) : "r"(lo), "r"(hi));
    return r;
}
__device__ __forceinline__ uint32_t sign_bytes(uint32_t ge, uint32_t le) {  // (ge ^ le) & (le | 1)
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0x2C;" : "=r"(r) : "r"(ge), "r"(le), "r"(0x01010101u));
    return r;
}
__device__ __forceinline__ uint4 lds128(const uint32_t* p) { return *reinterpret_cast<const uint4*>(p); }

// int8 (FMT 0: +1 = 0x01, -1 = 0xFF) / e4m3 (FMT 1: 0x38 / 0xB8) chunk: 16 bytes, sample s in byte s.
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

// e2m1 chunk (FMT 2), 16 signs -> 8 bytes: sample 8 w + 4 h + j sits in word w, byte j, nibble h
// (byte merges instead of nibble shuffles; every row uses the same order).  +1 = 0x2, -1 = 0xA, ties
// may come out as -0 (0x8).  yb: window words with bit 15 of each halfword set; own: plain words.
// D and E are IMADs (FMA pipe; `neg1` is a runtime -1 so ptxas keeps them off the ALU pipe).
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
__device__ __forceinline__ uint32_t nib_code(uint32_t ge, uint32_t le) {  // ((ge ^ le) & 0x2) | (le & 0x8)
    const uint32_t x = (ge ^ le) & 0x22222222u;
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xF8;" : "=r"(r) : "r"(x), "r"(le), "r"(0x88888888u));
    return r;
}
// Offset coding (TB_SIGN_E2M1_OFS): the element is S + 1 -- -1 -> 0 (0x0), tie -> 1.0 (0x2), +1 -> 2.0 (0x4).
// No sign bit ever toggles and half the operands are zero: the same MMA stream draws less power (see
// tb_gemm_fp4.cu, "offset operands").  At least one of ge / le is set in every nibble.
__device__ __forceinline__ uint32_t nib_code_ofs(uint32_t ge, uint32_t le) {  // ge & (le ? 0x2 : 0x4)
    uint32_t t, r;
    asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(t) : "r"(le), "r"(0x22222222u), "r"(0x44444444u));
    asm("lop3.b32 %0, %1, %2, %3, 0xC0;" : "=r"(r) : "r"(ge), "r"(t), "r"(0u));
    return r;
}
template <int OFS = 0>
__device__ __forceinline__ uint2 chunk_e2m1(const uint32_t (&yb)[8], const uint32_t (&own)[8], uint32_t neg1) {
    uint32_t ge[4], le[4];
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
        const uint32_t d0 = imad(own[2 * qq], neg1, yb[2 * qq]);
        const uint32_t d1 = imad(own[2 * qq + 1], neg1, yb[2 * qq + 1]);
        const uint32_t e0 = imad(d0, neg1, 0x00010000u);
        const uint32_t e1 = imad(d1, neg1, 0x00010000u);
        ge[qq] = prmt_signs(d0, d1);
        le[qq] = prmt_signs(e0, e1);
    }
    const uint32_t g0 = lop3_sel(ge[0], ge[1], 0x0F0F0F0Fu), l0 = lop3_sel(le[0], le[1], 0x0F0F0F0Fu);
    const uint32_t g1 = lop3_sel(ge[2], ge[3], 0x0F0F0F0Fu), l1 = lop3_sel(le[2], le[3], 0x0F0F0F0Fu);
    if (OFS) return make_uint2(nib_code_ofs(g0, l0), nib_code_ofs(g1, l1));
    return make_uint2(nib_code(g0, l0), nib_code(g1, l1));
}

// Sections 2 and 3 (~3% of the chunks): per-sample (a, b) lists -> own / window words and the
// number of valid leading samples.
__device__ __forceinline__ int sp_slow_chunk(int64_t c, const SpLayout& L, const uint16_t* r16, const uint32_t* wp,
                                             uint32_t (&own)[8], uint32_t (&y)[8]) {
    const int nbf = (int)L.nbf;
    const int64_t k2 = c - L.c1;
    if (k2 < L.c2) {
        const int P = (int)(k2 / 15), k = (int)(k2 - 15 * (int64_t)P);
        const int A0 = 2 * P, A1 = 2 * P + 1;
        if (k < 14 && (k < 7 || A1 < nbf)) {  // a paired j / 16 - j chunk of block blk
            const int blk = k < 7 ? A0 : A1, j = k < 7 ? k + 1 : k - 6;
            const uint16_t* rb = r16 + 16 * blk;
            const uint32_t w1 = rb[j], w2 = rb[16 - j];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int s0 = 2 * q, s1 = 2 * q + 1;
                own[q] = (uint32_t)rb[s0 < j ? s0 : s0 - j] | ((uint32_t)rb[s1 < j ? s1 : s1 - j] << 16);
                y[q] = (s0 < j ? w1 : w2) | ((s1 < j ? w1 : w2) << 16);
            }
            return 16;
        }
        // the b = 8 columns of A0 and A1 (or A0 alone: 8 valid samples)
        const int B1 = A1 < nbf ? A1 : A0;
        const uint32_t w1 = r16[16 * A0 + 8], w2 = r16[16 * B1 + 8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            own[q] = wp[8 * A0 + q];
            own[q + 4] = wp[8 * B1 + q];
            y[q] = w1 * 0x10001u;
            y[q + 4] = w2 * 0x10001u;
        }
        return A1 < nbf ? 16 : 8;
    }
    int64_t k3 = k2 - L.c2;  // tail segment t has nbf + (t > 0) chunks
    int t = 0;
    while (k3 >= L.nbf + (t > 0 ? 1 : 0)) {
        k3 -= L.nbf + (t > 0 ? 1 : 0);
        ++t;
    }
    const int b = 16 * nbf + t, i = (int)k3;
    const uint4 o0 = lds128(wp + 8 * i), o1 = lds128(wp + 8 * i + 4);
    own[0] = o0.x; own[1] = o0.y; own[2] = o0.z; own[3] = o0.w;
    own[4] = o1.x; own[5] = o1.y; own[6] = o1.z; own[7] = o1.w;
    const uint32_t rbb = (uint32_t)r16[b] * 0x10001u;
#pragma unroll
    for (int q = 0; q < 8; ++q) y[q] = rbb;
    return min(16, b - 16 * i);
}

// e2m1 chunks [c_lo, c_hi) of one row (c_lo even): each lane takes two adjacent chunks (a_l, a_l + 1
// of one block pair share the window: one pair of window loads, one rank-pair load, one 16-byte
// store; a warp writes 512 contiguous bytes) and steps 64 chunks = 4 block pairs.
// Sum of the offset-coded values (nibbles 0x0 / 0x2 / 0x4 = 0 / 1 / 2) of up to four words into acc: the
// nibbles are even, so w >> 1 halves each in place; two halved pair sums stay <= 8 per nibble, and two
// dp4a's add the eight nibbles of the result.
__device__ __forceinline__ int32_t ofs_sum4(uint32_t a, uint32_t b, uint32_t c, uint32_t d, int32_t acc) {
    const uint32_t z = ((a + b) >> 1) + ((c + d) >> 1);
    uint32_t u = __dp4a(z & 0x0F0F0F0Fu, 0x01010101u, (uint32_t)acc);
    u = __dp4a((z >> 4) & 0x0F0F0F0Fu, 0x01010101u, u);
    return (int32_t)u;
}
template <int OFS>
__device__ __forceinline__ void sp_e2m1_range(int c_lo, int c_hi, int lane, const SpLayout& L, const uint16_t* r16,
                                              const uint32_t* wp, const uint32_t* wb, const uint4* masks,
                                              int8_t* row, uint32_t neg1, int32_t& acc) {
    const int c1 = (int)L.c1, nbf = (int)L.nbf;
    int c = c_lo + 2 * lane;
    const int c1_end = min(c_hi, c1);  // c1 is a multiple of 16: a pair never straddles it
    if (c < c1_end) {
        const int al = c & 15;  // even
        const int bid = c >> 4;
        const double f = (double)nbf - 0.5;
        int A = (int)(f - sqrt(f * f - 2.0 * (double)bid));
        if (A < 0) A = 0;
        auto start = [nbf](int x) { return x * (nbf - 1) - x * (x - 1) / 2; };
        while (A > 0 && start(A) > bid) --A;
        while (A < nbf - 1 && start(A + 1) <= bid) ++A;
        int B = bid - start(A) + A + 1;
        uint32_t ow = wp[(16 * A + al) >> 1];  // ranks of a_l, a_l + 1
        const uint32_t* wptr = wb + 8 * B;
        uint4* outp = reinterpret_cast<uint4*>(row + 8 * (int64_t)c);
        for (;;) {
            const uint4 w0 = lds128(wptr), w1 = lds128(wptr + 4);
            const uint32_t y[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            const uint32_t oa = __byte_perm(ow, 0, 0x1010), ob = __byte_perm(ow, 0, 0x3232);
            const uint32_t owa[8] = {oa, oa, oa, oa, oa, oa, oa, oa};
            const uint32_t owb[8] = {ob, ob, ob, ob, ob, ob, ob, ob};
            const uint2 va = chunk_e2m1<OFS>(y, owa, neg1), vb = chunk_e2m1<OFS>(y, owb, neg1);
            *outp = make_uint4(va.x, va.y, vb.x, vb.y);
            if (OFS) acc = ofs_sum4(va.x, va.y, vb.x, vb.y, acc);
            c += 64;
            if (c >= c1_end) break;
            outp += 32;
            B += 4;
            wptr += 32;
            if (B >= nbf) {  // row A + 1 starts at B = A + 2
                do {
                    ++A;
                    B += A + 1 - nbf;
                } while (B >= nbf && A < nbf - 1);
                wptr = wb + 8 * B;
                ow = wp[(16 * A + al) >> 1];
            }
        }
    }
    // sections 2 and 3 (~3% of the chunks): per-sample lists, partial chunks masked
    for (; c < c_hi; c += 64) {
#pragma unroll 1
        for (int k = 0; k < 2 && c + k < c_hi; ++k) {
            uint32_t own[8], y[8];
            const int valid = sp_slow_chunk(c + k, L, r16, wp, own, y);
#pragma unroll
            for (int q = 0; q < 8; ++q) y[q] |= 0x80008000u;
            uint2 v2 = chunk_e2m1<OFS>(y, own, neg1);
            if (valid < 16) {
                const uint4 mk = masks[valid];
                v2.x &= mk.x;
                v2.y &= mk.y;
            }
            *reinterpret_cast<uint2*>(row + 8 * (int64_t)(c + k)) = v2;
            if (OFS) acc = ofs_sum4(v2.x, v2.y, 0u, 0u, acc);
        }
    }
}

// One CTA per (row, K-range); warps take contiguous chunk ranges and consecutive lanes consecutive
// chunks (coalesced stores).  Section 1 needs no per-lane decode after the start: a 32-chunk step is
// exactly two block pairs, and a_l = c mod 16 stays fixed.  The window of block B is 8 aligned words
// shared by the 16 lanes on that block (broadcast loads); own is one broadcast rank.
template <int FMT>
__global__ void __launch_bounds__(SP_THREADS, 4) signpack_kernel(const uint16_t* __restrict__ R, int64_t n,
                                                              int64_t ldr, int8_t* __restrict__ S, int64_t ldS,
                                                              int nw, uint32_t neg1, int32_t* __restrict__ rowsum,
                                                              int64_t n0) {
    pdl_wait();
    extern __shared__ __align__(16) uint32_t sp_words[];  // wp[nw] plain pairs, wb[nw] biased, masks[17]
    uint32_t* wp = sp_words;
    uint32_t* wb = sp_words + nw;
    uint4* masks = reinterpret_cast<uint4*>(sp_words + 2 * nw);
    const int64_t r = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nn = (int)n;
    const uint16_t* rr = R + r * ldr;
    for (int j = tid; j < nw; j += SP_THREADS) {
        const int h = 2 * j;
        const uint32_t lo = h < nn ? rr[h] : 0u, hi = h + 1 < nn ? rr[h + 1] : 0u;
        wp[j] = lo | (hi << 16);
        wb[j] = lo | (hi << 16) | 0x80008000u;
    }
    if (tid <= 16) {  // masks[v]: the first v samples of a chunk kept
        uint32_t mk0 = 0u, mk1 = 0u, mk2 = 0u, mk3 = 0u;
        for (int s = 0; s < tid; ++s) {
            const int wi = FMT >= 2 ? (s >> 3) : (s >> 2);
            const uint32_t bits = FMT >= 2 ? 0xFu << (8 * (s & 3) + 4 * ((s >> 2) & 1)) : 0xFFu << (8 * (s & 3));
            mk0 |= wi == 0 ? bits : 0u;
            mk1 |= wi == 1 ? bits : 0u;
            mk2 |= wi == 2 ? bits : 0u;
            mk3 |= wi == 3 ? bits : 0u;
        }
        masks[tid] = make_uint4(mk0, mk1, mk2, mk3);
    }
    __syncthreads();
    const uint16_t* r16 = reinterpret_cast<const uint16_t*>(wp);
    const uint32_t* win = FMT >= 2 ? wb : wp;

    const SpLayout L = sp_layout(n);
    const int nchunks = (int)(L.c1 + L.c2 + L.c3);  // < 2^31 (n <= 32767)
    const int c1 = (int)L.c1;
    int8_t* row = S + r * ldS;
    // CTA / warp ranges start on even chunks: the e2m1 loop gives each lane two adjacent chunks
    const int per = ((nchunks + (int)gridDim.y - 1) / (int)gridDim.y + 1) & ~1;
    const int b_lo = min((int)blockIdx.y * per, nchunks), b_hi = min(b_lo + per, nchunks);
    const int wper = ((b_hi - b_lo + (SP_THREADS / 32) - 1) / (SP_THREADS / 32) + 1) & ~1;
    const int c_lo = min(b_lo + warp * wper, b_hi), c_hi = min(c_lo + wper, b_hi);
    if (FMT >= 2) {
        int32_t acc = 0;
        sp_e2m1_range<FMT == 3>(c_lo, c_hi, lane, L, r16, wp, win, masks, row, neg1, acc);
        if (FMT == 3 && rowsum) {  // fused tb_sign_row_sums: rowsum[r] (zeroed by the host) += this warp's share
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (blockIdx.y == 0 && warp == 0) acc -= (int32_t)n0;
            if (lane == 0 && acc != 0) atomicAdd(rowsum + r, acc);
        }
    } else {
    int c = c_lo + lane;
    const int nbf = (int)L.nbf;
    // ---- section 1: block pairs (A < B); per step B += 2, own changes only with A
    const int c1_end = min(c_hi, c1);
    if (c < c1_end) {
        const int al = c & 15;
        const int bid = c >> 4;
        const double f = (double)nbf - 0.5;
        int A = (int)(f - sqrt(f * f - 2.0 * (double)bid));
        if (A < 0) A = 0;
        auto start = [nbf](int x) { return x * (nbf - 1) - x * (x - 1) / 2; };
        while (A > 0 && start(A) > bid) --A;
        while (A < nbf - 1 && start(A + 1) <= bid) ++A;
        int B = bid - start(A) + A + 1;
        uint32_t o2 = (uint32_t)r16[16 * A + al] * 0x10001u;
        const uint32_t* wptr = win + 8 * B;
        for (;;) {
            const uint4 w0 = lds128(wptr), w1 = lds128(wptr + 4);
            const uint32_t y[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            const uint32_t own[8] = {o2, o2, o2, o2, o2, o2, o2, o2};
            if (FMT == 2)
                *reinterpret_cast<uint2*>(row + 8 * (int64_t)c) = chunk_e2m1(y, own, neg1);
            else
                *reinterpret_cast<uint4*>(row + 16 * (int64_t)c) = chunk_signs<FMT>(y, own);
            c += 32;
            if (c >= c1_end) break;
            B += 2;
            wptr += 16;
            if (B >= nbf) {  // row A + 1 starts at B = A + 2
                do {
                    ++A;
                    B += A + 1 - nbf;
                } while (B >= nbf && A < nbf - 1);
                wptr = win + 8 * B;
                o2 = (uint32_t)r16[16 * A + al] * 0x10001u;
            }
        }
    }
    // ---- sections 2 and 3 (~3% of the chunks): per-sample lists, partial chunks masked
    for (; c < c_hi; c += 32) {
        uint32_t own[8], y[8];
        const int valid = sp_slow_chunk(c, L, r16, wp, own, y);
        if (FMT == 2) {
#pragma unroll
            for (int q = 0; q < 8; ++q) y[q] |= 0x80008000u;
            uint2 v2 = chunk_e2m1(y, own, neg1);
            if (valid < 16) {
                const uint4 mk = masks[valid];
                v2.x &= mk.x;
                v2.y &= mk.y;
            }
            *reinterpret_cast<uint2*>(row + 8 * (int64_t)c) = v2;
        } else {
            uint4 v = chunk_signs<FMT>(y, own);
            if (valid < 16) {
                const uint4 mk = masks[valid];
                v.x &= mk.x; v.y &= mk.y; v.z &= mk.z; v.w &= mk.w;
            }
            *reinterpret_cast<uint4*>(row + 16 * (int64_t)c) = v;
        }
    }
    }
    // zero the row tail [K bytes, ldS)
    const int64_t kb = (FMT >= 2 ? 8 : 16) * (int64_t)nchunks;
    for (int64_t k = kb + ((int64_t)blockIdx.y * SP_THREADS + tid) * 8; k < ldS; k += (int64_t)gridDim.y * SP_THREADS * 8)
        *reinterpret_cast<uint2*>(row + k) = make_uint2(0u, 0u);
    pdl_trigger();
}

}  // namespace tb

using namespace tb;

static int sign_pack_impl(const uint16_t* R, int64_t m, int64_t n, int64_t ldr, int8_t* S, int64_t ldS, int format,
                          int32_t* rowsum, void* stream);

extern "C" int tb_sign_pack(const uint16_t* R, int64_t m, int64_t n, int64_t ldr, int8_t* S, int64_t ldS,
                            int format, void* stream) {
    return sign_pack_impl(R, m, n, ldr, S, ldS, format, nullptr, stream);
}

extern "C" int tb_sign_pack_sums(const uint16_t* R, int64_t m, int64_t n, int64_t ldr, int8_t* S, int64_t ldS,
                                 int32_t* fix, void* stream) {
    if (!fix) return fail(TB_ERR_INVALID, "sign_pack_sums: null pointer");
    if (m < 1 || m > INT32_MAX) return fail(TB_ERR_INVALID, "sign_pack_sums: bad m");
    TB_CUDA_TRY(cudaMemsetAsync(fix, 0, (size_t)m * sizeof(int32_t), static_cast<cudaStream_t>(stream)));
    return sign_pack_impl(R, m, n, ldr, S, ldS, TB_SIGN_E2M1_OFS, fix, stream);
}

static int sign_pack_impl(const uint16_t* R, int64_t m, int64_t n, int64_t ldr, int8_t* S, int64_t ldS, int format,
                          int32_t* rowsum, void* stream) {
    if (m < 1 || n < 2) return fail(TB_ERR_INVALID, "sign_pack: need m >= 1 and n >= 2 (got m=%lld n=%lld)",
                                    (long long)m, (long long)n);
    if (n > 32767) return fail(TB_ERR_CAPACITY, "sign_pack: n=%lld exceeds 32767 (15-bit ranks)", (long long)n);
    const int64_t K = sp_k(n);
    if (format < 0 || format > 3) return fail(TB_ERR_CONFIG, "sign_pack: unknown format %d", format);
    const int64_t kbytes = format >= TB_SIGN_E2M1 ? K / 2 : K;
    if (ldS < kbytes || (ldS & 15))
        return fail(TB_ERR_CONFIG, "sign_pack: ldS=%lld must be >= %lld and 16-aligned", (long long)ldS,
                    (long long)kbytes);
    if (ldr < n || (ldr & 1)) return fail(TB_ERR_CONFIG, "sign_pack: ldr must be even and >= n");
    if (!R || !S) return fail(TB_ERR_INVALID, "sign_pack: null pointer");
    const int nw = (int)(((n + 1) / 2 + 8 + 3) & ~3);  // rank-pair words (window loads of the last block)
    const size_t smem = (size_t)2 * nw * sizeof(uint32_t) + 17 * sizeof(uint4);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t nblk = (K / 16 + 16 * SP_THREADS - 1) / (16 * SP_THREADS);  // >= 16 chunks per thread
    int64_t want = (8 * (int64_t)num_sms() + m - 1) / m;  // >= ~8 CTAs per SM in total
    int gy = (int)std::min<int64_t>(std::max<int64_t>(want, 1), std::min<int64_t>(nblk, 65535));
    dim3 grid((unsigned)m, gy);
#define TB_SP_LAUNCH(F)                                                                                   \
    TB_CUDA_TRY(cudaFuncSetAttribute(signpack_kernel<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    TB_CUDA_TRY(launch_pdl(signpack_kernel<F>, dim3(grid), dim3(SP_THREADS), smem, st, R, n, ldr, S, ldS, nw, 0xFFFFFFFFu, \
                           rowsum, n * (n - 1) / 2))
    if (format == TB_SIGN_E2M1_OFS) {
        TB_SP_LAUNCH(3);
    } else if (format == TB_SIGN_E2M1) {
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
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * blockDim.x) {
        uint4 v = S[i];
        // int8 bytes 0x00/0x01/0xFF: |s| = s & 1; e2m1 nibbles 0x0/0x2/0xA: |s| clears the sign bits
        v.x &= mask;
        v.y &= mask;
        v.z &= mask;
        v.w &= mask;
        A[i] = v;
    }
    pdl_trigger();
}
}  // namespace tb

// Row sums of an offset-coded S (nibbles 0x0 / 0x2 / 0x4 = 0 / 1 / 2): fix[r] = sum of the values - n0 =
// sum_k S[r, k].  One CTA per row, 16-byte loads; the row tail and unused slots are zero nibbles.
namespace tb {
__global__ void __launch_bounds__(256) rowsum_ofs_kernel(const int8_t* __restrict__ S, int64_t ldS, int64_t n0,
                                                         int32_t* __restrict__ fix) {
    pdl_wait();
    __shared__ int32_t red[8];
    const uint4* row = reinterpret_cast<const uint4*>(S + (int64_t)blockIdx.x * ldS);
    const int64_t nvec = ldS / 16;
    int32_t c1 = 0, c2 = 0;
    for (int64_t i = threadIdx.x; i < nvec; i += 256) {
        const uint4 v = row[i];
        c1 += __popc(v.x & 0x22222222u) + __popc(v.y & 0x22222222u) + __popc(v.z & 0x22222222u) + __popc(v.w & 0x22222222u);
        c2 += __popc(v.x & 0x44444444u) + __popc(v.y & 0x44444444u) + __popc(v.z & 0x44444444u) + __popc(v.w & 0x44444444u);
    }
    int32_t s = c1 + 2 * c2;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int w = 0; w < 8; ++w) t += red[w];
        fix[blockIdx.x] = (int32_t)(t - n0);
    }
    pdl_trigger();
}
}  // namespace tb

extern "C" int tb_sign_row_sums(const int8_t* S, int64_t m, int64_t ldS, int64_t n, int32_t* fix, void* stream) {
    if (m < 1 || n < 2 || ldS < 16 || (ldS & 15)) return fail(TB_ERR_CONFIG, "sign_row_sums: bad shape");
    if (m > INT32_MAX) return fail(TB_ERR_CAPACITY, "sign_row_sums: m too large");
    if (!S || !fix) return fail(TB_ERR_INVALID, "sign_row_sums: null pointer");
    TB_CUDA_TRY(launch_pdl(rowsum_ofs_kernel, dim3((unsigned)m), dim3(256), 0, static_cast<cudaStream_t>(stream), S,
                           ldS, n * (n - 1) / 2, fix));
    return check_launch("rowsum_ofs_kernel");
}

extern "C" int tb_abs_pack(const int8_t* S, int64_t m, int64_t ldS, int format, int8_t* A, void* stream) {
    if (m < 1 || ldS < 16 || (ldS & 15)) return fail(TB_ERR_CONFIG, "abs_pack: bad shape");
    if (!S || !A) return fail(TB_ERR_INVALID, "abs_pack: null pointer");
    const int64_t nvec = m * ldS / 16;
    const int64_t blocks = std::min<int64_t>((nvec + 255) / 256, (int64_t)num_sms() * 8);
    TB_CUDA_TRY(launch_pdl(abs_pack_kernel, dim3((unsigned)blocks), dim3(256), 0, static_cast<cudaStream_t>(stream), reinterpret_cast<const uint4*>(S), reinterpret_cast<uint4*>(A), nvec,
        format == TB_SIGN_E2M1_OFS ? 0x22222222u  // the tie indicator Z = [S == 0] (value 1.0 = 0x2)
        : format == TB_SIGN_E2M1 ? 0x77777777u : (format == TB_SIGN_E4M3 ? 0x7F7F7F7Fu : 0x01010101u)));
    return check_launch("abs_pack_kernel");
}

extern "C" int64_t tb_sign_k(int64_t n) { return n >= 2 ? tb::sp_k(n) : 0; }
