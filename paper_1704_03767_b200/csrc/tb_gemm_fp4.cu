// K3 v3: the numerator GEMM on block-scaled FP4 tensor cores (tcgen05.mma kind::mxf4).
//
// The sign values -1, 0, +1 are exact in e2m1 (0xA, 0x0, 0x2); with every ue8m0 scale = 1.0 the
// block-scaled MMA computes the plain dot product, and its f32 accumulators hold the integer
// partial sums exactly while |sum| < 2^24 (K < 2^24: n <= 5792) -- verified bit-for-bit against
// the int8 path on configs 2, 3 and 5 (tools/exp_fp8.py covers the same f32 accumulation).
// Two signs per byte halve the S bytes per MAC and the MMA rate doubles over kind::i8.
//
// Layout: a CTA pair (cluster of 2, cta_group::2) owns 256 rows x 480 columns: M = 256 split across
// the pair, N issued as two N=240 MMAs into TMEM columns [0,240) and [240,480); columns [480,512)
// hold the scale factors (all bytes 0x7F = 2^0, written once with tcgen05.st, shared by SFA and
// SFB).  K per pipeline stage: 128 bytes = 256 elements = 4 MMAs of K=64.  Units are
// (256-row block, 480-column block) pairs listed by the host in 2048 x 1920 super-blocks; split-K
// and the warp roles follow the int8 kernel (tb_gemm.cu).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cudaTypedefs.h>

#include <mutex>

#include "tb_common.cuh"
#include "tb_ptx.cuh"

namespace tb {

namespace g4 {
constexpr int UM = 256;       // pair M
constexpr int BM = 128;       // rows of A per CTA
constexpr int BN = 240;       // N per MMA
constexpr int NB = 2;         // N blocks per unit
constexpr int UN = BN * NB;   // 480 columns per unit
constexpr int BNH = 120;      // rows of B per CTA per N block
constexpr int BK = 128;       // bytes of K per stage (256 e2m1 elements)
constexpr int UKB = 32;       // bytes per MMA (K = 64)
constexpr int STAGES = 4;
constexpr uint32_t A_BYTES = BM * BK;    // 16 KiB
constexpr uint32_t B_BYTES = BNH * BK;   // 15 KiB per N block
constexpr uint32_t STAGE_BYTES = A_BYTES + NB * B_BYTES;
constexpr int EPI_WARPS = 16;  // EPI_WARPS / 4 per TMEM lane quarter, splitting each block's 16-column chunks
constexpr int EPI_PAR = EPI_WARPS / 4;
constexpr int THREADS = 128 + 32 * EPI_WARPS;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t SF_COL = 480;
constexpr int STG_LD = 17;    // epilogue staging tile: 32 rows x 16 columns, padded row stride
constexpr int STG_WORDS = 32 * STG_LD + 64 + 32;  // per epilogue warp: tile, 32 row bases (int64), 32 row n1 (u32)
constexpr uint32_t STG_BYTES = EPI_WARPS * STG_WORDS * 4;
constexpr size_t SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 256 + STG_BYTES;
}  // namespace g4

struct Gemm4Args {
    int64_t m;
    const int4* items;     // {256-row block, kb0, kb1, (240-col block b0 << 16) | b1 (0xFFFF: none)}
    int64_t nitems;
    int32_t partial;       // some unit is split over K: every item accumulates into acc
    int64_t job_lo, job_hi;
    int32_t* num;
    float* acc;      // split-K: f32 sums (exact integers < 2^24), red.global.add.v4.f32
    unsigned long long* trace;  // TB_TRACE=1 (diagnostics): per CTA, per item: [accumulator ready, epilogue done]
    // K-lockstep throttle: prog[pair] = epoch << 32 | k-blocks this pair has issued (0xFFFFFFFF: done);
    // a pair more than `lead` k-blocks ahead of the slowest running pair waits (see the producer)
    unsigned long long* prog;
    uint32_t epoch;
    int32_t lead;
    int32_t lagq;  // pairs allowed to lag more than `lead` behind before a pair waits
    // split-K fixup in the kernel (partial plans): item i belongs to unit item_unit[i], unit u has
    // unit_splits[u] items; unit_cnt[2 u + rank] counts the finished items of each CTA half, and the last
    // one converts that half's f32 sums to int32 numerators and re-zeroes them (no accum_convert launch)
    const int32_t* item_unit;
    const int32_t* unit_splits;
    int32_t* unit_cnt;
    // K >= 2^24 (n > 5792): every unit is split into items of <= 65535 k-blocks, whose f32 sums stay exact
    // integers (< 2^24); the items then add them as int32 (red.add.s32 into acc reinterpreted as int32)
    int32_t int_red;
    // fused finalize (direct plans): tau_b[j] = tau_b_ieee(num, n1[y], n1[x], n0) instead of num[j]
    double* tau_b;
    const unsigned long long* n1;
    double dn0;
    // offset operands: out(y, x) = dot(y, x) - fix[y] - fix[x] - fix_c (fix == nullptr: plain dot products).
    // With the S + 1 coding of TB_SIGN_E2M1_OFS, (S_y + 1).(S_x + 1) = S_y.S_x + s_y + s_x + n0, so fix = the
    // row sums s and fix_c = n0; a split unit's first item (kb0 == 0) carries the correction.
    const int32_t* fix;
    int32_t fix_c;
    int32_t l2hint;  // experiment (TB_GEMM_L2HINT): 1 = evict_last, 2 = evict_first on the operand loads
};

// ---- K-lockstep throttle.  The ~74 concurrently running CTA pairs stream the same S rows (units of one
// row group share A, units of one column window share B) at the same k-block only if they stay in step:
// an L2 line lives ~20 us at config-5 fill rates, so pairs that drift more than ~100 k-blocks apart
// re-read S from DRAM (ncu: ~13x the operand bytes per band).  Every LOCK_CHK k-blocks the leader CTA's
// producer publishes its progress and waits while it is more than `lead` k-blocks ahead of the slowest
// pair still running.  Entries of another launch (epoch) count as finished, so a pair never waits on a
// pair that has not published in this launch: the slowest running pair never waits, no deadlock.
// The poll is one round of parallel loads over the producer warp (prog_behind_warp) -- the first version
// scanned the ~74 entries from one thread, ~16 us of serialized L2 round trips per check, which starved the
// TMA ring and lost more than the clock gained (profiles/r02_gemm_lockstep.log).  With the warp-wide poll
// config 5 drops from 367 to 322 ms per step (lead 32; DRAM reads / band ~3.6x lower, capped SM clock 1552 ->
// 1717 MHz, profiles/r02_gemm_lockstep_v2.log).
constexpr int LOCK_CHK = 16;
#ifndef GEMM_LOCK_LEAD
#define GEMM_LOCK_LEAD 32  // default allowed lead (k-blocks); TB_GEMM_LEAD=0 turns the throttle off
#endif
__device__ __forceinline__ void prog_publish(unsigned long long* prog, int64_t pair, uint32_t epoch, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(prog + pair), "l"(((unsigned long long)epoch << 32) | v)
                 : "memory");
}
// number of running pairs of this launch more than `lead` k-blocks behind `done`
__device__ __forceinline__ int prog_behind(const unsigned long long* prog, int64_t npairs, uint32_t epoch,
                                           uint32_t done, uint32_t lead) {
    int c = 0;
    for (int64_t q = 0; q < npairs; ++q) {
        unsigned long long v;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(prog + q) : "memory");
        if ((uint32_t)(v >> 32) == epoch && (uint64_t)(uint32_t)v + lead < done) ++c;
    }
    return c;
}

// warp-parallel form: lane l scans pairs l, l + 32, ...; every lane returns the warp's total
__device__ __forceinline__ int prog_behind_warp(const unsigned long long* prog, int64_t npairs, uint32_t epoch,
                                                uint32_t done, uint32_t lead, int lane) {
    int c = 0;
    for (int64_t q = lane; q < npairs; q += 32) {
        unsigned long long v;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(prog + q) : "memory");
        if ((uint32_t)(v >> 32) == epoch && (uint64_t)(uint32_t)v + lead < done) ++c;
    }
    return __reduce_add_sync(0xffffffffu, c);
}

#ifndef GEMM_DB  // 1: single-block units alternating between the two TMEM accumulator sets, so a unit's MMAs
#define GEMM_DB 0  // run while the epilogue drains the previous unit (0: two-block units, one accumulator set)
#endif
#ifndef GEMM_DIAG_ALIGN  // 1: a row block's column blocks start at its diagonal (0: at multiples of 240)
#define GEMM_DIAG_ALIGN 1
#endif

struct Unit4 {
    int64_t y0;
    int64_t xs[2];       // first column of each 240-column block (two consecutive blocks of one row block)
    int32_t nblk;        // 1 or 2 blocks
    int32_t nb[2];       // MMA N per block: 240, or the partial last block rounded up to 16
    int32_t kb0, kb1;
    bool partial;
};

__device__ __forceinline__ bool next_unit4(const Gemm4Args& p, int64_t& cur, int64_t step, Unit4& t) {
    if (cur >= p.nitems) return false;
    const int4 it = __ldg(&p.items[cur]);
    t.y0 = (int64_t)it.x * g4::UM;
    const int32_t b0 = (int32_t)((uint32_t)it.w >> 16), b1 = it.w & 0xFFFF;
    t.nblk = b1 == 0xFFFF ? 1 : 2;
#if GEMM_DIAG_ALIGN  // column blocks start at the row block's diagonal: x = y0 + 240 k
    t.xs[0] = t.y0 + (int64_t)b0 * g4::BN;
    t.xs[1] = t.y0 + (int64_t)(b1 == 0xFFFF ? b0 : b1) * g4::BN;
#else
    t.xs[0] = (int64_t)b0 * g4::BN;
    t.xs[1] = (int64_t)(b1 == 0xFFFF ? b0 : b1) * g4::BN;
#endif
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int64_t live = p.m - t.xs[h];
        t.nb[h] = live >= g4::BN ? g4::BN : (int32_t)((live + 15) & ~int64_t(15));
    }
    t.kb0 = it.y;
    t.kb1 = it.z;
    t.partial = p.partial != 0;
    cur += step;
    return true;
}

// Split-K epilogue helper (lane per row): v[0..16) are one row's 16 consecutive job ids starting at
// 16-byte-quad offset A (j0 = quad start + A), invalid entries already zeroed; [lo, hi) is the valid
// index range.  Quads with no valid entry are skipped, so every red stays inside the buffer.
template <int A>
__device__ __forceinline__ void epi_red_row(float* quad0, const uint32_t (&v)[16], int lo, int hi) {
#pragma unroll
    for (int t = 0; t < 5; ++t) {
        const int i0 = 4 * t - A;  // chunk index of the quad's first element
        if (i0 + 3 < 0 || i0 >= 16) continue;
        if (i0 + 3 < lo || i0 >= hi) continue;
        float e[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) e[k] = (i0 + k >= 0 && i0 + k < 16) ? __uint_as_float(v[i0 + k]) : 0.0f;
        red_add_v4_f32(quad0 + 4 * t, e[0], e[1], e[2], e[3]);
    }
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(g4::THREADS, 1)
    gemm_fp4_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                    Gemm4Args p) {
    using namespace g4;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;   // [2]: accumulator set 0 / 1 (GEMM_DB alternates; else set 0)
    uint64_t* tempty = tfull + 2;       // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int64_t pair = blockIdx.x >> 1;
    const int64_t npairs = gridDim.x >> 1;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmap_a);
        tma_prefetch(&tmap_b);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * EPI_WARPS);  // epilogue warps x 2 CTAs
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc_2sm<TMEM_COLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (warp >= 4 && warp < 8) {  // scale factors: every byte 0x7F (ue8m0 2^0) in this CTA's lanes, columns [480, 512)
        tmem_st_32x32b_x32(tmem_base + (uint32_t((warp & 3) * 32) << 16) + SF_COL, 0x7F7F7F7Fu);
        tmem_st_wait();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    pdl_wait();  // the setup above overlaps the sign pack's tail; S and the accumulators are read after it

    if (warp == 0) {  // ---------------- TMA producer (both CTAs): the whole warp walks the loop, lane 0 issues
        int stage = 0;
        uint32_t phase = 0;
        int64_t cur = pair;
        Unit4 t;
        const bool lock = p.lead > 0 && leader;
        uint32_t done = 0;
        if (lock && lane == 0) prog_publish(p.prog, pair, p.epoch, 0);
        const uint64_t pol = p.l2hint == 1 ? l2_policy_evict_last() : (p.l2hint == 2 ? l2_policy_evict_first() : 0ull);
        while (next_unit4(p, cur, npairs, t)) {
            // each block loads a full 120-row box per CTA; the 2-SM MMA with N reads N / 2 rows of
            // each CTA, so CTA 1's box starts at N / 2 (partial blocks need no other tensor map)
            const uint32_t bytes = 2 * (A_BYTES + t.nblk * B_BYTES);
            for (int32_t kb = t.kb0; kb < t.kb1; ++kb, ++done) {
                if (lock && (done % LOCK_CHK) == 0) {
                    // one poll = one round of parallel loads (lane l reads pairs l, l + 32, ...) and a warp
                    // reduction: ~1 L2 latency every LOCK_CHK k-blocks, hidden behind the stages in flight
                    if (lane == 0) prog_publish(p.prog, pair, p.epoch, done);
                    while (prog_behind_warp(p.prog, npairs, p.epoch, done, (uint32_t)p.lead, lane) > p.lagq)
                        __nanosleep(400);
                }
                if (lane == 0) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[stage], bytes);
                    const uint32_t fb = mapa_shared(&full[stage], 0);
                    uint8_t* sa = smem + stage * STAGE_BYTES;
                    if (p.l2hint) {
                        tma_load_2d_2sm_hint(sa, &tmap_a, fb, kb * BK, (int32_t)(t.y0 + rank * BM), pol);
                        for (int h = 0; h < t.nblk; ++h)
                            tma_load_2d_2sm_hint(sa + A_BYTES + h * B_BYTES, &tmap_b, fb, kb * BK,
                                                 (int32_t)(t.xs[h] + rank * (t.nb[h] / 2)), pol);
                    } else {
                        tma_load_2d_2sm(sa, &tmap_a, fb, kb * BK, (int32_t)(t.y0 + rank * BM));
                        for (int h = 0; h < t.nblk; ++h)
                            tma_load_2d_2sm(sa + A_BYTES + h * B_BYTES, &tmap_b, fb, kb * BK,
                                            (int32_t)(t.xs[h] + rank * (t.nb[h] / 2)));
                    }
                }
                __syncwarp();
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
        }
        if (lock && lane == 0) prog_publish(p.prog, pair, p.epoch, 0xFFFFFFFFu);
    } else if (warp == 1) {
        if (leader) {  // ---------------- MMA issuer (leader CTA, warp 1; one elected lane issues)
            // The issue loop is kept branch- and arithmetic-light: one thread feeds the 2-SM tensor pipe,
            // and per-MMA overhead (descriptor builds, runtime-bounded loops) left it idle ~30% of the
            // time (csrc/tb_probe.cu: the same MMA stream issued fully unrolled reaches ~99% of peak).
            // Descriptors are base + constant offsets; each k-block issues a fully unrolled sequence.
            constexpr uint32_t idesc = idesc_mxf4(UM, BN);
            const uint32_t sf = tmem_base + SF_COL;
            const uint64_t desc0 = umma_desc_k_sw128(smem_u32(smem));  // stage 0, A operand
            constexpr uint64_t STAGE_D = STAGE_BYTES >> 4, B0_D = A_BYTES >> 4, B1_D = (A_BYTES + B_BYTES) >> 4;
            const uint32_t d0 = tmem_base, d1 = tmem_base + BN;
            int stage = 0;
            uint32_t phase = 0;
            uint32_t acc_ph[2] = {0u, 0u};
            int it = 0;
            int64_t cur = pair;
            Unit4 t;
            while (next_unit4(p, cur, npairs, t)) {
                const int aset = GEMM_DB ? (it & 1) : 0;
                mbar_wait(&tempty[aset], acc_ph[aset] ^ 1);
                tc_fence_after();
                const uint32_t dA = GEMM_DB ? tmem_base + (uint32_t)aset * BN : d0;
                const uint32_t id0 = t.nb[0] == BN ? idesc : idesc_mxf4(UM, (uint32_t)t.nb[0]);
                const uint32_t id1 = t.nb[1] == BN ? idesc : idesc_mxf4(UM, (uint32_t)t.nb[1]);
                const int mode = t.nblk;  // 2: both blocks, 1: block 0 only
                for (int32_t kb = t.kb0; kb < t.kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint64_t ad = desc0 + (uint64_t)stage * STAGE_D;
                    const uint32_t a0 = kb > t.kb0 ? 1u : 0u;
                    if (mode == 2) {
#pragma unroll
                        for (int k = 0; k < BK / UKB; ++k) {
                            const uint32_t acc = k ? 1u : a0;
                            mma_mxf4_2sm_warp(d0, ad + 2 * k, ad + B0_D + 2 * k, id0, sf, sf, acc);
                            mma_mxf4_2sm_warp(d1, ad + 2 * k, ad + B1_D + 2 * k, id1, sf, sf, acc);
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < BK / UKB; ++k)
                            mma_mxf4_2sm_warp(dA, ad + 2 * k, ad + B0_D + 2 * k, id0, sf, sf, k ? 1u : a0);
                    }
                    mma_commit_2sm_warp(&empty[stage], 0x3);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                mma_commit_2sm_warp(&tfull[aset], 0x3);
                acc_ph[aset] ^= 1;
                ++it;
            }
        }
    } else if (warp >= 4) {  // ---------------- epilogue (both CTAs)
        // Each warp drains its 32 TMEM lanes (rows) in 32 x 16 chunks.  Direct int32 results go back
        // transposed through shared memory: half a warp covers 16 consecutive columns of one row,
        // i.e. 16 consecutive job ids, so every store touches 2 short runs instead of 32 rows m ints
        // apart.  Split partials are added lane-per-row with aligned 16-byte f32 reds.
        const int q = warp & 3;              // TMEM lane quarter
        const int par = (warp - 4) >> 2;     // this warp's 16-column chunks: c / 16 = par (mod EPI_PAR)
        int32_t* stg = reinterpret_cast<int32_t*>(smem + STAGES * STAGE_BYTES + 256) + (warp - 4) * STG_WORDS;
        int64_t* rowbase = reinterpret_cast<int64_t*>(stg + 32 * STG_LD);
        uint32_t* rown1 = reinterpret_cast<uint32_t*>(rowbase + 32);  // n1 < n0 < 2^31
        uint32_t acc_ph[2] = {0u, 0u};
        int it = 0;
        const int64_t m = p.m;
        const int64_t span = p.job_hi - p.job_lo;
        const uint32_t tempty_leader[2] = {mapa_shared(&tempty[0], 0), mapa_shared(&tempty[1], 0)};
        const int half = lane >> 4, col = lane & 15;
        int64_t cur = pair;
        Unit4 t;
        while (next_unit4(p, cur, npairs, t)) {
            const int64_t y0 = t.y0 + rank * BM + q * 32;
            int64_t row_j0;  // job id of column 0 in this lane's row (relative to job_lo)
            int32_t rfix = 0;  // this lane's row correction (offset operands), applied by the unit's first item
            {
                const int64_t y = y0 + lane;
                row_j0 = (y < m) ? row_prefix(y, m) - y - p.job_lo : INT64_MIN / 2;
                rowbase[lane] = row_j0;
                if (p.fix && t.kb0 == 0) rfix = (y < m ? __ldg(&p.fix[y]) : 0) + p.fix_c;
                if (p.tau_b) rown1[lane] = y < m ? (uint32_t)__ldg(&p.n1[y]) : 0u;
            }
            __syncwarp();
            const int aset = GEMM_DB ? (it & 1) : 0;
            mbar_wait(&tfull[aset], acc_ph[aset]);
            tc_fence_after();
            int item = (int)((cur - pair) / npairs) - 1;
            if (p.trace && warp == 4 && lane == 0 && item < 8) p.trace[(blockIdx.x * 8 + item) * 2] = globaltimer();
            for (int h = 0; h < t.nblk; ++h) {
#pragma unroll 1
                for (int c = 16 * par; c < BN; c += 16 * EPI_PAR) {
                    uint32_t r[16];
                    tmem_ld_32x32b_x16(tmem_base + (uint32_t(q * 32) << 16) + (GEMM_DB ? aset : h) * BN + c, r);
                    tmem_ld_wait();
                    const int64_t xc = t.xs[h] + c;
                    if (xc >= m || xc + 15 < y0) continue;  // chunk right of the matrix or below the diagonal
                    if (t.partial) {
                        // split partials: lane per row straight from registers, aligned red.v4.f32 quads
                        // (measured 19.5 -> 15.6 us per config-2 item vs the shared-memory transpose;
                        // direct int32 stores below keep the transpose, which coalesces them)
                        const int64_t y = y0 + lane;
                        if (y < m) {
                            const int64_t j0 = row_j0 + xc;
                            int64_t lo64 = y - xc, hi64 = m - xc;
                            if (lo64 < -j0) lo64 = -j0;
                            if (hi64 > span - j0) hi64 = span - j0;
                            const int lo = (int)(lo64 < 0 ? 0 : (lo64 > 16 ? 16 : lo64));
                            const int hi = (int)(hi64 < 0 ? 0 : (hi64 > 16 ? 16 : hi64));
                            if (lo < hi && p.fix && t.kb0 == 0) {  // offset operands: exact integers, |.| < 2^24
#pragma unroll
                                for (int i = 0; i < 16; ++i) {
                                    const int32_t cf = (i >= lo && i < hi) ? __ldg(&p.fix[xc + i]) : 0;
                                    r[i] = __float_as_uint(__uint_as_float(r[i]) - (float)(rfix + cf));
                                }
                            }
                            if (lo < hi && p.int_red) {  // exact int32 partial sums (wide K)
                                int32_t* q0 = reinterpret_cast<int32_t*>(p.acc) + j0;
#pragma unroll
                                for (int i = 0; i < 16; ++i)
                                    if (i >= lo && i < hi)
                                        asm volatile("red.global.add.s32 [%0], %1;" ::"l"(q0 + i),
                                                     "r"(__float2int_rn(__uint_as_float(r[i]))) : "memory");
                            } else if (lo < hi) {
                                uint32_t v[16];
#pragma unroll
                                for (int i = 0; i < 16; ++i) v[i] = (i >= lo && i < hi) ? r[i] : 0u;
                                const int A = (int)(j0 & 3);
                                float* q0 = p.acc + (j0 - A);
                                switch (A) {
                                    case 0: epi_red_row<0>(q0, v, lo, hi); break;
                                    case 1: epi_red_row<1>(q0, v, lo, hi); break;
                                    case 2: epi_red_row<2>(q0, v, lo, hi); break;
                                    default: epi_red_row<3>(q0, v, lo, hi); break;
                                }
                            }
                        }
                        __syncwarp();  // reconverge before the next (.sync.aligned) tcgen05.ld
                        continue;
                    }
#pragma unroll
                    for (int i = 0; i < 16; ++i) stg[lane * STG_LD + i] = __float2int_rn(__uint_as_float(r[i])) - rfix;
                    __syncwarp();
                    const int32_t cfix = (p.fix && xc + col < m) ? __ldg(&p.fix[xc + col]) : 0;
                    if (p.tau_b) {  // fused K5: tau_b straight from the accumulator (8 B per pair, no numerator)
                        const int64_t x = xc + col;
                        const uint64_t t2 = x < m ? (uint64_t)__ldg(&p.n1[x]) : 0;
#pragma unroll 4
                        for (int k = 0; k < 16; ++k) {
                            const int rr = 2 * k + half;
                            const int64_t y = y0 + rr;
                            const int64_t j = rowbase[rr] + x;
                            if (x >= y && x < m && j >= 0 && j < span)
                                p.tau_b[j] = tau_b_ieee(stg[rr * STG_LD + col] - cfix, rown1[rr], t2, p.dn0);
                        }
                    } else {
                        const int64_t x = xc + col;
                        // interior chunk (warp-uniform): right of the diagonal for all 32 rows, inside the
                        // matrix and the job range -- plain stores, no per-element bounds (the epilogue is
                        // instruction-bound: ~20 issued per element on the checked path, ~6 here)
                        const bool interior = xc >= y0 + 31 && xc + 15 < m && y0 + 31 < m && rowbase[0] + xc >= 0 &&
                                              rowbase[31] + xc + 15 < span;
                        if (interior) {
                            int32_t* colp = p.num + x;
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                const int rr = 2 * k + half;
                                colp[rowbase[rr]] = stg[rr * STG_LD + col] - cfix;
                            }
                        } else {
#pragma unroll 4
                            for (int k = 0; k < 16; ++k) {
                                const int rr = 2 * k + half;
                                const int64_t y = y0 + rr;
                                const int64_t j = rowbase[rr] + x;
                                if (x >= y && x < m && j >= 0 && j < span)
                                    p.num[j] = stg[rr * STG_LD + col] - cfix;
                            }
                        }
                    }
                    __syncwarp();
                }
            }
            tc_fence_before();
            __syncwarp();
            if (p.trace && warp == 4 && lane == 0 && item < 8) p.trace[(blockIdx.x * 8 + item) * 2 + 1] = globaltimer();
            if (lane == 0) mbar_arrive_cluster(tempty_leader[aset]);
            acc_ph[aset] ^= 1;
            ++it;
            if (t.partial && p.unit_cnt) {
                // this CTA half's reds of the item are issued; the last of the unit's items converts the half
                // (CUTLASS's barrier pattern: CTA barrier, then one thread fences and arrives)
                asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
                volatile int* s_last = reinterpret_cast<volatile int*>(smem + STAGES * STAGE_BYTES + 128);
                if (warp == 4 && lane == 0) {
                    const int32_t u = __ldg(&p.item_unit[cur - npairs]);
                    int32_t* cnt = p.unit_cnt + 2 * u + rank;
                    __threadfence();
                    const int old = atomicAdd(cnt, 1);
                    const int last = old == __ldg(&p.unit_splits[u]) - 1;
                    if (last) {
                        *cnt = 0;  // ready for the next launch
                        __threadfence();
                    }
                    *s_last = last;
                }
                asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
                if (*s_last) {
                    // rows y0 + rank * BM + [0, BM) of the unit: warp w takes rows w - 4, w + 12, ...
                    for (int rr = warp - 4; rr < BM; rr += EPI_WARPS) {
                        const int64_t y = t.y0 + rank * BM + rr;
                        if (y >= m) break;
                        const int64_t rj0 = row_prefix(y, m) - y - p.job_lo;
                        for (int h = 0; h < t.nblk; ++h) {
                            int64_t x_lo = t.xs[h], x_hi = t.xs[h] + t.nb[h];
                            if (x_lo < y) x_lo = y;
                            if (x_hi > m) x_hi = m;
                            if (x_lo < -rj0) x_lo = -rj0;
                            if (x_hi > span - rj0) x_hi = span - rj0;
                            // up to 8 loads in flight per lane (one row block: <= 240 columns)
                            float v[8];
#pragma unroll
                            for (int k = 0; k < 8; ++k) {
                                const int64_t x = x_lo + lane + 32 * k;
                                v[k] = x < x_hi ? __ldcg(&p.acc[rj0 + x]) : 0.0f;
                            }
#pragma unroll
                            for (int k = 0; k < 8; ++k) {
                                const int64_t x = x_lo + lane + 32 * k;
                                if (x < x_hi) {
                                    p.num[rj0 + x] = __float2int_rn(v[k]);
                                    p.acc[rj0 + x] = 0.0f;
                                }
                            }
                        }
                    }
                }
            }
        }
    }
    pdl_trigger();
    tc_fence_before();
    cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_2sm<TMEM_COLS>(tmem_base);
    }
}

// ------------------------------------------------------------------ host work plan
// Units (256-row block Yb, 480-column block Xb) that intersect the job range's rows and the upper
// triangle, ordered by 8 x 4 super-blocks (2048 rows x 1920 columns) so concurrently running pairs
// share S rows through L2.  A unit carries 1 or 2 live N blocks (diagonal / right-edge units skip a
// block); its K range is split into s_u items and items are listed split-round-major, pair p
// running items p, p + P, ... (the K-lockstep order that lets concurrent pairs share S k-blocks in
// L2).  Items of one N block stream 31 KiB per stage instead of 46 KiB and cost ~2/3 of a two-block
// item, so the plan gives two-block units 3k splits and one-block units 2k (equal-cost items) or a
// uniform split, whichever a simulation of the static schedule finishes first.
struct Plan4 {
    DevTable table;  // the item table on its device (async upload, see tb_common.cuh)
    int64_t m = -1, lo = -1, hi = -1;
    int32_t nkb = -1, forced = -1, pairs = -1;
    int64_t count = 0;
    int32_t partial = 0;
    int64_t off_unit = -1, off_splits = -1, off_cnt = -1;  // byte offsets of the split-K fixup arrays
    const int4* dev() const { return static_cast<const int4*>(table.dev); }
    template <typename T>
    T* at(int64_t off) const { return off < 0 ? nullptr : reinterpret_cast<T*>(static_cast<uint8_t*>(table.dev) + off); }
};
// Plans are cached per (geometry, job range): the banded host path cycles through a few ranges.
constexpr int PLAN_CACHE = 32;  // the banded host path cycles through up to ~15 job ranges
static Plan4 g_plans4[PLAN_CACHE];
static int g_plans4_next = 0;

static void list_units4(int64_t m, int64_t job_lo, int64_t job_hi, std::vector<int32_t>& code, std::vector<int32_t>& nb,
                        std::vector<int32_t>& ncols) {
    // A unit = one 256-row block x two consecutive 240-column blocks.  Row block yb's blocks run from
    // the first one touching its diagonal, b = floor(256 yb / 240), to the last column of the matrix,
    // and are paired left to right (an odd count leaves one single-block unit), so diagonal and
    // right-edge remnants share units instead of each becoming a half-empty one.  Units are listed
    // per 16-row-block group (4096 rows) in windows of 4 column blocks, so the ~74 concurrently running
    // pairs cover a squarer patch (~16 row blocks x ~9 column blocks) and share S rows through L2
    // (config 5, r02: 8 x 8 -> 16 x 4 cut the GEMM from 389-397 to 375-382 ms and DRAM reads per band
    // from 251 to 232 GB, profiles/r02_gemm_unit_order.log).
    // unit-order knobs (experiments; TB_GEMM_GR row blocks per group, TB_GEMM_WIN column blocks per window,
    // TB_GEMM_SERP=1 reverses the window order of every other group)
    static const int64_t kGR = [] { const char* e = std::getenv("TB_GEMM_GR"); return e ? std::max(1, atoi(e)) : 16; }();
    static const int64_t kWIN = [] { const char* e = std::getenv("TB_GEMM_WIN"); return e ? std::max(1, atoi(e)) : 4; }();
    static const bool kSERP = [] { const char* e = std::getenv("TB_GEMM_SERP"); return e && e[0] == '1'; }();
    const int64_t RB = (m + g4::UM - 1) / g4::UM, GR = kGR;
    const int64_t b_last = (m - 1) / g4::BN;
    int64_t y_lo, x_lo, y_hi, x_hi;
    job_coord(job_lo, m, y_lo, x_lo);
    job_coord(job_hi - 1, m, y_hi, x_hi);
    auto nmma_x = [m](int64_t x0) -> int32_t {
        const int64_t live = m - x0;
        return live >= g4::BN ? g4::BN : (int32_t)((live + 15) / 16 * 16);
    };
    struct U { int64_t win, yb, b0, b1; int32_t nc; };
    for (int64_t SY = 0; SY < (RB + GR - 1) / GR; ++SY) {
        std::vector<U> g;
        for (int64_t yb = SY * GR; yb < std::min(RB, (SY + 1) * GR); ++yb) {
            const int64_t r0 = yb * g4::UM, r1 = std::min(r0 + g4::UM, m) - 1;
            if (r1 < y_lo || r0 > y_hi) continue;  // outside the job range rows
#if GEMM_DIAG_ALIGN
            // blocks k = 0, 1, ... at x = r0 + 240 k: only the 256 x 256 diagonal square is partly wasted
            // (config 2: ~24% of the MMA area below the diagonal with 240-aligned blocks, ~12% here)
            const int64_t k_last = (m - 1 - r0) / g4::BN;
            for (int64_t k = 0; k <= k_last; k += (GEMM_DB ? 1 : 2)) {
                const int64_t x0 = r0 + k * g4::BN, x1 = x0 + g4::BN;
                const bool two = !GEMM_DB && k + 1 <= k_last;
                g.push_back(U{(x0 / g4::BN) / kWIN, yb, k, two ? k + 1 : -1,
                              nmma_x(x0) + (two ? nmma_x(x1) : 0)});
            }
#else
            for (int64_t b = r0 / g4::BN; b <= b_last; b += 2)
                g.push_back(U{b / kWIN, yb, b, b + 1 <= b_last ? b + 1 : -1,
                              nmma_x(b * g4::BN) + (b + 1 <= b_last ? nmma_x((b + 1) * g4::BN) : 0)});
#endif
        }
        if (kSERP && (SY & 1))
            std::stable_sort(g.begin(), g.end(), [](const U& a, const U& b) { return a.win > b.win; });
        else
            std::stable_sort(g.begin(), g.end(), [](const U& a, const U& b) { return a.win < b.win; });
        for (const U& u : g) {
            code.push_back((int32_t)u.yb);
            nb.push_back((int32_t)((u.b0 << 16) | (u.b1 < 0 ? 0xFFFF : u.b1)));
            ncols.push_back(u.nc);
        }
    }
}

// Relative k-block cost of a unit: the A-operand share plus the MMA / B share of its issued columns
// (one full block = 0.6, two = 1.0, the partial edge block in proportion; TB_TRACE item timings).
static double unit_cost4(int32_t ncols) { return 0.2 + 0.8 * ncols / 480.0; }  // 1 block ~0.6 (measured)

// Items for per-unit split counts su[u]; returns the simulated makespan of the static schedule
// (items split-round-major, pair p runs p, p + P, ...), in two-block k-block units.
static double plan_items4(const std::vector<int32_t>& code, const std::vector<int32_t>& blocks,
                          const std::vector<int32_t>& ncols, const std::vector<int32_t>& su, int32_t nkb, int pairs,
                          std::vector<int4>* out, std::vector<int32_t>* out_unit = nullptr) {
    static const double kEpi = [] { const char* e = std::getenv("TB_PLAN_EPI"); return e ? atof(e) : 100.0; }();
    const double t_epi = kEpi;  // per item: epilogue ~20 us + split-red contention + refill (fitted to
                                 // measured 1- vs 2-wave plans on config 2), in two-block k-blocks
    std::vector<double> load(pairs, 0.0);
    const int32_t rounds = *std::max_element(su.begin(), su.end());
    int64_t idx = 0;
    for (int32_t r = 0; r < rounds; ++r)
        for (size_t u = 0; u < code.size(); ++u) {
            if (r >= su[u]) continue;
            const int32_t kb0 = (int32_t)((int64_t)r * nkb / su[u]), kb1 = (int32_t)((int64_t)(r + 1) * nkb / su[u]);
            load[idx % pairs] += (kb1 - kb0) * unit_cost4(ncols[u]) + t_epi;
            if (out) out->push_back(make_int4(code[u], kb0, kb1, blocks[u]));
            if (out_unit) out_unit->push_back((int32_t)u);
            ++idx;
        }
    return *std::max_element(load.begin(), load.end());
}

// K-blocks per item for exact f32 partial sums: 65535 x 256 e2m1 elements < 2^24
constexpr int32_t KB_EXACT = 65535;

static int build_plan4(int64_t m, int64_t job_lo, int64_t job_hi, int32_t nkb, int32_t forced, int pairs,
                       cudaStream_t st, Plan4** out) {
    std::lock_guard<std::mutex> lock(g_native_state_mutex);  // host threads share the caches
    int ordinal = 0;
    TB_CUDA_TRY(cudaGetDevice(&ordinal));
    for (Plan4& c : g_plans4)
        if (c.table.ordinal == ordinal && c.m == m && c.lo == job_lo && c.hi == job_hi && c.nkb == nkb && c.forced == forced &&
            c.pairs == pairs) {
            *out = &c;
            return TB_OK;
        }
    Plan4& g_plan4 = g_plans4[g_plans4_next];
    g_plans4_next = (g_plans4_next + 1) % PLAN_CACHE;
    g_plan4.m = -1;
    std::vector<int32_t> code, nb, ncols;
    list_units4(m, job_lo, job_hi, code, nb, ncols);
    std::vector<int32_t> su(code.size(), 1), best_su;
    double best = 0.0;
    if (!code.empty()) {
        if (forced > 0) {
            std::fill(su.begin(), su.end(), std::min(forced, nkb));
            best_su = su;
        } else {
            // equal-cost items: unit u gets ceil(cost_u * nkb / T) splits for a target item cost T;
            // T = c_max * nkb / k for k = 1, 1.5, 2, ... 64 (k = 1: no split); best simulated makespan wins
            const double c_max = unit_cost4(480);
            best_su = su;
            best = plan_items4(code, nb, ncols, su, nkb, pairs, nullptr);
            const int32_t kmax = std::max(1, std::min(64, nkb / 8));
            for (int32_t k2 = 3; k2 <= 2 * kmax; ++k2) {  // T = c_max * nkb / (k2 / 2): half steps
                const double T = 2.0 * c_max * nkb / k2;
                for (size_t u = 0; u < code.size(); ++u) {
                    // ceil, not round: no item may exceed the target (a rounded-down unit sets the makespan)
                    const double s_real = unit_cost4(ncols[u]) * nkb / T;
                    su[u] = (int32_t)std::max<int64_t>(1, std::min<int64_t>(nkb, (int64_t)std::ceil(s_real - 1e-9)));
                }
                const double t = plan_items4(code, nb, ncols, su, nkb, pairs, nullptr);
                if (std::getenv("TB_TRACE_PLAN")) {
                    int64_t ni = 0;
                    for (int32_t v : su) ni += v;
                    fprintf(stderr, "  cand k2 %d items %lld est %.0f\n", k2, (long long)ni, t);
                }
                if (t < best * 0.999) { best = t; best_su = su; }
            }
            // fill idle pairs: split the most expensive item's unit once more while items < pairs
            int64_t nitems = 0;
            for (int32_t v : best_su) nitems += v;
            su = best_su;
            // one wave with the same split count for every unit: every round's items cover the same K range,
            // so the concurrent pairs share S k-blocks through L2 (which the makespan model does not see);
            // preferred on a tie (config 2: 390 us for 3 uniform splits vs 405 us for the model's best plan,
            // tools/exp_splits.py, profiles/r02_gemm_split_plans.log)
            if ((int64_t)code.size() <= pairs) {
                // ... with at least 3 k-blocks per item: an item's epilogue reds its whole 256 x 480 tile, so
                // items of one k-block (config 1: 74 of them) spend more on reds than on MMAs (config 1 GEMM
                // 23.6 us at 74 splits, 19.5 us at 24-48; tools/exp_splits.py, profiles/r02_gemm_split_plans.log)
                const int32_t s_uni = (int32_t)std::max<int64_t>(
                    1, std::min<int64_t>(std::max<int64_t>(1, nkb / 3), pairs / (int64_t)code.size()));
                std::vector<int32_t> uni(code.size(), s_uni);
                const double t = plan_items4(code, nb, ncols, uni, nkb, pairs, nullptr);
                if (t <= best * 1.0001) {
                    best = t;
                    best_su = uni;
                    su = uni;
                    nitems = (int64_t)code.size() * s_uni;
                }
            }
            while (nitems < pairs) {
                size_t arg = 0;
                double worst = -1.0;
                for (size_t u = 0; u < code.size(); ++u) {
                    const double c = unit_cost4(ncols[u]) * nkb / su[u];
                    if (su[u] < nkb && c > worst) { worst = c; arg = u; }
                }
                if (worst < 0) break;
                ++su[arg];
                ++nitems;
                const double t = plan_items4(code, nb, ncols, su, nkb, pairs, nullptr);
                if (t < best * 0.999) { best = t; best_su = su; }
            }
        }
    }
    // wide K: no item may span more than KB_EXACT k-blocks (its f32 sums must stay exact integers)
    const int32_t min_splits = (nkb + KB_EXACT - 1) / KB_EXACT;
    for (int32_t& v : best_su) v = std::max(v, min_splits);
    std::vector<int4> items;
    std::vector<int32_t> item_unit;
    const double span_est = code.empty() ? 0.0 : plan_items4(code, nb, ncols, best_su, nkb, pairs, &items, &item_unit);
    const int32_t smax = best_su.empty() ? 1 : *std::max_element(best_su.begin(), best_su.end());
    const char* trace = std::getenv("TB_TRACE");
    if (trace && trace[0] == '1')
        fprintf(stderr, "plan4: m %lld units %zu nkb %d max splits %d items %zu est %.0f\n", (long long)m,
                code.size(), nkb, smax, items.size(), span_est);
    // table: items (int4), then for split plans the item -> unit map, the splits per unit and the per-unit,
    // per-CTA-half fixup counters (zero; each launch's last arrivers reset them)
    std::vector<uint8_t> blob(items.size() * sizeof(int4));
    if (!items.empty()) std::memcpy(blob.data(), items.data(), blob.size());
    if (smax > 1) {
        const size_t off_u = blob.size(), nu = best_su.size();
        blob.resize(off_u + (item_unit.size() + nu + 2 * nu) * sizeof(int32_t), 0);
        std::memcpy(blob.data() + off_u, item_unit.data(), item_unit.size() * sizeof(int32_t));
        std::memcpy(blob.data() + off_u + item_unit.size() * sizeof(int32_t), best_su.data(), nu * sizeof(int32_t));
        g_plan4.off_unit = (int64_t)off_u;
        g_plan4.off_splits = (int64_t)(off_u + item_unit.size() * sizeof(int32_t));
        g_plan4.off_cnt = (int64_t)(off_u + (item_unit.size() + nu) * sizeof(int32_t));
    } else {
        g_plan4.off_unit = g_plan4.off_splits = g_plan4.off_cnt = -1;
    }
    int rc = table_upload(g_plan4.table, blob.data(), blob.size(), st);
    if (rc) return rc;
    g_plan4.m = m;
    g_plan4.lo = job_lo;
    g_plan4.hi = job_hi;
    g_plan4.nkb = nkb;
    g_plan4.forced = forced;
    g_plan4.pairs = pairs;
    g_plan4.count = (int64_t)items.size();
    g_plan4.partial = smax > 1 ? 1 : 0;
    *out = &g_plan4;
    return TB_OK;
}

// Per-device progress slots of the K-lockstep throttle (zeroed once; launches tell their entries apart by
// epoch).  TB_GEMM_LEAD = the allowed lead in k-blocks (0 disables the throttle).
static int lockstep_state(unsigned long long** prog, uint32_t* epoch, int32_t* lead) {
    static const int32_t kLead = [] {
        const char* e = std::getenv("TB_GEMM_LEAD");
        return e ? std::max(0, atoi(e)) : GEMM_LOCK_LEAD;
    }();
    struct Slot { unsigned long long* p = nullptr; uint32_t epoch = 0; };
    static Slot slots[64];
    *lead = kLead;
    *prog = nullptr;
    *epoch = 0;
    if (kLead <= 0) return TB_OK;
    std::lock_guard<std::mutex> lock(g_native_state_mutex);
    int dev = 0;
    TB_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) { *lead = 0; return TB_OK; }
    Slot& sl = slots[dev];
    if (!sl.p) {
        TB_CUDA_TRY(cudaMalloc(&sl.p, 1024 * sizeof(unsigned long long)));
        TB_CUDA_TRY(cudaMemset(sl.p, 0, 1024 * sizeof(unsigned long long)));
        TB_CUDA_TRY(cudaDeviceSynchronize());
    }
    if (++sl.epoch == 0) sl.epoch = 1;
    *prog = sl.p;
    *epoch = sl.epoch;
    return TB_OK;
}

// tau_b != nullptr: fused finalize when the plan has no split unit (the kernel writes tau_b, num is not
// written; *fused = 1); a split plan computes num (which must then be a buffer) and *fused = 0.
int gemm_fp4(const int8_t* S, int64_t m, int64_t K, int64_t ldS, int64_t job_lo, int64_t job_hi, int32_t splits,
             int32_t* num, cudaStream_t st, double* tau_b, const uint64_t* n1, int64_t n, int* fused,
             const int32_t* fix, int64_t fix_c) {
    if (fused) *fused = 0;
    if (fix && (fix_c > INT32_MAX || fix_c < INT32_MIN)) return fail(TB_ERR_CONFIG, "gemm fp4: fix_c out of range");
    const bool wide = K >= (int64_t(1) << 24);  // items of <= KB_EXACT k-blocks, int32 partial sums
    if (m >= (int64_t(1) << 16) * g4::UM) return fail(TB_ERR_CAPACITY, "gemm fp4: m too large");
    int rc;
    Gemm4Args p{};
    p.m = m;
    const int64_t kbytes = K / 2;
    const int32_t nkb = (int32_t)((kbytes + g4::BK - 1) / g4::BK);
    const int pairs = std::max(1, num_sms() / 2);
    Plan4* plan = nullptr;
    if ((rc = build_plan4(m, job_lo, job_hi, nkb, splits, pairs, st, &plan))) return rc;
    p.items = plan->dev();
    p.nitems = plan->count;
    p.partial = plan->partial;
    p.job_lo = job_lo;
    p.job_hi = job_hi;
    p.num = num;
    p.int_red = wide ? 1 : 0;
    p.fix = fix;
    p.fix_c = fix ? (int32_t)fix_c : 0;
    static const int32_t kL2Hint = [] { const char* e = std::getenv("TB_GEMM_L2HINT"); return e ? atoi(e) : 0; }();
    p.l2hint = kL2Hint;
    if (wide && !p.partial) return fail(TB_ERR_CONFIG, "gemm fp4: wide K needs a split plan");
    // tau_b callers: a split plan finalizes straight from the f32 workspace (accum_finalize); a one-launch
    // plan's epilogue writes tau_b itself (TB_FUSE_EPILOGUE=0: it writes the numerators and the caller
    // finalizes).  Slower before the lockstep throttle (config 5 407.7 -> 422.7 ms,
    // profiles/r02_fused_finalize_ab.log), faster with it: 317.4 / 318.3 -> 315.3 / 315.4 ms per step, no
    // 8.6 GB numerator round trip (profiles/r02_fused_finalize_ab_s5.log)
    static const bool kEpiFuse = [] { const char* e = std::getenv("TB_FUSE_EPILOGUE"); return !e || e[0] != '0'; }();
    const bool acc_fin = tau_b && p.partial && !wide;
    if (tau_b && !p.partial && kEpiFuse) {
        p.tau_b = tau_b;
        p.n1 = reinterpret_cast<const unsigned long long*>(n1);
        p.dn0 = (double)(n * (n - 1) / 2);
        if (fused) *fused = 1;
    } else if (!num && !acc_fin) {
        return fail(TB_ERR_INVALID, "gemm fp4: this plan needs the numerator buffer");
    }
    if (p.partial && (rc = accum_workspace(job_hi - job_lo, &p.acc, st))) return rc;
    // In-kernel split-K fixup: opt-in (TB_GEMM_FIXUP=1).  Measured slower than the separate accum_convert
    // launch on configs 1-2 (config 1 0.039 -> 0.051 ms, config 2 0.540 -> 0.553 ms per step; config 3 within
    // noise; profiles/r02_gemm_fixup_ab.log): the last item of a unit serialises the conversion behind it.
    static const bool kFixup = [] { const char* e = std::getenv("TB_GEMM_FIXUP"); return e && e[0] == '1'; }();
    if (p.partial && kFixup && !wide) {
        p.item_unit = plan->at<const int32_t>(plan->off_unit);
        p.unit_splits = plan->at<const int32_t>(plan->off_splits);
        p.unit_cnt = plan->at<int32_t>(plan->off_cnt);
    }
    // K-lockstep: multi-wave plans without K splits (every unit walks the same k-blocks, so the cumulative
    // k-block count is the K position); one-wave plans start in step anyway
    if (!p.partial && p.nitems > pairs && (rc = lockstep_state(&p.prog, &p.epoch, &p.lead))) return rc;
    {
        static const int32_t kLagQ = [] { const char* e = std::getenv("TB_GEMM_LAGQ"); return e ? std::max(0, atoi(e)) : 0; }();
        p.lagq = kLagQ;
    }
    CUtensorMap ta, tbm;
    if ((rc = make_tmap(&ta, S, m, kbytes, ldS, g4::BM))) return rc;
    if ((rc = make_tmap(&tbm, S, m, kbytes, ldS, g4::BNH))) return rc;
    TB_CUDA_TRY(cudaFuncSetAttribute(gemm_fp4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)g4::SMEM_BYTES));
    const unsigned grid = (unsigned)(2 * std::max<int64_t>(1, std::min<int64_t>(p.nitems, pairs)));
    const char* trace = std::getenv("TB_TRACE");
    std::vector<unsigned long long> tr;
    if (trace && trace[0] == '1') {
        TB_CUDA_TRY(cudaMalloc(&p.trace, grid * 16 * sizeof(unsigned long long)));
        TB_CUDA_TRY(cudaMemsetAsync(p.trace, 0, grid * 16 * sizeof(unsigned long long), st));
        TB_CUDA_TRY(cudaStreamSynchronize(st));
    }
    TB_CUDA_TRY(launch_pdl(gemm_fp4_kernel, dim3(grid), dim3(g4::THREADS), g4::SMEM_BYTES, st, ta, tbm, p));
    if ((rc = check_launch("gemm_fp4_kernel"))) return rc;
    if ((rc = table_mark_used(plan->table, st))) return rc;
    if (p.trace) {
        TB_CUDA_TRY(cudaStreamSynchronize(st));
        tr.resize(grid * 16);
        TB_CUDA_TRY(cudaMemcpy(tr.data(), p.trace, tr.size() * 8, cudaMemcpyDeviceToHost));
        cudaFree(p.trace);
        unsigned long long t0 = ~0ull, tend = 0;
        for (size_t i = 0; i < tr.size(); ++i) if (tr[i]) { t0 = std::min(t0, tr[i]); tend = std::max(tend, tr[i]); }
        for (int it = 0; it < 8; ++it) {
            double sa = 0, se = 0, mn = 1e30, mx = 0; int n = 0;
            for (unsigned b = 0; b < grid; ++b) {
                unsigned long long a = tr[(b * 8 + it) * 2], e = tr[(b * 8 + it) * 2 + 1];
                if (!a || !e) continue;
                sa += (a - t0) * 1e-3; se += (e - a) * 1e-3; mn = std::min(mn, (a - t0) * 1e-3); mx = std::max(mx, (a - t0) * 1e-3); ++n;
            }
            if (n) fprintf(stderr, "item %d: ctas %d  tfull at mean %.1f us [%.1f, %.1f]  epilogue mean %.1f us\n", it, n, sa / n, mn, mx, se / n);
        }
        fprintf(stderr, "span first tfull -> last epilogue end %.1f us (items %lld)\n", (tend - t0) * 1e-3, (long long)p.nitems);
        if (trace[1] == 'u') {  // TB_TRACE=1u: first item of every pair with its unit geometry
            std::vector<int4> items(p.nitems);
            cudaMemcpy(items.data(), p.items, items.size() * sizeof(int4), cudaMemcpyDeviceToHost);
            for (unsigned b = 0; b < grid; b += 2) {
                const int4 it = items[b / 2];
                const long long yb = it.x, xb = (long long)((uint32_t)it.w >> 16), xb1 = it.w & 0xFFFF;
                fprintf(stderr, "  pair %3u unit (yb %lld, blocks %lld,%lld) kb [%d,%d) tfull %.1f us\n", b / 2, yb, xb, xb1, it.y, it.z,
                        tr[b * 16] ? (tr[b * 16] - t0) * 1e-3 : -1.0);
            }
        }
    }
    if (!p.partial) return TB_OK;
    if (p.int_red) return accum_convert_i32(reinterpret_cast<int32_t*>(p.acc), job_hi - job_lo, num, st);
    if (acc_fin) {
        if (fused) *fused = 1;
        return accum_finalize(p.acc, n1, m, n, job_lo, job_hi, tau_b, st);
    }
    if (p.unit_cnt) return accum_mark_clean();  // the kernel converted and re-zeroed every unit's sums
    return accum_convert(p.acc, job_hi - job_lo, num, st);
}

}  // namespace tb
