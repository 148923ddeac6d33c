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
#include <cstdlib>
#include <vector>
#include <cudaTypedefs.h>

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
constexpr int THREADS = 256;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t SF_COL = 480;
constexpr size_t SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 256;
}  // namespace g4

struct Gemm4Args {
    int64_t m;
    const int32_t* units;  // (row block << 16) | column block, rasterised
    int64_t nunits;        // per split
    int32_t splits;
    int32_t nkb;           // 128-byte K blocks
    int64_t job_lo, job_hi;
    int32_t* num;
};

struct Unit4 {
    int64_t y0, x0;
    int32_t h_lo;
    int32_t kb0, kb1;
    bool partial;
};

__device__ __forceinline__ bool next_unit4(const Gemm4Args& p, int64_t& cur, int64_t step, Unit4& t) {
    if (cur >= p.nunits * p.splits) return false;
    const int32_t s = (int32_t)(cur / p.nunits);
    const int64_t i = cur - (int64_t)s * p.nunits;
    const int32_t e = p.units[i];
    t.y0 = (int64_t)(e >> 16) * g4::UM;
    t.x0 = (int64_t)(e & 0xFFFF) * g4::UN;
    t.h_lo = (t.x0 + g4::BN - 1 < t.y0) ? 1 : 0;
    t.kb0 = (int32_t)((int64_t)s * p.nkb / p.splits);
    t.kb1 = (int32_t)((int64_t)(s + 1) * p.nkb / p.splits);
    t.partial = p.splits > 1;
    cur += step;
    return true;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(g4::THREADS, 1)
    gemm_fp4_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                    Gemm4Args p) {
    using namespace g4;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

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
        mbar_init(tfull, 1);
        mbar_init(tempty, 8);  // 4 epilogue warps x 2 CTAs
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc_2sm<TMEM_COLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (warp >= 4) {  // scale factors: every byte 0x7F (ue8m0 2^0) in this CTA's lanes, columns [480, 512)
        tmem_st_32x32b_x32(tmem_base + (uint32_t((warp & 3) * 32) << 16) + SF_COL, 0x7F7F7F7Fu);
        tmem_st_wait();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer (both CTAs)
            int stage = 0;
            uint32_t phase = 0;
            int64_t cur = pair;
            Unit4 t;
            while (next_unit4(p, cur, npairs, t)) {
                const uint32_t bytes = 2 * (A_BYTES + (NB - t.h_lo) * B_BYTES);
                for (int32_t kb = t.kb0; kb < t.kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[stage], bytes);
                    const uint32_t fb = mapa_shared(&full[stage], 0);
                    uint8_t* sa = smem + stage * STAGE_BYTES;
                    tma_load_2d_2sm(sa, &tmap_a, fb, kb * BK, (int32_t)(t.y0 + rank * BM));
                    for (int h = t.h_lo; h < NB; ++h)
                        tma_load_2d_2sm(sa + A_BYTES + h * B_BYTES, &tmap_b, fb, kb * BK,
                                        (int32_t)(t.x0 + h * BN + rank * BNH));
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {  // ---------------- MMA issuer (leader CTA, one thread)
            constexpr uint32_t idesc = idesc_mxf4(UM, BN);
            const uint32_t sf = tmem_base + SF_COL;
            int stage = 0;
            uint32_t phase = 0;
            uint32_t acc_phase = 0;
            int64_t cur = pair;
            Unit4 t;
            while (next_unit4(p, cur, npairs, t)) {
                mbar_wait(tempty, acc_phase ^ 1);
                tc_fence_after();
                for (int32_t kb = t.kb0; kb < t.kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
                    const uint64_t adesc = umma_desc_k_sw128(sa);
#pragma unroll
                    for (int k = 0; k < BK / UKB; ++k) {
                        const uint32_t acc = (kb > t.kb0 || k > 0) ? 1u : 0u;
                        for (int h = t.h_lo; h < NB; ++h) {
                            const uint64_t bdesc = umma_desc_k_sw128(sa + A_BYTES + h * B_BYTES);
                            mma_mxf4_2sm(tmem_base + h * BN, adesc + 2 * k, bdesc + 2 * k, idesc, sf, sf, acc);
                        }
                    }
                    mma_commit_2sm(&empty[stage], 0x3);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                mma_commit_2sm(tfull, 0x3);
                acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {  // ---------------- epilogue (both CTAs)
        const int q = warp & 3;
        uint32_t acc_phase = 0;
        const int64_t m = p.m;
        const int64_t span = p.job_hi - p.job_lo;
        const uint32_t tempty_leader = mapa_shared(tempty, 0);
        int64_t cur = pair;
        Unit4 t;
        while (next_unit4(p, cur, npairs, t)) {
            mbar_wait(tfull, acc_phase);
            tc_fence_after();
            const int64_t y = t.y0 + rank * BM + q * 32 + lane;
            const int64_t base = row_prefix(y, m) - y - p.job_lo;
            for (int h = t.h_lo; h < NB; ++h) {
#pragma unroll 1
                for (int c = 0; c < BN; c += 16) {
                    uint32_t r[16];
                    tmem_ld_32x32b_x16(tmem_base + (uint32_t(q * 32) << 16) + h * BN + c, r);
                    tmem_ld_wait();
                    if (y < m) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const int64_t x = t.x0 + h * BN + c + i;
                            const int64_t j = base + x;
                            if (x >= y && x < m && j >= 0 && j < span) {
                                const int32_t v = __float2int_rn(__uint_as_float(r[i]));
                                if (t.partial)
                                    atomicAdd(&p.num[j], v);
                                else
                                    p.num[j] = v;
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader);
            acc_phase ^= 1;
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_2sm<TMEM_COLS>(tmem_base);
    }
}

struct Unit4Table {
    int64_t m = -1, lo = -1, hi = -1;
    int32_t* dev = nullptr;
    int64_t count = 0, cap = 0;
};
static Unit4Table g_units4;

// Units (256-row block Yb, 480-column block Xb) that intersect the job range's rows and the upper
// triangle, ordered by 8 x 4 super-blocks (2048 rows x 1920 columns) so concurrently running pairs
// share S rows through L2.
static int build_units4(int64_t m, int64_t job_lo, int64_t job_hi, cudaStream_t st, const int32_t** out,
                        int64_t* count) {
    if (g_units4.m == m && g_units4.lo == job_lo && g_units4.hi == job_hi) {
        *out = g_units4.dev;
        *count = g_units4.count;
        return TB_OK;
    }
    const int64_t RB = (m + g4::UM - 1) / g4::UM, CB = (m + g4::UN - 1) / g4::UN;
    const int64_t GR = 8, GC = 4;
    int64_t y_lo, x_lo, y_hi, x_hi;
    job_coord(job_lo, m, y_lo, x_lo);
    job_coord(job_hi - 1, m, y_hi, x_hi);
    std::vector<int32_t> v;
    for (int64_t SY = 0; SY < (RB + GR - 1) / GR; ++SY)
        for (int64_t SX = 0; SX < (CB + GC - 1) / GC; ++SX)
            for (int64_t yb = SY * GR; yb < std::min(RB, (SY + 1) * GR); ++yb)
                for (int64_t xb = SX * GC; xb < std::min(CB, (SX + 1) * GC); ++xb) {
                    const int64_t r0 = yb * g4::UM, r1 = std::min(r0 + g4::UM, m) - 1;
                    if (xb * g4::UN + g4::UN - 1 < r0) continue;  // entirely below the diagonal
                    if (r1 < y_lo || r0 > y_hi) continue;          // outside the job range rows
                    v.push_back((int32_t)((yb << 16) | xb));
                }
    if ((int64_t)v.size() > g_units4.cap) {
        if (g_units4.dev) cudaFree(g_units4.dev);
        g_units4.dev = nullptr;
        TB_CUDA_TRY(cudaMalloc(&g_units4.dev, std::max<size_t>(v.size(), 1) * sizeof(int32_t)));
        g_units4.cap = (int64_t)v.size();
    }
    if (!v.empty())
        TB_CUDA_TRY(cudaMemcpyAsync(g_units4.dev, v.data(), v.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    TB_CUDA_TRY(cudaStreamSynchronize(st));
    g_units4.m = m;
    g_units4.lo = job_lo;
    g_units4.hi = job_hi;
    g_units4.count = (int64_t)v.size();
    *out = g_units4.dev;
    *count = g_units4.count;
    return TB_OK;
}

int gemm_fp4(const int8_t* S, int64_t m, int64_t K, int64_t ldS, int64_t job_lo, int64_t job_hi, int32_t splits,
             int32_t* num, cudaStream_t st) {
    if (K >= (int64_t(1) << 24)) return fail(TB_ERR_CAPACITY, "gemm fp4: K=%lld needs exact f32 sums (< 2^24)", (long long)K);
    if (m >= (int64_t(1) << 16) * g4::UM) return fail(TB_ERR_CAPACITY, "gemm fp4: m too large");
    int rc;
    const int32_t* units = nullptr;
    int64_t nunits = 0;
    if ((rc = build_units4(m, job_lo, job_hi, st, &units, &nunits))) return rc;
    Gemm4Args p{};
    p.m = m;
    p.units = units;
    p.nunits = nunits;
    const int64_t kbytes = K / 2;
    p.nkb = (int32_t)((kbytes + g4::BK - 1) / g4::BK);
    const int pairs = std::max(1, num_sms() / 2);
    if (splits <= 0) splits = pick_splits(nunits, p.nkb, pairs);
    if (splits > p.nkb) splits = p.nkb;
    p.splits = splits;
    p.job_lo = job_lo;
    p.job_hi = job_hi;
    p.num = num;
    if (splits > 1) TB_CUDA_TRY(cudaMemsetAsync(num, 0, (job_hi - job_lo) * sizeof(int32_t), st));
    CUtensorMap ta, tbm;
    if ((rc = make_tmap(&ta, S, m, kbytes, ldS, g4::BM))) return rc;
    if ((rc = make_tmap(&tbm, S, m, kbytes, ldS, g4::BNH))) return rc;
    TB_CUDA_TRY(cudaFuncSetAttribute(gemm_fp4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)g4::SMEM_BYTES));
    const int64_t work = nunits * splits;
    const unsigned grid = (unsigned)(2 * std::max<int64_t>(1, std::min<int64_t>(work, pairs)));
    gemm_fp4_kernel<<<grid, g4::THREADS, g4::SMEM_BYTES, st>>>(ta, tbm, p);
    return check_launch("gemm_fp4_kernel");
}

}  // namespace tb
