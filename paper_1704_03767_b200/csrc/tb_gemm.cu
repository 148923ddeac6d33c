// K3: the numerator GEMM num(y, x) = S_y . S_x on tcgen05 tensor cores.
//
// n_c - n_d = sum_{a<b} sign(u_b - u_a) sign(v_b - v_a) (kernel_naive.py:26-44)
// is a dot product of the two rows' {-1,0,+1} sign vectors, so the all-pairs
// numerator matrix is the SYRK S S^T over K = n(n-1)/2, exact in int32.
//
// This file holds the int8 (kind::i8) / e4m3 (kind::f8f6f4) generation of the GEMM, used when the
// FP4 path's f32 sums could overflow 2^24 (K >= 2^24, n > ~5790; tb_gemm_fp4.cu is the default), the
// SIMT dp4a cross-check kernel and the shared TMA helpers.
//  * units = 256-row x 512-column blocks of the upper triangle (512-tiles decoded on device with the
//    reference bijection, pairindex.py:58-65), rasterised in 2048 x 2048 super-blocks, split-K;
//  * a persistent grid of CTA pairs (cta_group::2) walks units split-major so concurrently running
//    pairs stream the same K-slab of S through L2;
//  * warp 0: TMA producer (128-byte swizzled K-major boxes, 4-stage mbarrier ring); warp 1 of the
//    leader CTA: single-thread tcgen05.mma issuer (M=256, two N=256 blocks, K=32 per instruction);
//    warps 4-7 of both CTAs: epilogue (tcgen05.ld -> masked store / red.add in job-id order);
//  * split-K partials are integer, so atomic accumulation is deterministic.
#include <algorithm>
#include <cstdlib>
#include <vector>
#include <cudaTypedefs.h>

#include <mutex>

#include "tb_common.cuh"
#include "tb_ptx.cuh"

namespace tb {

namespace gemm2 {
constexpr int TILE = 512;
constexpr int UM = 256;       // pair M
constexpr int BM = 128;       // rows of A per CTA
constexpr int BN = 256;       // N per MMA
constexpr int BNH = 128;      // rows of B per CTA per N block
constexpr int BK = 128;
constexpr int UK = 32;
constexpr int STAGES = 4;
constexpr uint32_t A_BYTES = BM * BK;        // 16 KiB
constexpr uint32_t B_BYTES = BNH * BK;       // 16 KiB per N block
constexpr uint32_t STAGE_BYTES = A_BYTES + 2 * B_BYTES;
constexpr int THREADS = 256;
constexpr uint32_t TMEM_COLS = 512;
constexpr size_t SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 256;
}  // namespace gemm2

struct Gemm2Args {
    int64_t m;
    int64_t w;             // 512-tile matrix width
    const int32_t* units;  // tile_id * 2 + half, rasterised
    int64_t nunits;        // per split
    int32_t splits;
    int32_t nkb;
    int64_t job_lo, job_hi;
    int32_t* num;
    int32_t atomic;
    int32_t fp8;             // experiment: e4m3 operands, f32 accumulators (kind::f8f6f4)
};

struct Unit2 {
    int64_t y0, x0;   // pair rows y0..y0+255, columns x0..x0+511
    int32_t h_lo;     // first N block needed (1 if block 0 is entirely below the diagonal)
    int32_t kb0, kb1;
    bool partial;     // covers only part of K: accumulate atomically
};

__device__ __forceinline__ Unit2 unit_geometry(const Gemm2Args& p, int64_t i) {
    const int32_t e = p.units[i];
    int64_t Y, X;
    job_coord(e >> 1, p.w, Y, X);
    Unit2 o;
    o.y0 = Y * gemm2::TILE + (e & 1) * gemm2::UM;
    o.x0 = X * gemm2::TILE;
    o.h_lo = (o.x0 + gemm2::BN - 1 < o.y0) ? 1 : 0;
    return o;
}

// Work sequence of one CTA pair: units u = pair, pair + npairs, ... of the split-major list
// (unit i, K split s).
struct WorkIter {
    int64_t cur, end, step;
};
__device__ __forceinline__ WorkIter work_begin(const Gemm2Args& p, int64_t pair, int64_t npairs) {
    WorkIter w;
    w.cur = pair;
    w.end = p.nunits * p.splits;
    w.step = npairs;
    return w;
}
__device__ __forceinline__ bool work_next(const Gemm2Args& p, WorkIter& w, Unit2& t) {
    if (w.cur >= w.end) return false;
    const int32_t s = (int32_t)(w.cur / p.nunits);
    const int64_t i = w.cur - (int64_t)s * p.nunits;
    t = unit_geometry(p, i);
    t.kb0 = (int32_t)((int64_t)s * p.nkb / p.splits);
    t.kb1 = (int32_t)((int64_t)(s + 1) * p.nkb / p.splits);
    t.partial = p.splits > 1;
    w.cur += w.step;
    return true;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(gemm2::THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmap, Gemm2Args p) {
    using namespace gemm2;
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
        tma_prefetch(&tmap);
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
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer (both CTAs)
            int stage = 0;
            uint32_t phase = 0;
            WorkIter wi = work_begin(p, pair, npairs);
            Unit2 t;
            while (work_next(p, wi, t)) {
                const uint32_t bytes = 2 * (A_BYTES + (2 - t.h_lo) * B_BYTES);
                for (int32_t kb = t.kb0; kb < t.kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[stage], bytes);
                    const uint32_t fb = mapa_shared(&full[stage], 0);
                    uint8_t* sa = smem + stage * STAGE_BYTES;
                    tma_load_2d_2sm(sa, &tmap, fb, kb * BK, (int32_t)(t.y0 + rank * BM));
                    for (int h = t.h_lo; h < 2; ++h)
                        tma_load_2d_2sm(sa + A_BYTES + h * B_BYTES, &tmap, fb, kb * BK,
                                        (int32_t)(t.x0 + h * BN + rank * BNH));
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {  // ---------------- MMA issuer (leader CTA, warp 1; one elected lane issues)
            // warp-uniform loop, base + offset descriptors, unrolled MMAs (see tb_gemm_fp4.cu)
            const uint32_t idesc = p.fp8 ? idesc_f8(UM, BN) : idesc_i8(UM, BN);
            const uint64_t desc0 = umma_desc_k_sw128(smem_u32(smem));  // stage 0, A operand
            constexpr uint64_t STAGE_D = STAGE_BYTES >> 4, B0_D = A_BYTES >> 4, B1_D = (A_BYTES + B_BYTES) >> 4;
            int stage = 0;
            uint32_t phase = 0;
            uint32_t acc_phase = 0;
            WorkIter wi = work_begin(p, pair, npairs);
            Unit2 t;
            while (work_next(p, wi, t)) {
                mbar_wait(tempty, acc_phase ^ 1);
                tc_fence_after();
                for (int32_t kb = t.kb0; kb < t.kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint64_t ad = desc0 + (uint64_t)stage * STAGE_D;
                    const uint32_t a0 = kb > t.kb0 ? 1u : 0u;
                    if (p.fp8) {
#pragma unroll
                        for (int k = 0; k < BK / UK; ++k) {
                            if (t.h_lo == 0) mma_f8_2sm_warp(tmem_base, ad + 2 * k, ad + B0_D + 2 * k, idesc, k ? 1u : a0);
                            mma_f8_2sm_warp(tmem_base + BN, ad + 2 * k, ad + B1_D + 2 * k, idesc, k ? 1u : a0);
                        }
                    } else if (t.h_lo == 0) {
#pragma unroll
                        for (int k = 0; k < BK / UK; ++k) {
                            mma_i8_2sm_warp(tmem_base, ad + 2 * k, ad + B0_D + 2 * k, idesc, k ? 1u : a0);
                            mma_i8_2sm_warp(tmem_base + BN, ad + 2 * k, ad + B1_D + 2 * k, idesc, k ? 1u : a0);
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < BK / UK; ++k)
                            mma_i8_2sm_warp(tmem_base + BN, ad + 2 * k, ad + B1_D + 2 * k, idesc, k ? 1u : a0);
                    }
                    mma_commit_2sm_warp(&empty[stage], 0x3);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                mma_commit_2sm_warp(tfull, 0x3);
                acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {  // ---------------- epilogue (both CTAs)
        const int q = warp & 3;
        uint32_t acc_phase = 0;
        const int64_t m = p.m;
        const int64_t span = p.job_hi - p.job_lo;
        const uint32_t tempty_leader = mapa_shared(tempty, 0);
        WorkIter wi = work_begin(p, pair, npairs);
        Unit2 t;
        while (work_next(p, wi, t)) {
            mbar_wait(tfull, acc_phase);
            tc_fence_after();
            const int64_t y = t.y0 + rank * BM + q * 32 + lane;
            const int64_t base = row_prefix(y, m) - y - p.job_lo;
            for (int h = t.h_lo; h < 2; ++h) {
#pragma unroll 1
                for (int c = 0; c < BN; c += 32) {
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) + h * BN + c, r);
                    tmem_ld_wait();
                    if (y < m) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const int64_t x = t.x0 + h * BN + c + i;
                            const int64_t j = base + x;
                            if (x >= y && x < m && j >= 0 && j < span) {
                                const int32_t val = p.fp8 ? __float2int_rn(__uint_as_float(r[i])) : (int32_t)r[i];
                                if (t.partial)
                                    atomicAdd(&p.num[j], val);
                                else
                                    p.num[j] = val;
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

// ------------------------------------------------------------------ SIMT dp4a cross-check
// 32 x 32 output block per CTA, K staged through shared memory 64 bytes at a time.
__global__ void __launch_bounds__(256) gemm_simt_kernel(const int8_t* __restrict__ S, int64_t m, int64_t K,
                                                        int64_t ldS, int64_t job_lo, int64_t job_hi,
                                                        int32_t* __restrict__ num) {
    __shared__ int32_t sa[32][17];
    __shared__ int32_t sb[32][17];
    const int64_t Y0 = (int64_t)blockIdx.y * 32, X0 = (int64_t)blockIdx.x * 32;
    if (X0 + 31 < Y0) return;  // strictly below the diagonal
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    int32_t acc[4] = {0, 0, 0, 0};
    const int64_t kw = (K + 3) / 4;  // words; bytes past K are zero (sign_pack contract)
    for (int64_t w0 = 0; w0 < kw; w0 += 16) {
        for (int e = threadIdx.x; e < 32 * 16; e += 256) {
            int rr = e >> 4, ww = e & 15;
            int64_t word = w0 + ww;
            int32_t va = 0, vb = 0;
            if (word < kw) {
                if (Y0 + rr < m) va = reinterpret_cast<const int32_t*>(S + (Y0 + rr) * ldS)[word];
                if (X0 + rr < m) vb = reinterpret_cast<const int32_t*>(S + (X0 + rr) * ldS)[word];
            }
            sa[rr][ww] = va;
            sb[rr][ww] = vb;
        }
        __syncthreads();
#pragma unroll
        for (int ww = 0; ww < 16; ++ww) {
            const int32_t b = sb[tx][ww];
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i] = __dp4a(sa[ty + 8 * i][ww], b, acc[i]);
        }
        __syncthreads();
    }
    const int64_t x = X0 + tx;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t y = Y0 + ty + 8 * i;
        if (y < m && x < m && x >= y) {
            const int64_t j = row_prefix(y, m) + x - y;
            if (j >= job_lo && j < job_hi) num[j - job_lo] = acc[i];
        }
    }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

int make_tmap(CUtensorMap* map, const int8_t* S, int64_t m, int64_t K, int64_t ldS, uint32_t box_rows) {
    auto enc = get_encode();
    if (!enc) return fail(TB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)m};
    cuuint64_t strides[1] = {(cuuint64_t)ldS};
    cuuint32_t box[2] = {(cuuint32_t)gemm2::BK, box_rows};  // 128-byte K boxes (SW128 atom width)
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(S), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(TB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return TB_OK;
}

static int check_job_args(int64_t m, int64_t K, int64_t ldS, int64_t job_lo, int64_t job_hi) {
    if (m < 1 || K < 1) return fail(TB_ERR_INVALID, "gemm: need m >= 1 and K >= 1");
    if (ldS < K || (ldS & 15)) return fail(TB_ERR_CONFIG, "gemm: ldS must be >= K and a multiple of 16");
    const int64_t total = m * (m + 1) / 2;
    if (job_lo < 0 || job_hi < job_lo || job_hi > total)
        return fail(TB_ERR_CONFIG, "gemm: job range [%lld, %lld) outside [0, %lld)", (long long)job_lo,
                    (long long)job_hi, (long long)total);
    return TB_OK;
}


// Rasterised unit table for the 2-SM kernel: (tile id on the 512-tile matrix) * 2 + half, ordered
// by 4 x 4 super-tiles, row-halves outer, so ~74 concurrently running pairs share A and B rows
// through L2.  Cached per (m, job range).
struct UnitTable {
    DevTable table;  // the unit table on its device (async upload, see tb_common.cuh)
    int64_t m = -1, lo = -1, hi = -1;
    int64_t count = 0;
};
static UnitTable g_unit_cache[32];  // per (m, job range): the banded host path cycles through a few
static int g_unit_next = 0;

static int build_units(int64_t m, int64_t job_lo, int64_t job_hi, cudaStream_t st, const int32_t** out,
                       int64_t* count, DevTable** table) {
    std::lock_guard<std::mutex> lock(g_native_state_mutex);  // host threads share the caches
    int ordinal = 0;
    TB_CUDA_TRY(cudaGetDevice(&ordinal));
    for (UnitTable& c : g_unit_cache)
        if (c.table.ordinal == ordinal && c.m == m && c.lo == job_lo && c.hi == job_hi) {
            *out = static_cast<const int32_t*>(c.table.dev);
            *count = c.count;
            *table = &c.table;
            return TB_OK;
        }
    UnitTable& g_units = g_unit_cache[g_unit_next];
    g_unit_next = (g_unit_next + 1) % 32;
    g_units.m = -1;
    const int64_t T = gemm2::TILE, G = 4;
    const int64_t w = (m + T - 1) / T;
    const int64_t W = (w + G - 1) / G;
    int64_t y_lo, x_lo, y_hi, x_hi;
    job_coord(job_lo, m, y_lo, x_lo);
    job_coord(job_hi - 1, m, y_hi, x_hi);
    std::vector<int32_t> v;
    for (int64_t SY = 0; SY < W; ++SY)
        for (int64_t SX = SY; SX < W; ++SX)
            for (int64_t LY = 0; LY < G; ++LY)
                for (int64_t r = 0; r < 2; ++r)
                    for (int64_t LX = 0; LX < G; ++LX) {
                        const int64_t Y = SY * G + LY, X = SX * G + LX;
                        if (Y > X || X >= w) continue;
                        const int64_t r0 = Y * T + r * gemm2::UM;
                        if (r0 >= m) continue;
                        const int64_t r1 = std::min(r0 + gemm2::UM, m) - 1;  // last row of the unit
                        if (r1 < y_lo || r0 > y_hi) continue;                 // outside the job range rows
                        if (X * T + T - 1 < r0) continue;                      // entirely below the diagonal
                        const int64_t tid = row_prefix(Y, w) + X - Y;
                        if (tid * 2 + 1 > INT32_MAX) return fail(TB_ERR_CAPACITY, "gemm: too many tiles");
                        v.push_back((int32_t)(tid * 2 + r));
                    }
    int rc = table_upload(g_units.table, v.data(), v.size() * sizeof(int32_t), st);
    if (rc) return rc;
    g_units.m = m;
    g_units.lo = job_lo;
    g_units.hi = job_hi;
    g_units.count = (int64_t)v.size();
    *out = static_cast<const int32_t*>(g_units.table.dev);
    *count = g_units.count;
    *table = &g_units.table;
    return TB_OK;
}

// Split-K choice: minimise waves(U*s / pairs) * (nkb/s * t_kb + t_epi).
int32_t pick_splits(int64_t units, int32_t nkb, int pairs) {
    const double t_kb = 1.0, t_epi = 40.0;  // k-block of the 2-SM kernel ~0.5 us; epilogue ~20 us
    int32_t best = 1;
    double best_t = 1e300;
    for (int32_t s = 1; s <= std::max(1, nkb / 8) && s <= 64; ++s) {
        const int64_t waves = (units * s + pairs - 1) / pairs;
        const double t = waves * ((double)nkb / s * t_kb + t_epi + (s > 1 ? t_epi : 0.0));
        if (t < best_t * 0.999) { best_t = t; best = s; }
    }
    return best;
}

static int gemm_v2(const int8_t* S, int64_t m, int64_t K, int64_t ldS, int64_t job_lo, int64_t job_hi,
                   int32_t splits, int format, int32_t* num, cudaStream_t st) {
    int rc;
    const int32_t* units = nullptr;
    int64_t nunits = 0;
    DevTable* table = nullptr;
    if ((rc = build_units(m, job_lo, job_hi, st, &units, &nunits, &table))) return rc;
    Gemm2Args p{};
    p.m = m;
    p.w = (m + gemm2::TILE - 1) / gemm2::TILE;
    p.units = units;
    p.nunits = nunits;
    p.nkb = (int32_t)((K + gemm2::BK - 1) / gemm2::BK);
    const int pairs = std::max(1, num_sms() / 2);
    // (a stream-K schedule was measured slower here -- its pairs sit at different K offsets and lose
    // the K-lockstep L2 reuse of S: config 2 GEMM 975 vs 874 us -- so the split-major static one stays)
    if (splits <= 0) splits = pick_splits(nunits, p.nkb, pairs);
    if (splits > p.nkb) splits = p.nkb;
    p.splits = splits;
    p.job_lo = job_lo;
    p.job_hi = job_hi;
    p.num = num;
    p.atomic = splits > 1;
    p.fp8 = format == TB_SIGN_E4M3 ? 1 : 0;
    if (p.atomic) TB_CUDA_TRY(cudaMemsetAsync(num, 0, (job_hi - job_lo) * sizeof(int32_t), st));
    CUtensorMap tm;
    if ((rc = make_tmap(&tm, S, m, K, ldS, gemm2::BM))) return rc;
    TB_CUDA_TRY(cudaFuncSetAttribute(gemm_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)gemm2::SMEM_BYTES));
    const int64_t work = nunits * splits;
    const unsigned grid = (unsigned)(2 * std::max<int64_t>(1, std::min<int64_t>(work, pairs)));
    gemm_tc2_kernel<<<grid, gemm2::THREADS, gemm2::SMEM_BYTES, st>>>(tm, p);
    if ((rc = check_launch("gemm_tc2_kernel"))) return rc;
    return table_mark_used(*table, st);
}

}  // namespace tb

using namespace tb;

namespace tb {
int gemm_fp4(const int8_t* S, int64_t m, int64_t K, int64_t ldS, int64_t job_lo, int64_t job_hi, int32_t splits,
             int32_t* num, cudaStream_t st, double* tau_b = nullptr, const uint64_t* n1 = nullptr, int64_t n = 0,
             int* fused = nullptr, const int32_t* fix = nullptr, int64_t fix_c = 0);
}
static bool is_e2m1(int format) { return format == TB_SIGN_E2M1 || format == TB_SIGN_E2M1_OFS; }

extern "C" int tb_gemm_pairs_fix(const int8_t* S, int64_t m, int64_t K, int64_t ldS, int format, int64_t job_lo,
                                 int64_t job_hi, int32_t splits, const int32_t* fix, int64_t fix_c, int32_t* num,
                                 void* stream) {
    if (format < TB_SIGN_I8 || format > TB_SIGN_E2M1_OFS) return fail(TB_ERR_CONFIG, "gemm: unknown format %d", format);
    if (fix && !is_e2m1(format)) return fail(TB_ERR_CONFIG, "gemm: offset operands (fix) need an e2m1 format");
    // the S + 1 coding quadruples the sums: exact f32 only while 4 K < 2^24
    if (format == TB_SIGN_E2M1_OFS && (!fix || 4 * K >= (int64_t(1) << 24)))
        return fail(TB_ERR_CONFIG, "gemm: TB_SIGN_E2M1_OFS needs the row sums (fix) and 4 K < 2^24 (K=%lld)", (long long)K);
    int rc = check_job_args(m, is_e2m1(format) ? K / 2 : K, ldS, job_lo, job_hi);
    if (rc) return rc;
    if (!S || !num) return fail(TB_ERR_INVALID, "gemm: null pointer");
    if (job_hi == job_lo) return TB_OK;
    if (m > (int64_t)INT32_MAX - gemm2::TILE) return fail(TB_ERR_CAPACITY, "gemm: m too large for TMA coordinates");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (is_e2m1(format))
        return gemm_fp4(S, m, K, ldS, job_lo, job_hi, splits, num, st, nullptr, nullptr, 0, nullptr, fix, fix_c);
    return gemm_v2(S, m, K, ldS, job_lo, job_hi, splits, format, num, st);
}

extern "C" int tb_gemm_pairs(const int8_t* S, int64_t m, int64_t K, int64_t ldS, int format, int64_t job_lo,
                             int64_t job_hi, int32_t splits, int32_t* num, void* stream) {
    return tb_gemm_pairs_fix(S, m, K, ldS, format, job_lo, job_hi, splits, nullptr, 0, num, stream);
}

extern "C" int tb_gemm_tau_b(const int8_t* S, int64_t m, int64_t K, int64_t ldS, int format, int64_t job_lo,
                             int64_t job_hi, int32_t splits, const uint64_t* n1_rows, int64_t n, int32_t* num_ws,
                             double* tau_b, void* stream) {
    return tb_gemm_tau_b_fix(S, m, K, ldS, format, job_lo, job_hi, splits, nullptr, 0, n1_rows, n, num_ws, tau_b, stream);
}

extern "C" int tb_gemm_tau_b_fix(const int8_t* S, int64_t m, int64_t K, int64_t ldS, int format, int64_t job_lo,
                                 int64_t job_hi, int32_t splits, const int32_t* fix, int64_t fix_c,
                                 const uint64_t* n1_rows, int64_t n, int32_t* num_ws, double* tau_b, void* stream) {
    if (format < TB_SIGN_I8 || format > TB_SIGN_E2M1_OFS) return fail(TB_ERR_CONFIG, "gemm_tau_b: unknown format %d", format);
    if (fix && !is_e2m1(format)) return fail(TB_ERR_CONFIG, "gemm_tau_b: offset operands (fix) need an e2m1 format");
    if (format == TB_SIGN_E2M1_OFS && (!fix || 4 * K >= (int64_t(1) << 24)))
        return fail(TB_ERR_CONFIG, "gemm_tau_b: TB_SIGN_E2M1_OFS needs the row sums (fix) and 4 K < 2^24");
    int rc = check_job_args(m, is_e2m1(format) ? K / 2 : K, ldS, job_lo, job_hi);
    if (rc) return rc;
    if (!S || !n1_rows || !tau_b) return fail(TB_ERR_INVALID, "gemm_tau_b: null pointer");
    if (n < 2) return fail(TB_ERR_INVALID, "gemm_tau_b: need n >= 2");
    if (job_hi == job_lo) return TB_OK;
    if (m > (int64_t)INT32_MAX - gemm2::TILE) return fail(TB_ERR_CAPACITY, "gemm: m too large for TMA coordinates");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int fused = 0;
    if (is_e2m1(format)) {
        if ((rc = gemm_fp4(S, m, K, ldS, job_lo, job_hi, splits, num_ws, st, tau_b, n1_rows, n, &fused, fix, fix_c)))
            return rc;
    } else {
        if (!num_ws) return fail(TB_ERR_INVALID, "gemm_tau_b: the int8 path needs the numerator workspace");
        if ((rc = gemm_v2(S, m, K, ldS, job_lo, job_hi, splits, format, num_ws, st))) return rc;
    }
    if (fused) return TB_OK;
    return tb_finalize(num_ws, n1_rows, m, n, job_lo, job_hi, nullptr, tau_b, stream);
}

extern "C" int tb_gemm_pairs_simt(const int8_t* S, int64_t m, int64_t K, int64_t ldS, int64_t job_lo,
                                  int64_t job_hi, int32_t* num, void* stream) {
    int rc = check_job_args(m, K, ldS, job_lo, job_hi);
    if (rc) return rc;
    if (!S || !num) return fail(TB_ERR_INVALID, "gemm_simt: null pointer");
    if (job_hi == job_lo) return TB_OK;
    const int64_t nb = (m + 31) / 32;
    if (nb > 65535) return fail(TB_ERR_CAPACITY, "gemm_simt: m too large for the cross-check kernel");
    dim3 grid((unsigned)nb, (unsigned)nb);
    gemm_simt_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(S, m, K, ldS, job_lo, job_hi, num);
    return check_launch("gemm_simt_kernel");
}
