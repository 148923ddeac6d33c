// Roofline probe (diagnostics, not part of the drop-in ABI): the INT32 issue peak the merge path's
// roofline is quoted against ("measure it with a dependency-free IADD3/LOP3
// microbenchmark").  Every thread runs 8 independent IADD3 chains and 8 independent LOP3 chains;
// one lane-instruction = one INT32 op, the unit of the merge path's 4 * n * ceil(log2 n) per pair.
#include <cstdint>
#include <cuda_runtime.h>

#include "tb_common.cuh"
#include "tb_ptx.cuh"

namespace {

__device__ __forceinline__ uint32_t iadd3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm volatile("add.u32 %0, %1, %2;\n\tadd.u32 %0, %0, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

__global__ void __launch_bounds__(256) int32_probe_kernel(uint32_t* out, int iters, uint32_t seed) {
    uint32_t a[8], b[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        a[k] = threadIdx.x * (k + 1) + seed;
        b[k] = threadIdx.x ^ (seed + 977u * k);
    }
    const uint32_t c = seed | 1u;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            a[k] = iadd3(a[k], b[(k + 1) & 7], c);
            b[k] = lop3(b[k], a[(k + 3) & 7], c);
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= a[k] ^ b[k];
    if (s == 0x12345678u) out[0] = s;  // keeps the chains alive
}

// The issue ceiling of a kernel that splits its integer work over both integer-capable pipes, as K4 does
// (ALU: IADD3 / LOP3 / min / max / SEL ...; FMA: IMAD): per iteration 8 IADD3 + 8 LOP3 chains on the ALU
// pipe and 16 independent IMAD chains on the FMA pipe (mad.lo with a runtime multiplier, so ptxas cannot
// turn it into shifts / adds).  Each pipe accepts one warp instruction per 2 cycles per SM sub-partition
// and the scheduler issues one per cycle, so a 50/50 mix is bounded by issue: 128 lane-ops / clk / SM.
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

__global__ void __launch_bounds__(256) int32_mixed_probe_kernel(uint32_t* out, int iters, uint32_t seed, uint32_t mul) {
    uint32_t a[8], b[8], f[16];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        a[k] = threadIdx.x * (k + 1) + seed;
        b[k] = threadIdx.x ^ (seed + 977u * k);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) f[k] = threadIdx.x + 31u * k + seed;
    const uint32_t c = seed | 1u;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            a[k] = iadd3(a[k], b[(k + 1) & 7], c);
            f[2 * k] = imad(f[2 * k], mul, c);
            b[k] = lop3(b[k], a[(k + 3) & 7], c);
            f[2 * k + 1] = imad(f[2 * k + 1], mul, a[k]);
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= a[k] ^ b[k];
#pragma unroll
    for (int k = 0; k < 16; ++k) s ^= f[k];
    if (s == 0x12345678u) out[0] = s;  // keeps the chains alive
}

// tcgen05.mma.cta_group::2.kind::mxf4.block_scale, M=256, the GEMM's two N=240 accumulators issued
// alternately, back to back from shared memory by one thread per CTA pair (no TMA, no epilogue):
// the MMA pipe's sustained rate for the numerator GEMM's instruction stream.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mxf4_probe_kernel(int iters) {
    using namespace tb;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 64 * 1024);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    const int warp = threadIdx.x >> 5;
    const bool leader = cluster_ctarank() == 0;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc_2sm<512>(slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *slot;
    tmem_st_32x32b_x32(tmem + (uint32_t(warp * 32) << 16) + 480, 0x7F7F7F7Fu);
    tmem_st_wait();
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (leader && threadIdx.x == 0) {
        constexpr uint32_t idesc = idesc_mxf4(256, 240);
        const uint32_t sf = tmem + 480;
        const uint64_t adesc = umma_desc_k_sw128(smem_u32(smem));
        const uint64_t bdesc = umma_desc_k_sw128(smem_u32(smem + 16384));
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                for (int h = 0; h < 2; ++h) mma_mxf4_2sm(tmem + h * 240, adesc + 2 * k, bdesc + 2 * k, idesc, sf, sf, 1u);
        mma_commit_2sm(bar, 0x3);
        mbar_wait(bar, 0);
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc_2sm<512>(tmem);
    }
}


// Sparse variant (throughput probe for a 2:4-structured-sparse operand A): tcgen05.mma.sp ... kind::mxf4
// (logical K = 128 per instruction: A holds 64 kept e2m1 values per row + 2-of-4 metadata in TMEM, B the
// full 128), M = 256, two N accumulators alternating.  Operand values are irrelevant to the rate; the
// metadata holds a valid pattern (kept indices 0, 1 of every group of four).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mxf4_sparse_probe_kernel(int iters, int N) {
    using namespace tb;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 64 * 1024);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    const int warp = threadIdx.x >> 5;
    const bool leader = cluster_ctarank() == 0;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc_2sm<512>(slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *slot;
    const uint32_t sf_col = 2u * N, meta_col = 480;
    tmem_st_32x32b_x32(tmem + (uint32_t(warp * 32) << 16) + sf_col, 0x7F7F7F7Fu);
    tmem_st_wait();
    tmem_st_32x32b_x32(tmem + (uint32_t(warp * 32) << 16) + meta_col, 0x44444444u);
    tmem_st_wait();
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (leader && threadIdx.x == 0) {
        const uint32_t idesc = idesc_mxf4(256, (uint32_t)N) | (1u << 2);  // sparse flag; K = 128 (k_size 0)
        const uint32_t sf = tmem + sf_col, meta = tmem + meta_col;
        const uint64_t adesc = umma_desc_k_sw128(smem_u32(smem));
        const uint64_t bdesc = umma_desc_k_sw128(smem_u32(smem + 16384));
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int k = 0; k < 2; ++k)
                for (int h = 0; h < 2; ++h)
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.sp.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, [%7], %3, [%5], [%6], p;\n\t}"
                        ::"r"(tmem + h * N), "l"(adesc + 2 * k), "l"(bdesc + 4 * k), "r"(idesc), "r"(1u), "r"(sf),
                        "r"(sf), "r"(meta)
                        : "memory");
        mma_commit_2sm(bar, 0x3);
        mbar_wait(bar, 0);
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc_2sm<512>(tmem);
    }
}
}  // namespace

// Returns the FLOP/s (2 per MAC) of the MMA stream above on every SM pair, best of `reps`; 0 on error.
extern "C" double tb_probe_mxf4_flops(int reps) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int pairs = sms / 2, iters = 4096;
    const size_t smem = 64 * 1024 + 2048;
    if (cudaFuncSetAttribute(mxf4_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 0.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps + 1; ++r) {
        cudaEventRecord(e0);
        mxf4_probe_kernel<<<2 * pairs, 128, smem>>>(r == 0 ? 64 : iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (cudaGetLastError() != cudaSuccess) return 0.0;
    const double flops = 2.0 * 256 * 240 * 64 * 8.0 * iters * pairs;
    return flops / (best * 1e-3);
}

// Returns INT32 lane-ops per second (IADD3 + LOP3 mix; ptxas fuses each add pair into one IADD3),
// best of `reps` launches on the current device; 0 on error.
extern "C" double tb_probe_int32_ops(int reps) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint32_t* out = nullptr;
    if (cudaMalloc(&out, 4) != cudaSuccess) return 0.0;
    const int iters = 4096, blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps + 1; ++r) {
        cudaEventRecord(e0);
        int32_probe_kernel<<<blocks, threads>>>(out, iters, 12345u + r);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;  // first launch is warm-up
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess) return 0.0;
    const double ops = (double)blocks * threads * iters * 16.0;  // 8 IADD3 + 8 LOP3 per iteration
    return ops / (best * 1e-3);
}

// Lane-ops/s of the mixed ALU + FMA integer probe (the issue ceiling K4's instruction mix is quoted
// against next to the ALU-only figure above).
extern "C" double tb_probe_int32_mixed_ops(int reps) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint32_t* out = nullptr;
    if (cudaMalloc(&out, 4) != cudaSuccess) return 0.0;
    const int iters = 4096, blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps + 1; ++r) {
        cudaEventRecord(e0);
        int32_mixed_probe_kernel<<<blocks, threads>>>(out, iters, 12345u + r, 0x9E3779B1u + r);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess) return 0.0;
    const double ops = (double)blocks * threads * iters * 32.0;  // 8 IADD3 + 8 LOP3 + 16 IMAD per iteration
    return ops / (best * 1e-3);
}

// FLOP/s (2 per logical MAC) of the sparse MMA stream above (N per accumulator), best of `reps`; 0 on error.
extern "C" double tb_probe_mxf4_sparse_flops(int reps, int N) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int pairs = sms / 2, iters = 4096;
    const size_t smem = 64 * 1024 + 2048;
    if (cudaFuncSetAttribute(mxf4_sparse_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 0.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps + 1; ++r) {
        cudaEventRecord(e0);
        mxf4_sparse_probe_kernel<<<2 * pairs, 128, smem>>>(r == 0 ? 64 : iters, N);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (cudaGetLastError() != cudaSuccess) return 0.0;
    const double flops = 2.0 * 256 * N * 128 * 4.0 * iters * pairs;
    return flops / (best * 1e-3);
}
