// Microbenchmark (diagnostics): sustained rate of tcgen05.mma.cta_group::2.kind::mxf4.block_scale
// issued back to back by one thread per CTA pair from shared memory (no TMA, no epilogue), for the
// GEMM's shapes.  Answers: is the ~71% tensor-active rate of gemm_fp4_kernel the MMA pipe's own limit?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1704_03767_b200/csrc/tb_common.cuh"
#include "../../paper_1704_03767_b200/csrc/tb_ptx.cuh"

using namespace tb;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe_kernel(int iters, int nblocks, int N, int per_commit, unsigned long long* cycles) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 64 * 1024);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool leader = cluster_ctarank() == 0;
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
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
        const uint32_t idesc = idesc_mxf4(256, (uint32_t)N);
        const uint32_t sf = tmem + 480;
        const uint64_t adesc = umma_desc_k_sw128(smem_u32(smem));
        const uint64_t bdesc = umma_desc_k_sw128(smem_u32(smem + 16384));
        const unsigned long long t0 = clock64();
        uint32_t phase = 0;
        for (int it = 0; it < iters; ++it) {
#pragma unroll 1
            for (int k = 0; k < 4; ++k)
                for (int h = 0; h < nblocks; ++h)
                    mma_mxf4_2sm(tmem + h * N, adesc + 2 * k, bdesc + 2 * k, idesc, sf, sf, 1u);
            if (per_commit && ((it + 1) % per_commit) == 0) {  // the GEMM's per-stage commit + wait pattern
                mma_commit_2sm(bar, 0x3);
                mbar_wait(bar, phase);
                phase ^= 1;
            }
        }
        mma_commit_2sm(bar, 0x3);
        mbar_wait(bar, phase);
        cycles[blockIdx.x / 2] = clock64() - t0;
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) { tc_fence_after(); tmem_dealloc_2sm<512>(tmem); }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int pairs = sms / 2;
    unsigned long long* d_cyc;
    cudaMalloc(&d_cyc, pairs * sizeof(unsigned long long));
    const size_t smem = 64 * 1024 + 2048;
    cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    struct Cfg { int nblocks, N, per_commit; const char* name; };
    const Cfg cfgs[] = {{2, 240, 0, "2 x N=240"}, {1, 240, 0, "1 x N=240"}, {3, 160, 0, "3 x N=160"},
                        {4, 120, 0, "4 x N=120"}, {2, 224, 0, "2 x N=224"}, {6, 80, 0, "6 x N=80"},
                        {5, 96, 0, "5 x N=96"}, {3, 144, 0, "3 x N=144"}};
    for (const Cfg& c : cfgs) {
        const int iters = 4096;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        probe_kernel<<<2 * pairs, 128, smem>>>(64, c.nblocks, c.N, c.per_commit, d_cyc);  // warm-up
        cudaEventRecord(e0);
        probe_kernel<<<2 * pairs, 128, smem>>>(iters, c.nblocks, c.N, c.per_commit, d_cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaError_t err = cudaGetLastError();
        float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 256 * c.N * 64 * 4.0 * c.nblocks * iters * pairs;
        unsigned long long cyc[128];
        cudaMemcpy(cyc, d_cyc, pairs * 8, cudaMemcpyDeviceToHost);
        double mean = 0; for (int i = 0; i < pairs; ++i) mean += cyc[i]; mean /= pairs;
        const double per_mma = mean / (4.0 * c.nblocks * iters);
        printf("%-38s %s: %.3f ms  %.0f TFLOP/s  %.1f cycles per MMA (ideal %.1f at 16384 MAC/cyc/SM)\n", c.name,
               cudaGetErrorString(err), ms, flops / ms / 1e9, per_mma, 128.0 * c.N * 64 / 16384.0);
    }
    return 0;
}
