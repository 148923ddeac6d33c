// Which pipe runs FMNMX on sm_100a?  Throughput of independent IMNMX, FMNMX and a 1:1 mix.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(unsigned* out, int iters, unsigned seed) {
    unsigned a[8], b[8];
    float fa[8], fb[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = seed * (i + 1) + threadIdx.x;
        b[i] = seed ^ (i * 77 + threadIdx.x);
        fa[i] = __uint_as_float((a[i] & 0x7FFFFF) | 0x3F800000u);
        fb[i] = __uint_as_float((b[i] & 0x7FFFFF) | 0x3F800000u);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0 || MODE == 2) {
                const unsigned lo = min(a[i], b[i]), hi = max(a[i], b[i]);
                a[i] = lo + 1; b[i] = hi;
            }
            if (MODE == 1 || MODE == 2) {
                const float lo = fminf(fa[i], fb[i]), hi = fmaxf(fa[i], fb[i]);
                fa[i] = hi; fb[i] = lo + 1.0f;
            }
        }
    }
    unsigned s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i] ^ b[i] ^ __float_as_uint(fa[i]) ^ __float_as_uint(fb[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    unsigned* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
    const int iters = 20000;
    const char* names[3] = {"IMNMX x2 (+IADD) per pair", "FMNMX x2 (+FADD) per pair", "mix: both per pair"};
    for (int mode = 0; mode < 3; ++mode) {
        cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(s);
            if (mode == 0) k<0><<<148 * 8, 256>>>(out, iters, 12345);
            if (mode == 1) k<1><<<148 * 8, 256>>>(out, iters, 12345);
            if (mode == 2) k<2><<<148 * 8, 256>>>(out, iters, 12345);
            cudaEventRecord(e); cudaEventSynchronize(e);
            float ms; cudaEventElapsedTime(&ms, s, e);
            if (rep == 2) printf("%-28s %8.3f ms\n", names[mode], ms);
        }
    }
    return 0;
}
