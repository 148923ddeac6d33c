// K2: sign pack.  S[r, k(a,b)] = sign(x[r,b] - x[r,a]) as int8, plus the
// per-row tied-pair count n1 = n0 - sum |S| (the n1/n2 scans of
// kernel_sorted.py:163-176, done once per variable instead of once per pair).
//
// One CTA owns (row r, a strided set of 8 KiB chunks of k).  The row's values
// sit in shared memory; consecutive threads produce consecutive bytes of k
// (so consecutive threads read consecutive x[b] -- conflict-free), bytes are
// staged in shared memory and written out with 16-byte coalesced stores.
// HBM-bound on the S write (m * ldS bytes).
#include "tb_common.cuh"

namespace tb {

constexpr int SP_THREADS = 256;
constexpr int SP_CHUNK = 8192;

template <typename T>
__global__ void __launch_bounds__(SP_THREADS) signpack_kernel(const T* __restrict__ x, int64_t m, int64_t n,
                                                              int64_t ldx, int8_t* __restrict__ S, int64_t ldS,
                                                              int64_t K, unsigned long long* __restrict__ nz,
                                                              int32_t* __restrict__ flags) {
    extern __shared__ __align__(16) uint8_t sp_smem[];
    T* xs = reinterpret_cast<T*>(sp_smem);
    uint8_t* stage = sp_smem + ((n * (int64_t)sizeof(T) + 15) & ~int64_t(15));
    const int64_t r = blockIdx.x;
    const int tid = threadIdx.x;

    bool bad = false;
    for (int64_t i = tid; i < n; i += SP_THREADS) {
        T v = x[r * ldx + i];
        bad |= (v != v);  // NaN has no rank (ranks.py:56-57)
        xs[i] = v;
    }
    if (bad) atomicOr(flags, 1);
    __syncthreads();

    uint32_t cnt = 0;
    const int64_t nchunks = (ldS + SP_CHUNK - 1) / SP_CHUNK;
    for (int64_t c = blockIdx.y; c < nchunks; c += gridDim.y) {
        const int64_t k0 = c * SP_CHUNK;
        const int64_t kend = min(k0 + SP_CHUNK, K);
        int64_t k = k0 + tid;
        if (k < kend) {
            int64_t a, b;
            k_decode(k, n, a, b);
            T xa = xs[a];
            for (;;) {
                T xb = xs[b];
                int s = (xb > xa) - (xb < xa);
                stage[k - k0] = static_cast<uint8_t>(static_cast<int8_t>(s));
                cnt += (s != 0);
                k += SP_THREADS;
                if (k >= kend) break;
                b += SP_THREADS;
                bool moved = false;
                while (b >= n) {  // carry into the next a-segments
                    int64_t over = b - n;
                    ++a;
                    b = a + 1 + over;
                    moved = true;
                }
                if (moved) xa = xs[a];
            }
        }
        const int64_t cend = min(k0 + SP_CHUNK, ldS);
        for (int64_t z = max(kend, k0) + tid; z < cend; z += SP_THREADS) stage[z - k0] = 0;
        __syncthreads();
        uint4* dst = reinterpret_cast<uint4*>(S + r * ldS + k0);
        const uint4* src = reinterpret_cast<const uint4*>(stage);
        const int64_t nv = (cend - k0) >> 4;
        for (int64_t i = tid; i < nv; i += SP_THREADS) dst[i] = src[i];
        __syncthreads();
    }
    // block reduction of the untied-pair count
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((tid & 31) == 0 && cnt) atomicAdd(&nz[r], (unsigned long long)cnt);
}

__global__ void nz_to_n1_kernel(unsigned long long* n1, int64_t m, unsigned long long n0) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < m) n1[r] = n0 - n1[r];
}

}  // namespace tb

using namespace tb;

extern "C" int tb_sign_pack(const void* x, int dtype, int64_t m, int64_t n, int64_t ldx, int8_t* S, int64_t ldS,
                            uint64_t* n1, int32_t* flags, void* stream) {
    if (m < 1 || n < 2) return fail(TB_ERR_INVALID, "sign_pack: need m >= 1 and n >= 2 (got m=%lld n=%lld)",
                                    (long long)m, (long long)n);
    if (n > TB_MAX_N) return fail(TB_ERR_CAPACITY, "sign_pack: n=%lld exceeds %d", (long long)n, TB_MAX_N);
    const int64_t K = n * (n - 1) / 2;
    if (ldS < K || (ldS & 15)) return fail(TB_ERR_CONFIG, "sign_pack: ldS=%lld must be >= K=%lld and 16-aligned",
                                           (long long)ldS, (long long)K);
    if (ldx < n) return fail(TB_ERR_CONFIG, "sign_pack: ldx < n");
    if (!x || !S || !n1 || !flags) return fail(TB_ERR_INVALID, "sign_pack: null pointer");
    size_t esz = dtype == TB_DTYPE_F64 ? 8 : 4;
    size_t smem = ((n * esz + 15) & ~size_t(15)) + SP_CHUNK;
    if (smem > 200 * 1024) return fail(TB_ERR_CAPACITY, "sign_pack: row of n=%lld does not fit shared memory", (long long)n);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TB_CUDA_TRY(cudaMemsetAsync(n1, 0, m * sizeof(uint64_t), st));
    const int64_t nchunks = (ldS + SP_CHUNK - 1) / SP_CHUNK;
    int64_t want = (8 * (int64_t)num_sms() + m - 1) / m;  // >= ~8 CTAs per SM in total
    int gy = (int)std::min<int64_t>(std::max<int64_t>(want, 1), std::min<int64_t>(nchunks, 65535));
    dim3 grid((unsigned)m, gy);
    auto* nz = reinterpret_cast<unsigned long long*>(n1);
    switch (dtype) {
        case TB_DTYPE_I32:
            cudaFuncSetAttribute(signpack_kernel<int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            signpack_kernel<int32_t><<<grid, SP_THREADS, smem, st>>>((const int32_t*)x, m, n, ldx, S, ldS, K, nz, flags);
            break;
        case TB_DTYPE_F32:
            cudaFuncSetAttribute(signpack_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            signpack_kernel<float><<<grid, SP_THREADS, smem, st>>>((const float*)x, m, n, ldx, S, ldS, K, nz, flags);
            break;
        case TB_DTYPE_F64:
            cudaFuncSetAttribute(signpack_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            signpack_kernel<double><<<grid, SP_THREADS, smem, st>>>((const double*)x, m, n, ldx, S, ldS, K, nz, flags);
            break;
        default:
            return fail(TB_ERR_INVALID, "sign_pack: unknown dtype %d", dtype);
    }
    int rc = check_launch("signpack_kernel");
    if (rc) return rc;
    nz_to_n1_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(nz, m, (unsigned long long)K);
    return check_launch("nz_to_n1_kernel");
}

// |S| (0/1 int8) for the full-count GEMM, 16 bytes per thread.
namespace tb {
__global__ void abs_pack_kernel(const uint4* __restrict__ S, uint4* __restrict__ A, int64_t nvec) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * blockDim.x) {
        uint4 v = S[i];
        // bytes are 0x00, 0x01 or 0xFF: |s| = s & 1
        v.x &= 0x01010101u;
        v.y &= 0x01010101u;
        v.z &= 0x01010101u;
        v.w &= 0x01010101u;
        A[i] = v;
    }
}
}  // namespace tb

extern "C" int tb_abs_pack(const int8_t* S, int64_t m, int64_t ldS, int8_t* A, void* stream) {
    if (m < 1 || ldS < 16 || (ldS & 15)) return fail(TB_ERR_CONFIG, "abs_pack: bad shape");
    if (!S || !A) return fail(TB_ERR_INVALID, "abs_pack: null pointer");
    const int64_t nvec = m * ldS / 16;
    const int64_t blocks = std::min<int64_t>((nvec + 255) / 256, (int64_t)num_sms() * 8);
    abs_pack_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const uint4*>(S), reinterpret_cast<uint4*>(A), nvec);
    return check_launch("abs_pack_kernel");
}
