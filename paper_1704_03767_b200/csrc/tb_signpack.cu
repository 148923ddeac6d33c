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
constexpr int SP_DCHUNK = 64;  // offsets d handled per work item

// Row value i lives at shared index i + i/16: lanes reading indices 16 apart hit distinct banks.
__device__ __forceinline__ int spad(int i) { return i + (i >> 4); }

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

// One warp = 32 consecutive 16-sample groups (a0 = 16 g) x a run of SP_DCHUNK offsets d.  A lane
// keeps its own 16 values and a 32-value sliding window x[a0 + d ..] in registers: per d it loads
// one new value, emits 16 signs as one uint4 (the warp writes 512 contiguous bytes), slides.
template <typename T>
__global__ void __launch_bounds__(SP_THREADS) signpack_kernel(const T* __restrict__ x, int64_t m, int64_t n,
                                                              int64_t ldx, int8_t* __restrict__ S, int64_t ldS,
                                                              int64_t K, unsigned long long* __restrict__ nz,
                                                              int32_t* __restrict__ flags) {
    extern __shared__ __align__(16) uint8_t sp_smem[];
    T* xs = reinterpret_cast<T*>(sp_smem);
    const int64_t r = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31;
    const int nn = (int)n;
    const int slack = nn + 48;  // window reads run up to 31 past n (masked)

    bool bad = false;
    for (int i = tid; i < slack; i += SP_THREADS) {
        T v = i < nn ? x[r * ldx + i] : T(0);
        bad |= (v != v);  // NaN has no rank (ranks.py:56-57)
        xs[spad(i)] = v;
    }
    if (bad) atomicOr(flags, 1);
    __syncthreads();

    int8_t* row = S + r * ldS;
    uint32_t cnt = 0;
    const int ngroups = (nn - 1 + 15) >> 4;          // groups with a0 < n - 1
    const int gblocks = (ngroups + 31) >> 5;
    const int nchunks = (nn - 1 + SP_DCHUNK - 1) / SP_DCHUNK;
    const int items = nchunks * gblocks;
    const int warps = SP_THREADS / 32;
    for (int it = blockIdx.y * warps + (tid >> 5); it < items; it += gridDim.y * warps) {
        const int c = it / gblocks, gb = it - c * gblocks;
        const int g = gb * 32 + lane;
        const int a0 = g * 16;
        const int d_lo = 1 + c * SP_DCHUNK;
        const int d_hi = min(1 + (c + 1) * SP_DCHUNK, nn - a0);  // group g exists while a0 < n - d
        if (d_lo >= d_hi) continue;
        T own[16], win[32];
#pragma unroll
        for (int i = 0; i < 16; ++i) own[i] = xs[spad(a0 + i)];
#pragma unroll
        for (int i = 0; i < 16; ++i) win[i] = xs[spad(a0 + d_lo + i)];
        int64_t off = diag_off(d_lo, n) + 16 * g;
        for (int db = d_lo; db < d_hi; db += 16) {
#pragma unroll
            for (int i = 0; i < 16; ++i) win[16 + i] = xs[spad(a0 + db + 16 + i)];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int d = db + j;
                if (d < d_hi) {
                    const int lim = nn - d - a0;  // samples a0 + i valid for i < lim
                    uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const T xb = win[i + j], xa = own[i];
                        const uint32_t gt = xb > xa, lt = xb < xa;
                        const uint32_t byte = (i < lim) ? (gt | (lt * 0xFFu)) : 0u;
                        w[i >> 2] |= byte << ((i & 3) * 8);
                    }
                    *reinterpret_cast<uint4*>(row + off) = make_uint4(w[0], w[1], w[2], w[3]);
                    cnt += __popc(w[0] & 0x01010101u) + __popc(w[1] & 0x01010101u) +
                           __popc(w[2] & 0x01010101u) + __popc(w[3] & 0x01010101u);
                    off += 16 * ((nn - d + 15) >> 4);
                }
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) win[i] = win[16 + i];
        }
    }
    // zero the row tail [K, ldS)
    for (int64_t k = K + ((int64_t)blockIdx.y * SP_THREADS + tid) * 16; k < ldS; k += (int64_t)gridDim.y * SP_THREADS * 16)
        *reinterpret_cast<uint4*>(row + k) = make_uint4(0u, 0u, 0u, 0u);
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0 && cnt) atomicAdd(&nz[r], (unsigned long long)cnt);
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
    const int64_t K = diag_k(n);
    if (ldS < K || (ldS & 15)) return fail(TB_ERR_CONFIG, "sign_pack: ldS=%lld must be >= K=%lld and 16-aligned",
                                           (long long)ldS, (long long)K);
    if (ldx < n) return fail(TB_ERR_CONFIG, "sign_pack: ldx < n");
    if (!x || !S || !n1 || !flags) return fail(TB_ERR_INVALID, "sign_pack: null pointer");
    size_t esz = dtype == TB_DTYPE_F64 ? 8 : 4;
    size_t smem = ((size_t)(n + 48 + (n + 48) / 16 + 1) * esz + 15) & ~size_t(15);
    if (smem > 200 * 1024) return fail(TB_ERR_CAPACITY, "sign_pack: row of n=%lld does not fit shared memory", (long long)n);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TB_CUDA_TRY(cudaMemsetAsync(n1, 0, m * sizeof(uint64_t), st));
    const int64_t items = ((n - 1 + SP_DCHUNK - 1) / SP_DCHUNK) * (((n - 1 + 15) / 16 + 31) / 32);
    const int64_t nblk = (items + SP_THREADS / 32 - 1) / (SP_THREADS / 32);
    int64_t want = (8 * (int64_t)num_sms() + m - 1) / m;  // >= ~8 CTAs per SM in total
    int gy = (int)std::min<int64_t>(std::max<int64_t>(want, 1), std::min<int64_t>(nblk, 65535));
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
    nz_to_n1_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(nz, m, (unsigned long long)(n * (n - 1) / 2));
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

extern "C" int64_t tb_sign_k(int64_t n) { return n >= 2 ? tb::diag_k(n) : 0; }
