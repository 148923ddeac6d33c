// Host side of the compact record stream (tb_records_compact): expands (numerator, n3) pairs into the
// reference's 48-byte CELL_DTYPE records (engine.py:45-55) in emission order (pairindex.py:116-129), on
// host threads (a persistent pool) with streaming stores.  compute_all_pairs runs it for some passes while the copy engine
// streams full records for the others, so a pass reaches the sink over two paths at once: PCIe carries
// 8 bytes per record instead of 48 for the expanded ones.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>
#include <immintrin.h>
#include <unistd.h>

#include "tb_common.cuh"

namespace tb {

// Where n3 comes from: the 8-byte stream (uint2: numerator, n3), or a 4-byte numerator stream plus the
// tied rows' table (n3 of a pair is 0 unless both variables are tied: tidx[i], tidx[j] >= 0 index the
// nt tied rows, n3t holds their pairs in the tied rows' own job-id order).
struct N3Src {
    const int32_t* tidx = nullptr;
    const int64_t* n3t = nullptr;
    int64_t nt = 0;
};

// Four records at a time (AVX2): the six fields of records j .. j+3 of row i as 4 x 64-bit vectors, transposed
// into the 24 quadwords of four consecutive 48-byte records (6 unpacks + 6 lane permutes + 6 stores).  Rows
// whose n3 comes from the tied-row table stay on the scalar loop.  Returns the first j not written.
static const bool g_has_avx2 = __builtin_cpu_supports("avx2");
static const int64_t g_prefetch_ahead = [] {
    // bytes ahead of the stores (0 = off).  The ring's lines come back from L3 on every lap; asking for them
    // in write state ahead of the stores took the config-5 call from 487-491 to 412-438 ms (expansion 387 ->
    // 293-339 ms; profiles/r02_plugin_prefetch.log)
    const char* e = std::getenv("TB_EXPAND_PREFETCH");
    return e ? (int64_t)std::max(0, atoi(e)) : (int64_t)512;
}();

template <bool NUM_ONLY, bool STREAM>
__attribute__((target("avx2"))) static inline int64_t expand_row_avx2(const void* cmpv, int64_t pos, int64_t i,
                                                                     int64_t jb, int64_t c1, const uint64_t* n1,
                                                                     uint64_t n1i, int64_t n0, int naive,
                                                                     uint8_t* out) {
    const __m256i vn1 = _mm256_set1_epi64x((int64_t)n1i);
    const __m256i vbase = _mm256_set1_epi64x(n0 - (int64_t)n1i);
    const __m256i zero = _mm256_setzero_si256();
    const __m256i sbit = _mm256_set1_epi64x((int64_t)0x8000000000000000ull);
    __m256i ij = _mm256_add_epi64(_mm256_set1_epi64x((int64_t)(uint64_t)(uint32_t)i),
                                  _mm256_slli_epi64(_mm256_add_epi64(_mm256_set1_epi64x(jb), _mm256_set_epi64x(3, 2, 1, 0)), 32));
    const __m256i ij_step = _mm256_set1_epi64x((int64_t)4 << 32);
    int64_t j = jb;
    for (; j + 4 <= c1; j += 4, pos += 4, ij = _mm256_add_epi64(ij, ij_step)) {
        __m256i num, n3;
        if constexpr (NUM_ONLY) {
            num = _mm256_cvtepi32_epi64(_mm_loadu_si128(reinterpret_cast<const __m128i*>(static_cast<const int32_t*>(cmpv) + pos)));
            n3 = zero;
        } else {
            const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(static_cast<const uint2*>(cmpv) + pos));
            n3 = _mm256_srli_epi64(v, 32);
            const __m256i lo = _mm256_and_si256(v, _mm256_set1_epi64x(0xFFFFFFFFll));
            const __m256i s31 = _mm256_set1_epi64x(0x80000000ll);
            num = _mm256_sub_epi64(_mm256_xor_si256(lo, s31), s31);  // sign-extend the low 32 bits
        }
        __m256i nd, n2, n1v;
        if (naive) {
            nd = n2 = n1v = n3 = zero;
        } else {
            n1v = vn1;
            n2 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(n1 + j));
            // nd = (n0 - n1 - n2 + n3 - num) / 2, C division (toward zero): add 1 to negatives, shift, keep the sign
            __m256i t = _mm256_sub_epi64(_mm256_add_epi64(_mm256_sub_epi64(vbase, n2), n3), num);
            const __m256i neg = _mm256_cmpgt_epi64(zero, t);
            t = _mm256_sub_epi64(t, neg);
            nd = _mm256_or_si256(_mm256_srli_epi64(t, 1), _mm256_and_si256(t, sbit));
        }
        const __m256i A = _mm256_unpacklo_epi64(ij, num), B = _mm256_unpackhi_epi64(ij, num);
        const __m256i C = _mm256_unpacklo_epi64(nd, n1v), D = _mm256_unpackhi_epi64(nd, n1v);
        const __m256i E = _mm256_unpacklo_epi64(n2, n3), F = _mm256_unpackhi_epi64(n2, n3);
        const __m256i v0 = _mm256_permute2x128_si256(A, C, 0x20), v1 = _mm256_permute2x128_si256(E, B, 0x20);
        const __m256i v2 = _mm256_permute2x128_si256(D, F, 0x20), v3 = _mm256_permute2x128_si256(A, C, 0x31);
        const __m256i v4 = _mm256_permute2x128_si256(E, B, 0x31), v5 = _mm256_permute2x128_si256(D, F, 0x31);
        uint8_t* r = out + 48 * pos;
        if constexpr (!STREAM) {  // ring slots: fetch the next lines for writing ahead of the stores (TB_EXPAND_PREFETCH)
            if (g_prefetch_ahead > 0) {
                __builtin_prefetch(r + g_prefetch_ahead, 1, 3);
                __builtin_prefetch(r + g_prefetch_ahead + 64, 1, 3);
                __builtin_prefetch(r + g_prefetch_ahead + 128, 1, 3);
            }
        }
        if constexpr (STREAM) {  // records are 16-byte aligned only: 128-bit non-temporal halves
            __m128i* r16 = reinterpret_cast<__m128i*>(r);
            const __m256i vs[6] = {v0, v1, v2, v3, v4, v5};
            for (int k = 0; k < 6; ++k) {
                _mm_stream_si128(r16 + 2 * k, _mm256_castsi256_si128(vs[k]));
                _mm_stream_si128(r16 + 2 * k + 1, _mm256_extracti128_si256(vs[k], 1));
            }
        } else {
            __m256i* r32 = reinterpret_cast<__m256i*>(r);
            _mm256_storeu_si256(r32, v0);
            _mm256_storeu_si256(r32 + 1, v1);
            _mm256_storeu_si256(r32 + 2, v2);
            _mm256_storeu_si256(r32 + 3, v3);
            _mm256_storeu_si256(r32 + 4, v4);
            _mm256_storeu_si256(r32 + 5, v5);
        }
    }
    return j;
}

// Records of tiles [t0, t1) (record offsets relative to the pass's first tile base0).
// STREAM: non-temporal stores (records bound for DRAM: slots far larger than the last-level cache);
// otherwise plain stores, for destinations small enough to stay cache-resident (the pass ring).
template <bool NUM_ONLY, bool STREAM>
static void expand_tiles(const void* cmpv, const uint64_t* n1, int64_t m, int64_t n0, int64_t q, int64_t w,
                         int64_t t0, int64_t t1, int64_t base0, int naive, uint8_t* out, N3Src tab) {
    const uint2* cmp = static_cast<const uint2*>(cmpv);
    const int32_t* nums = static_cast<const int32_t*>(cmpv);
    int64_t pos = cells_before_tile(t0, m, q, w) - base0;
    int64_t ty, tx;
    job_coord(t0, w, ty, tx);
    for (int64_t t = t0; t < t1; ++t) {
        const int64_t r0 = ty * q, c0 = tx * q;
        const int64_t r1 = std::min(r0 + q, m), c1 = std::min(c0 + q, m);
        for (int64_t i = r0; i < r1; ++i) {
            const int64_t jb = std::max(i, c0);
            const uint64_t n1i = naive ? 0 : n1[i];
            const int64_t ti = NUM_ONLY && !naive && tab.tidx ? tab.tidx[i] : -1;
            const int64_t trow = ti >= 0 ? ti * (2 * tab.nt - ti + 1) / 2 - ti : 0;  // tied job id of (ti, tj) = trow + tj
            int64_t j = jb;
            if (g_has_avx2 && ti < 0 && c1 - jb >= 4) {
                j = expand_row_avx2<NUM_ONLY, STREAM>(cmpv, pos, i, jb, c1, n1, n1i, n0, naive, out);
                pos += j - jb;
            }
            for (; j < c1; ++j, ++pos) {
                int64_t num;
                uint64_t n3 = 0;
                if constexpr (NUM_ONLY) {
                    num = nums[pos];
                    if (ti >= 0) {
                        const int64_t tj = tab.tidx[j];
                        if (tj >= 0) n3 = (uint64_t)tab.n3t[trow + tj];
                    }
                } else {
                    const uint2 v = cmp[pos];
                    num = (int32_t)v.x;
                    n3 = v.y;
                }
                uint64_t nd = 0, n2 = 0, n1v = 0;
                if (naive) {
                    n3 = 0;
                } else {
                    n1v = n1i;
                    n2 = n1[j];
                    nd = (uint64_t)(((int64_t)n0 - (int64_t)n1v - (int64_t)n2 + (int64_t)n3 - num) / 2);
                }
                __m128i* r = reinterpret_cast<__m128i*>(out + 48 * pos);
                const __m128i v0 = _mm_set_epi64x(num, (int64_t)((uint64_t)(uint32_t)i | ((uint64_t)(uint32_t)j << 32)));
                const __m128i v1 = _mm_set_epi64x((int64_t)n1v, (int64_t)nd);
                const __m128i v2 = _mm_set_epi64x((int64_t)n3, (int64_t)n2);
                if constexpr (STREAM) {
                    _mm_stream_si128(r, v0);
                    _mm_stream_si128(r + 1, v1);
                    _mm_stream_si128(r + 2, v2);
                } else {
                    _mm_store_si128(r, v0);
                    _mm_store_si128(r + 1, v1);
                    _mm_store_si128(r + 2, v2);
                }
            }
        }
        // next tile in id order: along the tile row, then the next row's diagonal tile
        if (++tx >= w) {
            ++ty;
            tx = ty;
        }
    }
    if constexpr (STREAM) _mm_sfence();  // streaming stores are weakly ordered: drain them before the thread reports done
}

// Persistent expansion workers: a config-5 call expands ~400 batches; spawning a dozen std::threads per
// batch cost more than the batch's own page of work at the small end.  One call at a time owns the pool
// (concurrent callers queue on `call_mu`); the caller thread runs part 0 itself.
class ExpandPool {
  public:
    void run(int parts, const std::function<void(int)>& fn) {
        std::lock_guard<std::mutex> call(call_mu_);
        ensure(parts - 1);
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            next_ = 1;
            parts_ = parts;
            pending_ = parts - 1;
            ++gen_;
        }
        cv_.notify_all();
        fn(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }

  private:
    void ensure(int n) {
        while ((int)workers_.size() < n) workers_.emplace_back([this] { loop(); });
    }
    void loop() {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> lk(mu_);
        for (;;) {
            cv_.wait(lk, [&] { return gen_ != seen && next_ < parts_; });
            const int part = next_++;
            if (next_ >= parts_) seen = gen_;
            const std::function<void(int)>* fn = fn_;
            lk.unlock();
            (*fn)(part);
            lk.lock();
            if (--pending_ == 0) done_cv_.notify_all();
        }
    }
    std::mutex call_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    std::vector<std::thread> workers_;
    const std::function<void(int)>* fn_ = nullptr;
    int next_ = 0, parts_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
};

// One pool per process, never destroyed (workers live for the process).  A fork()ed child inherits the pool
// object but not its threads, so a child builds its own (the parent's copy is abandoned, not touched).
static ExpandPool& expand_pool() {
    static std::mutex mu;
    static ExpandPool* pool = nullptr;
    static pid_t owner = 0;
    std::lock_guard<std::mutex> lk(mu);
    if (!pool || owner != getpid()) {
        pool = new ExpandPool();
        owner = getpid();
    }
    return *pool;
}

}  // namespace tb

using namespace tb;

// 0: streaming stores (default), 1: plain stores (cache-resident destinations)
static std::atomic<int> g_expand_plain{0};
extern "C" int tb_expand_store_mode(int plain) {
    return g_expand_plain.exchange(plain ? 1 : 0);
}

template <bool NUM_ONLY>
static int expand_impl(const void* compact, const uint64_t* n1_rows, int64_t m, int64_t n, int64_t q,
                       int64_t tile_lo, int64_t ntiles, int naive, void* records, int nthreads, N3Src tab) {
    if (m < 1 || q < 1 || n < 1) return fail(TB_ERR_CONFIG, "expand_records: need m, q, n >= 1");
    const int64_t w = (m + q - 1) / q, tt = w * (w + 1) / 2;
    if (ntiles < 0 || tile_lo < 0 || tile_lo + ntiles > tt) return fail(TB_ERR_CONFIG, "expand_records: bad tile range");
    if (ntiles == 0) return TB_OK;
    if (!compact || !records || (!naive && !n1_rows)) return fail(TB_ERR_INVALID, "expand_records: null pointer");
    if ((reinterpret_cast<uintptr_t>(records) & 15) != 0) return fail(TB_ERR_INVALID, "expand_records: records not 16-byte aligned");
    const int64_t n0 = n * (n - 1) / 2;
    const int64_t base0 = cells_before_tile(tile_lo, m, q, w);
    uint8_t* out = static_cast<uint8_t*>(records);
    const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(nthreads, ntiles));
    const bool plain = g_expand_plain.load(std::memory_order_relaxed) != 0;
    auto run = [&](int64_t a, int64_t b) {
        if (plain) expand_tiles<NUM_ONLY, false>(compact, n1_rows, m, n0, q, w, a, b, base0, naive, out, tab);
        else expand_tiles<NUM_ONLY, true>(compact, n1_rows, m, n0, q, w, a, b, base0, naive, out, tab);
    };
    if (nt == 1) {
        run(tile_lo, tile_lo + ntiles);
    } else {
        const std::function<void(int)> part = [&](int k) {
            run(tile_lo + ntiles * k / nt, tile_lo + ntiles * (k + 1) / nt);
        };
        expand_pool().run(nt, part);
    }
    _mm_sfence();
    return TB_OK;
}

// ---- pass ring: one compact batch expanded pass by pass into a small ring of pass buffers.
// The big record slots are DRAM-bound (non-temporal stores, ~150-195 GB/s on the B200 boxes' 16 cores, less
// next to a D2H); a ring of a few pass buffers stays in the cores' caches, so the plain stores never reach
// DRAM before the sink has seen the pass (tools/probe_expand_ring.py).  The pool is entered once per batch;
// its workers run the passes back to back, each taking the same share of every pass (the same ring bytes
// every lap: they stay in that core's L2), synchronised only by two counters: ctl[0] = passes produced,
// ctl[1] = passes the consumer released (ctl[2] != 0 aborts).
static inline int64_t ctl_load(const int64_t* p) { return __atomic_load_n(p, __ATOMIC_ACQUIRE); }

template <typename Cond>
static bool ring_spin(const int64_t* ctl, Cond ok) {
    for (int64_t spins = 0;; ++spins) {
        if (ok()) return true;
        if (ctl_load(ctl + 2) != 0) return false;
        if (spins < 2000) _mm_pause();
        else if (spins < 4000) std::this_thread::yield();
        else usleep(50);
    }
}

extern "C" int tb_ring_wait(const int64_t* ctl, int64_t seq) {
    if (!ctl) return fail(TB_ERR_INVALID, "ring_wait: null control block");
    return ring_spin(ctl, [&] { return ctl_load(ctl) > seq; }) ? TB_OK : TB_ERR_ABORTED;
}

extern "C" int tb_expand_ring(const void* compact, int width, const uint64_t* n1_rows, const int32_t* tidx,
                              const int64_t* n3t, int64_t nt_rows, int64_t m, int64_t n, int64_t q,
                              const int64_t* pass_tile, int64_t npass, int naive, void* ring, int64_t slot_bytes,
                              int64_t nslots, int64_t seq0, int64_t* ctl, int nthreads) {
    if (m < 1 || q < 1 || n < 1) return fail(TB_ERR_CONFIG, "expand_ring: need m, q, n >= 1");
    if (width != 4 && width != 8) return fail(TB_ERR_CONFIG, "expand_ring: width must be 4 or 8");
    if (npass < 0 || nslots < 1 || slot_bytes < 0 || seq0 < 0) return fail(TB_ERR_CONFIG, "expand_ring: bad ring geometry");
    if (npass == 0) return TB_OK;
    if (!compact || !ring || !ctl || !pass_tile || (!naive && !n1_rows))
        return fail(TB_ERR_INVALID, "expand_ring: null pointer");
    if ((reinterpret_cast<uintptr_t>(ring) & 15) != 0 || (slot_bytes & 15) != 0)
        return fail(TB_ERR_INVALID, "expand_ring: ring slots not 16-byte aligned");
    if (width == 4 && (nt_rows < 0 || nt_rows > m || (nt_rows > 0 && (!tidx || !n3t))))
        return fail(TB_ERR_INVALID, "expand_ring: bad tied-row table");
    const int64_t w = (m + q - 1) / q, tt = w * (w + 1) / 2;
    for (int64_t p = 0; p < npass; ++p)
        if (pass_tile[p] < 0 || pass_tile[p + 1] < pass_tile[p] || pass_tile[p + 1] > tt)
            return fail(TB_ERR_CONFIG, "expand_ring: bad pass tile ranges");
    const int64_t n0 = n * (n - 1) / 2;
    const int64_t base_batch = cells_before_tile(pass_tile[0], m, q, w);
    std::vector<int64_t> base(npass + 1);
    for (int64_t p = 0; p <= npass; ++p)
        base[p] = pass_tile[p] >= tt ? m * (m + 1) / 2 : cells_before_tile(pass_tile[p], m, q, w);
    for (int64_t p = 0; p < npass; ++p)
        if ((base[p + 1] - base[p]) * 48 > slot_bytes) return fail(TB_ERR_CAPACITY, "expand_ring: a pass exceeds the ring slot");
    N3Src tab;
    tab.tidx = (width == 4 && nt_rows > 0) ? tidx : nullptr;
    tab.n3t = n3t;
    tab.nt = width == 4 ? nt_rows : 0;
    const int nthr = (int)std::max<int64_t>(1, nthreads);
    // Every pass is cut into SUB chunks per worker.  A worker expands its own chunks first (the same ring
    // bytes every lap: they stay in its core's L2), then takes unclaimed chunks of workers that fell behind
    // -- from their last chunk backwards, so a worker that is merely a little late keeps its share.  On a
    // quiet host nothing is stolen; when a worker loses its core for a while (12 workers, the producer, the
    // consumer and the writer share 16 cores) the pass no longer waits for it.  TB_EXPAND_STEAL=0: off.
    static const bool kSteal = [] { const char* e = std::getenv("TB_EXPAND_STEAL"); return !e || e[0] != '0'; }();
    constexpr int SUB = 4;
    const int C = nthr * SUB;
    std::vector<std::atomic<uint8_t>> claimed((size_t)npass * C);
    for (auto& c : claimed) c.store(0, std::memory_order_relaxed);
    std::vector<std::atomic<int>> done(npass);
    for (auto& d : done) d.store(0, std::memory_order_relaxed);
    std::atomic<int> aborted{0};
    std::mutex pub_mu;
    int64_t published = 0;  // passes [0, published) are visible to the consumer (guarded by pub_mu)
    const std::function<void(int)> part = [&](int k) {
        for (int64_t p = 0; p < npass; ++p) {
            const int64_t seq = seq0 + p;
            if (!ring_spin(ctl, [&] { return seq - ctl_load(ctl + 1) < nslots; })) {
                aborted.store(1);
                return;
            }
            const int64_t t_lo = pass_tile[p], nti = pass_tile[p + 1] - t_lo;
            uint8_t* out = static_cast<uint8_t*>(ring) + (seq % nslots) * slot_bytes;
            const uint8_t* src = static_cast<const uint8_t*>(compact) + (base[p] - base_batch) * width;
            auto chunk = [&](int c) {
                std::atomic<uint8_t>& flag = claimed[(size_t)p * C + c];
                if (flag.load(std::memory_order_relaxed) != 0 || flag.exchange(1, std::memory_order_acq_rel) != 0) return;
                const int64_t a = t_lo + nti * c / C, b = t_lo + nti * (c + 1) / C;
                if (a < b) {
                    if (width == 4) expand_tiles<true, false>(src, n1_rows, m, n0, q, w, a, b, base[p], naive, out, tab);
                    else expand_tiles<false, false>(src, n1_rows, m, n0, q, w, a, b, base[p], naive, out, tab);
                }
                if (done[p].fetch_add(1, std::memory_order_acq_rel) == C - 1) {
                    // pass p is complete; publish it and any complete passes behind a late one, in order
                    std::lock_guard<std::mutex> lk(pub_mu);
                    while (published < npass && done[published].load(std::memory_order_acquire) == C) {
                        ++published;
                        __atomic_store_n(ctl, seq0 + published, __ATOMIC_RELEASE);
                    }
                }
            };
            for (int s2 = 0; s2 < SUB; ++s2) chunk(k * SUB + s2);
            if (kSteal)
                for (int off = 1; off < nthr; ++off) {
                    const int v = (k + off) % nthr;
                    for (int s2 = SUB - 1; s2 >= 0; --s2) chunk(v * SUB + s2);
                }
        }
    };
    if (nthr == 1) part(0);
    else expand_pool().run(nthr, part);
    return aborted.load() ? TB_ERR_ABORTED : TB_OK;
}

extern "C" int tb_expand_records(const void* compact, const uint64_t* n1_rows, int64_t m, int64_t n, int64_t q,
                                 int64_t tile_lo, int64_t ntiles, int naive, void* records, int nthreads) {
    return expand_impl<false>(compact, n1_rows, m, n, q, tile_lo, ntiles, naive, records, nthreads, N3Src{});
}

extern "C" int tb_expand_records_num(const int32_t* nums, const uint64_t* n1_rows, const int32_t* tidx,
                                     const int64_t* n3t, int64_t nt, int64_t m, int64_t n, int64_t q, int64_t tile_lo,
                                     int64_t ntiles, int naive, void* records, int nthreads) {
    if (nt < 0 || nt > m || (nt > 0 && (!tidx || !n3t)))
        return fail(TB_ERR_INVALID, "expand_records_num: bad tied-row table");
    N3Src tab;
    tab.tidx = nt > 0 ? tidx : nullptr;
    tab.n3t = n3t;
    tab.nt = nt;
    return expand_impl<true>(nums, n1_rows, m, n, q, tile_lo, ntiles, naive, records, nthreads, tab);
}

// Pageable host array -> device through two pinned staging buffers: the pool's threads fill one buffer
// (parallel memcpy) while the copy engine drains the other in <= 4 MiB pieces.  One call for the whole
// upload, so a Python caller holds no GIL while it runs (compute_all_pairs' early upload overlaps the
// main thread's planning).  Replaces the host side of the reference's dataset hand-off to its workers
// (engine.py:338-352: the rank matrix is shared with the worker threads as is).
extern "C" int tb_h2d_staged(const void* src, void* dst, int64_t nbytes, void* stage_a, void* stage_b,
                             int64_t stage_bytes, int nthreads, void* stream) {
    if (nbytes < 0 || stage_bytes < (1 << 20)) return fail(TB_ERR_CONFIG, "h2d_staged: bad sizes");
    if (nbytes == 0) return TB_OK;
    if (!src || !dst || !stage_a || !stage_b) return fail(TB_ERR_INVALID, "h2d_staged: null pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t* stage[2] = {static_cast<uint8_t*>(stage_a), static_cast<uint8_t*>(stage_b)};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    bool used[2] = {false, false};
    int rc = TB_OK;
    for (int b = 0; b < 2; ++b)
        if (cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming) != cudaSuccess) rc = fail(TB_ERR_CUDA, "h2d_staged: event");
    const uint8_t* s8 = static_cast<const uint8_t*>(src);
    uint8_t* d8 = static_cast<uint8_t*>(dst);
    const int nt = std::max(1, nthreads);
    int k = 0;
    for (int64_t o = 0; o < nbytes && rc == TB_OK; o += stage_bytes, ++k) {
        const int b = k & 1;
        const int64_t n = std::min(stage_bytes, nbytes - o);
        if (used[b] && cudaEventSynchronize(ev[b]) != cudaSuccess) { rc = fail(TB_ERR_CUDA, "h2d_staged: sync"); break; }
        const std::function<void(int)> part = [&](int t) {
            const int64_t a = n * t / nt, e = n * (t + 1) / nt;
            memcpy(stage[b] + a, s8 + o + a, (size_t)(e - a));
        };
        if (nt == 1) part(0);
        else expand_pool().run(nt, part);
        for (int64_t q = 0; q < n; q += (4 << 20)) {
            const int64_t e = std::min(n, q + (int64_t)(4 << 20));
            if (cudaMemcpyAsync(d8 + o + q, stage[b] + q, (size_t)(e - q), cudaMemcpyHostToDevice, st) != cudaSuccess) {
                rc = fail(TB_ERR_CUDA, "h2d_staged: copy");
                break;
            }
        }
        if (rc == TB_OK && cudaEventRecord(ev[b], st) != cudaSuccess) rc = fail(TB_ERR_CUDA, "h2d_staged: record");
        used[b] = true;
    }
    for (int b = 0; b < 2; ++b) {
        if (used[b]) cudaEventSynchronize(ev[b]);  // the staging buffers are free again on return
        if (ev[b]) cudaEventDestroy(ev[b]);
    }
    return rc;
}
