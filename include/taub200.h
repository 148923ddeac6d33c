/*
 * taub200 -- C ABI of the B200 (sm_100a) all-pairs Kendall tau engine.
 *
 * Plain extern "C": raw device pointers, sizes and a cudaStream_t passed as
 * void*.  All memory is caller-allocated; every call is asynchronous on the
 * given stream and returns a status code.  Status codes map one-to-one onto
 * the reference exception hierarchy (src/taucorr/errors.py:4-24):
 *
 *   TB_OK             0
 *   TB_ERR_INVALID    1  -> InvalidInputError     (errors.py:8-9)
 *   TB_ERR_CAPACITY   2  -> CapacityExceededError (errors.py:12-17)
 *   TB_ERR_CONFIG     3  -> ConfigError           (errors.py:23-24)
 *   TB_ERR_CUDA       4  -> RuntimeError (CUDA launch/driver failure)
 *   TB_ERR_ABORTED    5  -> (host pass ring only) the caller raised the ring's abort flag
 *
 * tb_last_error() returns the message of the last failing call on the calling
 * thread.
 *
 * Ordering contract: "job ids" are the reference's diagonal-inclusive
 * upper-triangle numbering J_m(y, x) = y(2m - y + 1)/2 + x - y
 * (src/taucorr/pairindex.py:20-31).  Every per-pair output buffer holds the
 * contiguous job-id range [job_lo, job_hi) at offset j - job_lo, which is
 * also the unit of multi-GPU sharding (pairindex.py:68-80 semantics).
 *
 * Citations are into /root/reference/pkg/.
 */
#ifndef TAUB200_H
#define TAUB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TB_ABI_VERSION 1

#define TB_OK 0
#define TB_ERR_INVALID 1
#define TB_ERR_CAPACITY 2
#define TB_ERR_CONFIG 3
#define TB_ERR_CUDA 4
#define TB_ERR_ABORTED 5

#define TB_DTYPE_I32 0
#define TB_DTYPE_F32 1
#define TB_DTYPE_F64 2

/* Sign-matrix element formats (S of tb_sign_pack / tb_gemm_pairs):
 *   TB_SIGN_I8    int8 -1/0/+1, one per byte      -> tcgen05 kind::i8 (exact int32 sums)
 *   TB_SIGN_E4M3  e4m3 -1/0/+1, one per byte      -> tcgen05 kind::f8f6f4 (f32 sums; experiment)
 *   TB_SIGN_E2M1  e2m1 -1/0/+1, two per byte      -> tcgen05 kind::mxf4, unit scales (f32 sums,
 *                 exact while K < 2^24, i.e. n <= 5792); the default GEMM format */
#define TB_SIGN_I8 0
#define TB_SIGN_E4M3 1
#define TB_SIGN_E2M1 2
/*   TB_SIGN_E2M1_OFS  e2m1 S + 1 (0 / 1 / 2 for -1 / tie / +1; unused slots 0), same layout as
 *                 TB_SIGN_E2M1.  (S_y + 1).(S_x + 1) = S_y.S_x + s_y + s_x + n0 with s = the row sums of S
 *                 (tb_sign_row_sums), so tb_gemm_pairs_fix(fix = s, fix_c = n0) returns the same numerators.
 *                 Exact while 4 K < 2^24 (n <= 2896).  Non-negative, half-zero operands toggle fewer
 *                 tensor-pipe bits than +-1: the power-capped GEMM of a long run is ~12% faster (DESIGN 3). */
#define TB_SIGN_E2M1_OFS 3

/* Largest n the device paths accept: the int32 numerator holds |n_c - n_d| <=
 * n(n-1)/2 < 2^31 exactly up to here.  Larger n raises
 * TB_ERR_CAPACITY (the reference's packed-capacity convention, ranks.py:64-76). */
#define TB_MAX_N 65536

typedef struct {
    int32_t abi_version;
    int32_t device;
    int32_t sm_count;
    int32_t cc_major;
    int32_t cc_minor;
    int32_t tcgen05_i8; /* 1 when the tcgen05 kind::i8 GEMM can run (sm_100a) */
    int64_t smem_optin;
} tb_caps;

const char *tb_last_error(void);
int tb_query(int device, tb_caps *caps);
/* Number of kernels this library has launched since load (all threads, all devices): the
 * launch-count evidence bench.py reports as gpu_launches. */
int64_t tb_launch_count(void);

/*
 * K0 rank transform (rank_transform, src/taucorr/ranks.py:37-61, for all rows
 * at once): dense 0-based ranks, ties share a rank, -0.0 == +0.0.
 *   x     [m, ldx] values (TB_DTYPE_*), n <= 8192 (the GEMM path)
 *   R     [m, ldr] uint16 ranks out (ldr >= n, multiple of 8; [n, ldr) zeroed)
 *   n1    [m] uint64 per-row tied-pair count sum_t t(t-1)/2 (kernel_sorted.py:163-176)
 *   flags device int32; bit 0 is set when a NaN was seen (ranks.py:56-57)
 */
int tb_rank_rows(const void *x, int dtype, int64_t m, int64_t n, int64_t ldx, uint16_t *R, int64_t ldr,
                 uint64_t *n1, int32_t *flags, void *stream);

/*
 * K0w rank transform for rows of any width (rank_transform, src/taucorr/ranks.py:37-61; the per-row loop
 * of dataio.py:194-196): dense 0-based int32 ranks, ties share a rank, -0.0 == +0.0, +-inf orderable.
 * The merge path's input stage (raw values -> tb_presort); one CTA per row, stable LSD radix sort.
 *   x         [m, ldx] values (TB_DTYPE_*), any n >= 1
 *   R         [m, ldr] ranks out: int32, or uint16 when r_u16 != 0 (n <= 65536; the sign pack's input for
 *             GEMM-path rows wider than tb_rank_rows takes; [n, ldr) zeroed)
 *   n1        [m] uint64 tied-pair count sum_t t(t-1)/2 per row (kernel_sorted.py:163-176)
 *   flags     device int32; bit 0 set when a NaN was seen (ranks.py:56-57)
 *   workspace device scratch of >= tb_rank_dense_workspace(m, n, dtype) bytes (for the current device)
 */
int64_t tb_rank_dense_workspace(int64_t m, int64_t n, int dtype);
int tb_rank_dense(const void *x, int dtype, int64_t m, int64_t n, int64_t ldx, void *R, int r_u16, int64_t ldr,
                  uint64_t *n1, int32_t *flags, void *workspace, int64_t ws_bytes, void *stream);

/*
 * K2 sign pack.  Replaces the per-pair sign enumeration of naive_numerator
 * (src/taucorr/kernel_naive.py:26-44), materialising each variable's sign
 * vector once.
 *   R     [m, ldr] uint16 dense ranks (< 2^15; tb_rank_rows output), ldr even
 *   S     [m, ldS] signs sign(R[r, b] - R[r, a]) of the n(n-1)/2 sample pairs a < b, one fixed
 *         order for every row (any order gives S_u.S_v = n_c - n_d), in 16-pair chunks (16 bytes
 *         int8/e4m3, 8 bytes e2m1).  "Block" order, nbf = n / 16 full 16-sample blocks:
 *           1. pairs between full blocks A < B (row-major), chunk a_l of (A, B) = (16A + a_l, 16B + s);
 *           2. pairs inside a full block: columns j and 16 - j share a chunk (s < j: (s, j), else
 *              (s - j, 16 - j)), the column-8 halves of blocks 2P and 2P + 1 share one;
 *           3. pairs ending at a tail sample b >= 16 nbf: a = 0 .. b-1 in chunks of 16.
 *         Unused slots (the tail of a section-3 segment, a lone column-8 half) are zero.
 *         K = tb_sign_k(n) = n(n-1)/2 + O(n/16) elements: K bytes for TB_SIGN_I8/E4M3, K/2 bytes
 *         for TB_SIGN_E2M1; the row tail up to ldS is zeroed; ldS (bytes) must be a multiple of 16.
 *         TB_SIGN_E2M1 stores chunk sample 8w + 4h + j in 32-bit word w, byte j, nibble h, and may
 *         write ties as -0 (0x8).
 */
int64_t tb_sign_k(int64_t n);
int tb_sign_pack(const uint16_t *R, int64_t m, int64_t n, int64_t ldr, int8_t *S, int64_t ldS, int format,
                 void *stream);

/*
 * K3 numerator GEMM on tcgen05 tensor cores (TMA-fed, TMEM accumulators, 2-SM
 * CTA pairs): num[j - job_lo] = S_y . S_x = n_c - n_d for every job id j in
 * [job_lo, job_hi).  Replaces the per-cell numerator of _tiles_naive
 * (src/taucorr/engine.py:170-188).  Exact: int32 sums (TB_SIGN_I8) or f32 sums
 * of +-1 below 2^24 (TB_SIGN_E2M1 requires K < 2^24).  K is the element count
 * (tb_sign_k(n)); format selects kind::i8 / f8f6f4 / mxf4.
 * splits: K-split factor (0 = automatic).  With splits > 1 the kernel
 * accumulates atomically; the library zeroes num first.
 */
int tb_gemm_pairs(const int8_t *S, int64_t m, int64_t K, int64_t ldS, int format, int64_t job_lo, int64_t job_hi,
                  int32_t splits, int32_t *num, void *stream);

/* The same GEMM over offset operands (e2m1 formats): num[j - job_lo] = S_y . S_x - fix[y] - fix[x] - fix_c,
 * fix[m] int32 on the device (NULL = tb_gemm_pairs).  TB_SIGN_E2M1_OFS numerators: fix = tb_sign_row_sums,
 * fix_c = n0 = n(n-1)/2; its tie-indicator matrix (tb_abs_pack of an OFS matrix, Z = [S == 0]) with
 * fix = n1 per row and fix_c = -n0 returns |S_y|.|S_x| = n0 - n1_y - n1_x + Z_y.Z_x, tb_full_counts' absdot. */
int tb_gemm_pairs_fix(const int8_t *S, int64_t m, int64_t K, int64_t ldS, int format, int64_t job_lo,
                      int64_t job_hi, int32_t splits, const int32_t *fix, int64_t fix_c, int32_t *num, void *stream);

/* fix[r] = sum_k S[r, k] of a TB_SIGN_E2M1_OFS matrix (the nibble values' sum minus n0): the Kendall
 * numerator of row r against the sample order, the correction term of tb_gemm_pairs_fix. */
int tb_sign_row_sums(const int8_t *S, int64_t m, int64_t ldS, int64_t n, int32_t *fix, void *stream);
/* tb_sign_pack(TB_SIGN_E2M1_OFS) and tb_sign_row_sums in one launch: the pack sums the values it writes
 * (fix is zeroed on the stream first), saving the extra pass over S. */
int tb_sign_pack_sums(const uint16_t *R, int64_t m, int64_t n, int64_t ldr, int8_t *S, int64_t ldS, int32_t *fix,
                      void *stream);

/* |S| for the full-count mode: A[r, k] = |S[r, k]| (0/1 int8), same layout.
 * The second GEMM A A^T gives n_c + n_d per pair (SURVEY 8 identities).
 * TB_SIGN_E2M1_OFS: A = the tie indicator Z = [S == 0] instead (unused slots stay 0), see tb_gemm_pairs_fix. */
int tb_abs_pack(const int8_t *S, int64_t m, int64_t ldS, int format, int8_t *A, void *stream);

/* Full counts on the GEMM path from num = S_y.S_x and absdot = |S_y|.|S_x|:
 * n_d = (absdot - num) / 2 and n3 = absdot - n0 + n1_y + n1_x (the CELL_DTYPE
 * fields of src/taucorr/engine.py:45-55).  nd / n3 may be NULL.  absdot may be NULL when no variable of
 * the range has ties (every n1 = 0): then |S_y|.|S_x| = n0 - n1_y - n1_x exactly (n3 = 0) and the
 * second GEMM is skipped. */
int tb_full_counts(const int32_t *num, const int32_t *absdot, const uint64_t *n1_rows, int64_t m, int64_t n,
                   int64_t job_lo, int64_t job_hi, uint64_t *nd, uint64_t *n3, void *stream);

/* Sparse full counts: after tb_full_counts' closed form (absdot NULL), overwrite n_d / n3 of the pairs of
 * two tied variables from the |S| GEMM over the tied rows only (absdot_t: job-id order of the nt tied rows
 * rows_t, ascending).  Processes tied job ids [tj_lo, tj_hi); pairs outside [job_lo, job_hi) are skipped.
 * n3 is zero for every pair with an untied variable, so this equals the full |S| GEMM path. */
int tb_tied_counts(const int32_t *absdot_t, const int32_t *rows_t, int64_t nt, const uint64_t *n1_rows, int64_t m,
                   int64_t n, int64_t job_lo, int64_t job_hi, int64_t tj_lo, int64_t tj_hi, const int32_t *num,
                   uint64_t *nd, uint64_t *n3, void *stream);

/*
 * Reference record stream: the 48-byte CELL_DTYPE records (src/taucorr/engine.py:45-55:
 * i, j, numerator, n_d, n1, n2, n3) of tiles [tile_lo, tile_lo + ntiles) of the q x q tile matrix in the
 * reference's emission order (pairindex.py:116-129; the per-tile loops of engine.py:170-238), gathered on the
 * device from job-id-ordered counts (num / nd / n3 indexed by job id - job_lo, n1 per row).  Every cell of
 * the tiles must have its job id in [job_lo, job_hi) (else TB_ERR_CONFIG).  Record k of the pass is the
 * k-th cell of the tiles in emission order (offsets are closed forms, see tb_tile_cells).  naive != 0
 * writes the naive kernel's zero counts.  Replaces the host-side record assembly of compute_all_pairs
 * (engine.py:366-376) and _pass_geometry (engine.py:261-276).
 */
int tb_records(const int32_t *num, const int64_t *nd, const int64_t *n3, const int64_t *n1_rows, int64_t m,
               int64_t q, int64_t job_lo, int64_t job_hi, int64_t tile_lo, int64_t ntiles, int naive, void *records,
               void *stream);

/*
 * Compact record stream: the records of tb_records as 8 bytes each -- (int32 numerator, uint32 n3) in the
 * same emission order -- for passes whose records are rebuilt on the host by tb_expand_records (PCIe
 * carries 1/6 of the bytes).  Same arguments and checks as tb_records; naive != 0 writes n3 = 0.
 */
int tb_records_compact(const int32_t *num, const int64_t *n3, int64_t m, int64_t q, int64_t job_lo, int64_t job_hi,
                       int64_t tile_lo, int64_t ntiles, int naive, void *compact, void *stream);

/*
 * Host-only: expand the compact stream of tiles [tile_lo, tile_lo + ntiles) into the 48-byte CELL_DTYPE
 * records tb_records would have written (byte-identical): i, j from the tile order, n1 = n1_rows[i],
 * n2 = n1_rows[j] (host array), n_d = (n0 - n1 - n2 + n3 - numerator) / 2 (result.py:42), n0 = n(n-1)/2.
 * records must be 16-byte aligned; nthreads host threads with streaming stores.  No device work.
 */
int tb_expand_records(const void *compact, const uint64_t *n1_rows, int64_t m, int64_t n, int64_t q,
                      int64_t tile_lo, int64_t ntiles, int naive, void *records, int nthreads);

/* The numerator alone (int32, 4 bytes per record, emission order) for runs whose n3 is known on the host:
 * n3 = 0 for every pair with an untied variable, and the tied rows' pairs come from a table
 * (tb_expand_records_num).  Same checks as tb_records. */
int tb_records_num(const int32_t *num, int64_t m, int64_t q, int64_t job_lo, int64_t job_hi, int64_t tile_lo,
                   int64_t ntiles, int32_t *out, void *stream);

/* Host-only: 48-byte records from the 4-byte numerator stream; tidx[m] maps a row to its index among the nt
 * tied rows (-1: untied), n3t[nt(nt+1)/2] holds n3 of the tied rows' pairs in their own job-id order.
 * nt = 0: no tied pair (tidx / n3t unused). */
int tb_expand_records_num(const int32_t *nums, const uint64_t *n1_rows, const int32_t *tidx, const int64_t *n3t,
                          int64_t nt, int64_t m, int64_t n, int64_t q, int64_t tile_lo, int64_t ntiles, int naive,
                          void *records, int nthreads);

/* Host-only: store policy of tb_expand_records / tb_expand_records_num.  0 (default): non-temporal stores,
 * for record slots far larger than the host's last-level cache; 1: plain stores, for a small ring of pass
 * buffers that stays cache-resident (the records are handed to the sink hot).  Returns the previous mode. */
int tb_expand_store_mode(int plain);

/* Host-only: one compact batch (width 4: tb_records_num stream + tied-row table as tb_expand_records_num;
 * width 8: tb_records_compact stream) expanded pass by pass into a ring of nslots pass buffers of slot_bytes
 * each, with plain stores, so the records stay cache-resident until the sink has seen them
 * (compute_all_pairs hands each pass to the sink as a view of its ring slot: engine.py:353-416 recycles
 * pass buffers the same way).  Pass p covers tiles [pass_tile[p], pass_tile[p + 1]) and is ring pass
 * seq0 + p of the run, written to ring + ((seq0 + p) % nslots) * slot_bytes.  ctl is the run's control block
 * (int64[3], zeroed by the caller): ctl[0] = passes produced (stored by this call, in order, once every
 * worker finished the pass), ctl[1] = passes released by the consumer (this call waits while
 * seq - ctl[1] >= nslots), ctl[2] != 0 aborts (TB_ERR_ABORTED).  Blocks until the batch is expanded. */
int tb_expand_ring(const void *compact, int width, const uint64_t *n1_rows, const int32_t *tidx, const int64_t *n3t,
                   int64_t nt, int64_t m, int64_t n, int64_t q, const int64_t *pass_tile, int64_t npass, int naive,
                   void *ring, int64_t slot_bytes, int64_t nslots, int64_t seq0, int64_t *ctl, int nthreads);

/* Host-only: block until ring pass seq is produced (ctl[0] > seq); TB_ERR_ABORTED if ctl[2] != 0. */
int tb_ring_wait(const int64_t *ctl, int64_t seq);

/* Cells (records) in tiles [tile_lo, tile_hi) of the q x q tile matrix over m variables, diagonal
 * included -- the sum of tile_cell_count (pairindex.py:107-112) in closed form; -1 on bad arguments.
 * Host-only, no device work. */
int64_t tb_tile_cells(int64_t m, int64_t q, int64_t tile_lo, int64_t tile_hi);

/* Same contract on CUDA cores (dp4a, TB_SIGN_I8 only); a GPU-side cross-check, not the product path. */
int tb_gemm_pairs_simt(const int8_t *S, int64_t m, int64_t K, int64_t ldS, int64_t job_lo, int64_t job_hi,
                       int32_t *num, void *stream);

/*
 * K5 fp64 finalize: derive_taus (src/taucorr/result.py:62-82) over the job
 * range.  tau_a = num / n0; tau_b = num / sqrt((n0 - n1_y) * (n0 - n1_x)), NaN
 * where the denominator is 0.  IEEE round-to-nearest div/sqrt, no
 * contraction: bit-identical to the reference.  tau_a / tau_b may be NULL.
 */
int tb_finalize(const int32_t *num, const uint64_t *n1_rows, int64_t m, int64_t n, int64_t job_lo,
                int64_t job_hi, double *tau_a, double *tau_b, void *stream);

/* K3 + K5 fused: tau_b of job ids [job_lo, job_hi) straight from the GEMM epilogue (8 B per pair written,
 * no numerator round trip through HBM), the same IEEE sequence as tb_finalize.  When the plan splits a
 * unit over K (few units: small m) or the format is int8, the numerators go to num_ws (job_hi - job_lo
 * int32, may be NULL only when neither happens) and tb_finalize runs after the GEMM.  Replaces the
 * numerator + derive_taus sequence (kernel_naive.py:26-44, result.py:62-82) for tau_b-only callers. */
int tb_gemm_tau_b(const int8_t *S, int64_t m, int64_t K, int64_t ldS, int format, int64_t job_lo, int64_t job_hi,
                  int32_t splits, const uint64_t *n1_rows, int64_t n, int32_t *num_ws, double *tau_b, void *stream);
/* tb_gemm_tau_b over offset operands (fix / fix_c as in tb_gemm_pairs_fix). */
int tb_gemm_tau_b_fix(const int8_t *S, int64_t m, int64_t K, int64_t ldS, int format, int64_t job_lo,
                      int64_t job_hi, int32_t splits, const int32_t *fix, int64_t fix_c, const uint64_t *n1_rows,
                      int64_t n, int32_t *num_ws, double *tau_b, void *stream);

/*
 * K1 presort for the merge path (large n): per variable, the position of
 * every observation in ascending-rank order (u-order), the rank sequence in
 * that order, the tie count n1 and the largest tie group.  Replaces step 1
 * of sorted_counts (src/taucorr/kernel_sorted.py:95-127, 163-176), once per
 * variable instead of once per pair.
 *   ranks   [m, n] int32 dense ranks (0 <= rank < n)
 *   pos     [m, n] int32 out: pos[r, e] = position of element e in u-order
 *   sorted  [m, n] int32 out: sorted[r, p] = rank at position p
 *   keys    [m, n] uint16 out: min-rank (competition rank) of every element, i.e. the number of
 *           elements of the row with a strictly smaller rank; the merge keys of tb_merge_pairs
 *   n1      [m] uint64 out;  maxgrp [m] int32 out (largest tie group)
 *   work    [m, n] int32 out: compact tie-group list, work[r, 2k] = first
 *           u-order position and work[r, 2k+1] = length of the k-th rank value
 *           held by >= 2 observations, k < ngroups[r]
 *   ngroups [m] int32 out
 *   flags   device int32; bit 1 is set when a rank is outside [0, n) (the
 *           caller raises InvalidInputError, as Dataset validation does)
 */
int tb_presort(const int32_t *ranks, int64_t m, int64_t n, int32_t *pos, int32_t *sorted, uint16_t *keys,
               uint64_t *n1, int32_t *maxgrp, int32_t *work, int32_t *ngroups, int32_t *flags, void *stream);

/*
 * K4 Knight merge-inversion counts (large n): for every job id in
 * [job_lo, job_hi): n_d (discordant pairs, strict), n3 (joint ties) and the
 * numerator n0 - n1 - n2 + n3 - 2 n_d (src/taucorr/result.py:42).  Replaces
 * steps 1-5 of sorted_counts (src/taucorr/kernel_sorted.py:195-212).
 * keys, pos, sorted, n1_rows, maxgrp, groups and ngroups are tb_presort's outputs.
 * nd / n3 may be NULL.  workspace: device scratch of >= tb_merge_workspace(n) bytes (for the current
 * device), used by pairs whose u variable has a tie group larger than 64 (the O(n log n) segmented count).
 */
int64_t tb_merge_workspace(int64_t n);
int tb_merge_pairs(const uint16_t *keys, const int32_t *pos, const int32_t *sorted, const uint64_t *n1_rows,
                   const int32_t *maxgrp, const int32_t *groups, const int32_t *ngroups, int64_t m, int64_t n,
                   int64_t job_lo, int64_t job_hi, int32_t *num, uint64_t *nd, uint64_t *n3, void *workspace,
                   int64_t ws_bytes, void *stream);

/* Host utility: upload nbytes of pageable host memory to the device through two pinned staging buffers
 * (stage_bytes each, >= 1 MiB), filled by nthreads host threads while the copy engine drains the other;
 * the copies are enqueued on stream and complete before the call returns. */
int tb_h2d_staged(const void *src, void *dst, int64_t nbytes, void *stage_a, void *stage_b, int64_t stage_bytes,
                  int nthreads, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* TAUB200_H */
