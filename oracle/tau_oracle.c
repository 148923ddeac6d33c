/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C) of the reference `taucorr` algorithms on the
 * all-pairs Kendall tau hot path.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline -- never as the product.
 *
 * Parity pinning: every function here is checked (tests/test_oracle_golden.py)
 * against golden vectors produced by importing the reference package itself
 * (oracle/gen_golden.py writes tests/golden/).
 *
 * Citations are into /root/reference/pkg/ (src/taucorr/... and tests/...).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Brute-force definition scan: tests/conftest.py:16-42 (_pair_scan).       */
/* out = {nc, nd, n1, n2, n3}.                                              */
/* ------------------------------------------------------------------------ */
void orc_pair_scan(const int32_t *u, const int32_t *v, int64_t n, int64_t *out)
{
    int64_t nc = 0, nd = 0, n1 = 0, n2 = 0, n3 = 0;
    for (int64_t i = 0; i < n; i++) {
        for (int64_t j = i + 1; j < n; j++) {
            int64_t du = (int64_t)u[i] - (int64_t)u[j];
            int64_t dv = (int64_t)v[i] - (int64_t)v[j];
            /* sign of the product, without overflow */
            int s = ((du > 0) - (du < 0)) * ((dv > 0) - (dv < 0));
            if (s > 0) nc++;
            else if (s < 0) nd++;
            if (du == 0) n1++;
            if (dv == 0) {
                n2++;
                if (du == 0) n3++;
            }
        }
    }
    out[0] = nc; out[1] = nd; out[2] = n1; out[3] = n2; out[4] = n3;
}

/* Quadratic numerator, kernel_naive.py:26-44 (sum of sign products). */
int64_t orc_naive_numerator(const int32_t *u, const int32_t *v, int64_t n)
{
    int64_t total = 0;
    for (int64_t i = 1; i < n; i++) {
        int64_t a = u[i], b = v[i], acc = 0;
        for (int64_t j = 0; j < i; j++) {
            int64_t du = a - u[j], dv = b - v[j];
            acc += ((du > 0) - (du < 0)) * ((dv > 0) - (dv < 0));
        }
        total += acc;
    }
    return total;
}

/* ------------------------------------------------------------------------ */
/* GSE merge-sort kernel: kernel_sorted.py:30-212.                          */
/* ------------------------------------------------------------------------ */

/* _merge_lex, kernel_sorted.py:30-57: stable merge by (u, v). */
static void merge_lex(const int32_t *au, const int32_t *av, int32_t *bu, int32_t *bv,
                      int64_t left, int64_t mid, int64_t right)
{
    int64_t l = left, r = mid, p = left;
    while (l < mid && r < right) {
        int32_t ru = au[r], lu = au[l];
        if (ru < lu || (ru == lu && av[r] < av[l])) {
            bu[p] = ru; bv[p] = av[r]; r++;
        } else {
            bu[p] = lu; bv[p] = av[l]; l++;
        }
        p++;
    }
    while (l < mid) { bu[p] = au[l]; bv[p] = av[l]; l++; p++; }
    while (r < right) { bu[p] = au[r]; bv[p] = av[r]; r++; p++; }
}

/* _merge_by_v, kernel_sorted.py:60-92: merge on v, counting right<left
 * events weighted by the unconsumed left-run length (strict <). */
static int64_t merge_by_v(const int32_t *au, const int32_t *av, int32_t *bu, int32_t *bv,
                          int64_t left, int64_t mid, int64_t right)
{
    int64_t nd = 0, l = left, r = mid, p = left;
    while (l < mid && r < right) {
        if (av[r] < av[l]) {
            nd += mid - l;
            bu[p] = au[r]; bv[p] = av[r]; r++;
        } else {
            bu[p] = au[l]; bv[p] = av[l]; l++;
        }
        p++;
    }
    while (l < mid) { bu[p] = au[l]; bv[p] = av[l]; l++; p++; }
    while (r < right) { bu[p] = au[r]; bv[p] = av[r]; r++; p++; }
    return nd;
}

/* Bottom-up merge sort driver shared by _sort_pairs_lex (:95-127) and
 * _sort_pairs_by_v (:130-160). */
static int64_t sort_pairs(int32_t *u, int32_t *v, int32_t *su, int32_t *sv, int64_t n, int by_v)
{
    int32_t *au = u, *av = v, *bu = su, *bv = sv;
    int in_place = 1;
    int64_t nd = 0;
    for (int64_t width = 1; width < n; width *= 2) {
        for (int64_t l = 0; l < n; l += 2 * width) {
            int64_t m = l + width < n ? l + width : n;
            int64_t r = l + 2 * width < n ? l + 2 * width : n;
            if (by_v) nd += merge_by_v(au, av, bu, bv, l, m, r);
            else merge_lex(au, av, bu, bv, l, m, r);
        }
        int32_t *t = au; au = bu; bu = t;
        t = av; av = bv; bv = t;
        in_place = !in_place;
    }
    if (!in_place) {
        memcpy(u, au, (size_t)n * sizeof(int32_t));
        memcpy(v, av, (size_t)n * sizeof(int32_t));
    }
    return nd;
}

/* _tie_pairs, kernel_sorted.py:163-176. */
static int64_t tie_pairs(const int32_t *keys, int64_t n)
{
    int64_t total = 0, run = 1;
    for (int64_t i = 1; i < n; i++) {
        if (keys[i] == keys[i - 1]) run++;
        else { total += run * (run - 1) / 2; run = 1; }
    }
    return total + run * (run - 1) / 2;
}

/* _joint_tie_pairs, kernel_sorted.py:179-192. */
static int64_t joint_tie_pairs(const int32_t *u, const int32_t *v, int64_t n)
{
    int64_t total = 0, run = 1;
    for (int64_t i = 1; i < n; i++) {
        if (u[i] == u[i - 1] && v[i] == v[i - 1]) run++;
        else { total += run * (run - 1) / 2; run = 1; }
    }
    return total + run * (run - 1) / 2;
}

/* sorted_counts, kernel_sorted.py:195-212.  scratch: 4*n int32.
 * out = {n_d, n1, n2, n3}. */
void orc_sorted_counts(const int32_t *u, const int32_t *v, int64_t n, int32_t *scratch, int64_t *out)
{
    int32_t *wu = scratch, *wv = scratch + n, *su = scratch + 2 * n, *sv = scratch + 3 * n;
    memcpy(wu, u, (size_t)n * sizeof(int32_t));
    memcpy(wv, v, (size_t)n * sizeof(int32_t));
    sort_pairs(wu, wv, su, sv, n, 0);               /* step 1 */
    int64_t n1 = tie_pairs(wu, n);                  /* step 2 */
    int64_t n3 = joint_tie_pairs(wu, wv, n);
    int64_t nd = sort_pairs(wu, wv, su, sv, n, 1);  /* step 3 */
    int64_t n2 = tie_pairs(wv, n);                  /* step 4 */
    out[0] = nd; out[1] = n1; out[2] = n2; out[3] = n3;
}

/* ------------------------------------------------------------------------ */
/* Packed (VSE-semantics) kernel: kernel_vectorized.py:445-523, scalar.      */
/* Keys are (u << 16) | v with 15-bit ranks (ranks.py:79-95); step 3 masks  */
/* to the low 15 bits (kernel_vectorized.py:519-520).  Same counts as GSE.  */
/* ------------------------------------------------------------------------ */
static int64_t merge_keys(const int32_t *a, int32_t *b, int64_t left, int64_t mid, int64_t right, int count)
{
    int64_t nd = 0, l = left, r = mid, p = left;
    while (l < mid && r < right) {
        int32_t x = a[l], y = a[r];
        if (y < x) { if (count) nd += mid - l; b[p++] = y; r++; }
        else { b[p++] = x; l++; }
    }
    while (l < mid) b[p++] = a[l++];
    while (r < right) b[p++] = a[r++];
    return nd;
}

/* Seeded runs of 16 (kernel_vectorized.py:403-442): insertion sort per block
 * while counting strict inversions, then bottom-up merges. */
static int64_t sort_keys(int32_t *a, int32_t *b, int64_t n, int count)
{
    const int64_t W = 16;
    int64_t nd = 0;
    for (int64_t base = 0; base < n; base += W) {
        int64_t hi = base + W < n ? base + W : n;
        for (int64_t i = base + 1; i < hi; i++) {
            int32_t key = a[i];
            int64_t j = i - 1;
            while (j >= base && a[j] > key) { a[j + 1] = a[j]; j--; if (count) nd++; }
            a[j + 1] = key;
        }
    }
    int32_t *src = a, *dst = b;
    int in_place = 1;
    for (int64_t width = W; width < n; width *= 2) {
        for (int64_t l = 0; l < n; l += 2 * width) {
            int64_t m = l + width < n ? l + width : n;
            int64_t r = l + 2 * width < n ? l + 2 * width : n;
            nd += merge_keys(src, dst, l, m, r, count);
        }
        int32_t *t = src; src = dst; dst = t;
        in_place = !in_place;
    }
    if (!in_place) memcpy(a, src, (size_t)n * sizeof(int32_t));
    return nd;
}

/* vectorized_counts, kernel_vectorized.py:507-523.  Caller guarantees
 * n <= 32767 and 0 <= rank < 2^15 (ranks.py:64-76).  scratch: 2*n int32. */
void orc_packed_counts(const int32_t *u, const int32_t *v, int64_t n, int32_t *scratch, int64_t *out)
{
    int32_t *pa = scratch, *pb = scratch + n;
    for (int64_t i = 0; i < n; i++) pa[i] = (int32_t)(((uint32_t)u[i] << 16) | (uint32_t)v[i]);
    sort_keys(pa, pb, n, 0);
    int64_t n1 = 0, n3 = 0, run_u = 1, run_j = 1;   /* _packed_tie_pairs :477-504 */
    for (int64_t i = 1; i < n; i++) {
        if ((pa[i] >> 16) == (pa[i - 1] >> 16)) run_u++;
        else { n1 += run_u * (run_u - 1) / 2; run_u = 1; }
        if (pa[i] == pa[i - 1]) run_j++;
        else { n3 += run_j * (run_j - 1) / 2; run_j = 1; }
    }
    n1 += run_u * (run_u - 1) / 2;
    n3 += run_j * (run_j - 1) / 2;
    for (int64_t i = 0; i < n; i++) pa[i] &= 0x7FFF;
    int64_t nd = sort_keys(pa, pb, n, 1);
    int64_t n2 = tie_pairs(pa, n);
    out[0] = nd; out[1] = n1; out[2] = n2; out[3] = n3;
}

/* ------------------------------------------------------------------------ */
/* Finalize: result.py:35-59 (result_from_counts) and :62-82 (derive_taus). */
/* ------------------------------------------------------------------------ */
void orc_derive_taus(const int64_t *num, const uint64_t *n1, const uint64_t *n2, int64_t count,
                     int64_t n, double *tau_a, double *tau_b)
{
    int64_t n0 = n * (n - 1) / 2;
    double dn0 = (double)n0;
    for (int64_t k = 0; k < count; k++) {
        double x = (double)num[k];
        tau_a[k] = x / dn0;
        double t1 = (double)n1[k], t2 = (double)n2[k];
        volatile double prod = (dn0 - t1) * (dn0 - t2);  /* no contraction */
        double denom = sqrt(prod);
        tau_b[k] = denom > 0 ? x / denom : NAN;
    }
}

/* ------------------------------------------------------------------------ */
/* Geometry: pairindex.py:20-80.                                             */
/* ------------------------------------------------------------------------ */
int64_t orc_row_prefix(int64_t y, int64_t m) { return y * (2 * m - y + 1) / 2; }

/* job_coord, pairindex.py:34-55 (float guess + integer correction). */
void orc_job_coord(int64_t j, int64_t m, int64_t *yo, int64_t *xo)
{
    double disc = (double)m * (double)m + (double)m + 0.25 - 2.0 * ((double)j + 1.0);
    int64_t y = (int64_t)ceil((double)m - 0.5 - sqrt(disc));
    if (y < 0) y = 0;
    else if (y > m - 1) y = m - 1;
    while (orc_row_prefix(y, m) > j) y--;
    while (orc_row_prefix(y + 1, m) <= j) y++;
    *yo = y;
    *xo = j + y - orc_row_prefix(y, m);
}

/* ------------------------------------------------------------------------ */
/* Threaded all-pairs driver over an explicit pair list (the CPU baseline:  */
/* the reference engine's static round-robin split, engine.py:172, 378-396). */
/* kernel: 0 = sorted (GSE), 1 = packed (VSE semantics), 2 = naive.          */
/* out_counts: npairs x 4 int64 {n_d, n1, n2, n3}; out_num: numerator.      */
/* ------------------------------------------------------------------------ */
typedef struct {
    const int32_t *ranks;
    int64_t n;
    const int64_t *pi, *pj;
    int64_t npairs;
    int kernel, tid, nthreads;
    int64_t *out_num, *out_counts;
} job_t;

static void *worker(void *arg)
{
    job_t *jb = (job_t *)arg;
    int64_t n = jb->n, n0 = n * (n - 1) / 2;
    int32_t *scratch = (int32_t *)malloc((size_t)(4 * n + 16) * sizeof(int32_t));
    for (int64_t k = jb->tid; k < jb->npairs; k += jb->nthreads) {
        const int32_t *u = jb->ranks + jb->pi[k] * n;
        const int32_t *v = jb->ranks + jb->pj[k] * n;
        int64_t c[4] = {0, 0, 0, 0};
        int64_t num;
        if (jb->kernel == 2) {
            num = orc_naive_numerator(u, v, n);
        } else {
            if (jb->kernel == 1) orc_packed_counts(u, v, n, scratch, c);
            else orc_sorted_counts(u, v, n, scratch, c);
            num = n0 - c[1] - c[2] + c[3] - 2 * c[0];   /* result.py:42 */
        }
        jb->out_num[k] = num;
        if (jb->out_counts) memcpy(jb->out_counts + 4 * k, c, sizeof(c));
    }
    free(scratch);
    return NULL;
}

int orc_all_pairs(const int32_t *ranks, int64_t n, const int64_t *pi, const int64_t *pj,
                  int64_t npairs, int kernel, int nthreads, int64_t *out_num, int64_t *out_counts)
{
    if (nthreads < 1) nthreads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    job_t *jobs = (job_t *)malloc(sizeof(job_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; t++) {
        jobs[t] = (job_t){ranks, n, pi, pj, npairs, kernel, t, nthreads, out_num, out_counts};
        pthread_create(&th[t], NULL, worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
    return 0;
}
