/*
 * tsdown_oracle.c -- CPU restatement of the reference MinMaxLTTB path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker (and the
 * `bench.py --impl reference` / `cpu_baseline` CPU arm).  Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline leg may load it.  The
 * product path (paper_2305_00332_b200/) never links or calls it.
 *
 * Every function restates one reference symbol of package `tsdown`
 * (/root/reference/pkg/src/tsdown/...), cited file:line.  The arithmetic is
 * kept exactly as the reference's: int64 total-order keys for the extrema
 * (first occurrence on ties, blocks of 64 as in _kernels.py:28-60) and strict
 * IEEE fp64 for LTTB (in-order sums, no FMA -- build with -ffp-contract=off).
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py writes the tests/golden fixtures).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_BLOCK 64 /* _kernels.py:19 */

/* _kernels.py:18,22-25: monotone int64 key of a float64 bit pattern. */
static inline int64_t or_order_key(int64_t bits) {
    return bits ^ ((bits >> 63) & (int64_t)0x7FFFFFFFFFFFFFFFLL);
}

/* core.py:161-175: bounds[b] = start + floor(b*L/k), b = 0..k.  Returns 0 on
 * success, -1 for InvalidPartition (k < 1 or k > L). */
int or_partition(int64_t start, int64_t end, int64_t k, int64_t *bounds) {
    int64_t len = end - start;
    if (k < 1 || k > len) return -1;
    for (int64_t b = 0; b <= k; ++b) bounds[b] = start + (b * len) / k;
    return 0;
}

/* _kernels.py:28-60: first-occurrence argmin/argmax of bits[lo:hi] in key
 * order, scanned in blocks of 64 with strict comparisons across blocks. */
void or_argminmax_range(const int64_t *bits, int64_t lo, int64_t hi,
                        int64_t *imn_out, int64_t *imx_out) {
    int64_t first = or_order_key(bits[lo]);
    int64_t mn = first, mx = first, imn = lo, imx = lo;
    int64_t j = lo + 1;
    while (j < hi) {
        int64_t e = j + OR_BLOCK < hi ? j + OR_BLOCK : hi;
        int64_t bmn = mn, bmx = mx;
        for (int64_t t = j; t < e; ++t) {
            int64_t key = or_order_key(bits[t]);
            bmn = key < bmn ? key : bmn;
            bmx = key > bmx ? key : bmx;
        }
        if (bmn < mn) {
            mn = bmn;
            for (int64_t t = j; t < e; ++t)
                if (or_order_key(bits[t]) == bmn) { imn = t; break; }
        }
        if (bmx > mx) {
            mx = bmx;
            for (int64_t t = j; t < e; ++t)
                if (or_order_key(bits[t]) == bmx) { imx = t; break; }
        }
        j = e;
    }
    *imn_out = imn;
    *imx_out = imx;
}

/* _kernels.py:63-78: per-bucket extrema; nthreads > 1 mirrors the prange
 * variant (_kernels.py:71-78; disjoint buckets, identical output). */
void or_extrema_by_bucket(const double *ys, const int64_t *bounds, int64_t k,
                          int64_t *out_min, int64_t *out_max, int nthreads) {
    const int64_t *bits = (const int64_t *)ys; /* ys.view(int64): downsamplers.py:56 */
#ifdef _OPENMP
    if (nthreads > 1) {
#pragma omp parallel for schedule(static) num_threads(nthreads)
        for (int64_t b = 0; b < k; ++b)
            or_argminmax_range(bits, bounds[b], bounds[b + 1], &out_min[b], &out_max[b]);
        return;
    }
#else
    (void)nthreads;
#endif
    for (int64_t b = 0; b < k; ++b)
        or_argminmax_range(bits, bounds[b], bounds[b + 1], &out_min[b], &out_max[b]);
}

/* downsamplers.py:60-69: (min(imin,imax), max(...)) per bucket, dropping the
 * second when equal.  Returns the number written (k..2k). */
int64_t or_interleave_minmax(const int64_t *idx_min, const int64_t *idx_max,
                             int64_t k, int64_t *out) {
    int64_t m = 0;
    for (int64_t b = 0; b < k; ++b) {
        int64_t lo = idx_min[b] < idx_max[b] ? idx_min[b] : idx_max[b];
        int64_t hi = idx_min[b] < idx_max[b] ? idx_max[b] : idx_min[b];
        out[m++] = lo;
        if (hi != lo) out[m++] = hi;
    }
    return m;
}

/* _kernels.py:81-119: sequential LTTB selection, strict IEEE fp64.
 * bounds has nb = n_out-1 entries covering [1, n-1); out has n_out slots. */
void or_lttb_select(const double *xs, const double *ys, int64_t n,
                    const int64_t *bounds, int64_t nb, int64_t *out) {
    int64_t k = nb - 1;
    out[0] = 0;
    out[k + 1] = n - 1;
    int64_t prev = 0;
    for (int64_t b = 0; b < k; ++b) {
        double cx, cy;
        if (b + 1 < k) {
            int64_t nlo = bounds[b + 1], nhi = bounds[b + 2];
            double sx = 0.0, sy = 0.0;
            for (int64_t j = nlo; j < nhi; ++j) { sx += xs[j]; sy += ys[j]; }
            cx = sx / (double)(nhi - nlo);
            cy = sy / (double)(nhi - nlo);
        } else {
            cx = xs[n - 1];
            cy = ys[n - 1];
        }
        double ax = xs[prev], ay = ys[prev];
        int64_t best = bounds[b];
        double best_area = -1.0;
        for (int64_t j = bounds[b]; j < bounds[b + 1]; ++j) {
            double area = fabs((ax - cx) * (ys[j] - ay) - (ax - xs[j]) * (cy - ay));
            if (area > best_area) { best_area = area; best = j; }
        }
        out[b + 1] = best;
        prev = best;
    }
}

/* downsamplers.py:115-132: lttb(series, n_out) -> n_out indices.
 * Returns 0, or -1 (NOutOfRange), -2 (allocation failure). */
int or_lttb(const double *xs, const double *ys, int64_t n, int64_t n_out, int64_t *out) {
    if (n_out < 3 || n_out > n) return -1;
    int64_t *bounds = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_out - 1));
    if (!bounds) return -2;
    or_partition(1, n - 1, n_out - 2, bounds);
    or_lttb_select(xs, ys, n, bounds, n_out - 1, out);
    free(bounds);
    return 0;
}

/* downsamplers.py:72-92: minmax(series, n_out).  out must hold n_out slots.
 * Returns the count, or -1 NOutOfRange, -3 OddNOut, -2 allocation failure. */
int64_t or_minmax(const double *ys, int64_t n, int64_t n_out, int64_t *out, int nthreads) {
    if (n_out < 3 || n_out > n) return -1;
    if (n_out % 2) return -3;
    int64_t k = n_out / 2;
    int64_t *bounds = (int64_t *)malloc(sizeof(int64_t) * (size_t)(3 * k + 1));
    if (!bounds) return -2;
    int64_t *imin = bounds + k + 1, *imax = imin + k;
    or_partition(0, n, k, bounds);
    or_extrema_by_bucket(ys, bounds, k, imin, imax, nthreads);
    int64_t m = or_interleave_minmax(imin, imax, k, out);
    free(bounds);
    return m;
}

/* downsamplers.py:135-161: minmax_preselect.  out must hold 2 + 2k slots,
 * k = (n_out-2)*(r_ps/2).  Returns m, or -1 NOutOfRange, -4
 * BadPreselectionRatio, -5 RatioTooLargeForSeries, -2 allocation failure. */
int64_t or_minmax_preselect(const double *ys, int64_t n, int64_t n_out, int64_t r_ps,
                            int64_t *out, int nthreads) {
    if (n_out < 3 || n_out > n) return -1;
    if (r_ps < 2 || r_ps % 2) return -4;
    int64_t k = (n_out - 2) * (r_ps / 2);
    if (k > n - 2) return -5;
    int64_t *bounds = (int64_t *)malloc(sizeof(int64_t) * (size_t)(3 * k + 1));
    if (!bounds) return -2;
    int64_t *imin = bounds + k + 1, *imax = imin + k;
    or_partition(1, n - 1, k, bounds);
    or_extrema_by_bucket(ys, bounds, k, imin, imax, nthreads);
    out[0] = 0;
    int64_t m = or_interleave_minmax(imin, imax, k, out + 1);
    out[m + 1] = n - 1;
    free(bounds);
    return m + 2;
}

/* downsamplers.py:164-179: r_ps = 1 contract (MinMax with forced endpoints).
 * out must hold n_out slots.  Returns the count or a negative code. */
int64_t or_minmax_with_endpoints(const double *ys, int64_t n, int64_t n_out,
                                 int64_t *out, int nthreads) {
    int64_t m = or_minmax(ys, n, n_out, out, nthreads);
    if (m < 0) return m;
    if (out[0] != 0) {
        if (m < n_out) {
            memmove(out + 1, out, sizeof(int64_t) * (size_t)m);
            out[0] = 0;
            ++m;
        } else {
            out[0] = 0;
        }
    }
    if (out[m - 1] != n - 1) {
        if (m < n_out) out[m++] = n - 1;
        else out[m - 1] = n - 1;
    }
    return m;
}

/* downsamplers.py:182-209: minmaxlttb.  out must hold n_out slots.
 * Returns the count (n_out when r_ps >= 2) or a negative code. */
int64_t or_minmaxlttb(const double *xs, const double *ys, int64_t n, int64_t n_out,
                      int64_t r_ps, int64_t *out, int nthreads) {
    if (r_ps == 1) return or_minmax_with_endpoints(ys, n, n_out, out, nthreads);
    if (n_out < 3 || n_out > n) return -1;
    if (r_ps < 2 || r_ps % 2) return -4;
    int64_t k = (n_out - 2) * (r_ps / 2);
    if (k > n - 2) return -5;
    int64_t cap = 2 + 2 * k;
    int64_t *pre = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cap + n_out));
    double *sx = (double *)malloc(sizeof(double) * (size_t)cap * 2);
    if (!pre || !sx) { free(pre); free(sx); return -2; }
    int64_t *pos = pre + cap;
    int64_t m = or_minmax_preselect(ys, n, n_out, r_ps, pre, nthreads);
    if (m < 0) { free(pre); free(sx); return m; }
    double *sy = sx + cap;
    for (int64_t i = 0; i < m; ++i) { sx[i] = xs[pre[i]]; sy[i] = ys[pre[i]]; } /* series.take */
    int rc = or_lttb(sx, sy, m, n_out, pos);
    if (rc == 0)
        for (int64_t i = 0; i < n_out; ++i) out[i] = pre[pos[i]];
    free(pre);
    free(sx);
    return rc < 0 ? rc : n_out;
}

/* downsamplers.py:95-112: m4.  out must hold n_out slots.  Returns the count,
 * or -1 NOutOfRange, -6 NOutNotDivisibleBy4, -2 allocation failure. */
int64_t or_m4(const double *ys, int64_t n, int64_t n_out, int64_t *out, int nthreads) {
    if (n_out < 3 || n_out > n) return -1;
    if (n_out % 4) return -6;
    int64_t k = n_out / 4;
    int64_t *bounds = (int64_t *)malloc(sizeof(int64_t) * (size_t)(3 * k + 1));
    if (!bounds) return -2;
    int64_t *imin = bounds + k + 1, *imax = imin + k;
    or_partition(0, n, k, bounds);
    or_extrema_by_bucket(ys, bounds, k, imin, imax, nthreads);
    int64_t m = 0;
    for (int64_t b = 0; b < k; ++b) {
        int64_t q[4] = {bounds[b], imin[b], imax[b], bounds[b + 1] - 1};
        /* quad.sort(axis=1), then keep entries differing from their left neighbour */
        for (int i = 1; i < 4; ++i)
            for (int j = i; j > 0 && q[j - 1] > q[j]; --j) { int64_t t = q[j]; q[j] = q[j - 1]; q[j - 1] = t; }
        out[m++] = q[0];
        for (int i = 1; i < 4; ++i) if (q[i] != q[i - 1]) out[m++] = q[i];
    }
    free(bounds);
    return m;
}

/* ---- chunked (typed-input) oracle: SURVEY §8(c) --------------------------
 * Inputs in their storage dtype (y: f32/f64; x: i64/f64/f32); every element
 * is converted to f64 exactly as TimeSeries does (core.py:48-53) but one
 * sub-bucket at a time, so a 2e9-point series never needs an f64 copy. */
enum { OR_F32 = 0, OR_F64 = 1, OR_I64 = 2, OR_I32 = 3 };

static inline double or_load(const void *p, int dt, int64_t i) {
    switch (dt) {
    case OR_F32: return (double)((const float *)p)[i];
    case OR_F64: return ((const double *)p)[i];
    case OR_I64: return (double)((const int64_t *)p)[i];
    default: return (double)((const int32_t *)p)[i];
    }
}

/* minmax_preselect over typed y; same return codes as or_minmax_preselect. */
int64_t or_minmax_preselect_typed(const void *ys, int ydt, int64_t n, int64_t n_out,
                                  int64_t r_ps, int64_t *out, int nthreads) {
    if (n_out < 3 || n_out > n) return -1;
    if (r_ps < 2 || r_ps % 2) return -4;
    int64_t k = (n_out - 2) * (r_ps / 2);
    if (k > n - 2) return -5;
    int64_t *bounds = (int64_t *)malloc(sizeof(int64_t) * (size_t)(3 * k + 1));
    if (!bounds) return -2;
    int64_t *imin = bounds + k + 1, *imax = imin + k;
    or_partition(1, n - 1, k, bounds);
    int64_t smax = 0;
    for (int64_t b = 0; b < k; ++b)
        if (bounds[b + 1] - bounds[b] > smax) smax = bounds[b + 1] - bounds[b];
    int failed = 0;
#ifdef _OPENMP
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1)
#endif
    {
        double *buf = (double *)malloc(sizeof(double) * (size_t)smax);
        if (!buf) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            failed = 1;
        }
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int64_t b = 0; b < k; ++b) {
            if (!buf) continue;
            int64_t lo = bounds[b], hi = bounds[b + 1];
            for (int64_t i = lo; i < hi; ++i) buf[i - lo] = or_load(ys, ydt, i);
            int64_t a, c;
            or_argminmax_range((const int64_t *)buf, 0, hi - lo, &a, &c);
            imin[b] = a + lo;
            imax[b] = c + lo;
        }
        free(buf);
    }
    if (failed) { free(bounds); return -2; }
    out[0] = 0;
    int64_t m = or_interleave_minmax(imin, imax, k, out + 1);
    out[m + 1] = n - 1;
    free(bounds);
    return m + 2;
}

/* minmaxlttb over typed x/y (r_ps >= 2): chunked preselection, then the
 * reference LTTB over the gathered f64 sub-series. */
int64_t or_minmaxlttb_typed(const void *xs, int xdt, const void *ys, int ydt, int64_t n,
                            int64_t n_out, int64_t r_ps, int64_t *out, int nthreads) {
    if (n_out < 3 || n_out > n) return -1;
    if (r_ps < 2 || r_ps % 2) return -4;
    int64_t k = (n_out - 2) * (r_ps / 2);
    if (k > n - 2) return -5;
    int64_t cap = 2 + 2 * k;
    int64_t *pre = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cap + n_out));
    double *sx = (double *)malloc(sizeof(double) * (size_t)cap * 2);
    if (!pre || !sx) { free(pre); free(sx); return -2; }
    int64_t *pos = pre + cap;
    int64_t m = or_minmax_preselect_typed(ys, ydt, n, n_out, r_ps, pre, nthreads);
    if (m < 0) { free(pre); free(sx); return m; }
    double *sy = sx + cap;
    for (int64_t i = 0; i < m; ++i) { sx[i] = or_load(xs, xdt, pre[i]); sy[i] = or_load(ys, ydt, pre[i]); }
    int rc = or_lttb(sx, sy, m, n_out, pos);
    if (rc == 0)
        for (int64_t i = 0; i < n_out; ++i) out[i] = pre[pos[i]];
    free(pre);
    free(sx);
    return rc < 0 ? rc : n_out;
}

/* One rank's share of the bucket-range sharded preselection (the multi-GPU
 * single-series path): sub-buckets [b0, b1) of partition(1, n-1, k)
 * (core.py:161-175 over downsamplers.py:149-155), over a shard holding global
 * elements [lo, lo + len), emitted as in minmax_preselect (:156-160): 0 first
 * when emit_first, the interleaved pairs (:60-69) in global indices, n-1 last
 * when emit_last.  Returns the count written to out. */
int64_t or_shard_preselect_typed(const void *ys, int ydt, int64_t lo, int64_t len, int64_t n,
                                 int64_t n_out, int64_t r_ps, int64_t b0, int64_t b1,
                                 int emit_first, int emit_last, int64_t *out, int nthreads) {
    if (n_out < 3 || n_out > n) return -1;
    if (r_ps < 2 || r_ps % 2) return -4;
    int64_t k = (n_out - 2) * (r_ps / 2);
    if (k > n - 2) return -5;
    if (b0 < 0 || b1 > k || b1 < b0) return -1;
    int64_t nb = b1 - b0;
    int64_t *bounds = (int64_t *)malloc(sizeof(int64_t) * (size_t)(3 * nb + 3));
    if (!bounds) return -2;
    int64_t *imin = bounds + nb + 1, *imax = imin + nb + 1;
    int64_t smax = 1;
    for (int64_t b = 0; b <= nb; ++b) bounds[b] = 1 + ((b0 + b) * (n - 2)) / k;
    for (int64_t b = 0; b < nb; ++b)
        if (bounds[b + 1] - bounds[b] > smax) smax = bounds[b + 1] - bounds[b];
    int failed = 0;
    for (int64_t b = 0; b <= nb; ++b)
        if (bounds[b] < lo || bounds[b] > lo + len) failed = 1; /* the shard must cover its buckets */
    if (failed) { free(bounds); return -1; }
#ifdef _OPENMP
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1)
#endif
    {
        double *buf = (double *)malloc(sizeof(double) * (size_t)smax);
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int64_t b = 0; b < nb; ++b) {
            if (!buf) continue;
            int64_t a0 = bounds[b], a1 = bounds[b + 1];
            for (int64_t i = a0; i < a1; ++i) buf[i - a0] = or_load(ys, ydt, i - lo);
            int64_t a, c;
            or_argminmax_range((const int64_t *)buf, 0, a1 - a0, &a, &c);
            imin[b] = a + a0;
            imax[b] = c + a0;
        }
        if (!buf) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            failed = 1;
        }
        free(buf);
    }
    if (failed) { free(bounds); return -2; }
    int64_t m = 0;
    if (emit_first) out[m++] = 0;
    m += or_interleave_minmax(imin, imax, nb, out + m);
    if (emit_last) out[m++] = n - 1;
    free(bounds);
    return m;
}

int or_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
