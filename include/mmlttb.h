/*
 * mmlttb.h -- C ABI of the B200-native MinMaxLTTB path (libmmlttb.so).
 *
 * Drop-in boundary for the reference package `tsdown`
 * (/root/reference/pkg/src/tsdown).  The reference's only native boundary is
 * two numba kernels called with caller-allocated int64 outputs
 * (downsamplers.py:56 and :131):
 *
 *   _extrema_by_bucket(bits, bounds, out_min, out_max)   _kernels.py:63-78
 *   _lttb_select(xs, ys, bounds, out)                    _kernels.py:81-119
 *
 * mmlttb_extrema_by_bucket / mmlttb_lttb_select replace those one-for-one.
 * The fused entry points below replace the Python compositions around them
 * (minmax_preselect downsamplers.py:135-161, minmaxlttb :182-209, lttb
 * :115-132, minmax :72-92, m4 :95-112, every_nth :44-47) so that a whole call
 * is a few stream-ordered kernel launches with no host round trip.
 *
 * Conventions
 *  - every pointer argument is a DEVICE pointer unless stated otherwise;
 *  - inputs are read-only; outputs/workspace are caller-allocated;
 *  - `stream` is a cudaStream_t passed as void*; all work is enqueued on it
 *    and nothing synchronises the host;
 *  - batched calls take B series: series s of y starts at y + s*y_ld
 *    elements; x_ld == 0 means one x shared by every series;
 *  - return 0 on success, a negative MM_E* code otherwise
 *    (mmlttb_last_error() gives the message; per-thread).
 *  - O(1) argument validation mirrors the reference's checks only
 *    defensively; the Python layer raises the reference's exception classes
 *    (errors.py) in the reference's order before calling in.
 */
#ifndef MMLTTB_H
#define MMLTTB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* element dtype codes */
enum { MM_F32 = 0, MM_F64 = 1, MM_I64 = 2, MM_I32 = 3 };

/* return codes */
enum {
    MM_OK = 0,
    MM_EINVAL = -1,      /* bad argument (n_out / r_ps / sizes / dtype)  */
    MM_ECUDA = -2,       /* CUDA launch or runtime error                 */
    MM_EWORKSPACE = -3,  /* workspace smaller than mmlttb_workspace_bytes */
    MM_ERANGE = -4       /* index arithmetic would overflow int64        */
};

/* operation codes for mmlttb_workspace_bytes */
enum { MM_OP_MINMAXLTTB = 0, MM_OP_PRESELECT = 1, MM_OP_LTTB = 2, MM_OP_MINMAX = 3, MM_OP_M4 = 4 };

int mmlttb_version(void);
const char *mmlttb_last_error(void);

/* Instrumentation (bench/profiling).  mmlttb_launch_count: kernels this
 * library has launched since load.  mmlttb_stage_timer(1): fused
 * minmaxlttb calls on this host thread record CUDA events on their stream at
 * the K1 | K2 | K3 stage boundaries; mmlttb_stage_timer_read synchronises on
 * them, writes the summed device milliseconds of the three stages to ms3[3]
 * and the number of timed calls, then clears. */
int64_t mmlttb_launch_count(void);
/* Exact bucket re-scans the large-bucket LTTB repair walk has performed since
 * load (synchronises the device; statistics for tests/bench only). */
int64_t mmlttb_repair_scans(void);
int mmlttb_stage_timer(int enable);
int mmlttb_stage_timer_read(double *ms3, int64_t *calls);
/* Launch trace: while enabled, the names of the kernels this host thread
 * launches are recorded; mmlttb_trace_read copies them comma-separated into
 * buf (NUL-terminated, truncated to len-1), returns the full length and
 * clears.  Stage boundaries are also NVTX ranges (no-ops without a tool). */
int mmlttb_trace(int enable);
int64_t mmlttb_trace_read(char *buf, int64_t len);

/* Deferred status word (non-finite y), for callers that keep their inputs on
 * the device and do not want a host sync per call.  mmlttb_status_arm()
 * returns a ticket >= 0 and arms this host thread: its next mmlttb_minmaxlttb
 * / mmlttb_minmax_preselect / mmlttb_minmax / mmlttb_m4 call stores that
 * call's status from the device into a pinned, device-mapped host slot (the
 * single-series K23 launch does it from its own CTA 0; other paths add one
 * 1-thread kernel after their last launch).  mmlttb_status_poll(ticket,
 * block) returns 2 while the slot is not yet written (block = 0; block = 1
 * synchronises the device first), else 1 if that call saw NaN/inf in y (the
 * reference's NonFiniteValue, core.py:80-94) or 0 if not; MM_EINVAL if the
 * armed call failed or the ticket was overwritten (the ring has 1024 slots).
 * A call made while its stream is capturing a graph does not deliver a
 * status (the slot then reads as clean).  mmlttb_status_ring()
 * exposes the 1024-slot ring (host view) for callers that poll it directly:
 * slot ticket % 1024 holds ((ticket + 1) << 3) | 4 * failed | 2 * captured | status bit
 * once written. */
int64_t mmlttb_status_arm(void);
const volatile unsigned long long *mmlttb_status_ring(void);
int mmlttb_status_poll(int64_t ticket, int block);

/* Bytes of device workspace an operation needs for B series of N points. */
int64_t mmlttb_workspace_bytes(int op, int64_t B, int64_t N, int64_t n_out, int64_t r_ps, int y_dtype);

/* minmaxlttb(series, n_out, r_ps)  -- downsamplers.py:182-209.
 * r_ps even >= 2: out[s*n_out + i], exactly n_out indices per series,
 * out_count[s] = n_out.  r_ps == 1: the _minmax_with_endpoints contract
 * (downsamplers.py:164-179): <= n_out indices, count in out_count[s].
 * x is only gathered at the <= 2 + (n_out-2)*r_ps preselected points. */
int mmlttb_minmaxlttb(const void *x, int x_dtype, int64_t x_ld,
                      const void *y, int y_dtype, int64_t y_ld,
                      int64_t B, int64_t N, int64_t n_out, int64_t r_ps,
                      int64_t *out, int64_t *out_count,
                      void *workspace, int64_t workspace_bytes, void *stream);

/* minmax_preselect(series, n_out, r_ps)  -- downsamplers.py:135-161.
 * out has 2 + 2k slots per series (k = (n_out-2)*r_ps/2); out_count[s] = m. */
int mmlttb_minmax_preselect(const void *y, int y_dtype, int64_t y_ld,
                            int64_t B, int64_t N, int64_t n_out, int64_t r_ps,
                            int64_t *out, int64_t out_ld, int64_t *out_count,
                            void *workspace, int64_t workspace_bytes, void *stream);

/* lttb(series, n_out)  -- downsamplers.py:115-132: exactly n_out indices. */
int mmlttb_lttb(const void *x, int x_dtype, int64_t x_ld,
                const void *y, int y_dtype, int64_t y_ld,
                int64_t B, int64_t N, int64_t n_out, int64_t *out,
                void *workspace, int64_t workspace_bytes, void *stream);

/* minmax(series, n_out) -- downsamplers.py:72-92 (n_out even).
 * m4(series, n_out)     -- downsamplers.py:95-112 (n_out % 4 == 0).
 * out has n_out slots per series; out_count[s] = number written. */
int mmlttb_minmax(const void *y, int y_dtype, int64_t y_ld, int64_t B, int64_t N, int64_t n_out,
                  int64_t *out, int64_t *out_count, void *workspace, int64_t workspace_bytes, void *stream);
int mmlttb_m4(const void *y, int y_dtype, int64_t y_ld, int64_t B, int64_t N, int64_t n_out,
              int64_t *out, int64_t *out_count, void *workspace, int64_t workspace_bytes, void *stream);

/* every_nth(series, n_out) -- downsamplers.py:44-47: out[i] = i*N // n_out. */
int mmlttb_every_nth(int64_t N, int64_t n_out, int64_t *out, void *stream);

/* _extrema_by_bucket(bits, bounds, out_min, out_max) -- _kernels.py:63-78.
 * bounds: k+1 ascending device int64 positions; max_bucket_len: an upper
 * bound on bounds[b+1]-bounds[b] (the caller built the partition).  y is the
 * float64 (or float32) series itself -- no int64 view is needed. */
int64_t mmlttb_extrema_workspace_bytes(int64_t k, int64_t max_bucket_len);
int mmlttb_extrema_by_bucket(const void *y, int y_dtype, const int64_t *bounds, int64_t k,
                             int64_t max_bucket_len, int64_t *out_min, int64_t *out_max,
                             void *workspace, int64_t workspace_bytes, void *stream);

/* _lttb_select(xs, ys, bounds, out) -- _kernels.py:81-119.  bounds has
 * nb = n_out-1 device entries covering [1, n-1); out has n_out slots. */
int64_t mmlttb_lttb_select_workspace_bytes(int64_t n, int64_t nb);
int mmlttb_lttb_select(const void *xs, int x_dtype, const void *ys, int y_dtype, int64_t n,
                       const int64_t *bounds, int64_t nb, int64_t *out,
                       void *workspace, int64_t workspace_bytes, void *stream);

/* ---- single-series multi-GPU path (bucket-range sharding) --
 * A rank owns sub-buckets [b0, b1) of partition(1, N-1, k) and the y (and x)
 * elements [lo, hi) they cover, stored at y_shard/x_shard (element lo at
 * offset 0).  emit_first / emit_last add global index 0 / N-1 (ranks 0 and
 * G-1).  Writes <= 2*(b1-b0)+2 entries (global index, x as f64, y as f64)
 * and the count into out_count[0]. */
int64_t mmlttb_shard_workspace_bytes(int64_t N, int64_t n_out, int64_t r_ps, int64_t b0, int64_t b1);
int mmlttb_shard_preselect(const void *x_shard, int x_dtype, const void *y_shard, int y_dtype,
                           int64_t lo, int64_t N, int64_t n_out, int64_t r_ps, int64_t b0, int64_t b1,
                           int emit_first, int emit_last,
                           int64_t *out_idx, double *out_x, double *out_y, int64_t *out_count,
                           void *workspace, int64_t workspace_bytes, void *stream);

/* Concatenate G gathered shard lists (each cap entries, counts[g] valid) in
 * rank order into one preselected set (out_idx/out_x/out_y, total in
 * out_m[0]).  Device-side: no host sync on the counts. */
int mmlttb_merge_shards(const int64_t *idx, const double *xs, const double *ys, const int64_t *counts,
                        int64_t G, int64_t cap, int64_t *out_idx, double *out_x, double *out_y,
                        int64_t *out_m, void *stream);

/* Same merge straight from the gathered packed messages: buf is [G][3*cap+1]
 * int64 rows (idx[cap] | x bits[cap] | y bits[cap] | count), i.e. the
 * all_gather of what mmlttb_shard_preselect wrote at (buf, buf+cap,
 * buf+2cap, buf+3cap); no unpacking copies. */
int mmlttb_merge_packed(const int64_t *buf, int64_t G, int64_t cap, int64_t *out_idx, double *out_x, double *out_y,
                        int64_t *out_m, void *stream);

/* Device-initiated exchange over peer memory (NVLink stores + epoch flags)
 * in place of the NCCL all_gather: each rank's symmetric buffer is int64
 * [2][G][3*cap+1] (slot = epoch & 1, row = writer rank) with a uint32 signal
 * pad [2G] (data flags, then acks); peer_bufs / peer_pads are device arrays
 * of the G peers' addresses (e.g. torch symmetric memory buffer_ptrs_dev /
 * signal_pad_ptrs_dev).  publish: wait for peer g's ack of epoch-2, store the
 * set into peer g's row, release its flag.  merge: acquire all G flags of
 * this epoch, concatenate the rows in rank order, ack the writers. */
int mmlttb_p2p_publish(const int64_t *idx, const double *xs, const double *ys, const int64_t *count, int64_t cap,
                       const uint64_t *peer_bufs, const uint64_t *peer_pads, const uint32_t *own_pad, int64_t G,
                       int64_t rank, uint32_t epoch, void *stream);
int mmlttb_p2p_merge(const int64_t *own_buf, const uint32_t *own_pad, const uint64_t *peer_pads, int64_t G,
                     int64_t rank, int64_t cap, uint32_t epoch, int64_t *out_idx, double *out_x, double *out_y,
                     int64_t *out_m, void *stream);

/* LTTB over preselected sets: series s has m[s] points (device counts)
 * pre_x/pre_y (f64, row stride ld) and maps position p -> pre_idx[p].
 * out[s*n_out + i] = pre_idx[lttb position].  r_ps bounds the bucket size
 * (m[s] <= 2 + (n_out-2)*r_ps). */
int64_t mmlttb_lttb_preselected_workspace_bytes(int64_t B, int64_t n_out, int64_t r_ps);
int mmlttb_lttb_preselected(const int64_t *pre_idx, const double *pre_x, const double *pre_y,
                            const int64_t *m, int64_t B, int64_t ld, int64_t n_out, int64_t r_ps,
                            int64_t *out, void *workspace, int64_t workspace_bytes, void *stream);

/* TSB1 ingest (seriesio.py:20-21,75-95): n interleaved f64 (x, y) pairs (device
 * buffer, 16-byte aligned) -> x[n], y[n]. */
int mmlttb_deinterleave_f64(const void *pairs, int64_t n, double *x, double *y, void *stream);

/* ---- evaluation step after the path ----------------
 * rasterize (raster.py:87-118, _kernels.py:122-163): draws points idx[0..n)
 * (or 0..n when idx is null) of (x, y) as the reference's anti-aliased width-2
 * polyline onto a w x h uint8 canvas mapping [x0,x1] x [y0,y1]; bit-identical
 * pixels.  conv_mask (metrics.py:69-82): dilated union of both images' ink.
 * pixel_metrics (metrics.py:85-132): out4 = {pem(margin), dssim, mse, mask
 * size}; pem and the SSIM map are exact, the dssim/mse means are summed in a
 * fixed order (not numpy's pairwise order). */
int64_t mmlttb_raster_workspace_bytes(int64_t n, int64_t w, int64_t h);
int mmlttb_rasterize(const void *x, int x_dtype, const void *y, int y_dtype, const int64_t *idx, int64_t n,
                     double x0, double x1, double y0, double y1, int64_t w, int64_t h, uint8_t *pixels,
                     void *workspace, int64_t workspace_bytes, void *stream);
int mmlttb_conv_mask(const uint8_t *a, const uint8_t *b, int64_t h, int64_t w, int kernel, uint8_t *mask, void *stream);
int mmlttb_pixel_metrics(const uint8_t *a, const uint8_t *b, const uint8_t *mask, int64_t h, int64_t w, int margin,
                         double *out4, void *workspace, int64_t workspace_bytes, void *stream);

/* TimeSeries invariants (core.py:80-94) on device: bit 0 set if any x or y
 * is NaN/inf, bit 1 if x decreases anywhere.  flags: one device int32,
 * zeroed by this call. */
int mmlttb_validate(const void *x, int x_dtype, const void *y, int y_dtype, int64_t N,
                    int32_t *flags, void *stream);
/* The same for B series in one launch: row s is x + s*x_ld (x_ld 0: one
 * shared x) and y + s*y_ld; flags[s] gets row s's bits (flags: B device
 * int32, zeroed by this call).  A batch is B TimeSeries built in row order,
 * so the first row with a nonzero word decides the error, and within a row
 * bit 0 wins (core.py:89-92). */
int mmlttb_validate_batch(const void *x, int x_dtype, int64_t x_ld, const void *y, int y_dtype, int64_t y_ld,
                          int64_t B, int64_t N, int32_t *flags, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MMLTTB_H */
