// raster.cuh -- line-chart rasterizer and pixel metrics on the device
// (the step after the path in evaluation.run_evaluation).
//
// Rasterizer (raster.py:87-118, _kernels.py:122-163): the reference walks the
// segments in order and accumulates 255*coverage into each pixel of the
// segment's bounding box.  Here one thread owns one pixel and walks, in the
// same segment order, exactly the segments whose boxes contain it (their
// column spans are monotone in the segment index because x is sorted, so the
// candidates are one contiguous range found by binary search).  Every
// contribution uses the reference's operation sequence with separately
// rounded fp64 ops, so the accumulated value -- and the uint8 pixel -- is
// bit-identical.
//
// Metrics (metrics.py:69-132): conv_mask (binary dilation), pem (integer
// counts: exact), and the 8x8 uniform-window SSIM: the window sums of the
// integer-valued images are exact in fp64 whatever the summation order, so
// the SSIM map is bit-identical; only the final masked means (dssim, mse) use
// a different (deterministic) summation order than numpy's pairwise sum.
#pragma once
#include "kernels.cuh"

namespace mm {

struct RasterCoordArgs {
  const void* x; int xdt;
  const void* y; int ydt;
  const int64_t* idx;   // optional subset (strictly increasing)
  int64_t n;            // points drawn
  double x0, x1, y0, y1;
  int64_t w, h;
  double* us; double* vs;
  int* box;             // [n-1][4] lox, hix, loy, hiy
};

// us = (xs - x0) / (x1 - x0) * width; vs = (y1 - ys) / (y1 - y0) * height
// (raster.py:112-113), then each segment's pixel box (_kernels.py:137-140)
__global__ void k_raster_coords(RasterCoordArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const int64_t j = a.idx ? a.idx[i] : i;
  const double xv = load_any(a.x, a.xdt, j), yv = load_any(a.y, a.ydt, j);
  a.us[i] = __dmul_rn(__ddiv_rn(__dsub_rn(xv, a.x0), __dsub_rn(a.x1, a.x0)), (double)a.w);
  a.vs[i] = __dmul_rn(__ddiv_rn(__dsub_rn(a.y1, yv), __dsub_rn(a.y1, a.y0)), (double)a.h);
}

__global__ void k_raster_boxes(RasterCoordArgs a) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s + 1 >= a.n) return;
  const double x0 = a.us[s], y0 = a.vs[s], x1 = a.us[s + 1], y1 = a.vs[s + 1];
  const double lx = floor(__dsub_rn(fmin(x0, x1), 1.5)), hx = ceil(__dadd_rn(fmax(x0, x1), 1.5));
  const double ly = floor(__dsub_rn(fmin(y0, y1), 1.5)), hy = ceil(__dadd_rn(fmax(y0, y1), 1.5));
  // int(...) then clip: values are clamped first so the conversion never overflows
  const double big = 2147483000.0;
  int lox = (int)fmax(fmin(lx, big), -big), hix = (int)fmax(fmin(hx, big), -big);
  int loy = (int)fmax(fmin(ly, big), -big), hiy = (int)fmax(fmin(hy, big), -big);
  lox = max(lox, 0);
  hix = min(hix, (int)a.w - 1);
  loy = max(loy, 0);
  hiy = min(hiy, (int)a.h - 1);
  int* b = a.box + 4 * s;
  b[0] = lox; b[1] = hix; b[2] = loy; b[3] = hiy;
}

// one thread per pixel: its ordered contributions (_kernels.py:144-163)
__global__ void k_rasterize(const double* __restrict__ us, const double* __restrict__ vs, const int* __restrict__ box,
                            int64_t n, int64_t w, int64_t h, unsigned char* __restrict__ pix) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= w * h) return;
  const int r = (int)(p / w), c = (int)(p % w);
  const int64_t ns = n - 1;
  // first segment whose right edge reaches column c (hix non-decreasing)
  int64_t lo = 0, hi = ns;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (box[4 * mid + 1] < c) lo = mid + 1; else hi = mid;
  }
  const int64_t sa = lo;
  // one past the last segment whose left edge is <= c (lox non-decreasing)
  lo = sa; hi = ns;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (box[4 * mid] <= c) lo = mid + 1; else hi = mid;
  }
  const int64_t sb = lo;
  const double px = (double)c + 0.5, py = (double)r + 0.5;
  double acc = 0.0;
  for (int64_t s = sa; s < sb; ++s) {
    const int* b = box + 4 * s;
    if (c < b[0] || c > b[1] || r < b[2] || r > b[3]) continue;
    const double x0 = us[s], y0 = vs[s], x1 = us[s + 1], y1 = vs[s + 1];
    const double dx = __dsub_rn(x1, x0), dy = __dsub_rn(y1, y0);
    const double seg2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
    double t = 0.0;
    if (seg2 > 0.0) {
      t = __ddiv_rn(__dadd_rn(__dmul_rn(__dsub_rn(px, x0), dx), __dmul_rn(__dsub_rn(py, y0), dy)), seg2);
      if (t < 0.0) t = 0.0;
      else if (t > 1.0) t = 1.0;
    }
    const double qx = __dadd_rn(x0, __dmul_rn(t, dx)), qy = __dadd_rn(y0, __dmul_rn(t, dy));
    const double ex = __dsub_rn(px, qx), ey = __dsub_rn(py, qy);
    const double d = __dsqrt_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)));
    double cov = __dsub_rn(1.5, d);
    if (cov > 0.0) {
      if (cov > 1.0) cov = 1.0;
      acc = __dadd_rn(acc, __dmul_rn(255.0, cov));
    }
  }
  pix[p] = (unsigned char)fmin(rint(acc), 255.0);  // np.minimum(np.rint(acc), 255).astype(uint8)
}

// conv_mask (metrics.py:69-82): ink of either image, dilated by a k x k square
__global__ void k_conv_mask(const unsigned char* a, const unsigned char* b, int64_t h, int64_t w, int k,
                            unsigned char* mask) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= w * h) return;
  const int r = (int)(p / w), c = (int)(p % w), e = k / 2;
  unsigned char m = 0;
  for (int i = max(0, r - e); i <= min((int)h - 1, r + e) && !m; ++i)
    for (int j = max(0, c - e); j <= min((int)w - 1, c + e); ++j)
      if (a[i * w + j] | b[i * w + j]) { m = 1; break; }
  mask[p] = m;
}

__device__ __forceinline__ int reflect_idx(int i, int n) {  // scipy.ndimage mode='reflect'
  if (i < 0) return -i - 1;
  if (i >= n) return 2 * n - i - 1;
  return i;
}

// pass 1: uniform_filter1d(size 8) along axis 0 of fa, fb, fa^2, fb^2, fa*fb
// (window [r-4, r+3]); the sums are integers, so exact in fp64.
__global__ void k_ssim_rows(const unsigned char* a, const unsigned char* b, int64_t h, int64_t w, double* m5) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= w * h) return;
  const int r = (int)(p / w), c = (int)(p % w);
  double s[5] = {0, 0, 0, 0, 0};
  for (int d = -4; d <= 3; ++d) {
    const int rr = reflect_idx(r + d, (int)h);
    const double fa = a[rr * w + c], fb = b[rr * w + c];
    s[0] += fa; s[1] += fb; s[2] += fa * fa; s[3] += fb * fb; s[4] += fa * fb;
  }
  for (int q = 0; q < 5; ++q) m5[q * w * h + p] = s[q] / 8.0;
}

// pass 2 along axis 1, then the SSIM map (metrics.py:98-114) and the masked
// dssim / squared-error terms; per-block partial sums in a fixed order
__global__ void k_ssim_cols(const unsigned char* a, const unsigned char* b, const unsigned char* mask, int64_t h,
                            int64_t w, const double* m5, double* part /* [blocks][2] */) {
  __shared__ double s_d[256], s_e[256];
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double vd = 0.0, ve = 0.0;
  if (p < w * h && mask[p]) {
    const int r = (int)(p / w), c = (int)(p % w);
    double s[5] = {0, 0, 0, 0, 0};
    for (int d = -4; d <= 3; ++d) {
      const int cc = reflect_idx(c + d, (int)w);
      for (int q = 0; q < 5; ++q) s[q] += m5[q * w * h + (int64_t)r * w + cc];
    }
    const double mu_a = s[0] / 8.0, mu_b = s[1] / 8.0;
    const double var_a = __dsub_rn(s[2] / 8.0, __dmul_rn(mu_a, mu_a));
    const double var_b = __dsub_rn(s[3] / 8.0, __dmul_rn(mu_b, mu_b));
    const double cov = __dsub_rn(s[4] / 8.0, __dmul_rn(mu_a, mu_b));
    // _SSIM_C1 = (0.01*255.0)**2, _SSIM_C2 = (0.03*255.0)**2 as Python evaluates them
    const double C1 = 0x1.a028f5c28f5c4p+2, C2 = 0x1.d42e147ae147ap+5;
    const double num = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, mu_a), mu_b), C1), __dadd_rn(__dmul_rn(2.0, cov), C2));
    const double den = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(mu_a, mu_a), __dmul_rn(mu_b, mu_b)), C1),
                                 __dadd_rn(__dadd_rn(var_a, var_b), C2));
    vd = __ddiv_rn(__dsub_rn(1.0, __ddiv_rn(num, den)), 2.0);
    const double df = __ddiv_rn((double)a[p] - (double)b[p], 255.0);
    ve = __dmul_rn(df, df);
  }
  s_d[threadIdx.x] = vd;
  s_e[threadIdx.x] = ve;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (threadIdx.x < o) { s_d[threadIdx.x] += s_d[threadIdx.x + o]; s_e[threadIdx.x] += s_e[threadIdx.x + o]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { part[2 * blockIdx.x] = s_d[0]; part[2 * blockIdx.x + 1] = s_e[0]; }
}

// final: counts (exact) and the fixed-order sums -> pem, dssim, mse
__global__ void k_metrics_final(const unsigned char* a, const unsigned char* b, const unsigned char* mask, int64_t n,
                                int margin, const double* part, int64_t nparts, double* out3) {
  __shared__ unsigned long long s_cnt[256], s_exc[256];
  __shared__ double s_d[256], s_e[256];
  unsigned long long cnt = 0, exc = 0;
  for (int64_t p = threadIdx.x; p < n; p += 256)
    if (mask[p]) {
      ++cnt;
      exc += abs((int)a[p] - (int)b[p]) > margin;
    }
  double d = 0.0, e = 0.0;
  for (int64_t q = threadIdx.x; q < nparts; q += 256) { d += part[2 * q]; e += part[2 * q + 1]; }
  s_cnt[threadIdx.x] = cnt; s_exc[threadIdx.x] = exc; s_d[threadIdx.x] = d; s_e[threadIdx.x] = e;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (threadIdx.x < o) {
      s_cnt[threadIdx.x] += s_cnt[threadIdx.x + o]; s_exc[threadIdx.x] += s_exc[threadIdx.x + o];
      s_d[threadIdx.x] += s_d[threadIdx.x + o]; s_e[threadIdx.x] += s_e[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double size = (double)s_cnt[0];
    out3[0] = s_cnt[0] ? (double)s_exc[0] / size : 0.0;  // pem  (metrics.py:85-95)
    out3[1] = s_cnt[0] ? s_d[0] / size : 0.0;             // dssim (:117-123)
    out3[2] = s_cnt[0] ? s_e[0] / size : 0.0;             // mse  (:126-132)
    out3[3] = size;
  }
}

}  // namespace mm
