// lttb_launch.cu -- K3 (LTTB) planning and launch: tables + scan / jump (K3a), large-bucket K3c.
#include "lttb_impl.cuh"  // planning helpers (templates are instantiated in lttb_x_*.cu)

namespace mmh {

// ---- K3 planning --------------------------------------------------------
// Buckets of <= 64 points: exact transition tables over all points (K3a).
// Larger buckets: candidate tables + full verification + repair (K3c).

int64_t lttb_ws(int64_t B, int64_t n_out, int64_t s) {
  const int64_t k3 = n_out - 2;
  if (use_tables(s)) return up(B * tab_ld(k3, smax_for(s)));
  return up(B * k3 * (int64_t)sizeof(double2)) + up(B * k3 * HMAX * 8) + up(B * k3 * 4) + up(B * tab_ld(k3, HMAX)) +
         up(B * (k3 + 2) * 8) + up(B * k3 * 8) + up(B * k3 * 4) + up(B * k3 * (int64_t)sizeof(double2)) +
         up(B * k3 * 8) + up(B * k3 * 4) + up(B * 4) + up(B * k3 * (int64_t)sizeof(double2)) +
         up(B * k3 * (int64_t)sizeof(XAff)) + up(B * k3 * (int64_t)sizeof(double2)) +
         (B == 1 ? up((3 * k3 + 3) * 4) + up(k3 * flat_cp_max(k3) * K3C_FLAT_PART) + up(k3 * 4) +
                    up(std::min<int64_t>(k3, mm::K3S_K3MAX) * (int64_t)mm::K3S_GCAP * 8) : 0);
}

int launch_lttb_f32(LttbArgs a, int ydt, int64_t s, cudaStream_t st);
int launch_lttb_f64(LttbArgs a, int ydt, int64_t s, cudaStream_t st);
int launch_lttb_i64(LttbArgs a, int ydt, int64_t s, cudaStream_t st);
int launch_lttb_i32(LttbArgs a, int ydt, int64_t s, cudaStream_t st);
int64_t repair_scans_f32();
int64_t repair_scans_f64();
int64_t repair_scans_i64();
int64_t repair_scans_i32();

// a.tables must point at lttb_ws(B, n_out, s) bytes of workspace
int launch_lttb(LttbArgs a, int xdt, int ydt, int64_t s, cudaStream_t st) {
  switch (xdt) {
    case MM_F32: return launch_lttb_f32(a, ydt, s, st);
    case MM_F64: return launch_lttb_f64(a, ydt, s, st);
    case MM_I64: return launch_lttb_i64(a, ydt, s, st);
    case MM_I32: return launch_lttb_i32(a, ydt, s, st);
  }
  return fail(MM_EINVAL, "x dtype");
}

// K3s phase timestamps (tools/k3s_check.py --prof): [G][8] %globaltimer values
unsigned long long* k3s_prof_buffer() {
  static const bool on = env_i64("MMLTTB_K3S_PROF", 0) != 0;
  static unsigned long long* buf = nullptr;
  if (on && !buf) {
    if (cudaMalloc(&buf, (K3S_GMAX * 8 + 64) * sizeof(unsigned long long)) != cudaSuccess) buf = nullptr;
    if (buf) cudaMemset(buf + K3S_GMAX * 8, 0, 64 * 8);
  }
  return on ? buf : nullptr;
}

int64_t repair_scans_read() {
  const int64_t v[4] = {repair_scans_f32(), repair_scans_f64(), repair_scans_i64(), repair_scans_i32()};
  int64_t t = 0;
  for (int64_t x : v) {
    if (x < 0) return -1;
    t += x;
  }
  return t;
}

}  // namespace mmh

extern "C" int64_t mmlttb_debug_k3s_prof(unsigned long long* host, int64_t n) {
  unsigned long long* b = mmh::k3s_prof_buffer();
  if (!b || n > mm::K3S_GMAX * 8 + 64) return -1;
  if (cudaMemcpy(host, b, (size_t)n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return n;
}
