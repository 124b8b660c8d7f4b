// capi.cu -- host dispatch behind include/mmlttb.h (extern "C", no torch).
//
// Each entry validates its O(1) arguments defensively (the Python layer has
// already raised the reference's exception classes in the reference's order),
// carves the caller's workspace, and enqueues 1-4 kernels on the caller's
// stream.  Nothing here synchronises the host.  The kernel launchers live in
// k1_launch.cu / lttb_launch.cu / fused_launch.cu / post_launch.cu (host.cuh).
#include "host.cuh"
#include <chrono>
#include "k23.cuh"
#include "raster.cuh"

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: a no-op unless a tool (nsys / ncu) is attached

namespace mmh {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

std::atomic<int64_t> g_launches{0};
// launch trace (mmlttb_trace): kernel names of this thread's calls, for
// bench.py's launch list and roofline labels
thread_local bool g_trace_on = false;
thread_local std::string g_trace;

int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (g_trace_on) {
    if (!g_trace.empty()) g_trace += ',';
    g_trace += what;
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MM_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return MM_OK;
}

// Host-path profiler (tuning builds only: -DMMLTTB_HOSTPROF via MMLTTB_NVCC_EXTRA):
// cumulative host time between marks of the single-series minmaxlttb path.
#ifdef MMLTTB_HOSTPROF
thread_local double g_hp_acc[16];
thread_local std::chrono::high_resolution_clock::time_point g_hp_t;
#define HP_MARK(i)                                                                              \
  do {                                                                                          \
    auto _n = std::chrono::high_resolution_clock::now();                                        \
    if (i > 0) g_hp_acc[i] += std::chrono::duration<double, std::micro>(_n - g_hp_t).count();  \
    g_hp_t = _n;                                                                                \
  } while (0)
#else
#define HP_MARK(i) do {} while (0)
#endif

// Stage timer: events recorded on the caller's stream at K1|K2|K3 boundaries
// of the fused entries (bench.py reads per-kernel device time from these).
struct StageTimer {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<std::array<cudaEvent_t, 4>> calls;
  std::array<cudaEvent_t, 4> cur{};
};
thread_local StageTimer g_timer;

// NVTX range per stage of a fused entry (K1 | K2 | K3), matching the events
void stage_mark(cudaStream_t st, int i) {
  static const char* names[3] = {"mmlttb K1 extrema", "mmlttb K2 compact", "mmlttb K3 lttb"};
  if (i > 0) nvtxRangePop();
  if (i < 3) nvtxRangePushA(names[i]);
  if (!g_timer.on) return;
  if (g_timer.used == g_timer.pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    g_timer.pool.push_back(e);
  }
  cudaEvent_t e = g_timer.pool[g_timer.used++];
  cudaEventRecord(e, st);
  g_timer.cur[i] = e;
  if (i == 3) g_timer.calls.push_back(g_timer.cur);
}

// ---- shared pieces of the fused entries ----------------------------------
// sizes for minmaxlttb / preselect on B series
int64_t preselect_ws(int64_t B, int64_t N, int64_t n_out, int64_t r_ps, int ydt, bool with_lttb) {
  const int64_t k = (n_out - 2) * (r_ps / 2);
  const int64_t S = cdiv(N - 2, k);
  const ExPlan p = plan_extrema(B * k, S, ydt, B, true, with_lttb && k23_ok(B, k, n_out, r_ps) && dyn_chunk_elems() > 0);
  const int64_t cap = 2 + 2 * k;
  int64_t bytes = ex_ws(B * k, p) + up(B * 8);
  if (with_lttb) bytes += 3 * up(B * cap * 8) + lttb_ws(B, n_out, r_ps) + k23_ws() + up(4 * (K23_STAT + B * k));
  return bytes;
}


template <typename XT, typename YT>
void pairs_t(const PairArgs& pa, dim3 g, cudaStream_t st) {
  k_compact_pairs<XT, YT, PAIR_NT, PAIR_ITEMS><<<g, PAIR_NT, 0, st>>>(pa);
}

// K2 launch; pa.out_x == null means no gather (x/y dtypes then irrelevant)
int launch_pairs(PairArgs pa, int64_t B, cudaStream_t st) {
  const int64_t tiles = std::max<int64_t>(1, cdiv(pa.nb, PAIR_NT * PAIR_ITEMS));
  if (B > 65535) return fail(MM_ERANGE, "batch > 65535 series");
  const dim3 g((unsigned)tiles, (unsigned)B);
  const bool y32 = pa.ydt == MM_F32;
  if (!pa.out_x) {  // no gather: x unused; y only read for the endpoint finite check
    pa.x = nullptr;
    y32 ? pairs_t<double, float>(pa, g, st) : pairs_t<double, double>(pa, g, st);
    return check_launch("k_compact_pairs");
  }
  switch (pa.xdt) {
    case MM_F32: y32 ? pairs_t<float, float>(pa, g, st) : pairs_t<float, double>(pa, g, st); break;
    case MM_F64: y32 ? pairs_t<double, float>(pa, g, st) : pairs_t<double, double>(pa, g, st); break;
    case MM_I64: y32 ? pairs_t<long long, float>(pa, g, st) : pairs_t<long long, double>(pa, g, st); break;
    default: y32 ? pairs_t<int, float>(pa, g, st) : pairs_t<int, double>(pa, g, st); break;
  }
  return check_launch("k_compact_pairs");
}

// First 256 bytes of every fused entry's workspace: status word (bit 0 =
// non-finite y seen), zeroed on the stream at entry (not between the chunks of
// one call split by batch_chunks, so the word ORs over the whole batch).
thread_local bool g_chunk_cont = false;
int* take_status(Carve& cv, cudaStream_t st) {
  int* p = cv.take<int>(1);
  if (p && !g_chunk_cont && cudaMemsetAsync(p, 0, sizeof(int), st) != cudaSuccess) return nullptr;
  return p;
}

// Batches above the 65,535-series grid.y limit of the per-series kernels run
// as stream-ordered chunks over the same workspace (each chunk needs no more
// than the whole batch's workspace).  f(s0, b) runs series [s0, s0 + b).
constexpr int64_t MAX_CHUNK_B = 65535;
template <typename F>
int batch_chunks(int64_t B, F f) {
  int rc = MM_OK;
  for (int64_t s0 = 0; s0 < B && rc == MM_OK; s0 += MAX_CHUNK_B) {
    g_chunk_cont = s0 > 0;
    rc = f(s0, std::min<int64_t>(MAX_CHUNK_B, B - s0));
  }
  g_chunk_cont = false;
  return rc;
}
inline const void* elem_off(const void* p, int dt, int64_t i) {
  return p ? (const void*)((const char*)p + i * esize(dt)) : nullptr;
}

int check_common(const void* y, int ydt, int64_t B, int64_t N, int64_t n_out) {
  if (!y) return fail(MM_EINVAL, "y is null");
  if (!ydt_ok(ydt)) return fail(MM_EINVAL, "y dtype must be f32 or f64");
  if (B < 1 || N < 2) return fail(MM_EINVAL, "need B >= 1 and N >= 2");
  if (n_out < 3 || n_out > N) return fail(MM_EINVAL, "n_out must be in [3, %lld]", (long long)N);
  return MM_OK;
}

// Deferred status: device-input callers learn of non-finite y (the
// reference's NonFiniteValue) without a host sync.  mmlttb_status_arm()
// hands out a slot of a pinned, device-mapped ring; the next status-producing
// call of this host thread stores (tag | status bit) there from the device:
// K23 (the single-series path) from its CTA 0 as part of the launch, every
// other path with one 1-thread kernel after its last launch.
constexpr int64_t STATUS_SLOTS = 1024;
struct StatusRing {
  std::mutex mu;
  volatile unsigned long long* host = nullptr;
};
StatusRing g_status;
struct StatusArm {
  unsigned long long* slot = nullptr;  // device view of the armed slot
  volatile unsigned long long* hslot = nullptr;  // host view
  unsigned long long tag = 0;
  bool consumed = false;
};
thread_local StatusArm g_arm;
constexpr unsigned long long TAG_FAILED = 4;  // host-written: the armed call failed

__global__ void k_status_mirror(const int* status, unsigned long long* slot, unsigned long long tag) {
  *(volatile unsigned long long*)slot = tag | (unsigned long long)(*status & 1);
}

inline unsigned long long ticket_tag(int64_t t) { return (unsigned long long)(t + 1) << 3; }

// Runs one status-producing entry; delivers the armed slot afterwards.
constexpr unsigned long long TAG_SKIPPED = 2;  // host-written: the armed call was captured into a graph
template <class F>
int with_status_slot(const void* workspace, void* stream, F&& f) {
  if (g_arm.slot) {  // a captured launch must not bake the slot into the graph
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing((cudaStream_t)stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      *g_arm.hslot = g_arm.tag | TAG_SKIPPED;
      g_arm = StatusArm{};
    }
  }
  int rc = f();
  StatusArm a = g_arm;
  g_arm = StatusArm{};
  if (!a.slot) return rc;
  if (rc == MM_OK && !a.consumed) {
    k_status_mirror<<<1, 1, 0, (cudaStream_t)stream>>>((const int*)workspace, a.slot, a.tag);
    rc = check_launch("k_status_mirror");
  }
  if (rc != MM_OK) *a.hslot = a.tag | TAG_FAILED;
  return rc;
}
unsigned long long* status_slot_take(unsigned long long* tag) {
  if (!g_arm.slot || g_arm.consumed) return nullptr;
  g_arm.consumed = true;
  *tag = g_arm.tag;
  return g_arm.slot;
}

}  // namespace mmh


extern "C" {

int mmlttb_version(void) { return 1; }

int64_t mmlttb_launch_count(void) { return g_launches.load(); }

int64_t mmlttb_repair_scans(void) {
  return repair_scans_read();
}

int mmlttb_trace(int enable) {
  g_trace_on = enable != 0;
  g_trace.clear();
  return MM_OK;
}

int64_t mmlttb_trace_read(char* buf, int64_t len) {
  const int64_t n = (int64_t)g_trace.size();
  if (buf && len > 0) {
    const int64_t c = std::min<int64_t>(n, len - 1);
    memcpy(buf, g_trace.data(), (size_t)c);
    buf[c] = 0;
  }
  g_trace.clear();
  return n;
}

const volatile unsigned long long* mmlttb_status_ring(void) {
  std::lock_guard<std::mutex> lk(g_status.mu);
  if (!g_status.host) {
    void* h = nullptr;
    if (cudaHostAlloc(&h, STATUS_SLOTS * sizeof(unsigned long long), cudaHostAllocMapped | cudaHostAllocPortable) !=
        cudaSuccess) {
      fail(MM_ECUDA, "status ring: cudaHostAlloc");
      return nullptr;
    }
    memset(h, 0, STATUS_SLOTS * sizeof(unsigned long long));
    g_status.host = (volatile unsigned long long*)h;
  }
  return g_status.host;
}

int64_t mmlttb_status_arm(void) {
  static std::atomic<int64_t> next{0};
  if (!g_status.host && !mmlttb_status_ring()) return MM_ECUDA;
  const int64_t t = next.fetch_add(1);
  const int64_t s = t % STATUS_SLOTS;
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, (void*)(g_status.host + s), 0) != cudaSuccess)
    return fail(MM_ECUDA, "status_arm: cudaHostGetDevicePointer");
  g_status.host[s] = 0;
  g_arm = StatusArm{(unsigned long long*)d, g_status.host + s, ticket_tag(t), false};
  return t;
}

int mmlttb_status_poll(int64_t ticket, int block) {
  if (ticket < 0 || !g_status.host) return fail(MM_EINVAL, "bad status ticket");
  const unsigned long long tag = ticket_tag(ticket);
  volatile unsigned long long* p = g_status.host + ticket % STATUS_SLOTS;
  unsigned long long v = *p;
  if ((v & ~7ull) != tag && block) {  // the slot is written by the call's last kernel
    if (cudaDeviceSynchronize() != cudaSuccess) return fail(MM_ECUDA, "status_poll: %s",
                                                            cudaGetErrorString(cudaGetLastError()));
    v = *p;
  }
  if ((v & ~7ull) != tag) {
    if (v != 0 && (v & ~7ull) > tag) return fail(MM_EINVAL, "expired status ticket");
    return block ? fail(MM_EINVAL, "status ticket never delivered") : 2;
  }
  if (v & TAG_FAILED) return fail(MM_EINVAL, "the armed call failed");
  return (int)(v & 1);  // (TAG_SKIPPED: no status, reads as 0)
}

int mmlttb_stage_timer(int enable) {
  g_timer.on = enable != 0;
  g_timer.used = 0;
  g_timer.calls.clear();
  return MM_OK;
}

int mmlttb_stage_timer_read(double* ms3, int64_t* calls) {
  for (int i = 0; i < 3; ++i) ms3[i] = 0.0;
  for (auto& c : g_timer.calls) {
    if (cudaEventSynchronize(c[3]) != cudaSuccess) return fail(MM_ECUDA, "cudaEventSynchronize");
    for (int i = 0; i < 3; ++i) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, c[i], c[i + 1]) != cudaSuccess) return fail(MM_ECUDA, "cudaEventElapsedTime");
      ms3[i] += ms;
    }
  }
  *calls = (int64_t)g_timer.calls.size();
  g_timer.used = 0;
  g_timer.calls.clear();
  return MM_OK;
}
const char* mmlttb_last_error(void) { return g_err.c_str(); }

int64_t mmlttb_workspace_bytes(int op, int64_t B, int64_t N, int64_t n_out, int64_t r_ps, int y_dtype) {
  if (B < 1 || N < 3 || n_out < 3 || n_out > N) return 0;
  switch (op) {
    case MM_OP_MINMAXLTTB:
      if (r_ps == 1) return mmlttb_workspace_bytes(MM_OP_MINMAX, B, N, n_out, 0, y_dtype);
      if (r_ps < 2 || r_ps % 2) return 0;
      return ALIGN + preselect_ws(B, N, n_out, r_ps, y_dtype, true);
    case MM_OP_PRESELECT:
      if (r_ps < 2 || r_ps % 2) return 0;
      return ALIGN + preselect_ws(B, N, n_out, r_ps, y_dtype, false);
    case MM_OP_LTTB:
      return lttb_ws(B, n_out, cdiv(N - 2, n_out - 2));
    case MM_OP_MINMAX:
    case MM_OP_M4: {
      const int64_t k = op == MM_OP_MINMAX ? n_out / 2 : n_out / 4;
      if (k < 1) return 0;
      return ALIGN + ex_ws(B * k, plan_extrema(B * k, cdiv(N, k), y_dtype, B, true));
    }
  }
  return 0;
}

static int preselect_entry(const void* y, int y_dtype, int64_t y_ld, int64_t B, int64_t N, int64_t n_out,
                            int64_t r_ps, int64_t* out, int64_t out_ld, int64_t* out_count, void* workspace,
                            int64_t workspace_bytes, void* stream) {
  int rc = check_common(y, y_dtype, B, N, n_out);
  if (rc) return rc;
  if (r_ps < 2 || r_ps % 2) return fail(MM_EINVAL, "r_ps must be even >= 2");
  const int64_t k = (n_out - 2) * (r_ps / 2);
  if (k > N - 2) return fail(MM_EINVAL, "sub-buckets exceed interior");
  if (!mul_ok(k, N)) return fail(MM_ERANGE, "k*N overflows int64");
  if (out_ld < 2 + 2 * k) return fail(MM_EINVAL, "out_ld < 2 + 2k");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t S = cdiv(N - 2, k);
  const ExPlan p = plan_extrema(B * k, S, y_dtype, B, true);
  Carve cv{(char*)workspace, workspace_bytes};
  int* status = take_status(cv, st);
  ExArgs ea{y, y_ld, B, 1, N - 2, k, nullptr, 0, k, p.C, p.chunk};
  if (!carve_ex(cv, B * k, p, ea) || !status) return fail(MM_EWORKSPACE, "workspace too small");
  if ((rc = launch_extrema(ea, y_dtype, st))) return rc;
  PairArgs pa{};
  pa.ext = ea.ext; pa.cnt8 = ea.cnt8; pa.nb = k;
  pa.emit_first = 0; pa.emit_last = N - 1;
  pa.out_idx = out; pa.out_ld = out_ld; pa.out_count = out_count;
  pa.y = y; pa.ydt = y_dtype; pa.y_ld = y_ld; pa.status = status;
  return launch_pairs(pa, B, st);
}

static int minmax_impl(const void* y, int ydt, int64_t y_ld, int64_t B, int64_t N, int64_t n_out, int m4,
                       int64_t force_n_out, int64_t* out, int64_t* out_count, void* ws, int64_t wsb,
                       cudaStream_t st) {
  int rc = check_common(y, ydt, B, N, n_out);
  if (rc) return rc;
  const int64_t k = m4 ? n_out / 4 : n_out / 2;
  if ((m4 && n_out % 4) || (!m4 && n_out % 2)) return fail(MM_EINVAL, "n_out divisibility");
  if (!mul_ok(k + 1, N)) return fail(MM_ERANGE, "k*N overflows int64");
  const ExPlan p = plan_extrema(B * k, cdiv(N, k), ydt, B, true);
  Carve cv{(char*)ws, wsb};
  int* status = take_status(cv, st);
  ExArgs ea{y, y_ld, B, 0, N, k, nullptr, 0, k, p.C, p.chunk};
  if (!carve_ex(cv, B * k, p, ea) || !status) return fail(MM_EWORKSPACE, "workspace too small");
  if ((rc = launch_extrema(ea, ydt, st))) return rc;
  if (!m4 && force_n_out == 0) {
    PairArgs pa{};
    pa.ext = ea.ext; pa.cnt8 = ea.cnt8; pa.nb = k;
    pa.emit_first = -1; pa.emit_last = -1;
    pa.out_idx = out; pa.out_ld = n_out; pa.out_count = out_count;
    pa.y = y; pa.ydt = ydt; pa.y_ld = y_ld; pa.status = status;
    return launch_pairs(pa, B, st);
  }
  CompactArgs ca{};
  ca.ext = ea.ext; ca.nb = k; ca.mode = m4 ? 1 : 0;
  ca.ydt = ydt; ca.status = status;
  ca.emit_first = -1; ca.emit_last = -1; ca.force_n_out = force_n_out; ca.last_index = N - 1;
  ca.start = 0; ca.len = N; ca.k = k; ca.b0 = 0;
  ca.out_idx = out; ca.out_ld = n_out; ca.out_count = out_count;
  k_compact<512><<<(unsigned)B, 512, 0, st>>>(ca);
  return check_launch("k_compact");
}

int mmlttb_minmax(const void* y, int y_dtype, int64_t y_ld, int64_t B, int64_t N, int64_t n_out, int64_t* out,
                  int64_t* out_count, void* workspace, int64_t workspace_bytes, void* stream) {
  return with_status_slot(workspace, stream, [&] {
    return batch_chunks(B, [&](int64_t s0, int64_t b) {
      return minmax_impl(elem_off(y, y_dtype, s0 * y_ld), y_dtype, y_ld, b, N, n_out, 0, 0, out + s0 * n_out,
                         out_count ? out_count + s0 : nullptr, workspace, workspace_bytes, (cudaStream_t)stream);
    });
  });
}

int mmlttb_m4(const void* y, int y_dtype, int64_t y_ld, int64_t B, int64_t N, int64_t n_out, int64_t* out,
              int64_t* out_count, void* workspace, int64_t workspace_bytes, void* stream) {
  return with_status_slot(workspace, stream, [&] {
    return batch_chunks(B, [&](int64_t s0, int64_t b) {
      return minmax_impl(elem_off(y, y_dtype, s0 * y_ld), y_dtype, y_ld, b, N, n_out, 1, 0, out + s0 * n_out,
                         out_count ? out_count + s0 : nullptr, workspace, workspace_bytes, (cudaStream_t)stream);
    });
  });
}

static int minmaxlttb_entry(const void* x, int x_dtype, int64_t x_ld, const void* y, int y_dtype, int64_t y_ld, int64_t B,
                      int64_t N, int64_t n_out, int64_t r_ps, int64_t* out, int64_t* out_count, void* workspace,
                      int64_t workspace_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (r_ps == 1) {  // downsamplers.py:204-205
    if (n_out % 2) return fail(MM_EINVAL, "r_ps=1 needs an even n_out");
    return minmax_impl(y, y_dtype, y_ld, B, N, n_out, 0, n_out, out, out_count, workspace, workspace_bytes, st);
  }
  int rc = check_common(y, y_dtype, B, N, n_out);
  if (rc) return rc;
  if (!x || !xdt_ok(x_dtype)) return fail(MM_EINVAL, "x missing or bad dtype");
  if (r_ps < 2 || r_ps % 2) return fail(MM_EINVAL, "r_ps must be 1 or even >= 2");
  const int64_t k = (n_out - 2) * (r_ps / 2);
  if (k > N - 2) return fail(MM_EINVAL, "sub-buckets exceed interior");
  if (!mul_ok(k, N)) return fail(MM_ERANGE, "k*N overflows int64");
  const int64_t S = cdiv(N - 2, k);
  const bool k23 = k23_ok(B, k, n_out, r_ps);
  const ExPlan p = plan_extrema(B * k, S, y_dtype, B, true, k23 && dyn_chunk_elems() > 0);
  const int64_t cap = 2 + 2 * k;
  HP_MARK(2);
  if (k23) {
    // one series: K1, then K2 + K3 in one cooperative launch (K23).  The only
    // zeroing of the call is one memset over K23's barrier words and K1's
    // arrival counters (adjacent); the status word is written, not ORed.
    Carve cv{(char*)workspace, workspace_bytes};
    int* status = cv.take<int>(1);
    unsigned* zr = cv.take<unsigned>(K23_STAT + B * k);
    unsigned* k23s = cv.take<unsigned>(k23_ws() / 4);
    ExArgs ea{y, y_ld, B, 1, N - 2, k, nullptr, 0, k, p.C, p.chunk};
    carve_ex(cv, B * k, p, ea);
    int64_t* pre = cv.take<int64_t>(B * cap);
    double* px = cv.take<double>(B * cap);
    double* py = cv.take<double>(B * cap);
    if (!cv.ok) return fail(MM_EWORKSPACE, "workspace too small (%lld bytes)", (long long)workspace_bytes);
    ea.arrivals = zr + K23_STAT;  // (the carve_ex slot stays unused)
    ea.arrivals_zeroed = 1;
    ea.ticket = p.E > 0 && dyn_chunk_elems() > 0 ? zr + 128 : nullptr;  // (zeroed with the rest)
    HP_MARK(3);
    if (cudaMemsetAsync(zr, 0, (size_t)(K23_STAT + B * k) * sizeof(unsigned), st) != cudaSuccess)
      return fail(MM_ECUDA, "memset");
    HP_MARK(4);
    stage_mark(st, 0);
    HP_MARK(5);
    if ((rc = launch_extrema(ea, y_dtype, st))) return rc;
    HP_MARK(6);
    stage_mark(st, 1);
    K23Args ka{};
    ka.ext = ea.ext; ka.cnt8 = ea.cnt8; ka.k = k; ka.N = N; ka.n_out = n_out;
    ka.x = x; ka.y = y; ka.pre = pre; ka.px = px; ka.py = py; ka.out = out; ka.status = status;
    ka.mirror = status_slot_take(&ka.mtag);
    ka.sync = zr;
    ka.stat = k23s;
    HP_MARK(7);
    if ((rc = launch_k23(ka, x_dtype, y_dtype, r_ps, st))) return rc;
    HP_MARK(8);
    stage_mark(st, 2);
    stage_mark(st, 3);
    HP_MARK(9);
    if (out_count) {
      k_fill<<<(unsigned)cdiv(B, 256), 256, 0, st>>>(out_count, B, n_out);
      return check_launch("k_fill");
    }
    return MM_OK;
  }
  Carve cv0{(char*)workspace, workspace_bytes};
  int* status = take_status(cv0, st);
  if (!status) return fail(MM_EWORKSPACE, "workspace too small");
  if (fused_ok(B, N, n_out, r_ps, y_dtype)) {  // one CTA per series, everything on chip
    FusedArgs fa{x, x_ld, y, y_ld, B, N, n_out, r_ps, out, status};
    stage_mark(st, 0);
    if ((rc = launch_fused(fa, x_dtype, y_dtype, st))) return rc;
    stage_mark(st, 1);
    stage_mark(st, 2);
    stage_mark(st, 3);
    if (out_count) {
      k_fill<<<(unsigned)cdiv(B, 256), 256, 0, st>>>(out_count, B, n_out);
      return check_launch("k_fill");
    }
    return MM_OK;
  }
  Carve cv = cv0;
  ExArgs ea{y, y_ld, B, 1, N - 2, k, nullptr, 0, k, p.C, p.chunk};
  carve_ex(cv, B * k, p, ea);
  int64_t* cnt = cv.take<int64_t>(B);
  int64_t* pre = cv.take<int64_t>(B * cap);
  double* px = cv.take<double>(B * cap);
  double* py = cv.take<double>(B * cap);
  unsigned char* lt = cv.take<unsigned char>(lttb_ws(B, n_out, r_ps));
  if (!cv.ok) return fail(MM_EWORKSPACE, "workspace too small (%lld bytes)", (long long)workspace_bytes);
  // K1: sub-bucket extrema over partition(1, N-1, k)  (downsamplers.py:149-155)
  stage_mark(st, 0);
  if ((rc = launch_extrema(ea, y_dtype, st))) return rc;
  stage_mark(st, 1);
  if (post_ok(k, n_out, r_ps)) {  // K2 + K3 in one CTA per series
    PostArgs qa{ea.ext, k, x, x_ld, y, y_ld, N, n_out, pre, px, py, cap, out, status};
    if ((rc = launch_post(qa, B, x_dtype, y_dtype, smax_for(r_ps), st))) return rc;
    stage_mark(st, 2);
    stage_mark(st, 3);
    if (out_count) {
      k_fill<<<(unsigned)cdiv(B, 256), 256, 0, st>>>(out_count, B, n_out);
      return check_launch("k_fill");
    }
    return MM_OK;
  }
  // K2: [0] + interleaved pairs + [N-1], gathered as f64 (:156-160, :207)
  PairArgs pa{};
  pa.ext = ea.ext; pa.cnt8 = ea.cnt8; pa.nb = k;
  pa.emit_first = 0; pa.emit_last = N - 1;
  pa.out_idx = pre; pa.out_ld = cap; pa.out_count = cnt;
  pa.x = x; pa.xdt = x_dtype; pa.x_ld = x_ld;
  pa.y = y; pa.ydt = y_dtype; pa.y_ld = y_ld;
  pa.out_x = px; pa.out_y = py; pa.status = status;
  if ((rc = launch_pairs(pa, B, st))) return rc;
  stage_mark(st, 2);
  // K3: LTTB over the compacted sub-series, mapped back (:208-209)
  LttbArgs la{};
  la.x = px; la.x_ld = cap; la.y = py; la.y_ld = cap;
  la.m_dev = cnt; la.n = 0; la.bounds = nullptr; la.map = pre; la.map_ld = cap;
  la.B = B; la.n_out = n_out; la.out = out; la.tables = lt;
  if ((rc = launch_lttb(la, MM_F64, MM_F64, r_ps, st))) return rc;
  stage_mark(st, 3);
  if (out_count) {  // every series yields exactly n_out (P9)
    k_fill<<<(unsigned)cdiv(B, 256), 256, 0, st>>>(out_count, B, n_out);
    return check_launch("k_fill");
  }
  return MM_OK;
}

static int lttb_entry(const void* x, int x_dtype, int64_t x_ld, const void* y, int y_dtype, int64_t y_ld, int64_t B,
                int64_t N, int64_t n_out, int64_t* out, void* workspace, int64_t workspace_bytes, void* stream) {
  int rc = check_common(y, y_dtype, B, N, n_out);
  if (rc) return rc;
  if (!x || !xdt_ok(x_dtype)) return fail(MM_EINVAL, "x missing or bad dtype");
  if (!mul_ok(n_out, N)) return fail(MM_ERANGE, "n_out*N overflows int64");
  const int64_t s = cdiv(N - 2, n_out - 2);
  if (workspace_bytes < lttb_ws(B, n_out, s)) return fail(MM_EWORKSPACE, "workspace too small");
  LttbArgs la{};
  la.x = x; la.x_ld = x_ld; la.y = y; la.y_ld = y_ld;
  la.m_dev = nullptr; la.n = N; la.bounds = nullptr; la.map = nullptr;
  la.B = B; la.n_out = n_out; la.out = out; la.tables = (unsigned char*)workspace;
  return launch_lttb(la, x_dtype, y_dtype, s, (cudaStream_t)stream);
}

int mmlttb_minmax_preselect(const void* y, int y_dtype, int64_t y_ld, int64_t B, int64_t N, int64_t n_out,
                            int64_t r_ps, int64_t* out, int64_t out_ld, int64_t* out_count, void* workspace,
                            int64_t workspace_bytes, void* stream) {
  return with_status_slot(workspace, stream, [&] {
    return batch_chunks(B, [&](int64_t s0, int64_t b) {
      return preselect_entry(elem_off(y, y_dtype, s0 * y_ld), y_dtype, y_ld, b, N, n_out, r_ps, out + s0 * out_ld,
                             out_ld, out_count ? out_count + s0 : nullptr, workspace, workspace_bytes, stream);
    });
  });
}

#ifdef MMLTTB_HOSTPROF
int mmlttb_hostprof_read(double* acc) {
  for (int i = 0; i < 16; ++i) { acc[i] = g_hp_acc[i]; g_hp_acc[i] = 0; }
  return MM_OK;
}
#endif

int mmlttb_minmaxlttb(const void* x, int x_dtype, int64_t x_ld, const void* y, int y_dtype, int64_t y_ld, int64_t B,
                      int64_t N, int64_t n_out, int64_t r_ps, int64_t* out, int64_t* out_count, void* workspace,
                      int64_t workspace_bytes, void* stream) {
  HP_MARK(0);
  return with_status_slot(workspace, stream, [&] {
    HP_MARK(1);
    return batch_chunks(B, [&](int64_t s0, int64_t b) {
      return minmaxlttb_entry(elem_off(x, x_dtype, s0 * x_ld), x_dtype, x_ld, elem_off(y, y_dtype, s0 * y_ld), y_dtype,
                              y_ld, b, N, n_out, r_ps, out + s0 * n_out, out_count ? out_count + s0 : nullptr,
                              workspace, workspace_bytes, stream);
    });
  });
}

int mmlttb_lttb(const void* x, int x_dtype, int64_t x_ld, const void* y, int y_dtype, int64_t y_ld, int64_t B,
                int64_t N, int64_t n_out, int64_t* out, void* workspace, int64_t workspace_bytes, void* stream) {
  return batch_chunks(B, [&](int64_t s0, int64_t b) {
    return lttb_entry(elem_off(x, x_dtype, s0 * x_ld), x_dtype, x_ld, elem_off(y, y_dtype, s0 * y_ld), y_dtype, y_ld,
                      b, N, n_out, out + s0 * n_out, workspace, workspace_bytes, stream);
  });
}

int mmlttb_every_nth(int64_t N, int64_t n_out, int64_t* out, void* stream) {
  if (n_out < 1 || !mul_ok(n_out, N)) return fail(MM_EINVAL, "bad n_out");
  k_every_nth<<<(unsigned)cdiv(n_out, 256), 256, 0, (cudaStream_t)stream>>>(N, n_out, out);
  return check_launch("k_every_nth");
}

int64_t mmlttb_extrema_workspace_bytes(int64_t k, int64_t max_bucket_len) {
  (void)max_bucket_len;
  return ex_ws(k, plan_extrema(k, 1, MM_F32));
}

int mmlttb_extrema_by_bucket(const void* y, int y_dtype, const int64_t* bounds, int64_t k, int64_t max_bucket_len,
                             int64_t* out_min, int64_t* out_max, void* workspace, int64_t workspace_bytes,
                             void* stream) {
  if (!y || !bounds || !ydt_ok(y_dtype) || k < 1 || max_bucket_len < 1) return fail(MM_EINVAL, "bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const ExPlan p = plan_extrema(k, max_bucket_len, y_dtype);
  Carve cv{(char*)workspace, workspace_bytes};
  ExArgs ea{y, 0, 1, 0, 1, 1, bounds, 0, k, p.C, p.chunk};
  if (!carve_ex(cv, k, p, ea)) return fail(MM_EWORKSPACE, "workspace too small");
  int rc = launch_extrema(ea, y_dtype, st);
  if (rc) return rc;
  k_finalize_extrema<<<(unsigned)cdiv(k, 256), 256, 0, st>>>(ea.ext, k, out_min, out_max);
  return check_launch("k_finalize_extrema");
}

int64_t mmlttb_lttb_select_workspace_bytes(int64_t n, int64_t nb) {
  (void)n;
  return lttb_ws(1, nb + 1, INT64_MAX / 4);
}

int mmlttb_lttb_select(const void* xs, int x_dtype, const void* ys, int y_dtype, int64_t n, const int64_t* bounds,
                       int64_t nb, int64_t* out, void* workspace, int64_t workspace_bytes, void* stream) {
  if (!xs || !ys || !bounds || !xdt_ok(x_dtype) || !ydt_ok(y_dtype) || nb < 2 || n < 2)
    return fail(MM_EINVAL, "bad arguments");
  if (workspace_bytes < mmlttb_lttb_select_workspace_bytes(n, nb)) return fail(MM_EWORKSPACE, "workspace too small");
  LttbArgs la{};
  la.x = xs; la.y = ys; la.n = n; la.bounds = bounds; la.B = 1; la.n_out = nb + 1; la.out = out;
  la.tables = (unsigned char*)workspace;
  // explicit bounds: bucket sizes are the caller's -> the general (K3c) path
  return launch_lttb(la, x_dtype, y_dtype, INT64_MAX / 4, (cudaStream_t)stream);
}

int64_t mmlttb_shard_workspace_bytes(int64_t N, int64_t n_out, int64_t r_ps, int64_t b0, int64_t b1) {
  const int64_t k = (n_out - 2) * (r_ps / 2);
  if (k < 1 || b1 <= b0) return ALIGN;
  return std::max(ex_ws(b1 - b0, plan_extrema(b1 - b0, cdiv(N - 2, k), MM_F32, 1, true)),
                  ex_ws(b1 - b0, plan_extrema(b1 - b0, cdiv(N - 2, k), MM_F64, 1, true)));
}

int mmlttb_shard_preselect(const void* x_shard, int x_dtype, const void* y_shard, int y_dtype, int64_t lo, int64_t N,
                           int64_t n_out, int64_t r_ps, int64_t b0, int64_t b1, int emit_first, int emit_last,
                           int64_t* out_idx, double* out_x, double* out_y, int64_t* out_count, void* workspace,
                           int64_t workspace_bytes, void* stream) {
  int rc = check_common(y_shard, y_dtype, 1, N, n_out);
  if (rc) return rc;
  if (!x_shard || !xdt_ok(x_dtype)) return fail(MM_EINVAL, "x missing or bad dtype");
  if (r_ps < 2 || r_ps % 2) return fail(MM_EINVAL, "r_ps must be even >= 2");
  const int64_t k = (n_out - 2) * (r_ps / 2);
  if (k > N - 2 || b0 < 0 || b1 > k || b1 < b0) return fail(MM_EINVAL, "bad bucket range");
  if (!mul_ok(k, N)) return fail(MM_ERANGE, "k*N overflows int64");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nb = b1 - b0;
  const ExPlan p = plan_extrema(std::max<int64_t>(nb, 1), cdiv(N - 2, k), y_dtype, 1, true);
  Carve cv{(char*)workspace, workspace_bytes};
  // virtual base: element i of the global series lives at y_shard[i - lo]
  const void* ybase = (const char*)y_shard - lo * esize(y_dtype);
  const void* xbase = (const char*)x_shard - lo * esize(x_dtype);
  ExArgs ea{ybase, 0, 1, 1, N - 2, k, nullptr, b0, nb, p.C, p.chunk};
  if (!carve_ex(cv, std::max<int64_t>(nb, 1), p, ea)) return fail(MM_EWORKSPACE, "workspace too small");
  if (nb > 0 && (rc = launch_extrema(ea, y_dtype, st))) return rc;
  PairArgs pa{};
  pa.ext = ea.ext; pa.cnt8 = ea.cnt8; pa.nb = nb;
  pa.emit_first = emit_first ? 0 : -1; pa.emit_last = emit_last ? N - 1 : -1;
  pa.out_idx = out_idx; pa.out_ld = 0; pa.out_count = out_count;
  pa.x = xbase; pa.xdt = x_dtype; pa.x_ld = 0;
  pa.y = ybase; pa.ydt = y_dtype; pa.y_ld = 0;
  pa.out_x = out_x; pa.out_y = out_y;
  return launch_pairs(pa, 1, st);
}

int mmlttb_merge_shards(const int64_t* idx, const double* xs, const double* ys, const int64_t* counts, int64_t G,
                        int64_t cap, int64_t* out_idx, double* out_x, double* out_y, int64_t* out_m, void* stream) {
  if (G < 1 || cap < 1) return fail(MM_EINVAL, "bad arguments");
  const dim3 grid((unsigned)cdiv(cap, MERGE_TILE), (unsigned)G);
  k_merge_shards<<<grid, 256, 0, (cudaStream_t)stream>>>(idx, xs, ys, counts, G, cap, out_idx, out_x, out_y, out_m);
  return check_launch("k_merge_shards");
}

int mmlttb_merge_packed(const int64_t* buf, int64_t G, int64_t cap, int64_t* out_idx, double* out_x, double* out_y,
                        int64_t* out_m, void* stream) {
  if (!buf || !out_idx || !out_x || !out_y || !out_m || G < 1 || cap < 1) return fail(MM_EINVAL, "bad arguments");
  const dim3 grid((unsigned)cdiv(cap, MERGE_TILE), (unsigned)G);
  k_merge_packed<<<grid, 256, 0, (cudaStream_t)stream>>>((const long long*)buf, G, cap, out_idx, out_x, out_y, out_m);
  return check_launch("k_merge_packed");
}

int mmlttb_p2p_publish(const int64_t* idx, const double* xs, const double* ys, const int64_t* count, int64_t cap,
                       const uint64_t* peer_bufs, const uint64_t* peer_pads, const uint32_t* own_pad, int64_t G,
                       int64_t rank, uint32_t epoch, void* stream) {
  if (!idx || !xs || !ys || !count || !peer_bufs || !peer_pads || !own_pad || G < 1 || rank < 0 || rank >= G ||
      cap < 1 || epoch == 0)
    return fail(MM_EINVAL, "bad arguments");
  k_p2p_publish<<<(unsigned)G, 256, 0, (cudaStream_t)stream>>>(idx, xs, ys, count, cap,
                                                              (const unsigned long long*)peer_bufs,
                                                              (const unsigned long long*)peer_pads, own_pad, G, rank,
                                                              epoch);
  return check_launch("k_p2p_publish");
}

int mmlttb_p2p_merge(const int64_t* own_buf, const uint32_t* own_pad, const uint64_t* peer_pads, int64_t G,
                     int64_t rank, int64_t cap, uint32_t epoch, int64_t* out_idx, double* out_x, double* out_y,
                     int64_t* out_m, void* stream) {
  if (!own_buf || !own_pad || !peer_pads || !out_idx || !out_x || !out_y || !out_m || G < 1 || cap < 1 || epoch == 0)
    return fail(MM_EINVAL, "bad arguments");
  k_p2p_merge<<<(unsigned)G, 256, 0, (cudaStream_t)stream>>>((const long long*)own_buf, own_pad,
                                                            (const unsigned long long*)peer_pads, G, rank, cap, epoch,
                                                            out_idx, out_x, out_y, out_m);
  return check_launch("k_p2p_merge");
}

int64_t mmlttb_lttb_preselected_workspace_bytes(int64_t B, int64_t n_out, int64_t r_ps) {
  return lttb_ws(B, n_out, r_ps);
}

int mmlttb_lttb_preselected(const int64_t* pre_idx, const double* pre_x, const double* pre_y, const int64_t* m,
                            int64_t B, int64_t ld, int64_t n_out, int64_t r_ps, int64_t* out, void* workspace,
                            int64_t workspace_bytes, void* stream) {
  if (!pre_idx || !pre_x || !pre_y || !m || B < 1 || n_out < 3 || r_ps < 1) return fail(MM_EINVAL, "bad arguments");
  if (workspace_bytes < lttb_ws(B, n_out, r_ps)) return fail(MM_EWORKSPACE, "workspace too small");
  LttbArgs la{};
  la.x = pre_x; la.x_ld = ld; la.y = pre_y; la.y_ld = ld;
  la.m_dev = m; la.map = pre_idx; la.map_ld = ld;
  la.B = B; la.n_out = n_out; la.out = out; la.tables = (unsigned char*)workspace;
  return launch_lttb(la, MM_F64, MM_F64, r_ps, (cudaStream_t)stream);
}

int mmlttb_deinterleave_f64(const void* pairs, int64_t n, double* x, double* y, void* stream) {
  if (!pairs || !x || !y || n < 0) return fail(MM_EINVAL, "bad arguments");
  if (n == 0) return MM_OK;
  if ((uintptr_t)pairs % 16) return fail(MM_EINVAL, "pairs must be 16-byte aligned");
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(n, 256), (int64_t)sm_count() * 32);
  k_deinterleave_f64<<<blocks, 256, 0, (cudaStream_t)stream>>>((const double2*)pairs, x, y, n);
  return check_launch("k_deinterleave_f64");
}

int64_t mmlttb_raster_workspace_bytes(int64_t n, int64_t w, int64_t h) {
  return up(n * 8) * 2 + up(std::max<int64_t>(n - 1, 1) * 16) + up(5 * w * h * 8) + up(cdiv(w * h, 256) * 16) + ALIGN;
}

int mmlttb_rasterize(const void* x, int x_dtype, const void* y, int y_dtype, const int64_t* idx, int64_t n, double x0,
                     double x1, double y0, double y1, int64_t w, int64_t h, uint8_t* pixels, void* workspace,
                     int64_t workspace_bytes, void* stream) {
  if (!x || !y || !pixels || n < 2 || w < 1 || h < 1 || !xdt_ok(x_dtype) || !xdt_ok(y_dtype) ||
      w * h > (int64_t)INT32_MAX)
    return fail(MM_EINVAL, "bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  Carve cv{(char*)workspace, workspace_bytes};
  RasterCoordArgs a{x, x_dtype, y, y_dtype, idx, n, x0, x1, y0, y1, w, h, nullptr, nullptr, nullptr};
  a.us = cv.take<double>(n);
  a.vs = cv.take<double>(n);
  a.box = cv.take<int>(4 * (n - 1));
  if (!cv.ok) return fail(MM_EWORKSPACE, "workspace too small");
  k_raster_coords<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(a);
  int rc = check_launch("k_raster_coords");
  if (rc) return rc;
  k_raster_boxes<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(a);
  if ((rc = check_launch("k_raster_boxes"))) return rc;
  k_rasterize<<<(unsigned)cdiv(w * h, 256), 256, 0, st>>>(a.us, a.vs, a.box, n, w, h, pixels);
  return check_launch("k_rasterize");
}

int mmlttb_conv_mask(const uint8_t* a, const uint8_t* b, int64_t h, int64_t w, int kernel, uint8_t* mask, void* stream) {
  if (!a || !b || !mask || kernel < 1 || kernel % 2 == 0 || w * h < 1) return fail(MM_EINVAL, "bad arguments");
  k_conv_mask<<<(unsigned)cdiv(w * h, 256), 256, 0, (cudaStream_t)stream>>>(a, b, h, w, kernel, mask);
  return check_launch("k_conv_mask");
}

int mmlttb_pixel_metrics(const uint8_t* a, const uint8_t* b, const uint8_t* mask, int64_t h, int64_t w, int margin,
                         double* out4, void* workspace, int64_t workspace_bytes, void* stream) {
  if (!a || !b || !mask || !out4 || h < 8 || w < 8 || margin < 0 || margin > 255) return fail(MM_EINVAL, "bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  Carve cv{(char*)workspace, workspace_bytes};
  double* m5 = cv.take<double>(5 * w * h);
  const int64_t nb = cdiv(w * h, 256);
  double* part = cv.take<double>(2 * nb);
  if (!cv.ok) return fail(MM_EWORKSPACE, "workspace too small");
  k_ssim_rows<<<(unsigned)nb, 256, 0, st>>>(a, b, h, w, m5);
  int rc = check_launch("k_ssim_rows");
  if (rc) return rc;
  k_ssim_cols<<<(unsigned)nb, 256, 0, st>>>(a, b, mask, h, w, m5, part);
  if ((rc = check_launch("k_ssim_cols"))) return rc;
  k_metrics_final<<<1, 256, 0, st>>>(a, b, mask, w * h, margin, part, nb, out4);
  return check_launch("k_metrics_final");
}

int mmlttb_validate_batch(const void* x, int x_dtype, int64_t x_ld, const void* y, int y_dtype, int64_t y_ld,
                          int64_t B, int64_t N, int32_t* flags, void* stream) {
  if (!x || !y || !flags || N < 1 || B < 1 || !xdt_ok(x_dtype) || !ydt_ok(y_dtype) || x_ld < 0 || y_ld < N ||
      (x_ld != 0 && x_ld < N))
    return fail(MM_EINVAL, "bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(flags, 0, (size_t)B * sizeof(int32_t), st) != cudaSuccess) return fail(MM_ECUDA, "memset");
  const bool al = ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0) && (x_ld * esize(x_dtype)) % 16 == 0 &&
                  (y_ld * esize(y_dtype)) % 16 == 0;  // 16-byte loads of 4 elements on every row
  const int64_t per = cdiv(al ? cdiv(N, 4) : N, 256);
  const int64_t want = (int64_t)sm_count() * 8;  // ~8 CTAs per SM over the whole batch
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(per, cdiv(want, B)));
  const unsigned gy = (unsigned)std::min<int64_t>(B, 65535);
  const dim3 g(gx, gy);
#define MM_V(XT, YT)                                                                                                \
  do {                                                                                                              \
    if (al) k_validate<XT, YT><<<g, 256, 0, st>>>((const XT*)x, (const YT*)y, N, x_ld, y_ld, B, (int*)flags);        \
    else k_validate_scalar<XT, YT><<<g, 256, 0, st>>>((const XT*)x, (const YT*)y, N, x_ld, y_ld, B, (int*)flags);    \
  } while (0)
  if (y_dtype == MM_F32) {
    switch (x_dtype) {
      case MM_F32: MM_V(float, float); break;
      case MM_F64: MM_V(double, float); break;
      case MM_I64: MM_V(long long, float); break;
      default: MM_V(int, float); break;
    }
  } else {
    switch (x_dtype) {
      case MM_F32: MM_V(float, double); break;
      case MM_F64: MM_V(double, double); break;
      case MM_I64: MM_V(long long, double); break;
      default: MM_V(int, double); break;
    }
  }
#undef MM_V
  return check_launch("k_validate");
}

int mmlttb_validate(const void* x, int x_dtype, const void* y, int y_dtype, int64_t N, int32_t* flags, void* stream) {
  return mmlttb_validate_batch(x, x_dtype, 0, y, y_dtype, N, 1, N, flags, stream);
}

}  // extern "C"
