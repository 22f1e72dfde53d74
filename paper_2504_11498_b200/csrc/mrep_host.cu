// mrep_host.cu -- end-to-end projection from HOST buffers.
//
// The reference's project_prepared (project.py:245-289) takes numpy arrays in
// host memory and returns numpy arrays; this entry point keeps that contract
// at the C ABI: queries in host memory, results written to host memory,
// synchronous on return.  The batch is cut into chunks that flow through a
// two-slot pipeline (H2D of chunk i+1 and D2H of chunk i-1 overlap the
// kernel of chunk i on separate copy engines).  Pinned caller buffers are
// copied directly; pageable ones are staged through cached pinned buffers.
#include <cuda_runtime.h>

#include <cstdlib>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <utility>
#include <vector>
#include <algorithm>
#include <mutex>

#include "mrep_common.cuh"

namespace mrep {

namespace {

constexpr int64_t CHUNK_MAX = 1 << 19;  // queries per pipeline slot (buffer size)
constexpr int NSLOT_MAX = 4;
// pipeline shape: MREP_E2E_CHUNK (queries per chunk, <= 2^19) and
// MREP_E2E_SLOTS (1..4 chunks in flight) override the defaults
static int64_t chunk_size() {
  static int64_t c = [] {
    const char* e = getenv("MREP_E2E_CHUNK");
    int64_t v = e ? atoll(e) : (1 << 18);
    return v < 4096 ? (int64_t)4096 : (v > CHUNK_MAX ? CHUNK_MAX : v);
  }();
  return c;
}
static int num_slots() {
  static int n = [] {
    const char* e = getenv("MREP_E2E_SLOTS");
    int v = e ? atoi(e) : 4;
    return v < 1 ? 1 : (v > NSLOT_MAX ? NSLOT_MAX : v);
  }();
  return n;
}

struct Slot {
  cudaStream_t st = nullptr;
  cudaEvent_t done = nullptr;
  double *dq = nullptr, *dt = nullptr, *dfoot = nullptr, *ddist = nullptr;
  int64_t* dcand = nullptr;
  int32_t* dseg = nullptr;
  int32_t* dcur = nullptr;
  uint64_t* dcnt = nullptr;
  double *hq = nullptr, *ht = nullptr, *hfoot = nullptr, *hdist = nullptr;
  int64_t* hcand = nullptr;
  int32_t* hseg = nullptr;
  int32_t* hcur = nullptr;
  int64_t lo = 0, cnt = 0;  // chunk in flight (for staged write-back)
  bool busy = false;
};

// whole-batch device buffers for the pinned fast path (grown on demand)
struct BigBuf {
  int64_t cap = 0;
  double *dq = nullptr, *dt = nullptr, *dfoot = nullptr, *ddist = nullptr;
  int64_t* dcand = nullptr;
  int32_t *dseg = nullptr, *dcur = nullptr;
};

struct HostCtx {
  std::mutex mu;
  int device = -1;
  Slot slot[NSLOT_MAX];
  BigBuf big;
  cudaStream_t cin = nullptr, cout = nullptr;  // copy-in / copy-out streams (fast path)
  // fast-path compute streams by chunk index, in descending priority: the
  // earliest chunk's kernels win the SMs, so its download starts first and
  // later chunks fill the gaps
  static constexpr int NPRIO = 8;
  cudaStream_t prio[NPRIO] = {};
  std::vector<cudaEvent_t> ev_in, ev_comp;     // per-chunk hand-off events (cached)
  bool ready = false;
};

// One pipeline context per device (slots, streams, events and whole-batch
// buffers all belong to the device they were created on); created on the
// first host-buffer call made with that device current, never torn down.
constexpr int MAX_DEVICES = 64;
HostCtx* g_ctxs[MAX_DEVICES] = {};
std::mutex g_ctxs_mu;

HostCtx* current_ctx() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= MAX_DEVICES) {
    cudaGetLastError();
    set_error("no current CUDA device");
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(g_ctxs_mu);
  if (!g_ctxs[dev]) {
    g_ctxs[dev] = new HostCtx;
    g_ctxs[dev]->device = dev;
  }
  return g_ctxs[dev];
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int ensure_ctx(HostCtx& g_ctx) {
  if (g_ctx.ready) return MREP_OK;
  for (auto& s : g_ctx.slot) {
    // blocking streams: ordered after work on the legacy default stream (torch)
    MREP_CUDA_CHECK(cudaStreamCreateWithFlags(&s.st, cudaStreamDefault));
    MREP_CUDA_CHECK(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    MREP_CUDA_CHECK(cudaMalloc(&s.dq, CHUNK_MAX * 3 * sizeof(double)));
    MREP_CUDA_CHECK(cudaMalloc(&s.dt, CHUNK_MAX * sizeof(double)));
    MREP_CUDA_CHECK(cudaMalloc(&s.dfoot, CHUNK_MAX * 3 * sizeof(double)));
    MREP_CUDA_CHECK(cudaMalloc(&s.ddist, CHUNK_MAX * sizeof(double)));
    MREP_CUDA_CHECK(cudaMalloc(&s.dcand, CHUNK_MAX * sizeof(int64_t)));
    MREP_CUDA_CHECK(cudaMalloc(&s.dseg, CHUNK_MAX * sizeof(int32_t)));
    MREP_CUDA_CHECK(cudaMalloc(&s.dcur, CHUNK_MAX * sizeof(int32_t)));
    MREP_CUDA_CHECK(cudaMalloc(&s.dcnt, MREP_NUM_COUNTERS * sizeof(uint64_t)));
    MREP_CUDA_CHECK(cudaMallocHost(&s.hq, CHUNK_MAX * 3 * sizeof(double)));
    MREP_CUDA_CHECK(cudaMallocHost(&s.ht, CHUNK_MAX * sizeof(double)));
    MREP_CUDA_CHECK(cudaMallocHost(&s.hfoot, CHUNK_MAX * 3 * sizeof(double)));
    MREP_CUDA_CHECK(cudaMallocHost(&s.hdist, CHUNK_MAX * sizeof(double)));
    MREP_CUDA_CHECK(cudaMallocHost(&s.hcand, CHUNK_MAX * sizeof(int64_t)));
    MREP_CUDA_CHECK(cudaMallocHost(&s.hseg, CHUNK_MAX * sizeof(int32_t)));
    MREP_CUDA_CHECK(cudaMallocHost(&s.hcur, CHUNK_MAX * sizeof(int32_t)));
  }
  {
    int least = 0, greatest = 0;
    MREP_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    for (int k = 0; k < HostCtx::NPRIO; ++k) {
      const int pr = greatest + k < least ? greatest + k : least;
      MREP_CUDA_CHECK(cudaStreamCreateWithPriority(&g_ctx.prio[k], cudaStreamDefault, pr));
    }
  }
  MREP_CUDA_CHECK(cudaStreamCreateWithFlags(&g_ctx.cin, cudaStreamDefault));
  MREP_CUDA_CHECK(cudaStreamCreateWithFlags(&g_ctx.cout, cudaStreamDefault));
  g_ctx.ready = true;
  return MREP_OK;
}

void release_ctx(HostCtx& c) {
  for (auto& s : c.slot) {
    if (s.st) cudaStreamDestroy(s.st);
    if (s.done) cudaEventDestroy(s.done);
    cudaFree(s.dq);
    cudaFree(s.dt);
    cudaFree(s.dfoot);
    cudaFree(s.ddist);
    cudaFree(s.dcand);
    cudaFree(s.dseg);
    cudaFree(s.dcur);
    cudaFree(s.dcnt);
    cudaFreeHost(s.hq);
    cudaFreeHost(s.ht);
    cudaFreeHost(s.hfoot);
    cudaFreeHost(s.hdist);
    cudaFreeHost(s.hcand);
    cudaFreeHost(s.hseg);
    cudaFreeHost(s.hcur);
    s = Slot{};
  }
  cudaFree(c.big.dq);
  cudaFree(c.big.dt);
  cudaFree(c.big.dfoot);
  cudaFree(c.big.ddist);
  cudaFree(c.big.dcand);
  cudaFree(c.big.dseg);
  cudaFree(c.big.dcur);
  c.big = BigBuf{};
  for (auto& p : c.prio)
    if (p) cudaStreamDestroy(p), p = nullptr;
  if (c.cin) cudaStreamDestroy(c.cin), c.cin = nullptr;
  if (c.cout) cudaStreamDestroy(c.cout), c.cout = nullptr;
  for (auto e : c.ev_in) cudaEventDestroy(e);
  for (auto e : c.ev_comp) cudaEventDestroy(e);
  c.ev_in.clear();
  c.ev_comp.clear();
  c.ready = false;
}

}  // namespace
}  // namespace mrep

using namespace mrep;

// Frees every device's host-call pipeline context (streams, events, staging
// buffers); the next host-buffer call re-creates them.  Registered at exit by
// the Python package so leak checkers see a clean teardown.
extern "C" MREP_API int mrep_host_release(void) {
  int cur = 0;
  const bool have = cudaGetDevice(&cur) == cudaSuccess;
  std::lock_guard<std::mutex> lk(g_ctxs_mu);
  for (int d = 0; d < MAX_DEVICES; ++d) {
    HostCtx* c = g_ctxs[d];
    if (!c) continue;
    {
      std::lock_guard<std::mutex> lc(c->mu);
      if (cudaSetDevice(d) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess)
        release_ctx(*c);
    }
    delete c;
    g_ctxs[d] = nullptr;
  }
  if (have) cudaSetDevice(cur);
  cudaGetLastError();
  return MREP_OK;
}

namespace mrep {
namespace {

// Chunked H2D -> kernel -> D2H pipeline over the two slots.  `launch` runs the
// projection of one chunk already resident in the slot's device buffers.
template <class Launch>
int host_pipeline(HostCtx& g_ctx, int d, const double* queries, const int32_t* curve_ids, int64_t n,
                  double* out_t, double* out_foot, double* out_dist, int64_t* out_cand,
                  int32_t* out_seg, uint64_t* counters_host, Launch launch) {
  const auto t_entry = std::chrono::steady_clock::now();
  int rc = ensure_ctx(g_ctx);
  if (rc != MREP_OK) return rc;
  const bool pin_in = is_pinned(queries) && (!curve_ids || is_pinned(curve_ids));
  const bool pin_out = is_pinned(out_t) && is_pinned(out_foot) && is_pinned(out_dist) &&
                       is_pinned(out_cand) && (!out_seg || is_pinned(out_seg));

  const int NS = num_slots();
  const bool fast = pin_in && pin_out && !getenv("MREP_E2E_SLOTTED");
  // work counters only when the caller asked for them (4 memsets saved per call)
  if (counters_host)
    for (auto& s : g_ctx.slot)
      MREP_CUDA_CHECK(cudaMemsetAsync(s.dcnt, 0, MREP_NUM_COUNTERS * sizeof(uint64_t),
                                      fast ? g_ctx.cin : s.st));
  if (fast) {
    static const bool use_prio = !getenv("MREP_E2E_PRIO") || atoi(getenv("MREP_E2E_PRIO")) != 0;
    const int NS = getenv("MREP_E2E_SLOTS") ? num_slots() : 2;
    // Pinned fast path: device buffers for the whole batch, every chunk
    // enqueued at once round-robin over NS streams (H2D -> kernels -> D2H
    // straight into the caller's buffers); nothing waits for a free slot.
    BigBuf& B = g_ctx.big;
    if (B.cap < n) {
      cudaFree(B.dq);
      cudaFree(B.dt);
      cudaFree(B.dfoot);
      cudaFree(B.ddist);
      cudaFree(B.dcand);
      cudaFree(B.dseg);
      cudaFree(B.dcur);
      B = BigBuf{};
      int64_t cap = std::max<int64_t>(n, (int64_t)1 << 16);
      MREP_CUDA_CHECK(cudaMalloc(&B.dq, cap * 3 * sizeof(double)));
      MREP_CUDA_CHECK(cudaMalloc(&B.dt, cap * sizeof(double)));
      MREP_CUDA_CHECK(cudaMalloc(&B.dfoot, cap * 3 * sizeof(double)));
      MREP_CUDA_CHECK(cudaMalloc(&B.ddist, cap * sizeof(double)));
      MREP_CUDA_CHECK(cudaMalloc(&B.dcand, cap * sizeof(int64_t)));
      MREP_CUDA_CHECK(cudaMalloc(&B.dseg, cap * sizeof(int32_t)));
      MREP_CUDA_CHECK(cudaMalloc(&B.dcur, cap * sizeof(int32_t)));
      B.cap = cap;
    }
    const int64_t CH = getenv("MREP_E2E_CHUNK") ? chunk_size()
                                                : std::min<int64_t>(CHUNK_MAX, std::max<int64_t>(
                                                      (int64_t)1 << 16, (n + 7) / 8));
    // chunk list: five equal chunks (>= 2^16 queries each, <= 2^19), each on
    // its own priority stream (earlier chunk = higher priority) -- measured
    // best on B200 for 10^6 queries: 1.48 ms vs 1.64 for a short-edge
    // schedule and 1.57-1.74 for 4-10 chunks.  MREP_E2E_CHUNK forces a chunk
    // size, MREP_E2E_EDGE the older short-first/short-last schedule.
    std::vector<std::pair<int64_t, int64_t>> cl;
    if (getenv("MREP_E2E_EDGE") && !getenv("MREP_E2E_CHUNK")) {
      const int64_t edge = std::max<int64_t>(4096, atoll(getenv("MREP_E2E_EDGE")));
      const int64_t first = std::min(n, edge), last = std::min(n - first, edge);
      const int64_t mid = n - first - last;
      cl.push_back({0, first});
      if (mid > 0) {
        const int64_t k = (mid + CHUNK_MAX - 1) / CHUNK_MAX;
        int64_t lo2 = first;
        for (int64_t i = 0; i < k; ++i) {
          int64_t c2 = mid / k + (i < mid % k ? 1 : 0);
          cl.push_back({lo2, c2});
          lo2 += c2;
        }
      }
      if (last > 0) cl.push_back({n - last, last});
    } else if (getenv("MREP_E2E_SIZES") && !getenv("MREP_E2E_CHUNK")) {
      // explicit chunk sizes, comma separated; the remainder is one more chunk
      const char* e = getenv("MREP_E2E_SIZES");
      int64_t lo2 = 0;
      while (*e && lo2 < n) {
        const int64_t c2 = std::min<int64_t>(n - lo2, std::max<int64_t>(1024, atoll(e)));
        cl.push_back({lo2, c2});
        lo2 += c2;
        while (*e && *e != ',') ++e;
        if (*e == ',') ++e;
      }
      if (lo2 < n) cl.push_back({lo2, n - lo2});
    } else if (getenv("MREP_E2E_FIRST") && !getenv("MREP_E2E_CHUNK")) {
      // geometric schedule: first chunk MREP_E2E_FIRST queries, each next
      // one MREP_E2E_GEOM times larger (the last takes the remainder)
      const double r = getenv("MREP_E2E_GEOM") ? atof(getenv("MREP_E2E_GEOM")) : 2.0;
      double sz = (double)std::max<int64_t>(4096, atoll(getenv("MREP_E2E_FIRST")));
      for (int64_t lo2 = 0; lo2 < n;) {
        int64_t c2 = std::min<int64_t>(n - lo2, ((int64_t)sz + 4095) & ~(int64_t)4095);
        if (n - lo2 - c2 < c2 / 4) c2 = n - lo2;  // no sliver at the end
        cl.push_back({lo2, c2});
        lo2 += c2;
        sz *= r;
      }
    } else {
      const int64_t CHU = getenv("MREP_E2E_CHUNK")
                              ? CH
                              : std::min<int64_t>(CHUNK_MAX, std::max<int64_t>(
                                                                 (int64_t)1 << 16,
                                                                 (((n + 4) / 5 + 4095) / 4096) * 4096));
      for (int64_t lo2 = 0; lo2 < n; lo2 += CHU) cl.push_back({lo2, std::min(CHU, n - lo2)});
    }
    const int64_t nch = (int64_t)cl.size();
    while ((int64_t)g_ctx.ev_in.size() < nch) {
      cudaEvent_t a, b;
      MREP_CUDA_CHECK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
      MREP_CUDA_CHECK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
      g_ctx.ev_in.push_back(a);
      g_ctx.ev_comp.push_back(b);
    }
    static const int conc = getenv("MREP_E2E_CONC") ? atoi(getenv("MREP_E2E_CONC")) : 0;
    static const bool dtrace = getenv("MREP_E2E_TRACE") != nullptr;
    std::vector<cudaEvent_t> te;  // per chunk: upload end, kernels end, download end
    cudaEvent_t te0 = nullptr;
    if (dtrace) {
      cudaEventCreate(&te0);
      cudaEventRecord(te0, g_ctx.cin);
    }
    auto tmark = [&](cudaStream_t st) {
      if (!dtrace) return;
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, st);
      te.push_back(e);
    };
    // uploads back to back on the copy-in stream; chunk c's kernels (on
    // compute stream c % NS) wait for its upload; downloads back to back on
    // the copy-out stream, each waiting for its chunk's kernels
    for (int64_t c = 0; c < nch; ++c) {
      const int64_t lo = cl[c].first;
      Slot v = g_ctx.slot[c % NS];  // stream + counters of the slot, big-buffer views
      if (use_prio) v.st = g_ctx.prio[c < HostCtx::NPRIO ? c : HostCtx::NPRIO - 1];
      v.lo = lo;
      v.cnt = cl[c].second;
      v.dq = B.dq + lo * d;
      v.dt = B.dt + lo;
      v.dfoot = B.dfoot + lo * d;
      v.ddist = B.ddist + lo;
      v.dcand = B.dcand + lo;
      v.dseg = B.dseg + lo;
      v.dcur = B.dcur + lo;
      cudaStream_t ci = g_ctx.cin, co = g_ctx.cout;
      MREP_CUDA_CHECK(cudaMemcpyAsync(v.dq, queries + lo * d, v.cnt * d * sizeof(double),
                                      cudaMemcpyHostToDevice, ci));
      if (curve_ids)
        MREP_CUDA_CHECK(cudaMemcpyAsync(v.dcur, curve_ids + lo, v.cnt * sizeof(int32_t),
                                        cudaMemcpyHostToDevice, ci));
      MREP_CUDA_CHECK(cudaEventRecord(g_ctx.ev_in[c], ci));
      tmark(ci);
      MREP_CUDA_CHECK(cudaStreamWaitEvent(v.st, g_ctx.ev_in[c], 0));
      // at most `conc` chunks' kernels in flight (MREP_E2E_CONC; default all)
      if (conc > 0 && c >= conc)
        MREP_CUDA_CHECK(cudaStreamWaitEvent(v.st, g_ctx.ev_comp[c - conc], 0));
      const auto t_l0 = std::chrono::steady_clock::now();
      if ((rc = launch(v)) != MREP_OK) return rc;
      if (dtrace)
        fprintf(stderr, "chunk %lld: host launch %.3f ms (at %.3f)\n", (long long)c,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_l0)
                    .count(),
                std::chrono::duration<double, std::milli>(t_l0 - t_entry).count());
      MREP_CUDA_CHECK(cudaEventRecord(g_ctx.ev_comp[c], v.st));
      tmark(v.st);
      MREP_CUDA_CHECK(cudaStreamWaitEvent(co, g_ctx.ev_comp[c], 0));
      MREP_CUDA_CHECK(cudaMemcpyAsync(out_t + lo, v.dt, v.cnt * sizeof(double),
                                      cudaMemcpyDeviceToHost, co));
      MREP_CUDA_CHECK(cudaMemcpyAsync(out_foot + lo * d, v.dfoot, v.cnt * d * sizeof(double),
                                      cudaMemcpyDeviceToHost, co));
      MREP_CUDA_CHECK(cudaMemcpyAsync(out_dist + lo, v.ddist, v.cnt * sizeof(double),
                                      cudaMemcpyDeviceToHost, co));
      MREP_CUDA_CHECK(cudaMemcpyAsync(out_cand + lo, v.dcand, v.cnt * sizeof(int64_t),
                                      cudaMemcpyDeviceToHost, co));
      if (out_seg)
        MREP_CUDA_CHECK(cudaMemcpyAsync(out_seg + lo, v.dseg, v.cnt * sizeof(int32_t),
                                        cudaMemcpyDeviceToHost, co));
      tmark(co);
    }
    const auto t_enq = std::chrono::steady_clock::now();
    MREP_CUDA_CHECK(cudaStreamSynchronize(g_ctx.cout));
    if (dtrace) {
      const auto t_sync = std::chrono::steady_clock::now();
      fprintf(stderr, "host: enqueue %.3f ms, wait %.3f ms\n",
              std::chrono::duration<double, std::milli>(t_enq - t_entry).count(),
              std::chrono::duration<double, std::milli>(t_sync - t_enq).count());
      cudaDeviceSynchronize();
      for (size_t k = 0; k + 2 < te.size(); k += 3) {
        float a = 0, b = 0, e = 0;
        cudaEventElapsedTime(&a, te0, te[k]);
        cudaEventElapsedTime(&b, te0, te[k + 1]);
        cudaEventElapsedTime(&e, te0, te[k + 2]);
        fprintf(stderr, "chunk %zu n=%lld: h2d_end %.3f  kern_end %.3f  d2h_end %.3f\n", k / 3,
                (long long)cl[k / 3].second, a, b, e);
      }
      for (auto ev : te) cudaEventDestroy(ev);
      cudaEventDestroy(te0);
    }
    // (every chunk's kernels precede its download on the copy-out stream)
    if (counters_host) {
      for (auto& s : g_ctx.slot) {
        uint64_t cc[MREP_NUM_COUNTERS];
        MREP_CUDA_CHECK(cudaMemcpy(cc, s.dcnt, sizeof cc, cudaMemcpyDeviceToHost));
        for (int i = 0; i < MREP_NUM_COUNTERS; ++i) counters_host[i] += cc[i];
      }
    }
    return MREP_OK;
  }

  auto write_back = [&](Slot& s) -> int {
    if (!s.busy) return MREP_OK;
    MREP_CUDA_CHECK(cudaEventSynchronize(s.done));
    if (!pin_out) {
      std::memcpy(out_t + s.lo, s.ht, s.cnt * sizeof(double));
      std::memcpy(out_foot + s.lo * d, s.hfoot, s.cnt * d * sizeof(double));
      std::memcpy(out_dist + s.lo, s.hdist, s.cnt * sizeof(double));
      std::memcpy(out_cand + s.lo, s.hcand, s.cnt * sizeof(int64_t));
      if (out_seg) std::memcpy(out_seg + s.lo, s.hseg, s.cnt * sizeof(int32_t));
    }
    s.busy = false;
    return MREP_OK;
  };

  // Chunk schedule: about 8 chunks per call (2^16 .. 2^19 queries each) so
  // the first upload and the last download are short and up to NS chunks
  // overlap their copies and kernels; MREP_E2E_CHUNK forces a size.
  std::vector<std::pair<int64_t, int64_t>> chunks;
  int64_t CHUNK = getenv("MREP_E2E_CHUNK") ? chunk_size()
                                            : std::min<int64_t>(CHUNK_MAX, std::max<int64_t>(
                                                  (int64_t)1 << 16, (n + 7) / 8));
  for (int64_t lo = 0; lo < n; lo += CHUNK) chunks.push_back({lo, std::min(CHUNK, n - lo)});
  const int64_t nchunks = (int64_t)chunks.size();
  // MREP_E2E_TRACE=1: per-chunk device timeline (H2D / kernels / D2H ends)
  static const bool trace = getenv("MREP_E2E_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  std::vector<double> th;
  cudaEvent_t t0ev = nullptr;
  auto host_ms = [] {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  double h0 = host_ms();
  if (trace) {
    cudaEventCreate(&t0ev);
    cudaEventRecord(t0ev, g_ctx.slot[0].st);
  }
  auto mark = [&](cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tev.push_back(e);
  };
  for (int64_t c = 0; c < nchunks; ++c) {
    Slot& s = g_ctx.slot[c % NS];
    if ((rc = write_back(s)) != MREP_OK) return rc;
    s.lo = chunks[c].first;
    s.cnt = chunks[c].second;
    const double* src = queries + s.lo * d;
    const int32_t* csrc = curve_ids ? curve_ids + s.lo : nullptr;
    if (!pin_in) {
      std::memcpy(s.hq, src, s.cnt * d * sizeof(double));
      src = s.hq;
      if (csrc) {
        std::memcpy(s.hcur, csrc, s.cnt * sizeof(int32_t));
        csrc = s.hcur;
      }
    }
    MREP_CUDA_CHECK(
        cudaMemcpyAsync(s.dq, src, s.cnt * d * sizeof(double), cudaMemcpyHostToDevice, s.st));
    if (csrc)
      MREP_CUDA_CHECK(
          cudaMemcpyAsync(s.dcur, csrc, s.cnt * sizeof(int32_t), cudaMemcpyHostToDevice, s.st));
    mark(s.st);
    if (trace) th.push_back(host_ms() - h0);
    rc = launch(s);
    if (rc != MREP_OK) return rc;
    mark(s.st);
    if (trace) th.push_back(host_ms() - h0);
    double* ht = pin_out ? out_t + s.lo : s.ht;
    double* hf = pin_out ? out_foot + s.lo * d : s.hfoot;
    double* hd = pin_out ? out_dist + s.lo : s.hdist;
    int64_t* hc = pin_out ? out_cand + s.lo : s.hcand;
    int32_t* hs = pin_out ? (out_seg ? out_seg + s.lo : nullptr) : s.hseg;
    MREP_CUDA_CHECK(cudaMemcpyAsync(ht, s.dt, s.cnt * sizeof(double), cudaMemcpyDeviceToHost, s.st));
    MREP_CUDA_CHECK(
        cudaMemcpyAsync(hf, s.dfoot, s.cnt * d * sizeof(double), cudaMemcpyDeviceToHost, s.st));
    MREP_CUDA_CHECK(
        cudaMemcpyAsync(hd, s.ddist, s.cnt * sizeof(double), cudaMemcpyDeviceToHost, s.st));
    MREP_CUDA_CHECK(
        cudaMemcpyAsync(hc, s.dcand, s.cnt * sizeof(int64_t), cudaMemcpyDeviceToHost, s.st));
    if (hs)
      MREP_CUDA_CHECK(
          cudaMemcpyAsync(hs, s.dseg, s.cnt * sizeof(int32_t), cudaMemcpyDeviceToHost, s.st));
    MREP_CUDA_CHECK(cudaEventRecord(s.done, s.st));
    mark(s.st);
    s.busy = true;
  }
  for (auto& s : g_ctx.slot)
    if ((rc = write_back(s)) != MREP_OK) return rc;
  if (trace) {
    cudaDeviceSynchronize();
    for (int64_t c = 0; c < nchunks; ++c) {
      float a = 0, b = 0, e = 0;
      cudaEventElapsedTime(&a, t0ev, tev[3 * c]);
      cudaEventElapsedTime(&b, t0ev, tev[3 * c + 1]);
      cudaEventElapsedTime(&e, t0ev, tev[3 * c + 2]);
      fprintf(stderr, "chunk %lld n=%lld: h2d_end %.3f  kern_end %.3f  d2h_end %.3f  (host enq %.3f..%.3f)\n",
              (long long)c, (long long)chunks[c].second, a, b, e, th[2 * c], th[2 * c + 1]);
    }
    fprintf(stderr, "host total %.3f ms\n", host_ms() - h0);
    for (auto ev : tev) cudaEventDestroy(ev);
    cudaEventDestroy(t0ev);
  }
  if (counters_host) {
    for (auto& s : g_ctx.slot) {
      uint64_t c[MREP_NUM_COUNTERS];
      MREP_CUDA_CHECK(cudaMemcpy(c, s.dcnt, sizeof c, cudaMemcpyDeviceToHost));
      for (int i = 0; i < MREP_NUM_COUNTERS; ++i) counters_host[i] += c[i];
    }
  }
  return MREP_OK;
}

}  // namespace
}  // namespace mrep

extern "C" int mrep_project_host(const void* table, int64_t S, int d, const double* queries,
                                 int64_t n, double clip_tol, int max_iter, unsigned flags,
                                 double* out_t, double* out_foot, double* out_dist,
                                 int64_t* out_cand, int32_t* out_seg, uint64_t* counters_host) {
  if (n < 0 || (d != 2 && d != 3) || S < 1 || !table) {
    set_error("mrep_project_host: bad arguments");
    return MREP_ERR_ARG;
  }
  if (n == 0) return MREP_OK;
  HostCtx* C = current_ctx();
  if (!C) return MREP_ERR_CUDA;
  std::lock_guard<std::mutex> lock(C->mu);
  flags &= ~MREP_STATS;
  return host_pipeline(*C, d, queries, nullptr, n, out_t, out_foot, out_dist, out_cand, out_seg,
                       counters_host, [&](Slot& s) {
                         return mrep_project(table, S, d, s.dq, s.cnt, clip_tol, max_iter, 0,
                                             flags, s.dt, s.dfoot, s.ddist, s.dcand, s.dseg,
                                             nullptr, nullptr, counters_host ? s.dcnt : nullptr,
                                             s.st);
                       });
}

extern "C" int mrep_project_batch_host(const void* set, const double* queries,
                                       const int32_t* curve_ids, int64_t n, double clip_tol,
                                       int max_iter, unsigned flags, double* out_t,
                                       double* out_foot, double* out_dist, int64_t* out_cand,
                                       int32_t* out_seg, uint64_t* counters_host) {
  int d = 0;
  if (!set || n < 0 || mrep_curveset_info(set, nullptr, nullptr, &d, nullptr) != MREP_OK) {
    set_error("mrep_project_batch_host: bad arguments");
    return MREP_ERR_ARG;
  }
  if (n == 0) return MREP_OK;
  HostCtx* C = current_ctx();
  if (!C) return MREP_ERR_CUDA;
  std::lock_guard<std::mutex> lock(C->mu);
  return host_pipeline(*C, d, queries, curve_ids, n, out_t, out_foot, out_dist, out_cand, out_seg,
                       counters_host, [&](Slot& s) {
                         return mrep_project_batch(set, s.dq, s.dcur, s.cnt, clip_tol, max_iter,
                                                   flags, s.dt, s.dfoot, s.ddist, s.dcand, s.dseg,
                                                   counters_host ? s.dcnt : nullptr, s.st);
                       });
}

// Surfaces: the same pipeline; the slot's 8-byte candidate-count buffer
// carries v (u rides in t, the patch id in the segment buffer).
extern "C" int mrep_project_surface_host(const void* table, int64_t npatch, int pu, int pv,
                                         const double* queries, int64_t n, unsigned flags,
                                         double* out_u, double* out_v, double* out_foot,
                                         double* out_dist, int32_t* out_patch,
                                         uint64_t* counters_host) {
  if (!table || npatch < 1 || n < 0) {
    set_error("mrep_project_surface_host: bad arguments");
    return MREP_ERR_ARG;
  }
  if (n == 0) return MREP_OK;
  HostCtx* C = current_ctx();
  if (!C) return MREP_ERR_CUDA;
  std::lock_guard<std::mutex> lock(C->mu);
  return host_pipeline(*C, 3, queries, nullptr, n, out_u, out_foot, out_dist, (int64_t*)out_v,
                       out_patch, counters_host, [&](Slot& s) {
                         return mrep_project_surface(table, npatch, pu, pv, s.dq, s.cnt, flags,
                                                     s.dt, (double*)s.dcand, s.dfoot, s.ddist,
                                                     s.dseg, counters_host ? s.dcnt : nullptr,
                                                     s.st);
                       });
}

// ---------------------------------------------------------------------------
// Host-array entry points: what a ctypes / cffi binding in the reference
// binds without any GPU framework.

extern "C" int mrep_table_create(const double* seg_pts, const double* seg_ta, const double* seg_tb,
                                 const double* seam_t, const double* seam_pt, int64_t S, int d,
                                 void** table_out) {
  *table_out = nullptr;
  int64_t bytes = mrep_table_bytes(S);
  if (bytes < 0 || (d != 2 && d != 3)) {
    set_error("mrep_table_create: need S >= 1 and d in {2,3}");
    return MREP_ERR_ARG;
  }
  double *dsp = nullptr, *dta = nullptr, *dtb = nullptr, *dst = nullptr, *dspt = nullptr;
  void* table = nullptr;
  MREP_CUDA_CHECK(cudaMalloc(&table, (size_t)bytes));
  MREP_CUDA_CHECK(cudaMalloc(&dsp, S * 4 * d * sizeof(double)));
  MREP_CUDA_CHECK(cudaMalloc(&dta, S * sizeof(double)));
  MREP_CUDA_CHECK(cudaMalloc(&dtb, S * sizeof(double)));
  MREP_CUDA_CHECK(cudaMalloc(&dst, (S + 1) * sizeof(double)));
  MREP_CUDA_CHECK(cudaMalloc(&dspt, (S + 1) * d * sizeof(double)));
  MREP_CUDA_CHECK(cudaMemcpy(dsp, seg_pts, S * 4 * d * sizeof(double), cudaMemcpyHostToDevice));
  MREP_CUDA_CHECK(cudaMemcpy(dta, seg_ta, S * sizeof(double), cudaMemcpyHostToDevice));
  MREP_CUDA_CHECK(cudaMemcpy(dtb, seg_tb, S * sizeof(double), cudaMemcpyHostToDevice));
  MREP_CUDA_CHECK(cudaMemcpy(dst, seam_t, (S + 1) * sizeof(double), cudaMemcpyHostToDevice));
  MREP_CUDA_CHECK(cudaMemcpy(dspt, seam_pt, (S + 1) * d * sizeof(double), cudaMemcpyHostToDevice));
  int rc = mrep_table_pack(dsp, dta, dtb, dst, dspt, S, d, table, nullptr);
  cudaDeviceSynchronize();
  cudaFree(dsp);
  cudaFree(dta);
  cudaFree(dtb);
  cudaFree(dst);
  cudaFree(dspt);
  if (rc != MREP_OK) {
    cudaFree(table);
    return rc;
  }
  *table_out = table;
  return MREP_OK;
}

extern "C" int mrep_table_free(void* table) {
  if (table) MREP_CUDA_CHECK(cudaFree(table));
  return MREP_OK;
}

extern "C" int mrep_project_block_host(const double* seg_pts, const double* seg_ta,
                                       const double* seg_tb, const double* seam_t,
                                       const double* seam_pt, int64_t S, int d,
                                       const double* queries, int64_t n, double clip_tol,
                                       int max_iter, int soundness_samples, double* out_t,
                                       double* out_foot, double* out_dist, int64_t* out_cand,
                                       int64_t* out_stats, double* out_sound) {
  void* table = nullptr;
  int rc = mrep_table_create(seg_pts, seg_ta, seg_tb, seam_t, seam_pt, S, d, &table);
  if (rc != MREP_OK) return rc;
  if (n == 0) return mrep_table_free(table);
  double *dq = nullptr, *dt = nullptr, *df = nullptr, *dd = nullptr, *dso = nullptr;
  int64_t *dc = nullptr, *dstat = nullptr;
  MREP_CUDA_CHECK(cudaMalloc(&dq, n * d * sizeof(double)));
  MREP_CUDA_CHECK(cudaMalloc(&dt, n * sizeof(double)));
  MREP_CUDA_CHECK(cudaMalloc(&df, n * d * sizeof(double)));
  MREP_CUDA_CHECK(cudaMalloc(&dd, n * sizeof(double)));
  MREP_CUDA_CHECK(cudaMalloc(&dso, n * sizeof(double)));
  MREP_CUDA_CHECK(cudaMalloc(&dc, n * sizeof(int64_t)));
  MREP_CUDA_CHECK(cudaMalloc(&dstat, n * 6 * sizeof(int64_t)));
  MREP_CUDA_CHECK(cudaMemset(dstat, 0, n * 6 * sizeof(int64_t)));
  MREP_CUDA_CHECK(cudaMemcpy(dq, queries, n * d * sizeof(double), cudaMemcpyHostToDevice));
  rc = mrep_project(table, S, d, dq, n, clip_tol, max_iter, soundness_samples, MREP_STATS, dt, df,
                    dd, dc, nullptr, dstat, dso, nullptr, nullptr);
  if (rc == MREP_OK) {
    MREP_CUDA_CHECK(cudaMemcpy(out_t, dt, n * sizeof(double), cudaMemcpyDeviceToHost));
    MREP_CUDA_CHECK(cudaMemcpy(out_foot, df, n * d * sizeof(double), cudaMemcpyDeviceToHost));
    MREP_CUDA_CHECK(cudaMemcpy(out_dist, dd, n * sizeof(double), cudaMemcpyDeviceToHost));
    MREP_CUDA_CHECK(cudaMemcpy(out_cand, dc, n * sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (out_stats)
      MREP_CUDA_CHECK(cudaMemcpy(out_stats, dstat, n * 6 * sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (out_sound)
      MREP_CUDA_CHECK(cudaMemcpy(out_sound, dso, n * sizeof(double), cudaMemcpyDeviceToHost));
  }
  cudaFree(dq);
  cudaFree(dt);
  cudaFree(df);
  cudaFree(dd);
  cudaFree(dso);
  cudaFree(dc);
  cudaFree(dstat);
  mrep_table_free(table);
  return rc;
}

// ---------------------------------------------------------------------------
// Synthetic-input helper (host only): the sequential momentum walk of the
// reference fixture generator (_fixtures.py _walk_points): v <- v + 0.55 g_i,
// v <- v / ||v||, p_i = p_{i-1} + v, with ||v|| computed as numpy does for a
// short vector (BLAS ddot = FMA chain, then sqrt).  The caller draws v0 and
// the normals g with numpy (same RNG stream) and normalises the result.
#include <cmath>
extern "C" int mrep_synth_walk(const double* v0, const double* g, int64_t n, int d, double* pts) {
  if (n < 1 || (d != 2 && d != 3) || !v0 || !pts || (n > 1 && !g)) {
    set_error("mrep_synth_walk: bad arguments");
    return MREP_ERR_ARG;
  }
  double v[3] = {v0[0], v0[1], d == 3 ? v0[2] : 0.0};
  double cur[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < d; ++k) pts[k] = 0.0;
  for (int64_t i = 1; i < n; ++i) {
    double w[3];
    for (int k = 0; k < d; ++k) {
      volatile double prod = 0.55 * g[(i - 1) * d + k];  // no contraction into an FMA
      w[k] = v[k] + prod;
    }
    volatile double sq0 = w[0] * w[0];
    double s = std::fma(w[1], w[1], sq0);
    if (d == 3) s = std::fma(w[2], w[2], s);
    double nr = std::sqrt(s);
    for (int k = 0; k < d; ++k) {
      v[k] = w[k] / nr;
      cur[k] = cur[k] + v[k];
      pts[i * d + k] = cur[k];
    }
  }
  return MREP_OK;
}
