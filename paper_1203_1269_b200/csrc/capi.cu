// capi.cu -- host runtime behind include/gpemu_b200.h.
//
// Owns device memory, the jitter-ladder batch executor, the batched GA driver
// and the C-ABI. Mirrors the reference's host logic (paths relative to
// /root/reference/proj/include/gpemu/):
//   Hyperparameters::validate   core.hpp:76-83
//   FitConfig::bounds_for       core.hpp:114-123
//   Backend::factorize_into     backend.hpp:102-120 (ladder; one factorization in the Ledger)
//   ProfileEvaluator            likelihood.hpp:74-158
//   ga_minimize                 optimizer.hpp:93-187 (candidate sequence reproduced exactly;
//                               each generation's population is ONE device batch)
//   fit_gp_detailed             likelihood.hpp:243-303 (stash: strict <, earliest slot wins)
//   model_at_theta / predict    likelihood.hpp:216-237, predictor.hpp:20-50
// There is no CPU fallback: every numeric result comes from the sm_100a kernels.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <memory>
#include <map>
#include <numeric>
#include <queue>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gpemu_b200.h"
#include "kernels.h"
#include "layout.cuh"

using namespace gpemu_dev;

namespace {

thread_local std::string g_last_error;

int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

struct CudaError {
  std::string msg;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError{std::string(what) + ": " + cudaGetErrorString(e)};
}

// NVTX ranges (header-only NVTX3: a no-op unless a tool such as nsys / ncu is attached): one per
// K1-K4 phase launch, per GA generation, per refine polish and per prediction call.
inline void nvtx_push(const char* name) { nvtxRangePushA(name); }
inline void nvtx_pop() { nvtxRangePop(); }
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtx_push(name); }
  ~NvtxRange() { nvtx_pop(); }
};

// Device -> host copy ordered on `s` (the engine's streams are non-blocking, so a legacy
// cudaMemcpy is not ordered after their work).
void d2h_sync(void* dst, const void* src, size_t bytes, cudaStream_t s, const char* what) {
  ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s), what);
  ck(cudaStreamSynchronize(s), what);
}

constexpr double kLadder[6] = {0.0, 1e-8, 1e-7, 1e-6, 1e-5, 1e-4};  // backend.hpp:77

// Plans whose whole batch is a few tile tasks per SM (latency-bound passes: n <= 384 at 100
// candidates) get a second set of slots for the speculative first ladder rung (run_batch).
constexpr size_t kSpecTaskCap = 600;
bool spec_slots_for(int NT, size_t max_batch) {
  return (size_t)NT * (NT + 1) / 2 * max_batch <= kSpecTaskCap;
}

// Device memory: one stream-ordered pool per device, owned by the library, that keeps freed
// blocks mapped (release threshold = max). A plan holds gigabytes (C3: 6.9 GB of factors and
// table); cudaMalloc / cudaFree of those per plan cost 1-700 ms each on the box, more than the
// GA fit itself at the paper's sizes, and the paper protocol builds a plan per replication.
// With the pool a new plan reuses the previous plan's pages. The pool is trimmed when an
// allocation would not fit otherwise and when a context is destroyed.
struct DevPool {
  cudaMemPool_t pool = nullptr;
  cudaStream_t stream = nullptr;  // allocation stream, synchronised after every allocation
};

DevPool& dev_pool(int dev) {
  static std::mutex mu;
  static DevPool pools[64];
  if (dev < 0 || dev >= 64) throw CudaError{"device index out of range"};
  std::lock_guard<std::mutex> lock(mu);
  DevPool& P = pools[dev];
  if (!P.pool) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    ck(cudaMemPoolCreate(&P.pool, &props), "cudaMemPoolCreate");
    uint64_t keep = UINT64_MAX;
    ck(cudaMemPoolSetAttribute(P.pool, cudaMemPoolAttrReleaseThreshold, &keep), "cudaMemPoolSetAttribute");
    int cur = 0;
    ck(cudaGetDevice(&cur), "cudaGetDevice");
    ck(cudaSetDevice(dev), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&P.stream, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaSetDevice(cur), "cudaSetDevice");
  }
  return P;
}

// Bytes the pool holds mapped but not handed out (free for the next plan).
size_t pool_idle_bytes(int dev) {
  DevPool& P = dev_pool(dev);
  uint64_t reserved = 0, used = 0;
  ck(cudaMemPoolGetAttribute(P.pool, cudaMemPoolAttrReservedMemCurrent, &reserved), "cudaMemPoolGetAttribute");
  ck(cudaMemPoolGetAttribute(P.pool, cudaMemPoolAttrUsedMemCurrent, &used), "cudaMemPoolGetAttribute");
  return reserved > used ? static_cast<size_t>(reserved - used) : 0;
}

void pool_trim(int dev) {
  DevPool& P = dev_pool(dev);
  ck(cudaStreamSynchronize(P.stream), "cudaStreamSynchronize");
  ck(cudaMemPoolTrimTo(P.pool, 0), "cudaMemPoolTrimTo");
}

// A pool allocation. Frees are stream-ordered on the owner's stream (`sp`: the owning
// context's current stream, bound by own()): every kernel that used the block was issued on
// that stream before the free, and the pool hands a freed block to the next allocation only
// after that stream's work reaches the free (the pool's default event-dependency reuse rules),
// so no device-wide synchronisation is needed. An unbound buffer (no owner) falls back to
// synchronising its device before the free.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t count = 0;
  int dev = -1;
  const cudaStream_t* sp = nullptr;
  void alloc(size_t c) {
    free();
    if (c == 0) c = 1;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    DevPool& P = dev_pool(dev);
    void* q = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync(&q, c * sizeof(T), P.pool, P.stream);
    if (e == cudaErrorMemoryAllocation) {  // idle pool pages are not enough: release them, retry
      (void)cudaGetLastError();
      ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
      ck(cudaMemPoolTrimTo(P.pool, 0), "cudaMemPoolTrimTo");
      e = cudaMallocFromPoolAsync(&q, c * sizeof(T), P.pool, P.stream);
    }
    ck(e, "cudaMallocFromPoolAsync");
    ck(cudaStreamSynchronize(P.stream), "cudaStreamSynchronize");  // usable from any stream
    p = static_cast<T*>(q);
    count = c;
  }
  void reserve(size_t c) {  // grow-only: keeps the allocation when it is large enough
    if (count < c) alloc(c);
  }
  void free() {
    if (p) {
      int cur = -1;
      cudaGetDevice(&cur);
      if (cur != dev) cudaSetDevice(dev);
      if (sp) {
        cudaFreeAsync(p, *sp);
      } else {
        cudaDeviceSynchronize();
        cudaFreeAsync(p, dev_pool(dev).stream);
      }
      if (cur != dev && cur >= 0) cudaSetDevice(cur);
    }
    p = nullptr;
    count = 0;
  }
  ~DevBuf() { free(); }
};

// Page-locked host staging (per-pass slot lists, jitters, statuses, records): copies from and
// to it are truly asynchronous and skip the driver's pageable bounce buffer, which matters for
// the latency-bound small designs (a C1 batch is ~0.35 ms).
template <typename T>
struct PinnedVec {
  T* p = nullptr;
  size_t n = 0;
  PinnedVec() = default;
  PinnedVec(const PinnedVec&) = delete;
  PinnedVec& operator=(const PinnedVec&) = delete;
  ~PinnedVec() {
    if (p) cudaFreeHost(p);
  }
  void assign(size_t count, T v) {
    if (count > n) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      n = 0;
      void* q = nullptr;
      ck(cudaMallocHost(&q, (count ? count : 1) * sizeof(T)), "cudaMallocHost");
      p = static_cast<T*>(q);
      n = count;
    }
    std::fill(p, p + count, v);
  }
  T* data() { return p; }
  const T* data() const { return p; }
  T* begin() { return p; }
  T& operator[](size_t i) { return p[i]; }
  const T& operator[](size_t i) const { return p[i]; }
};

// Binds buffers to the stream their users launch on (see DevBuf).
template <typename... B>
void own(const cudaStream_t* s, B&... bufs) {
  ((bufs.sp = s), ...);
}

// splitmix64 seed derivation (rng.hpp:12-25).
uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
uint64_t derive_seed(uint64_t base) { return mix64(base); }
uint64_t derive_seed(uint64_t base, uint64_t a) { return derive_seed(mix64(base ^ mix64(a))); }
uint64_t derive_seed(uint64_t base, uint64_t a, uint64_t b) {
  return derive_seed(mix64(base ^ mix64(a)), b);
}

// Rng mappings of rng.hpp:29-58 over std::mt19937_64.
struct Rng {
  std::mt19937_64 eng;
  explicit Rng(uint64_t seed) : eng(seed) {}
  double uniform01() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
  double uniform01_open_low() { return static_cast<double>((eng() >> 11) + 1) * 0x1.0p-53; }
  uint64_t below(uint64_t n) {
    return static_cast<uint64_t>((static_cast<__uint128_t>(eng()) * n) >> 64);
  }
  double normal() {
    const double u1 = uniform01_open_low();
    const double u2 = uniform01();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2);
  }
};

int validate_params(const double* theta, size_t d, double p, double nugget) {
  for (size_t k = 0; k < d; ++k) {
    if (!(theta[k] >= 0.0) || !std::isfinite(theta[k]))
      return set_error(GPEMU_VALIDATION, "Hyperparameters: theta entries must be finite and nonnegative");
  }
  if (!(p > 0.0) || !(p <= 2.0)) return set_error(GPEMU_VALIDATION, "Hyperparameters: p must be in (0, 2]");
  if (!(nugget >= 0.0) || !std::isfinite(nugget))
    return set_error(GPEMU_VALIDATION, "Hyperparameters: nugget must be finite and nonnegative");
  return GPEMU_OK;
}

int validate_unit_cube(const double* X, size_t rows, size_t d, const char* who) {
  for (size_t i = 0; i < rows * d; ++i) {
    const double x = X[i];
    if (!std::isfinite(x)) return set_error(GPEMU_VALIDATION, "%s: non-finite input coordinate", who);
    if (x < -1e-12 || x > 1.0 + 1e-12)
      return set_error(GPEMU_VALIDATION, "%s: coordinate %g outside the unit cube at row %zu", who, x, i / d);
  }
  return GPEMU_OK;
}

}  // namespace

struct gpemu_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  int engine = GPEMU_ENGINE_DAG;
  int num_sms = 148;
  uint64_t launches = 0;
  // Backend-level single-matrix calls (try_cholesky / factorize): a one-slot plan and an n x n
  // staging matrix reused across calls (the reference's fit through the plugin makes
  // thousands of them), rebuilt only when n changes.
  gpemu_plan* scratch = nullptr;
  DevBuf<double> scratch_a, scratch_l;
  // Plans and models free their device buffers on this context's stream, so a context
  // destroyed while some are alive is finalised when the last of them goes.
  std::mutex mu;
  int children = 0;
  bool closing = false;
};

struct gpemu_plan {
  gpemu_ctx* ctx = nullptr;
  int n = 0, d = 0, NT = 0, Npad = 0;
  double p = 1.95, nugget = 0.0;
  size_t max_batch = 0, nslots = 0;  // nslots = max_batch + 1 (stash slot)
  size_t slot_stride = 0;
  int epoch = 0;
  DevBuf<double> X, y, table, factors, borders, theta, jitter, out;
  DevBuf<int> status, slots, flags, counter, error;
  int precision = GPEMU_PRECISION_DOUBLE;
  DevBuf<float> factors_f, borders_f;  // single precision storage (table: `table`, double)
  DevBuf<unsigned long long> dag_prof;  // optional DAG phase counters
  // ticket orders of large launches by batch size (see ticket_order): a GA generation and its
  // jitter-ladder relaunches alternate between a few sizes
  std::map<int, std::unique_ptr<DevBuf<int>>> orders;
  uint64_t data_hash = 0;  // FNV-1a of (n, d, X, y): plans of one dataset on several devices
  DevBuf<int> trsv_flags, trsv_counter;  // blocked triangular solve (alpha)
  int trsv_epoch = 0;
  PinnedVec<double> h_jitter;
  PinnedVec<int> h_slots, h_status_all;
  PinnedVec<double> h_out;
  size_t last_B = 0;
  std::vector<int> last_ladder;  // ladder step per slot of the last batch (-1: failed)
  std::vector<int> fslot;        // slot holding each candidate's factor in the last batch
  PinnedVec<int> h_error;        // deadlock-guard word, read with each pass's statuses
  bool spec_slots = false;       // speculation slots [max_batch + 1, 2 max_batch + 1) (run_batch)
  bool spec_active = false;
  uint64_t r_builds = 0, factorizations = 0, solves = 0;
  // optional per-phase CUDA-event timing on the plan's stream (bench roofline)
  bool profile = false;
  struct Mark {
    int kind;
    cudaEvent_t a, b;
  };
  std::vector<Mark> marks;
  void bind() {  // stream-ordered frees on the context's stream (DevBuf)
    own(&ctx->stream, X, y, table, factors, borders, theta, jitter, out);
    own(&ctx->stream, status, slots, flags, counter, error);
    own(&ctx->stream, factors_f, borders_f);
    own(&ctx->stream, dag_prof, trsv_flags, trsv_counter);
    for (auto& o : orders) own(&ctx->stream, *o.second);
  }
  void mark_begin(int kind) {
    if (!profile) return;
    Mark m{kind, nullptr, nullptr};
    cudaEventCreate(&m.a);
    cudaEventCreate(&m.b);
    cudaEventRecord(m.a, ctx->stream);
    marks.push_back(m);
  }
  void mark_end() {
    if (!profile) return;
    cudaEventRecord(marks.back().b, ctx->stream);
  }
  void clear_marks() {
    for (auto& m : marks) {
      cudaEventDestroy(m.a);
      cudaEventDestroy(m.b);
    }
    marks.clear();
  }
  ~gpemu_plan() { clear_marks(); }
};

struct gpemu_model {
  gpemu_ctx* ctx = nullptr;
  int n = 0, d = 0, NT = 0;
  double p = 1.95, mu = 0.0, sigma2 = 0.0, vtv = 0.0, neg2 = 0.0, jitter = 0.0, log_det = 0.0;
  std::vector<double> theta;
  DevBuf<double> X, theta_d, alpha, tiles, u, v;
  // extension-mode workspace for the MSE (test-point row tiles)
  DevBuf<double> ext;
  DevBuf<int> ext_flags, ext_slot, counter, error;
  int ext_rt_cap = 0, epoch = 0;
  bool single = false;  // float model: yhat through the float corr_vector / dot (predict_f32)
  // predict scratch, grown on demand and reused across calls (no per-call cudaMalloc/Free)
  DevBuf<double> pred_xt, pred_y, pred_mse, pred_part;
  DevBuf<int> pred_bad;
  void bind() {  // stream-ordered frees on the context's stream (DevBuf)
    own(&ctx->stream, X, theta_d, alpha, tiles, u, v, ext);
    own(&ctx->stream, ext_flags, ext_slot, counter, error);
    own(&ctx->stream, pred_xt, pred_y, pred_mse, pred_part);
    own(&ctx->stream, pred_bad);
  }
};

// Releases a context's stream, scratch and idle pool pages.
static void ctx_finalize(gpemu_ctx* ctx) {
  delete ctx->scratch;
  ctx->scratch_a.free();
  ctx->scratch_l.free();
  cudaStreamSynchronize(ctx->stream);
  if (ctx->own) cudaStreamDestroy(ctx->own);
  const int dev = ctx->device;
  delete ctx;
  try {  // hand the idle pool pages back to the driver (other CUDA users in the process)
    pool_trim(dev);
  } catch (const CudaError&) {
  }
}


namespace {

void ctx_adopt(gpemu_ctx* c) {
  std::lock_guard<std::mutex> lock(c->mu);
  ++c->children;
}

// Deletes a plan / model, then finalises its context if that was destroyed meanwhile.
template <typename H>
void release(H* h) {
  if (!h) return;
  gpemu_ctx* c = h->ctx;
  delete h;
  if (!c) return;
  bool fin = false;
  {
    std::lock_guard<std::mutex> lock(c->mu);
    fin = --c->children == 0 && c->closing;
  }
  if (fin) ctx_finalize(c);
}

constexpr int kTraceTasks = 65536;  // DAG timeline capacity (diagnostics)
constexpr double kOrderQuantum = 0.0;  // us; ticket_order priority quantum (0: exact bottom level)
// ticket_order: exact priority only below this fraction of the longest path (large tile counts:
// the L2-friendly setting; small ones: the faster one)
constexpr double kOrderTailLarge = 0.4;  // NT >= 24
constexpr double kOrderTailSmall = 0.7;

// Ticket order for a large launch (B candidates x NT(NT+1)/2 tile tasks): a list schedule on
// P processors with estimated task times (OFF(I,j): ~4 + 18.5 j + 20 us, DIAG(j): ~8 + 18.6 j
// + 45 us, the measured per-K slopes), ready tasks taken by longest remaining path (bottom
// level), ties by candidate and
// tile. Every task is scheduled after its inputs, so the order is topological (the kernel's
// waits only target lower tickets) and the factor is the same; it only changes which task
// a free CTA takes next. Packed as bpos << 16 | I << 8 | j (NT <= 256, B < 32768).
std::vector<int> ticket_order(int B, int NT, int P) {
  const int T = NT * (NT + 1) / 2;
  auto id = [](int I, int j) { return I * (I + 1) / 2 + j; };
  std::vector<double> dur(T), bl(T, 0.0);
  std::vector<std::vector<int>> succ(T);
  std::vector<int> ndeps(T, 0), tI(T), tj(T);
  for (int I = 0; I < NT; ++I)
    for (int j = 0; j <= I; ++j) {
      const int t = id(I, j);
      tI[t] = I;
      tj[t] = j;
      dur[t] = I == j ? 53.0 + 18.6 * j : 24.0 + 18.5 * j;
      for (int K = 0; K < j; ++K) {  // operand tiles (I,K), (j,K)
        succ[id(j, K)].push_back(t);
        ++ndeps[t];
        if (I != j) {
          succ[id(I, K)].push_back(t);
          ++ndeps[t];
        }
      }
      if (I != j) {  // L(j,j)
        succ[id(j, j)].push_back(t);
        ++ndeps[t];
      }
    }
  for (int j = NT - 1; j >= 0; --j) {  // successors first: later columns, then this column's OFFs
    for (int I = NT - 1; I >= j; --I) {
      const int t = id(I == j ? j : I, j);
      double m = 0.0;
      for (int u : succ[t]) m = std::max(m, bl[u]);
      bl[t] = dur[t] + m;
    }
  }
  // Priority. Tasks whose bottom level is at least kOrderTail of the longest path (the first
  // ~30% of every candidate's chain) share one key and go candidate-major (lower candidate,
  // then lower column, then lower row): a candidate's ready column group is dispatched together,
  // so the OFF(., j) tasks sharing the B panel L(j, 0..j-1) and the A panels of consecutive
  // columns are read through L2. Below that, the exact bottom level orders the tail, which is
  // what the list schedule buys over the built-in column order. Measured at C3 (ncu, one
  // launch): exact bottom level everywhere 150.1 GB DRAM read, 5% L2 hits, 73.83 ms; with
  // kOrderTail = 0.4, 101.8 GB, 73.91 ms (same speed in alternating bench runs); candidate-major
  // everywhere 85.4 GB, +0.3%; the built-in column order 79.3 GB, +1.3%
  // (tools/order_quantum_sweep.sh). Round 2, with the operand-flag snapshot (GPEMU_ORDER_TAIL
  // sweep, alternating runs): 0.7 is the best of {0, 0.2, 0.4, 0.55, 0.7, 0.85} over C3
  // (73.26 ms vs 73.31 at 0.4), C2 (7.39 vs 7.53) and a 100-candidate n=1024 batch (2.09 vs 2.15).
  // Later in the round, at C3 the time no longer depends on it (71.23 ms at 0.4, 71.22 at 0.7)
  // while the DRAM reads do (101.7 GB at 0.4, 134.2 GB at 0.7; tools/order_tail_sweep.sh), so
  // NT >= 24 (n > 2944) uses 0.4 and smaller designs 0.7. GPEMU_ORDER_Q quantises the exact part (microseconds).
  const char* qenv = std::getenv("GPEMU_ORDER_Q");
  const double quantum = qenv ? std::atof(qenv) : kOrderQuantum;
  struct Ready {
    double key;
    int b, t, j, I;
    bool operator<(const Ready& o) const {  // max-heap on key, then lower b, j, I
      if (key != o.key) return key < o.key;
      if (b != o.b) return b > o.b;
      if (j != o.j) return j > o.j;
      return I > o.I;
    }
  };
  const char* tenv = std::getenv("GPEMU_ORDER_TAIL");
  const double tail_frac = tenv ? std::atof(tenv) : (NT >= 24 ? kOrderTailLarge : kOrderTailSmall);
  double max_bl = 0.0;
  for (int t = 0; t < T; ++t) max_bl = std::max(max_bl, bl[t]);
  auto mk = [&](int b, int t) {
    double key = quantum > 0.0 ? std::floor(bl[t] / quantum) : bl[t];
    if (tail_frac > 0.0 && bl[t] >= tail_frac * max_bl) key = 1e300;  // before the tail: candidate-major
    return Ready{key, b, t, tj[t], tI[t]};
  };
  struct Done {
    double time;
    int b, t;
    bool operator<(const Done& o) const { return time > o.time; }  // min-heap on time
  };
  std::priority_queue<Ready> ready;
  std::priority_queue<Done> running;
  std::vector<int> left((size_t)B * T);
  for (int b = 0; b < B; ++b)
    for (int t = 0; t < T; ++t) {
      left[(size_t)b * T + t] = ndeps[t];
      if (ndeps[t] == 0) ready.push(mk(b, t));
    }
  std::vector<int> order;
  order.reserve((size_t)B * T);
  int free_p = P;
  double now = 0.0;
  while (order.size() < (size_t)B * T) {
    while (free_p > 0 && !ready.empty()) {
      const Ready r = ready.top();
      ready.pop();
      order.push_back(r.b << 16 | tI[r.t] << 8 | tj[r.t]);
      running.push({now + dur[r.t], r.b, r.t});
      --free_p;
    }
    if (running.empty()) break;  // (cannot happen for a DAG)
    now = running.top().time;
    while (!running.empty() && running.top().time <= now) {
      const Done d = running.top();
      running.pop();
      ++free_p;
      for (int u : succ[d.t])
        if (--left[(size_t)d.b * T + u] == 0) ready.push(mk(d.b, u));
    }
  }
  return order;
}

void run_chol(gpemu_plan* pl, int nact) {
  DagLaunch a;
  a.factors = pl->factors.p;
  a.borders = pl->borders.p;
  a.slot_stride = pl->slot_stride;
  a.n = pl->n;
  a.NT = pl->NT;
  a.slots = pl->slots.p;
  a.nslots = nact;
  a.counter = pl->counter.p;
  a.flags = pl->flags.p;
  a.epoch = ++pl->epoch;
  a.status = pl->status.p;
  a.error = pl->error.p;
  a.prof = pl->dag_prof.p;
  if (a.prof) {
    a.trace = a.prof + (size_t)pl->ctx->num_sms * 24 + 256;
    a.trace_cap = kTraceTasks;
  }
  if (pl->precision == GPEMU_PRECISION_SINGLE) {
    a.factors = reinterpret_cast<double*>(pl->factors_f.p);
    a.borders = reinterpret_cast<double*>(pl->borders_f.p);
    a.prof = nullptr;
    a.trace = nullptr;
    launch_chol_dag_f32(a, pl->ctx->num_sms, pl->ctx->stream);
  } else if (pl->ctx->engine == GPEMU_ENGINE_SIMPLE) {
    launch_chol_simple(a, pl->ctx->stream);
  } else {
    const int T = pl->NT * (pl->NT + 1) / 2;
    const long long ntasks = (long long)nact * T;
    const int grid = (int)std::min<long long>(ntasks, pl->ctx->num_sms);
    const char* env = std::getenv("GPEMU_TICKET_ORDER");
    if (ntasks >= 16LL * grid && nact < (1 << 15) && pl->NT <= 256 && !(env && env[0] == '0')) {
      auto it = pl->orders.find(nact);
      if (it == pl->orders.end()) {
        if (pl->orders.size() >= 8) pl->orders.erase(pl->orders.begin());
        const std::vector<int> ord = ticket_order(nact, pl->NT, grid);
        auto buf = std::make_unique<DevBuf<int>>();
        own(&pl->ctx->stream, *buf);
        buf->alloc(ord.size());
        ck(cudaMemcpyAsync(buf->p, ord.data(), ord.size() * sizeof(int), cudaMemcpyHostToDevice,
                           pl->ctx->stream),
           "H2D ticket order");
        ck(cudaStreamSynchronize(pl->ctx->stream), "ticket order");
        it = pl->orders.emplace(nact, std::move(buf)).first;
      }
      a.order = it->second->p;
    }
    launch_chol_dag(a, pl->ctx->num_sms, pl->ctx->stream);
  }
  pl->ctx->launches += 1;
}

// Evaluates slots [0, B) whose thetas are already in pl->theta; runs the jitter
// ladder (backend.hpp:105-119) on the device, re-assembling R only for the
// candidates whose factorization failed. Leaves records in pl->out[0, B) and the slot holding
// each candidate's factor in pl->fslot.
// With tolerate_nonfinite a slot with a non-finite R entry is left with its status-2 record
// instead of failing the batch (speculative evaluations the caller may never use).
//
// Speculative first rung: on small designs a pass is bound by one candidate's serial chain,
// not by throughput, so a retry pass costs a whole second chain. A plan with speculation slots
// (kSpecTaskCap) evaluates, once the previous batch showed that most candidates climb the ladder,
// every candidate at jitter 0 in slot i AND at kJitterLadder[1] in slot max_batch + 1 + i in the
// same pass; a candidate that fails at 0 and succeeds at 1e-8 takes the second record and
// factor (bitwise what the reference's second attempt computes: the same R + 1e-8 I through the
// same kernels). Failures at both continue the ladder at 1e-7. One factorization per
// candidate in the Ledger either way.
int run_batch(gpemu_plan* pl, size_t B, bool tolerate_nonfinite = false) {
  cudaStream_t s = pl->ctx->stream;
  pl->last_B = B;
  pl->last_ladder.assign(B, -1);
  pl->fslot.resize(B);
  std::iota(pl->fslot.begin(), pl->fslot.end(), 0);
  const char* spec_env = std::getenv("GPEMU_SPEC_LADDER");  // "0": off (A/B and tests)
  const bool spec = pl->spec_slots && pl->spec_active && B <= pl->max_batch &&
                    !(spec_env && spec_env[0] == '0');
  const size_t SB = pl->max_batch + 1;  // first speculation slot
  const size_t used = spec ? SB + B : B;
  std::vector<int> active(B);
  std::iota(active.begin(), active.end(), 0);
  for (size_t i = 0; i < B; ++i) pl->h_jitter[i] = 0.0;
  if (spec) {
    for (size_t i = 0; i < B; ++i) {
      active.push_back((int)(SB + i));
      pl->h_jitter[SB + i] = kLadder[1];
    }
    ck(cudaMemcpyAsync(pl->theta.p + SB * pl->d, pl->theta.p, B * pl->d * sizeof(double),
                       cudaMemcpyDeviceToDevice, s),
       "D2D speculation theta");
  }
  ck(cudaMemcpyAsync(pl->jitter.p, pl->h_jitter.data(), used * sizeof(double), cudaMemcpyHostToDevice, s),
     "H2D jitter");
  for (int step = 0; step < 6 && !active.empty();) {
    const int nact = (int)active.size();
    if (step > 0 && pl->precision == GPEMU_PRECISION_SINGLE) {
      // In float a rung whose diagonal rounds to the previous rung's (1 + 1e-8 == 1 in float)
      // rebuilds the same matrix: that attempt fails again by construction, so it is skipped
      // (the recorded jitter and every value are those of the rung-by-rung ladder).
      const float diag_base = 1.0f + (float)pl->nugget;  // kernels_f32.cu assemble
      volatile float prev = diag_base + (float)kLadder[step - 1];
      volatile float cur = diag_base + (float)kLadder[step];
      if (prev == cur) {
        ++step;
        continue;
      }
    }
    if (step > 0) {
      for (int q = 0; q < nact; ++q) pl->h_jitter[active[q]] = kLadder[step];
      ck(cudaMemcpyAsync(pl->jitter.p, pl->h_jitter.data(), B * sizeof(double),
                         cudaMemcpyHostToDevice, s),
         "H2D jitter");
    }
    std::copy(active.begin(), active.end(), pl->h_slots.begin());
    ck(cudaMemcpyAsync(pl->slots.p, pl->h_slots.data(), nact * sizeof(int), cudaMemcpyHostToDevice, s),
       "H2D slots");
    nvtx_push("K1 assemble");
    pl->mark_begin(0);
    if (pl->precision == GPEMU_PRECISION_SINGLE)
      launch_assemble_f32(pl->table.p, pl->theta.p, pl->y.p, pl->n, pl->d, pl->nugget, pl->NT,
                          pl->slots.p, nact, pl->jitter.p, pl->factors_f.p, pl->slot_stride,
                          pl->borders_f.p, pl->status.p, s);
    else
      launch_assemble(pl->table.p, pl->theta.p, pl->y.p, pl->n, pl->d, pl->nugget, pl->NT,
                      pl->slots.p, nact, pl->jitter.p, pl->factors.p, pl->slot_stride,
                      pl->borders.p, pl->status.p, pl->ctx->num_sms, s);
    pl->mark_end();
    nvtx_pop();
    nvtx_push("K2 cholesky + border solves");
    pl->mark_begin(1);
    run_chol(pl, nact);
    pl->mark_end();
    nvtx_pop();
    nvtx_push("K3 finalize");
    pl->mark_begin(2);
    const int spec_off = (spec && step == 0) ? (int)SB : 0;  // records of rung 1 land in slot i
    if (pl->precision == GPEMU_PRECISION_SINGLE)
      launch_finalize_f32(pl->factors_f.p, pl->slot_stride, pl->borders_f.p, pl->status.p,
                          pl->jitter.p, pl->n, pl->NT, pl->slots.p, nact, pl->out.p, spec_off, s);
    else
      launch_finalize(pl->factors.p, pl->slot_stride, pl->borders.p, pl->status.p, pl->jitter.p,
                      pl->n, pl->NT, pl->slots.p, nact, pl->out.p, spec_off, s);
    pl->mark_end();
    nvtx_pop();
    pl->ctx->launches += 4;
    ck(cudaGetLastError(), "kernel launch");
    ck(cudaMemcpyAsync(pl->h_status_all.data(), pl->status.p, used * sizeof(int), cudaMemcpyDeviceToHost, s),
       "D2H status");
    ck(cudaMemcpyAsync(pl->h_error.data(), pl->error.p, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H error");
    ck(cudaStreamSynchronize(s), "batch");
    if (pl->h_error[0]) return set_error(GPEMU_CUDA, "chol_dag: dependency wait timed out (deadlock guard)");
    std::vector<int> failed;
    for (int q = 0; q < nact; ++q) {
      const int slot = active[q];
      if ((size_t)slot >= SB) continue;  // speculation slots are read with their candidate below
      const int st = pl->h_status_all[slot];
      if (st == 2) {
        if (tolerate_nonfinite) continue;
        return set_error(GPEMU_NONFINITE, "CorrelationPlan: non-finite correlation value");
      }
      if (st == 1) {
        if (spec && step == 0 && pl->h_status_all[SB + slot] == 0) {  // the second rung held
          pl->last_ladder[slot] = 1;
          pl->fslot[slot] = (int)(SB + slot);  // its record is already in out[slot] (finalize)
        } else {
          failed.push_back(slot);
        }
      } else {
        pl->last_ladder[slot] = step;
      }
    }
    active.swap(failed);
    step += (spec && step == 0) ? 2 : 1;  // the speculative pass covered rungs 0 and 1
  }
  if (pl->spec_slots) {  // speculate while most candidates climb the ladder (GA generations are alike)
    size_t climb = 0;
    for (size_t i = 0; i < B; ++i) climb += pl->last_ladder[i] != 0;
    if (!pl->spec_active && 2 * climb > B) pl->spec_active = true;
    else if (pl->spec_active && 4 * climb < B) pl->spec_active = false;
  }
  pl->r_builds += B;
  pl->factorizations += B;
  pl->solves += 2 * B;
  return GPEMU_OK;
}

int download_records(gpemu_plan* pl, size_t B) {
  ck(cudaMemcpyAsync(pl->h_out.data(), pl->out.p, B * REC_SIZE * sizeof(double),
                     cudaMemcpyDeviceToHost, pl->ctx->stream),
     "D2H out");
  ck(cudaStreamSynchronize(pl->ctx->stream), "D2H out");
  return GPEMU_OK;
}

// alpha = (R + jI)^-1 (y - mu 1) on the factor of `slot` (solve_full, backend.hpp:163-169;
// likelihood.hpp:226-230). The forward half is already in the factor's border rows:
// L^-1 (y - mu 1) = u - mu v, so one blocked backward solve (kernels_trsv.cu) gives alpha.
// d_alpha: Npad doubles. Two triangular solves in the Ledger, as the reference's solve_full.
void solve_alpha(gpemu_plan* pl, int slot, double mu, double* d_alpha) {
  NvtxRange range("K3 alpha (blocked backward solve)");
  cudaStream_t s = pl->ctx->stream;
  pl->trsv_flags.reserve(pl->NT);
  pl->trsv_counter.reserve(1);
  if (pl->trsv_epoch == 0)
    ck(cudaMemsetAsync(pl->trsv_flags.p, 0, pl->NT * sizeof(int), s), "memset trsv flags");
  const double* tiles = pl->factors.p + (size_t)slot * pl->slot_stride;
  const double* u = pl->borders.p + (size_t)slot * 2 * pl->Npad;
  launch_tile_trsv(tiles, pl->NT, u, u + pl->Npad, mu, pl->Npad, d_alpha, 1, pl->trsv_flags.p,
                   pl->trsv_counter.p, ++pl->trsv_epoch, pl->error.p, pl->ctx->num_sms, s);
  pl->ctx->launches += 1;
  ck(cudaGetLastError(), "tile_trsv launch");
  int err = 0;
  ck(cudaMemcpyAsync(&err, pl->error.p, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H error");
  ck(cudaStreamSynchronize(s), "solve_alpha");
  if (err) throw CudaError{"tile_trsv: dependency wait timed out (deadlock guard)"};
  pl->solves += 2;
}

gpemu_model* make_model(gpemu_plan* pl, int slot, const double* theta, const double* rec) {
  auto* m = new gpemu_model();
  ctx_adopt(pl->ctx);
  m->ctx = pl->ctx;
  m->bind();
  m->n = pl->n;
  m->d = pl->d;
  m->NT = pl->NT;
  m->p = pl->p;
  m->neg2 = rec[REC_NEG2];
  m->mu = rec[REC_MU];
  m->sigma2 = rec[REC_SIGMA2];
  m->vtv = rec[REC_VTV];
  m->jitter = rec[REC_JITTER];
  m->log_det = rec[REC_LOGDET];
  m->theta.assign(theta, theta + pl->d);
  cudaStream_t s = pl->ctx->stream;
  m->X.alloc((size_t)pl->n * pl->d);
  m->theta_d.alloc(pl->d);
  m->alpha.alloc(pl->Npad);  // the blocked solve writes whole 128-row blocks
  m->tiles.alloc(pl->slot_stride);
  m->u.alloc(pl->Npad);
  m->v.alloc(pl->Npad);
  ck(cudaMemcpyAsync(m->X.p, pl->X.p, (size_t)pl->n * pl->d * sizeof(double), cudaMemcpyDeviceToDevice, s), "model X");
  ck(cudaMemcpyAsync(m->theta_d.p, theta, pl->d * sizeof(double), cudaMemcpyHostToDevice, s), "model theta");
  if (pl->precision == GPEMU_PRECISION_SINGLE) {
    // float factor: alpha by the float solves (likelihood.hpp:228-229); the factor and the
    // border rows widened to double for the MSE extension DAG
    m->single = true;
    const float* ftiles = pl->factors_f.p + (size_t)slot * pl->slot_stride;
    launch_tiles_f32_to_f64(ftiles, pl->NT, m->tiles.p, s);
    std::vector<float> hb(2 * (size_t)pl->Npad);
    ck(cudaMemcpyAsync(hb.data(), pl->borders_f.p + (size_t)slot * 2 * pl->Npad, hb.size() * sizeof(float),
                       cudaMemcpyDeviceToHost, s), "D2H borders");
    ck(cudaStreamSynchronize(s), "borders");
    std::vector<double> hu(hb.begin(), hb.begin() + pl->Npad), hv(hb.begin() + pl->Npad, hb.end());
    // ordered on the ctx stream (a non-blocking stream is not ordered after legacy copies)
    ck(cudaMemcpyAsync(m->u.p, hu.data(), pl->Npad * sizeof(double), cudaMemcpyHostToDevice, s), "model u");
    ck(cudaMemcpyAsync(m->v.p, hv.data(), pl->Npad * sizeof(double), cudaMemcpyHostToDevice, s), "model v");
    launch_alpha_f32(ftiles, pl->n, pl->y.p, m->mu, m->alpha.p, s);
    pl->ctx->launches += 2;
    ck(cudaStreamSynchronize(s), "float model");
    pl->solves += 2;
    return m;
  }
  ck(cudaMemcpyAsync(m->tiles.p, pl->factors.p + (size_t)slot * pl->slot_stride,
                     pl->slot_stride * sizeof(double), cudaMemcpyDeviceToDevice, s),
     "model tiles");
  ck(cudaMemcpyAsync(m->u.p, pl->borders.p + (size_t)slot * 2 * pl->Npad,
                     pl->Npad * sizeof(double), cudaMemcpyDeviceToDevice, s),
     "model u");
  ck(cudaMemcpyAsync(m->v.p, pl->borders.p + (size_t)slot * 2 * pl->Npad + pl->Npad,
                     pl->Npad * sizeof(double), cudaMemcpyDeviceToDevice, s),
     "model v");
  solve_alpha(pl, slot, m->mu, m->alpha.p);
  return m;
}

}  // namespace

#define GPEMU_GUARD_BEGIN try {
#define GPEMU_GUARD_END                                        \
  }                                                            \
  catch (const CudaError& e) {                                 \
    return set_error(GPEMU_CUDA, "%s", e.msg.c_str());        \
  }                                                            \
  catch (const std::bad_alloc&) {                              \
    return set_error(GPEMU_ERROR, "host allocation failed");   \
  }

extern "C" {

const char* gpemu_last_error(void) { return g_last_error.c_str(); }
const char* gpemu_version(void) { return "gpemu_b200 0.1 (sm_100a)"; }

int gpemu_ctx_create(int device, gpemu_ctx** out) {
  GPEMU_GUARD_BEGIN
  if (!out) return set_error(GPEMU_VALIDATION, "ctx_create: null out");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return set_error(GPEMU_CUDA, "no CUDA device available (the B200 engine has no CPU fallback)");
  if (device < 0 || device >= count) return set_error(GPEMU_CONFIG, "ctx_create: bad device %d", device);
  ck(cudaSetDevice(device), "cudaSetDevice");
  cudaDeviceProp prop;
  ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major < 10)
    return set_error(GPEMU_CUDA, "device %s (sm_%d%d) is not Blackwell sm_100", prop.name, prop.major, prop.minor);
  auto* c = new gpemu_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  ck(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking), "cudaStreamCreate");
  c->stream = c->own;
  own(&c->stream, c->scratch_a, c->scratch_l);
  *out = c;
  return GPEMU_OK;
  GPEMU_GUARD_END
}

int gpemu_ctx_destroy(gpemu_ctx* ctx) {
  if (!ctx) return GPEMU_OK;
  {
    std::lock_guard<std::mutex> lock(ctx->mu);
    if (ctx->children > 0) {  // finalised by the last plan / model
      ctx->closing = true;
      return GPEMU_OK;
    }
  }
  ctx_finalize(ctx);
  return GPEMU_OK;
}

int gpemu_ctx_set_stream(gpemu_ctx* ctx, void* stream) {
  if (!ctx) return set_error(GPEMU_VALIDATION, "null ctx");
  // work (and stream-ordered frees) already issued on the old stream completes first
  cudaStreamSynchronize(ctx->stream);
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own;
  return GPEMU_OK;
}

int gpemu_ctx_set_engine(gpemu_ctx* ctx, int engine) {
  if (!ctx) return set_error(GPEMU_VALIDATION, "null ctx");
  if (engine != GPEMU_ENGINE_DAG && engine != GPEMU_ENGINE_SIMPLE)
    return set_error(GPEMU_CONFIG, "unknown engine %d", engine);
  ctx->engine = engine;
  return GPEMU_OK;
}

uint64_t gpemu_ctx_launch_count(const gpemu_ctx* ctx) { return ctx ? ctx->launches : 0; }
int gpemu_ctx_num_sms(const gpemu_ctx* ctx) { return ctx ? ctx->num_sms : 0; }

int gpemu_ctx_mem_info(gpemu_ctx* ctx, size_t* free_bytes, size_t* total_bytes) {
  GPEMU_GUARD_BEGIN
  if (!ctx) return set_error(GPEMU_VALIDATION, "null ctx");
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  size_t f = 0, tot = 0;
  ck(cudaMemGetInfo(&f, &tot), "cudaMemGetInfo");
  f += pool_idle_bytes(ctx->device);  // mapped by the engine's pool but free for the next plan
  if (free_bytes) *free_bytes = f;
  if (total_bytes) *total_bytes = tot;
  return GPEMU_OK;
  GPEMU_GUARD_END
}

size_t gpemu_plan_bytes(size_t n, size_t d, size_t max_batch, int precision) {
  const size_t NT = (n + TILE - 1) / TILE, tiles = NT * (NT + 1) / 2;
  const size_t elem = precision == GPEMU_PRECISION_SINGLE ? sizeof(float) : sizeof(double);
  const size_t slots = (spec_slots_for((int)NT, max_batch) ? 2 * max_batch : max_batch) + 1;
  return tiles * TILE_ELEMS * (d * sizeof(double) + slots * elem) + slots * 2 * NT * TILE * elem +
         slots * (NT + 1) * NT * sizeof(int) + (n * d + n) * sizeof(double);
}

// ---------------------------------------------------------------------------
int gpemu_build_corr(gpemu_ctx* ctx, const double* X, size_t n, size_t d, const double* theta,
                     double p, double nugget, double* R_out) {
  GPEMU_GUARD_BEGIN
  if (!ctx || !X || !theta || !R_out) return set_error(GPEMU_VALIDATION, "build_corr: null argument");
  int rc = validate_params(theta, d, p, nugget);
  if (rc) return rc;
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  DevBuf<double> dX, dT, dR;
  DevBuf<int> bad;
  own(&ctx->stream, dX, dT, dR, bad);
  dX.alloc(n * d);
  dT.alloc(d);
  dR.alloc(n * n);
  bad.alloc(1);
  cudaStream_t s = ctx->stream;
  ck(cudaMemcpyAsync(dX.p, X, n * d * sizeof(double), cudaMemcpyHostToDevice, s), "H2D X");
  ck(cudaMemcpyAsync(dT.p, theta, d * sizeof(double), cudaMemcpyHostToDevice, s), "H2D theta");
  ck(cudaMemsetAsync(bad.p, 0, sizeof(int), s), "memset");
  if (n > 0) launch_build_corr_rowmajor(dX.p, (int)n, (int)d, dT.p, p, nugget, dR.p, bad.p, s);
  ctx->launches += 1;
  ck(cudaGetLastError(), "build_corr launch");
  int hbad = 0;
  ck(cudaMemcpyAsync(R_out, dR.p, n * n * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H R");
  ck(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H bad");
  ck(cudaStreamSynchronize(s), "build_corr");
  if (hbad) return set_error(GPEMU_NONFINITE, "build_corr_matrix: non-finite correlation value");
  return GPEMU_OK;
  GPEMU_GUARD_END
}

int gpemu_corr_vector(gpemu_ctx* ctx, const double* xstar, const double* X, size_t n, size_t d,
                      const double* theta, double p, double* r_out) {
  GPEMU_GUARD_BEGIN
  if (!ctx || !xstar || !X || !theta || !r_out) return set_error(GPEMU_VALIDATION, "corr_vector: null argument");
  int rc = validate_params(theta, d, p, 0.0);
  if (rc) return rc;
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  DevBuf<double> dX, dT, dS, dR;
  DevBuf<int> bad;
  own(&ctx->stream, dX, dT, dS, dR, bad);
  dX.alloc(n * d);
  dT.alloc(d);
  dS.alloc(d);
  dR.alloc(n);
  bad.alloc(1);
  cudaStream_t s = ctx->stream;
  ck(cudaMemcpyAsync(dX.p, X, n * d * sizeof(double), cudaMemcpyHostToDevice, s), "H2D X");
  ck(cudaMemcpyAsync(dT.p, theta, d * sizeof(double), cudaMemcpyHostToDevice, s), "H2D theta");
  ck(cudaMemcpyAsync(dS.p, xstar, d * sizeof(double), cudaMemcpyHostToDevice, s), "H2D xstar");
  ck(cudaMemsetAsync(bad.p, 0, sizeof(int), s), "memset");
  if (n > 0) launch_corr_vectors(dS.p, 1, dX.p, (int)n, (int)d, dT.p, p, dR.p, bad.p, s);
  ctx->launches += 1;
  int hbad = 0;
  ck(cudaMemcpyAsync(r_out, dR.p, n * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H r");
  ck(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H bad");
  ck(cudaStreamSynchronize(s), "corr_vector");
  if (hbad) return set_error(GPEMU_NONFINITE, "corr_vector: non-finite correlation value");
  return GPEMU_OK;
  GPEMU_GUARD_END
}

// One Cholesky attempt of A (no ladder): Backend::try_cholesky (backend.hpp:174).
static int factor_once(gpemu_ctx* ctx, gpemu_plan& pl, const double* dR, double jit, int* st,
                       double* rec) {
  cudaStream_t s = ctx->stream;
  ck(cudaMemsetAsync(pl.status.p, 0, sizeof(int), s), "memset");
  ck(cudaMemsetAsync(pl.borders.p, 0, 2 * pl.Npad * sizeof(double), s), "memset");
  ck(cudaMemcpyAsync(pl.jitter.p, &jit, sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
  launch_rowmajor_to_tiles(dR, pl.n, pl.NT, jit, pl.factors.p, s);
  run_chol(&pl, 1);
  launch_finalize(pl.factors.p, pl.slot_stride, pl.borders.p, pl.status.p, pl.jitter.p, pl.n,
                  pl.NT, pl.slots.p, 1, pl.out.p, 0, s);
  ctx->launches += 2;
  ck(cudaMemcpyAsync(st, pl.status.p, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
  ck(cudaMemcpyAsync(rec, pl.out.p, REC_SIZE * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
  ck(cudaStreamSynchronize(s), "factorize");
  int err = 0;
  d2h_sync(&err, pl.error.p, sizeof(int), ctx->stream, "D2H error");
  if (err) return set_error(GPEMU_CUDA, "chol_dag: dependency wait timed out (deadlock guard)");
  return GPEMU_OK;
}

static void single_slot_plan(gpemu_ctx* ctx, gpemu_plan& pl, size_t n) {
  pl.ctx = ctx;
  pl.bind();
  pl.n = (int)n;
  pl.NT = (int)((n + TILE - 1) / TILE);
  pl.Npad = pl.NT * TILE;
  pl.slot_stride = (size_t)num_tiles(pl.NT) * TILE_ELEMS;
  cudaStream_t s = ctx->stream;
  pl.factors.alloc(pl.slot_stride);
  pl.borders.alloc(2 * pl.Npad);
  pl.jitter.alloc(1);
  pl.out.alloc(REC_SIZE);
  pl.status.alloc(1);
  pl.slots.alloc(1);
  pl.flags.alloc((size_t)(pl.NT + 1) * pl.NT);
  pl.counter.alloc(1);
  pl.error.alloc(1);
  ck(cudaMemsetAsync(pl.flags.p, 0, pl.flags.count * sizeof(int), s), "memset");
  ck(cudaMemsetAsync(pl.slots.p, 0, sizeof(int), s), "memset");
  ck(cudaMemsetAsync(pl.error.p, 0, sizeof(int), s), "memset");
}

// The context's reusable one-slot plan for n (see gpemu_ctx::scratch).
static gpemu_plan& scratch_plan(gpemu_ctx* ctx, size_t n) {
  if (!ctx->scratch || ctx->scratch->n != (int)n) {
    delete ctx->scratch;
    ctx->scratch = nullptr;
    auto* pl = new gpemu_plan();
    try {
      single_slot_plan(ctx, *pl, n);
    } catch (...) {
      delete pl;
      throw;
    }
    ctx->scratch = pl;
  }
  return *ctx->scratch;
}

int gpemu_try_cholesky(gpemu_ctx* ctx, double* A, size_t n) {
  GPEMU_GUARD_BEGIN
  if (!ctx || !A || n == 0) return set_error(GPEMU_VALIDATION, "try_cholesky: bad argument");
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  gpemu_plan& pl = scratch_plan(ctx, n);
  cudaStream_t s = ctx->stream;
  DevBuf<double>& dA = ctx->scratch_a;
  dA.reserve(n * n);
  ck(cudaMemcpyAsync(dA.p, A, n * n * sizeof(double), cudaMemcpyHostToDevice, s), "H2D A");
  int st = 0;
  double rec[REC_SIZE];
  int rc = factor_once(ctx, pl, dA.p, 0.0, &st, rec);
  if (rc) return rc;
  if (st != 0) return set_error(GPEMU_NOT_PD, "try_cholesky: pivot not strictly positive");
  launch_tiles_to_rowmajor(pl.factors.p, pl.n, pl.NT, dA.p, s);
  ctx->launches += 1;
  ck(cudaMemcpyAsync(A, dA.p, n * n * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H L");
  ck(cudaStreamSynchronize(s), "try_cholesky");
  return GPEMU_OK;
  GPEMU_GUARD_END
}

// Factorization workspace for the Backend-level API (one slot, no table).
int gpemu_factorize(gpemu_ctx* ctx, const double* R, size_t n, double* L_out, double* log_det,
                    double* jitter_used) {
  GPEMU_GUARD_BEGIN
  if (!ctx || !R || n == 0) return set_error(GPEMU_VALIDATION, "factorize: bad argument");
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  gpemu_plan& pl = scratch_plan(ctx, n);
  cudaStream_t s = ctx->stream;
  DevBuf<double>& dR = ctx->scratch_a;
  dR.reserve(n * n);
  ck(cudaMemcpyAsync(dR.p, R, n * n * sizeof(double), cudaMemcpyHostToDevice, s), "H2D R");
  for (int step = 0; step < 6; ++step) {
    const double jit = kLadder[step];
    int st = 0;
    double rec[REC_SIZE];
    int rc = factor_once(ctx, pl, dR.p, jit, &st, rec);
    if (rc) return rc;
    if (st == 0) {
      if (L_out) {
        DevBuf<double>& dL = ctx->scratch_l;
        dL.reserve(n * n);
        launch_tiles_to_rowmajor(pl.factors.p, pl.n, pl.NT, dL.p, s);
        ctx->launches += 1;
        ck(cudaMemcpyAsync(L_out, dL.p, n * n * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H L");
        ck(cudaStreamSynchronize(s), "factorize");
      }
      if (log_det) *log_det = rec[REC_LOGDET];
      if (jitter_used) *jitter_used = jit;
      return GPEMU_OK;
    }
  }
  return set_error(GPEMU_NOT_PD, "factorize: not positive definite at any jitter level (n = %zu)", n);
  GPEMU_GUARD_END
}

static int solve_common(gpemu_ctx* ctx, const double* L, size_t n, const double* b, double* x,
                        int upper) {
  GPEMU_GUARD_BEGIN
  if (!ctx || !L || !b || !x || n == 0) return set_error(GPEMU_VALIDATION, "solve: bad argument");
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  const int NT = (int)((n + TILE - 1) / TILE);
  cudaStream_t s = ctx->stream;
  DevBuf<double> dL, tiles, db, dx;
  DevBuf<int> flags, counter, error;
  own(&ctx->stream, dL, tiles, db, dx);
  own(&ctx->stream, flags, counter, error);
  dL.alloc(n * n);
  tiles.alloc((size_t)num_tiles(NT) * TILE_ELEMS);
  db.alloc(n);
  dx.alloc((size_t)NT * TILE);
  flags.alloc(NT);
  counter.alloc(1);
  error.alloc(1);
  ck(cudaMemsetAsync(flags.p, 0, NT * sizeof(int), s), "memset");
  ck(cudaMemsetAsync(error.p, 0, sizeof(int), s), "memset");
  ck(cudaMemcpyAsync(dL.p, L, n * n * sizeof(double), cudaMemcpyHostToDevice, s), "H2D L");
  ck(cudaMemcpyAsync(db.p, b, n * sizeof(double), cudaMemcpyHostToDevice, s), "H2D b");
  launch_rowmajor_to_tiles(dL.p, (int)n, NT, 0.0, tiles.p, s);
  launch_tile_trsv(tiles.p, NT, db.p, nullptr, 0.0, (int)n, dx.p, upper, flags.p, counter.p, 1,
                   error.p, ctx->num_sms, s);
  ctx->launches += 2;
  ck(cudaGetLastError(), "solve launch");
  int err = 0;
  ck(cudaMemcpyAsync(x, dx.p, n * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H x");
  ck(cudaMemcpyAsync(&err, error.p, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H error");
  ck(cudaStreamSynchronize(s), "solve");
  if (err) return set_error(GPEMU_CUDA, "tile_trsv: dependency wait timed out (deadlock guard)");
  return GPEMU_OK;
  GPEMU_GUARD_END
}

int gpemu_solve_lower(gpemu_ctx* ctx, const double* L, size_t n, const double* b, double* x) {
  return solve_common(ctx, L, n, b, x, 0);
}
int gpemu_solve_upper(gpemu_ctx* ctx, const double* L, size_t n, const double* b, double* x) {
  return solve_common(ctx, L, n, b, x, 1);
}

// ---------------------------------------------------------------------------
int gpemu_plan_create(gpemu_ctx* ctx, const double* X, const double* y, size_t n, size_t d,
                      double p, double nugget, size_t max_batch, gpemu_plan** out) {
  return gpemu_plan_create_ex(ctx, X, y, n, d, p, nugget, max_batch, GPEMU_PRECISION_DOUBLE, out);
}

int gpemu_plan_precision(const gpemu_plan* pl) { return pl ? pl->precision : -1; }

int gpemu_plan_create_ex(gpemu_ctx* ctx, const double* X, const double* y, size_t n, size_t d,
                         double p, double nugget, size_t max_batch, int precision, gpemu_plan** out) {
  GPEMU_GUARD_BEGIN
  if (precision != GPEMU_PRECISION_DOUBLE && precision != GPEMU_PRECISION_SINGLE)
    return set_error(GPEMU_CONFIG, "unknown precision %d (expected single|double)", precision);
  if (!ctx || !X || !y || !out) return set_error(GPEMU_VALIDATION, "plan_create: null argument");
  if (n < 2) return set_error(GPEMU_VALIDATION, "new_dataset: need at least 2 design points");
  if (d < 1) return set_error(GPEMU_VALIDATION, "new_dataset: need at least 1 input dimension");
  if (max_batch < 1) return set_error(GPEMU_VALIDATION, "plan_create: max_batch must be >= 1");
  int rc = validate_unit_cube(X, n, d, "new_dataset");
  if (rc) return rc;
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(y[i])) return set_error(GPEMU_VALIDATION, "new_dataset: non-finite output");
  std::vector<double> probe(d, 1.0);  // likelihood.hpp:89-90
  rc = validate_params(probe.data(), d, p, nugget);
  if (rc) return rc;
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  auto* pl = new gpemu_plan();
  pl->ctx = ctx;
  pl->bind();
  ctx_adopt(ctx);
  pl->n = (int)n;
  pl->d = (int)d;
  pl->p = p;
  pl->nugget = nugget;
  pl->NT = (int)((n + TILE - 1) / TILE);
  pl->Npad = pl->NT * TILE;
  pl->max_batch = max_batch;
  pl->spec_slots = spec_slots_for(pl->NT, max_batch);
  pl->nslots = (pl->spec_slots ? 2 * max_batch : max_batch) + 1;
  pl->slot_stride = (size_t)num_tiles(pl->NT) * TILE_ELEMS;
  try {
    pl->X.alloc(n * d);
    pl->y.alloc(n);
    pl->precision = precision;
    if (precision == GPEMU_PRECISION_SINGLE) {
      pl->table.alloc((size_t)num_tiles(pl->NT) * d * TILE_ELEMS);  // column-major, double
      pl->factors_f.alloc(pl->nslots * pl->slot_stride);
      pl->borders_f.alloc(pl->nslots * 2 * pl->Npad);
    } else {
      pl->table.alloc((size_t)num_tiles(pl->NT) * d * TILE_ELEMS);
      pl->factors.alloc(pl->nslots * pl->slot_stride);
      pl->borders.alloc(pl->nslots * 2 * pl->Npad);
    }
    pl->theta.alloc(pl->nslots * d);
    pl->jitter.alloc(pl->nslots);
    pl->out.alloc(pl->nslots * REC_SIZE);
    pl->status.alloc(pl->nslots);
    pl->slots.alloc(pl->nslots);
    pl->flags.alloc(pl->nslots * (size_t)(pl->NT + 1) * pl->NT);
    pl->counter.alloc(1);
    pl->error.alloc(1);
  } catch (const CudaError& e) {
    release(pl);
    return set_error(GPEMU_CUDA, "plan_create: device allocation failed (%s)", e.msg.c_str());
  }
  {
    uint64_t h = 1469598103934665603ull;
    auto mixb = [&h](const void* p, size_t bytes) {
      const unsigned char* c = static_cast<const unsigned char*>(p);
      for (size_t i = 0; i < bytes; ++i) h = (h ^ c[i]) * 1099511628211ull;
    };
    mixb(&n, sizeof(n));
    mixb(&d, sizeof(d));
    mixb(X, n * d * sizeof(double));
    mixb(y, n * sizeof(double));
    pl->data_hash = h;
  }
  cudaStream_t s = ctx->stream;
  ck(cudaMemcpyAsync(pl->X.p, X, n * d * sizeof(double), cudaMemcpyHostToDevice, s), "H2D X");
  ck(cudaMemcpyAsync(pl->y.p, y, n * sizeof(double), cudaMemcpyHostToDevice, s), "H2D y");
  ck(cudaMemsetAsync(pl->flags.p, 0, pl->flags.count * sizeof(int), s), "memset flags");
  ck(cudaMemsetAsync(pl->error.p, 0, sizeof(int), s), "memset error");
  ck(cudaMemsetAsync(pl->status.p, 0, pl->nslots * sizeof(int), s), "memset status");
  if (precision == GPEMU_PRECISION_SINGLE)
    launch_pow_table_f32(pl->X.p, pl->n, pl->d, p, pl->NT, pl->table.p, s);
  else
    launch_pow_table(pl->X.p, pl->n, pl->d, p, pl->NT, pl->table.p, s);
  ctx->launches += 1;
  ck(cudaGetLastError(), "pow_table launch");
  ck(cudaStreamSynchronize(s), "plan_create");
  pl->h_jitter.assign(pl->nslots, 0.0);
  pl->h_slots.assign(pl->nslots, 0);
  pl->h_status_all.assign(pl->nslots, 0);
  pl->h_out.assign(pl->nslots * REC_SIZE, 0.0);
  pl->h_error.assign(1, 0);
  *out = pl;
  return GPEMU_OK;
  GPEMU_GUARD_END
}

int gpemu_plan_destroy(gpemu_plan* plan) {
  release(plan);
  return GPEMU_OK;
}

size_t gpemu_plan_device_bytes(const gpemu_plan* pl) {
  if (!pl) return 0;
  return (pl->X.count + pl->y.count + pl->table.count + pl->factors.count + pl->borders.count +
          pl->theta.count + pl->jitter.count + pl->out.count) *
             sizeof(double) +
         (pl->factors_f.count + pl->borders_f.count) * sizeof(float) +
         (pl->status.count + pl->slots.count + pl->flags.count + 2) * sizeof(int);
}

int gpemu_eval_batch_device(gpemu_plan* pl, const double* d_theta, size_t B, double* d_out) {
  GPEMU_GUARD_BEGIN
  if (!pl || !d_theta) return set_error(GPEMU_VALIDATION, "eval_batch_device: null argument");
  if (B == 0) return GPEMU_OK;
  if (B > pl->max_batch) return set_error(GPEMU_VALIDATION, "eval_batch: B = %zu exceeds max_batch %zu", B, pl->max_batch);
  ck(cudaSetDevice(pl->ctx->device), "cudaSetDevice");
  cudaStream_t s = pl->ctx->stream;
  ck(cudaMemcpyAsync(pl->theta.p, d_theta, B * pl->d * sizeof(double), cudaMemcpyDeviceToDevice, s),
     "D2D theta");
  int rc = run_batch(pl, B);
  if (rc) return rc;
  if (d_out)
    ck(cudaMemcpyAsync(d_out, pl->out.p, B * REC_SIZE * sizeof(double), cudaMemcpyDeviceToDevice, s),
       "D2D out");
  return GPEMU_OK;
  GPEMU_GUARD_END
}

int gpemu_eval_batch(gpemu_plan* pl, const double* theta, size_t B, double* neg2, double* mu,
                     double* sigma2, double* jitter, double* log_det, int* slot_status) {
  GPEMU_GUARD_BEGIN
  if (!pl || (!theta && B)) return set_error(GPEMU_VALIDATION, "eval_batch: null argument");
  if (B == 0) return GPEMU_OK;
  if (B > pl->max_batch) return set_error(GPEMU_VALIDATION, "eval_batch: B = %zu exceeds max_batch %zu", B, pl->max_batch);
  ck(cudaSetDevice(pl->ctx->device), "cudaSetDevice");
  ck(cudaMemcpyAsync(pl->theta.p, theta, B * pl->d * sizeof(double), cudaMemcpyHostToDevice,
                     pl->ctx->stream),
     "H2D theta");
  int rc = run_batch(pl, B);
  if (rc) return rc;
  download_records(pl, B);
  for (size_t b = 0; b < B; ++b) {
    const double* r = &pl->h_out[b * REC_SIZE];
    if (neg2) neg2[b] = r[REC_NEG2];
    if (mu) mu[b] = r[REC_MU];
    if (sigma2) sigma2[b] = r[REC_SIGMA2];
    if (jitter) jitter[b] = r[REC_JITTER];
    if (log_det) log_det[b] = r[REC_LOGDET];
    if (slot_status) slot_status[b] = (int)r[REC_STATUS];
  }
  return GPEMU_OK;
  GPEMU_GUARD_END
}

int gpemu_plan_set_profiling(gpemu_plan* pl, int enable) {
  if (!pl) return set_error(GPEMU_VALIDATION, "null plan");
  cudaStreamSynchronize(pl->ctx->stream);
  pl->clear_marks();
  pl->profile = enable != 0;
  return GPEMU_OK;
}

int gpemu_plan_phase_ms(gpemu_plan* pl, int phase, double* total_ms, int* launches) {
  GPEMU_GUARD_BEGIN
  if (!pl || !total_ms) return set_error(GPEMU_VALIDATION, "null argument");
  ck(cudaStreamSynchronize(pl->ctx->stream), "phase_ms");
  double t = 0.0;
  int c = 0;
  for (auto& m : pl->marks) {
    if (m.kind != phase) continue;
    float ms = 0.0f;
    ck(cudaEventElapsedTime(&ms, m.a, m.b), "cudaEventElapsedTime");
    t += ms;
    ++c;
  }
  *total_ms = t;
  if (launches) *launches = c;
  return GPEMU_OK;
  GPEMU_GUARD_END
}

int gpemu_ticket_order(int B, int NT, int procs, int* out, size_t out_len) {
  GPEMU_GUARD_BEGIN
  if (B < 1 || B >= (1 << 15) || NT < 1 || NT > 256 || procs < 1 || !out)
    return set_error(GPEMU_VALIDATION, "ticket_order: bad arguments");
  const size_t need = (size_t)B * NT * (NT + 1) / 2;
  if (out_len < need) return set_error(GPEMU_VALIDATION, "ticket_order: out needs %zu entries", need);
  const std::vector<int> ord = ticket_order(B, NT, procs);
  std::copy(ord.begin(), ord.end(), out);
  return GPEMU_OK;
  GPEMU_GUARD_END
}

int gpemu_plan_dag_profile(gpemu_plan* pl, int enable, uint64_t* out, size_t out_len) {
  GPEMU_GUARD_BEGIN
  if (!pl) return set_error(GPEMU_VALIDATION, "null plan");
  const size_t len = (size_t)pl->ctx->num_sms * 24 + 256 + (size_t)kTraceTasks * 4;
  if (out && pl->dag_prof.p) {
    ck(cudaStreamSynchronize(pl->ctx->stream), "dag_profile");
    d2h_sync(out, pl->dag_prof.p, std::min(out_len, len) * sizeof(uint64_t), pl->ctx->stream,
             "D2H prof");
  }
  if (enable && !pl->dag_prof.p) {
    pl->dag_prof.alloc(len);
  }
  if (enable) ck(cudaMemsetAsync(pl->dag_prof.p, 0, len * sizeof(uint64_t), pl->ctx->stream), "memset prof");
  if (!enable) pl->dag_prof.free();
  return GPEMU_OK;
  GPEMU_GUARD_END
}

int gpemu_plan_last_factor(gpemu_plan* pl, size_t slot, double* L_out, double* log_det,
                           double* jitter_used) {
  GPEMU_GUARD_BEGIN
  if (!pl) return set_error(GPEMU_VALIDATION, "last_factor: null plan");
  if (slot >= pl->last_B) return set_error(GPEMU_VALIDATION, "last_factor: slot %zu not in the last batch", slot);
  if (pl->last_ladder[slot] < 0) return set_error(GPEMU_NOT_PD, "last_factor: slot %zu did not factorize", slot);
  const size_t fs = (size_t)pl->fslot[slot];  // the slot that holds this candidate's factor
  cudaStream_t s = pl->ctx->stream;
  if (L_out) {
    DevBuf<double> dL;
    own(&pl->ctx->stream, dL);
    dL.alloc((size_t)pl->n * pl->n);
    if (pl->precision == GPEMU_PRECISION_SINGLE)
      launch_tiles_f32_to_rowmajor(pl->factors_f.p + fs * pl->slot_stride, pl->n, pl->NT, dL.p, s);
    else
      launch_tiles_to_rowmajor(pl->factors.p + fs * pl->slot_stride, pl->n, pl->NT, dL.p, s);
    pl->ctx->launches += 1;
    ck(cudaMemcpyAsync(L_out, dL.p, (size_t)pl->n * pl->n * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H L");
  }
  double rec[REC_SIZE];
  ck(cudaMemcpyAsync(rec, pl->out.p + slot * REC_SIZE, sizeof(rec), cudaMemcpyDeviceToHost, s), "D2H rec");
  ck(cudaStreamSynchronize(s), "last_factor");
  if (log_det) *log_det = rec[REC_LOGDET];
  if (jitter_used) *jitter_used = kLadder[pl->last_ladder[slot]];
  return GPEMU_OK;
  GPEMU_GUARD_END
}

// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// The reference GA (optimizer.hpp:93-187) as a host state machine: population of the
// current generation out, its fitness in. Identical candidate sequence to the sequential
// reference for any evaluation order / batch split; also tracks the fit_gp_detailed stash
// (likelihood.hpp:257-273: strict <, earliest (generation, slot) wins).
struct gpemu_ga {
  int d = 0, P = 0, G = 0, gen = 0;
  gpemu_ga_config cfg{};
  uint64_t ga_seed = 0;
  double mut_prob = 0.0;
  std::vector<double> glo, ghi;
  std::vector<std::vector<double>> pop;
  std::vector<double> fitness;
  double best_value = INFINITY;  // GA incumbent (record_generation, optimizer.hpp:133-141)
  std::vector<double> best_point;
  double stash_value = INFINITY;  // evaluation stash
  int stash_gen = -1, stash_slot = -1;
  std::vector<double> trace_best, trace_genes;

  void init_population() {
    Rng init_rng(derive_seed(ga_seed, 0x1e17u));
    pop.assign(P, std::vector<double>(d));
    std::vector<int> perm(P);
    for (int k = 0; k < d; ++k) {
      std::iota(perm.begin(), perm.end(), 0);
      for (int i = P - 1; i > 0; --i) {
        const int j = (int)init_rng.below((uint64_t)i + 1);
        std::swap(perm[i], perm[j]);
      }
      const double width = ghi[k] - glo[k];
      for (int i = 0; i < P; ++i) {
        const double u = (perm[i] + init_rng.uniform01()) / P;
        pop[i][k] = glo[k] + width * u;
      }
    }
  }

  void thetas(double* out) const {  // likelihood.hpp:265
    for (int i = 0; i < P; ++i)
      for (int k = 0; k < d; ++k) out[(size_t)i * d + k] = std::pow(10.0, pop[i][k]);
  }

  // Records the generation (stash + trace) and breeds the next one.
  void tell(const double* f) {
    fitness.assign(f, f + P);
    for (int i = 0; i < P; ++i) {
      if (fitness[i] < stash_value) {
        stash_value = fitness[i];
        stash_gen = gen;
        stash_slot = i;
      }
    }
    int b = 0;
    for (int i = 1; i < P; ++i)
      if (fitness[i] < fitness[b]) b = i;
    if (fitness[b] < best_value) {
      best_value = fitness[b];
      best_point = pop[b];
    }
    trace_best.push_back(fitness[b]);
    trace_genes.insert(trace_genes.end(), pop[b].begin(), pop[b].end());
    ++gen;
    if (gen >= G) return;
    std::vector<std::vector<double>> next(P);
    std::vector<int> order(P);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int c) { return fitness[a] < fitness[c]; });
    for (int e = 0; e < cfg.elitism; ++e) next[e] = pop[order[e]];
    for (int slot = cfg.elitism; slot < P; ++slot) {
      Rng rng(derive_seed(ga_seed, (uint64_t)gen, (uint64_t)slot));
      auto tournament = [&]() -> const std::vector<double>& {
        const int a = (int)rng.below(P);
        const int c = (int)rng.below(P);
        const bool a_wins = fitness[a] < fitness[c] || (fitness[a] == fitness[c] && a <= c);
        return pop[a_wins ? a : c];
      };
      const auto& pa = tournament();
      const auto& pb = tournament();
      std::vector<double> child(d);
      if (rng.uniform01() < cfg.crossover_rate) {
        for (int k = 0; k < d; ++k) child[k] = rng.uniform01() < 0.5 ? pa[k] : pb[k];
      } else {
        child = pa;
      }
      for (int k = 0; k < d; ++k) {
        if (rng.uniform01() < mut_prob) child[k] += cfg.mutation_sigma * rng.normal();
        child[k] = std::clamp(child[k], glo[k], ghi[k]);
      }
      next[slot] = std::move(child);
    }
    pop = std::move(next);
  }
};

static int ga_setup(gpemu_ga* g, size_t d, const double* lo, const double* hi,
                    const gpemu_ga_config* gac, uint64_t seed) {
  const int P = gac->population, G = gac->generations;
  // GaConfig::validate (optimizer.hpp:29-38)
  if (P <= 0 || G <= 0) return set_error(GPEMU_VALIDATION, "GaConfig: population and generations must be positive");
  if (gac->crossover_rate < 0.0 || gac->crossover_rate > 1.0) return set_error(GPEMU_VALIDATION, "GaConfig: crossover_rate must be in [0,1]");
  if (!(gac->mutation_sigma > 0.0)) return set_error(GPEMU_VALIDATION, "GaConfig: mutation_sigma must be positive");
  if (gac->mutation_prob < 0.0 || gac->mutation_prob > 1.0) return set_error(GPEMU_VALIDATION, "GaConfig: mutation_prob must be in [0,1]");
  if (gac->elitism < 0 || gac->elitism >= P) return set_error(GPEMU_VALIDATION, "GaConfig: elitism must be in [0, population)");
  if (d == 0) return set_error(GPEMU_VALIDATION, "ga_minimize: empty bounds");
  g->d = (int)d;
  g->P = P;
  g->G = G;
  g->cfg = *gac;
  g->glo.resize(d);
  g->ghi.resize(d);
  // FitConfig::bounds_for (core.hpp:114-123) + log10 box (likelihood.hpp:247-251)
  for (size_t k = 0; k < d; ++k) {
    if (!(lo[k] > 0.0) || !(lo[k] < hi[k])) return set_error(GPEMU_VALIDATION, "FitConfig: theta bounds require 0 < lower < upper");
    g->glo[k] = std::log10(lo[k]);
    g->ghi[k] = std::log10(hi[k]);
    if (!(g->glo[k] < g->ghi[k]) || !std::isfinite(g->glo[k]) || !std::isfinite(g->ghi[k]))
      return set_error(GPEMU_VALIDATION, "ga_minimize: degenerate bounds");
  }
  g->ga_seed = derive_seed(seed, 0x9a5eedull);  // likelihood.hpp:276
  g->mut_prob = gac->mutation_prob > 0.0 ? gac->mutation_prob : 1.0 / (double)d;
  g->init_population();
  return GPEMU_OK;
}

int gpemu_ga_create(size_t d, const double* lo, const double* hi, const gpemu_ga_config* cfg,
                    uint64_t seed, gpemu_ga** out) {
  if (!lo || !hi || !cfg || !out) return set_error(GPEMU_VALIDATION, "ga_create: null argument");
  auto* g = new gpemu_ga();
  int rc = ga_setup(g, d, lo, hi, cfg, seed);
  if (rc) {
    delete g;
    return rc;
  }
  *out = g;
  return GPEMU_OK;
}

int gpemu_ga_destroy(gpemu_ga* g) {
  delete g;
  return GPEMU_OK;
}

int gpemu_ga_thetas(const gpemu_ga* g, double* thetas) {
  if (!g || !thetas) return set_error(GPEMU_VALIDATION, "ga_thetas: null argument");
  if (g->gen >= g->G) return set_error(GPEMU_VALIDATION, "ga_thetas: the GA is finished");
  g->thetas(thetas);
  return GPEMU_OK;
}

int gpemu_ga_tell(gpemu_ga* g, const double* fitness) {
  if (!g || !fitness) return set_error(GPEMU_VALIDATION, "ga_tell: null argument");
  if (g->gen >= g->G) return set_error(GPEMU_VALIDATION, "ga_tell: the GA is finished");
  g->tell(fitness);
  return GPEMU_OK;
}

int gpemu_ga_status(const gpemu_ga* g, int* generation, int* done, double* best_value,
                    double* best_theta, int* stash_generation, int* stash_slot,
                    double* trace_best, double* trace_genes) {
  if (!g) return set_error(GPEMU_VALIDATION, "ga_status: null argument");
  if (generation) *generation = g->gen;
  if (done) *done = g->gen >= g->G;
  if (best_value) *best_value = g->best_value;
  if (best_theta && !g->best_point.empty())
    for (int k = 0; k < g->d; ++k) best_theta[k] = std::pow(10.0, g->best_point[k]);
  if (stash_generation) *stash_generation = g->stash_gen;
  if (stash_slot) *stash_slot = g->stash_slot;
  if (trace_best) std::copy(g->trace_best.begin(), g->trace_best.end(), trace_best);
  if (trace_genes) std::copy(g->trace_genes.begin(), g->trace_genes.end(), trace_genes);
  return GPEMU_OK;
}

// ---------------------------------------------------------------------------
// Candidate sharding over several plans (one per device; optimizer.hpp:86-92 allows the
// population to be evaluated in parallel, :116-121). A generation's P candidates split into
// contiguous ranges of ceil(P/G); each plan evaluates its range in chunks of its max_batch on
// its own host thread, and the records come back in slot order. No device-to-device traffic:
// every plan holds the whole dataset and the winning factor stays on the device that made it.
namespace {

struct ShardOut {
  int rc = GPEMU_OK;
  std::string err;
  int best_i = -1;  // global candidate index of the shard's best below the threshold
  double best = INFINITY;
  std::vector<double> best_rec;
  double jitter_max = 0.0;
};

bool same_dataset(const gpemu_plan* a, const gpemu_plan* b) {
  return a->n == b->n && a->d == b->d && a->p == b->p && a->nugget == b->nugget &&
         a->precision == b->precision && a->data_hash == b->data_hash;
}

// Copies a slot's factor + border rows into the plan's stash slot (max_batch).
void keep_factor(gpemu_plan* pl, int slot) {
  cudaStream_t s = pl->ctx->stream;
  const size_t stash = pl->max_batch;
  if (pl->precision == GPEMU_PRECISION_SINGLE) {
    ck(cudaMemcpyAsync(pl->factors_f.p + stash * pl->slot_stride, pl->factors_f.p + (size_t)slot * pl->slot_stride,
                       pl->slot_stride * sizeof(float), cudaMemcpyDeviceToDevice, s), "stash factor");
    ck(cudaMemcpyAsync(pl->borders_f.p + stash * 2 * pl->Npad, pl->borders_f.p + (size_t)slot * 2 * pl->Npad,
                       2 * pl->Npad * sizeof(float), cudaMemcpyDeviceToDevice, s), "stash border");
  } else {
    ck(cudaMemcpyAsync(pl->factors.p + stash * pl->slot_stride, pl->factors.p + (size_t)slot * pl->slot_stride,
                       pl->slot_stride * sizeof(double), cudaMemcpyDeviceToDevice, s), "stash factor");
    ck(cudaMemcpyAsync(pl->borders.p + stash * 2 * pl->Npad, pl->borders.p + (size_t)slot * 2 * pl->Npad,
                       2 * pl->Npad * sizeof(double), cudaMemcpyDeviceToDevice, s), "stash border");
  }
}

// Evaluates candidates [c0, c1) of a generation on one plan, in chunks of max_batch; fitness
// lands in fitness[c0..c1). With keep, the shard's best candidate strictly below `threshold`
// (earliest wins ties, likelihood.hpp:267) has its factor saved in the stash slot before a
// later chunk reuses its slot.
void eval_shard(gpemu_plan* pl, const double* thetas, int c0, int c1, double threshold, bool keep,
                double* fitness, double* recs, ShardOut* out) {
  try {
    ck(cudaSetDevice(pl->ctx->device), "cudaSetDevice");
    cudaStream_t s = pl->ctx->stream;
    const int d = pl->d, MB = (int)pl->max_batch;
    double best = threshold;
    for (int a = c0; a < c1; a += MB) {
      const int cn = std::min(MB, c1 - a);
      ck(cudaMemcpyAsync(pl->theta.p, thetas + (size_t)a * d, (size_t)cn * d * sizeof(double),
                         cudaMemcpyHostToDevice, s),
         "H2D theta");
      const int rc = run_batch(pl, cn);
      if (rc) {
        out->rc = rc;
        out->err = g_last_error;
        return;
      }
      download_records(pl, cn);
      int chunk_best = -1;
      for (int q = 0; q < cn; ++q) {
        const int i = a + q;
        const double* r = &pl->h_out[(size_t)q * REC_SIZE];
        fitness[i] = r[REC_NEG2];
        if (recs) std::copy(r, r + REC_SIZE, recs + (size_t)i * REC_SIZE);
        if (pl->last_ladder[q] >= 0) out->jitter_max = std::max(out->jitter_max, kLadder[pl->last_ladder[q]]);
        if (fitness[i] < best) {
          best = fitness[i];
          out->best_i = i;
          chunk_best = q;
        }
      }
      if (chunk_best >= 0) {
        const double* r = &pl->h_out[(size_t)chunk_best * REC_SIZE];
        out->best = best;
        out->best_rec.assign(r, r + REC_SIZE);
        if (keep) keep_factor(pl, pl->fslot[chunk_best]);
      }
    }
  } catch (const CudaError& e) {
    out->rc = GPEMU_CUDA;
    out->err = e.msg;
  } catch (const std::bad_alloc&) {
    out->rc = GPEMU_ERROR;
    out->err = "host allocation failed";
  }
}

// Runs eval_shard for every plan (plan k gets range k of ceil(P/G)) on G host threads.
int eval_sharded(gpemu_plan* const* plans, int G, const double* thetas, int P, double threshold,
                 bool keep, double* fitness, double* recs, std::vector<ShardOut>& outs) {
  const int S = (P + G - 1) / G;
  outs.assign(G, ShardOut{});
  if (G == 1) {
    eval_shard(plans[0], thetas, 0, P, threshold, keep, fitness, recs, &outs[0]);
  } else {
    std::vector<std::thread> ts;
    for (int k = 0; k < G; ++k) {
      const int c0 = std::min(P, k * S), c1 = std::min(P, (k + 1) * S);
      ts.emplace_back(eval_shard, plans[k], thetas, c0, c1, threshold, keep, fitness, recs, &outs[k]);
    }
    for (auto& t : ts) t.join();
  }
  for (auto& o : outs)
    if (o.rc) return set_error(o.rc, "%s", o.err.c_str());
  return GPEMU_OK;
}

int check_plans(gpemu_plan* const* plans, int G, const char* who) {
  if (!plans || G < 1) return set_error(GPEMU_VALIDATION, "%s: need at least one plan", who);
  for (int k = 0; k < G; ++k) {
    if (!plans[k]) return set_error(GPEMU_VALIDATION, "%s: null plan %d", who, k);
    if (!same_dataset(plans[0], plans[k]))
      return set_error(GPEMU_VALIDATION, "%s: plan %d holds a different dataset / p / nugget / precision", who, k);
  }
  return GPEMU_OK;
}

}  // namespace

int gpemu_eval_batch_multi(gpemu_plan* const* plans, int G, const double* theta, size_t B,
                           double* neg2, double* mu, double* sigma2, double* jitter,
                           double* log_det, int* slot_status) {
  GPEMU_GUARD_BEGIN
  int rc = check_plans(plans, G, "eval_batch_multi");
  if (rc) return rc;
  if (!theta && B) return set_error(GPEMU_VALIDATION, "eval_batch_multi: null theta");
  if (B == 0) return GPEMU_OK;
  std::vector<double> fit(B), recs(B * REC_SIZE);
  std::vector<ShardOut> outs;
  rc = eval_sharded(plans, G, theta, (int)B, -INFINITY, false, fit.data(), recs.data(), outs);
  if (rc) return rc;
  for (size_t b = 0; b < B; ++b) {
    const double* r = &recs[b * REC_SIZE];
    if (neg2) neg2[b] = r[REC_NEG2];
    if (mu) mu[b] = r[REC_MU];
    if (sigma2) sigma2[b] = r[REC_SIGMA2];
    if (jitter) jitter[b] = r[REC_JITTER];
    if (log_det) log_det[b] = r[REC_LOGDET];
    if (slot_status) slot_status[b] = (int)r[REC_STATUS];
  }
  return GPEMU_OK;
  GPEMU_GUARD_END
}

int gpemu_fit_multi(gpemu_plan* const* plans, int G, const double* lo, const double* hi,
                    const gpemu_ga_config* gac, uint64_t seed, gpemu_fit_result* res,
                    double* theta_hat, double* alpha, double* trace_best, double* trace_genes,
                    gpemu_model** model_out) {
  GPEMU_GUARD_BEGIN
  int rc = check_plans(plans, G, "fit");
  if (rc) return rc;
  if (!lo || !hi || !gac) return set_error(GPEMU_VALIDATION, "fit: null argument");
  gpemu_ga ga;
  rc = ga_setup(&ga, plans[0]->d, lo, hi, gac, seed);
  if (rc) return rc;
  const int d = plans[0]->d, P = ga.P;
  std::vector<double> thetas((size_t)P * d), fitness(P), stash_theta(d), stash_rec(REC_SIZE, 0.0);
  int stash_dev = -1;
  double jitter_max = 0.0;
  std::vector<ShardOut> outs;
  while (ga.gen < ga.G) {
    nvtx_push("gpemu GA generation");
    // the objective (likelihood.hpp:264-273) over the generation: one batch per shard chunk
    ga.thetas(thetas.data());
    const double prev_stash = ga.stash_value;
    rc = eval_sharded(plans, G, thetas.data(), P, prev_stash, true, fitness.data(), nullptr, outs);
    nvtx_pop();
    if (rc) return rc;
    int best_i = -1, best_k = -1;
    double best = prev_stash;
    for (int k = 0; k < G; ++k) {  // shards in slot order: strict < keeps the earliest slot
      jitter_max = std::max(jitter_max, outs[k].jitter_max);
      if (outs[k].best_i >= 0 && outs[k].best < best) {
        best = outs[k].best;
        best_i = outs[k].best_i;
        best_k = k;
      }
    }
    if (best_i >= 0) {
      stash_dev = best_k;
      stash_rec = outs[best_k].best_rec;
      std::copy(&thetas[(size_t)best_i * d], &thetas[(size_t)best_i * d] + d, stash_theta.begin());
    }
    const int gen_now = ga.gen;
    ga.tell(fitness.data());
    const bool improved = ga.stash_value < prev_stash && ga.stash_gen == gen_now;
    if (improved != (best_i >= 0) || (improved && ga.stash_slot != best_i))
      return set_error(GPEMU_ERROR, "fit: evaluation stash diverged from the optimizer's");
  }
  for (int k = 0; k < G; ++k) ck(cudaStreamSynchronize(plans[k]->ctx->stream), "fit");
  if (!std::isfinite(ga.stash_value) || stash_dev < 0)
    return set_error(GPEMU_FIT, "fit_gp: every candidate failed factorization (n = %d)", plans[0]->n);
  if (ga.best_value != ga.stash_value)
    return set_error(GPEMU_ERROR, "fit_gp: optimizer incumbent diverged from evaluation stash");
  gpemu_plan* owner = plans[stash_dev];  // the model is built where the winning factor lives
  ck(cudaSetDevice(owner->ctx->device), "cudaSetDevice");
  gpemu_model* m = make_model(owner, (int)owner->max_batch, stash_theta.data(), stash_rec.data());
  if (theta_hat) std::copy(stash_theta.begin(), stash_theta.end(), theta_hat);
  if (alpha) d2h_sync(alpha, m->alpha.p, owner->n * sizeof(double), m->ctx->stream, "D2H alpha");
  if (trace_best) std::copy(ga.trace_best.begin(), ga.trace_best.end(), trace_best);
  if (trace_genes) std::copy(ga.trace_genes.begin(), ga.trace_genes.end(), trace_genes);
  if (res) {
    res->neg2_log_lik = stash_rec[REC_NEG2];
    res->mu_hat = stash_rec[REC_MU];
    res->sigma2_hat = stash_rec[REC_SIGMA2];
    res->jitter_max = jitter_max;
    res->r_builds = res->factorizations = res->triangular_solves = 0;
    for (int k = 0; k < G; ++k) {
      res->r_builds += plans[k]->r_builds;
      res->factorizations += plans[k]->factorizations;
      res->triangular_solves += plans[k]->solves;
    }
  }
  if (model_out) {
    *model_out = m;
  } else {
    release(m);
  }
  return GPEMU_OK;
  GPEMU_GUARD_END
}

int gpemu_fit(gpemu_plan* pl, const double* lo, const double* hi, const gpemu_ga_config* gac,
              uint64_t seed, gpemu_fit_result* res, double* theta_hat, double* alpha,
              double* trace_best, double* trace_genes, gpemu_model** model_out) {
  if (!pl) return set_error(GPEMU_VALIDATION, "fit: null argument");
  return gpemu_fit_multi(&pl, 1, lo, hi, gac, seed, res, theta_hat, alpha, trace_best, trace_genes,
                         model_out);
}

// bench.hpp:302-383 detail::refine_fit: coordinate-wise golden-section polish, `budget`
// sequential single-candidate device evaluations; on improvement the model is rebuilt at
// the refined theta (one more evaluation + alpha, as bench.hpp:363-382).
int gpemu_refine_fit(gpemu_plan* pl, const double* lo, const double* hi, const double* theta_fit,
                     double neg2_fit, int budget, double* theta_out, double* neg2_out,
                     int* evals_out, gpemu_model** model_out, double* scalars, double* alpha) {
  return gpemu_refine_fit_ex(pl, pl, lo, hi, theta_fit, neg2_fit, budget, theta_out, neg2_out,
                             evals_out, model_out, scalars, alpha);
}

// bench.hpp:302-383 with the polish evaluations on `pl` (double precision regardless of the
// run precision, bench.hpp:300-301) and the model rebuilt on `rebuild` in the run's own
// precision (bench.hpp:363-382).
int gpemu_refine_fit_ex(gpemu_plan* pl, gpemu_plan* rebuild, const double* lo, const double* hi,
                        const double* theta_fit, double neg2_fit, int budget, double* theta_out,
                        double* neg2_out, int* evals_out, gpemu_model** model_out, double* scalars,
                        double* alpha) {
  GPEMU_GUARD_BEGIN
  NvtxRange range("refine_fit polish");
  if (!rebuild) rebuild = pl;
  if (!pl || pl->d != rebuild->d || pl->n != rebuild->n)
    return set_error(GPEMU_VALIDATION, "refine_fit: polish and rebuild plans must share the dataset");
  if (!pl || !lo || !hi || !theta_fit) return set_error(GPEMU_VALIDATION, "refine_fit: null argument");
  const int d = pl->d;
  for (int k = 0; k < d; ++k)
    if (!(lo[k] > 0.0) || !(lo[k] < hi[k])) return set_error(GPEMU_VALIDATION, "FitConfig: theta bounds require 0 < lower < upper");
  cudaStream_t s = pl->ctx->stream;
  std::vector<double> best(d), g(d), theta(d);
  for (int k = 0; k < d; ++k) best[k] = std::log10(theta_fit[k]);
  double best_value = neg2_fit;
  int used = 0;
  int rc = GPEMU_OK;
  constexpr double kInvPhi = 0.6180339887498949;
  constexpr double kHalfWidth = 0.25;  // log10 units around the incumbent
  // the two golden-section moves (bench.hpp:302-383), shared by the polish and its speculation
  auto move_left = [&](double& a, double& b, double& x1, double& x2) {
    b = x2;
    x2 = x1;
    x1 = b - kInvPhi * (b - a);
    return x1;
  };
  auto move_right = [&](double& a, double& b, double& x1, double& x2) {
    a = x1;
    x1 = x2;
    x2 = a + kInvPhi * (b - a);
    return x2;
  };
  // Speculation: a coordinate's polish is 2 evaluations plus 2 golden-section steps, each
  // step choosing between two points known in advance, so the 2 + 2 + 4 points of its
  // decision tree are evaluated in ONE batch and the sequential algorithm below replays
  // against those records. Batch invariance makes every record bitwise the value a B=1
  // evaluation returns, so theta, -2logL and the evaluation count are the sequential
  // polish's; only the points the replay visits count (the plan's ledger is restored to
  // that count). Needs 8 slots; smaller plans evaluate one candidate at a time.
  const bool spec = pl->max_batch >= 8;
  const uint64_t led_r = pl->r_builds, led_f = pl->factorizations, led_s = pl->solves;
  // the ledger counts the polish's evaluations, not the speculative extras, on every exit path
  struct LedgerRestore {
    gpemu_plan* pl;
    bool on;
    uint64_t r, f, s;
    const int* used;
    void apply() {
      if (!on) return;
      on = false;
      pl->r_builds = r + *used;
      pl->factorizations = f + *used;
      pl->solves = s + 2 * (uint64_t)*used;
    }
    ~LedgerRestore() { apply(); }
  } led_restore{pl, spec, led_r, led_f, led_s, &used};
  double sp_x[8], sp_v[8];
  int sp_n = 0, sp_k = -1;
  auto speculate = [&](int k, double a, double b, double x1, double x2) {
    double pts[8];
    pts[0] = x1;
    pts[1] = x2;
    double aL = a, bL = b, x1L = x1, x2L = x2, aR = a, bR = b, x1R = x1, x2R = x2;
    pts[2] = move_left(aL, bL, x1L, x2L);
    pts[3] = move_right(aR, bR, x1R, x2R);
    {
      double a2 = aL, b2 = bL, y1 = x1L, y2 = x2L;
      pts[4] = move_left(a2, b2, y1, y2);
    }
    {
      double a2 = aL, b2 = bL, y1 = x1L, y2 = x2L;
      pts[5] = move_right(a2, b2, y1, y2);
    }
    {
      double a2 = aR, b2 = bR, y1 = x1R, y2 = x2R;
      pts[6] = move_left(a2, b2, y1, y2);
    }
    {
      double a2 = aR, b2 = bR, y1 = x1R, y2 = x2R;
      pts[7] = move_right(a2, b2, y1, y2);
    }
    std::vector<double> th((size_t)8 * d);
    for (int i = 0; i < 8; ++i)
      for (int q = 0; q < d; ++q) th[(size_t)i * d + q] = std::pow(10.0, q == k ? pts[i] : best[q]);
    ck(cudaMemcpyAsync(pl->theta.p, th.data(), th.size() * sizeof(double), cudaMemcpyHostToDevice, s),
       "H2D theta");
    rc = run_batch(pl, 8, /*tolerate_nonfinite=*/true);
    if (rc) return;
    download_records(pl, 8);
    sp_n = 0;
    for (int i = 0; i < 8; ++i) {
      // a non-finite point is left out: if the replay visits it, it is evaluated on its own
      // and fails as the sequential polish does
      if (pl->h_out[(size_t)i * REC_SIZE + REC_STATUS] == 2.0) continue;
      sp_x[sp_n] = pts[i];
      sp_v[sp_n] = pl->h_out[(size_t)i * REC_SIZE + REC_NEG2];
      ++sp_n;
    }
    sp_k = k;
  };
  auto eval_genes = [&](const std::vector<double>& genes, int k) -> double {
    ++used;
    double v = INFINITY;
    int hit = -1;
    if (sp_k == k)
      for (int i = 0; i < sp_n && hit < 0; ++i)
        if (sp_x[i] == genes[k]) hit = i;
    if (hit >= 0) {
      v = sp_v[hit];
    } else {
      for (int q = 0; q < d; ++q) theta[q] = std::pow(10.0, genes[q]);
      ck(cudaMemcpyAsync(pl->theta.p, theta.data(), d * sizeof(double), cudaMemcpyHostToDevice, s),
         "H2D theta");
      rc = run_batch(pl, 1);
      if (rc) return INFINITY;
      download_records(pl, 1);
      v = pl->h_out[REC_NEG2];
    }
    if (v < best_value) {
      best_value = v;
      best = genes;
    }
    return v;
  };
  int k = 0;
  while (used < budget) {
    g = best;
    double a = std::max(std::log10(lo[k]), best[k] - kHalfWidth);
    double b = std::min(std::log10(hi[k]), best[k] + kHalfWidth);
    double x1 = b - kInvPhi * (b - a);
    double x2 = a + kInvPhi * (b - a);
    sp_k = -1;
    if (spec && budget - used >= 2) {
      speculate(k, a, b, x1, x2);
      if (rc) return rc;
    }
    g[k] = x1;
    double f1 = eval_genes(g, k);
    if (rc) return rc;
    if (used >= budget) break;
    g[k] = x2;
    double f2 = eval_genes(g, k);
    if (rc) return rc;
    for (int step = 0; step < 2 && used < budget; ++step) {
      if (f1 <= f2) {
        f2 = f1;
        g[k] = move_left(a, b, x1, x2);
        f1 = eval_genes(g, k);
      } else {
        f1 = f2;
        g[k] = move_right(a, b, x1, x2);
        f2 = eval_genes(g, k);
      }
      if (rc) return rc;
    }
    k = (k + 1) % d;
  }
  led_restore.apply();  // before the model rebuild adds its own evaluation
  for (int q = 0; q < d; ++q) theta[q] = std::pow(10.0, best[q]);
  if (theta_out) std::copy(theta.begin(), theta.end(), theta_out);
  if (neg2_out) *neg2_out = best_value;
  if (evals_out) *evals_out = used;
  if (model_out) {
    *model_out = nullptr;
    if (best_value < neg2_fit) {
      gpemu_plan* rb = rebuild;
      ck(cudaMemcpyAsync(rb->theta.p, theta.data(), d * sizeof(double), cudaMemcpyHostToDevice,
                         rb->ctx->stream), "H2D theta");
      rc = run_batch(rb, 1);
      if (rc) return rc;
      download_records(rb, 1);
      if (std::isfinite(rb->h_out[REC_NEG2]) && rb->h_out[REC_NEG2] < neg2_fit) {
        gpemu_model* m = make_model(rb, rb->fslot[0], theta.data(), rb->h_out.data());
        if (scalars) {
          scalars[0] = m->neg2;
          scalars[1] = m->mu;
          scalars[2] = m->sigma2;
          scalars[3] = m->jitter;
        }
        if (alpha) d2h_sync(alpha, m->alpha.p, pl->n * sizeof(double), m->ctx->stream, "D2H alpha");
        *model_out = m;
      }
    }
  }
  return GPEMU_OK;
  GPEMU_GUARD_END
}

int gpemu_model_at_theta(gpemu_plan* pl, const double* theta, gpemu_model** model_out,
                         double* scalars, double* alpha) {
  GPEMU_GUARD_BEGIN
  if (!pl || !theta) return set_error(GPEMU_VALIDATION, "model_at_theta: null argument");
  cudaStream_t s = pl->ctx->stream;
  ck(cudaMemcpyAsync(pl->theta.p, theta, pl->d * sizeof(double), cudaMemcpyHostToDevice, s), "H2D theta");
  int rc = run_batch(pl, 1);
  if (rc) return rc;
  download_records(pl, 1);
  const double* r = pl->h_out.data();
  if (!std::isfinite(r[REC_NEG2]))
    return set_error(GPEMU_NOT_PD, "model_at_theta: factorization failed at the requested theta");
  gpemu_model* m = make_model(pl, pl->fslot[0], theta, r);
  if (scalars) {
    scalars[0] = m->neg2;
    scalars[1] = m->mu;
    scalars[2] = m->sigma2;
    scalars[3] = m->jitter;
  }
  if (alpha) d2h_sync(alpha, m->alpha.p, pl->n * sizeof(double), m->ctx->stream, "D2H alpha");
  if (model_out) {
    *model_out = m;
  } else {
    release(m);
  }
  return GPEMU_OK;
  GPEMU_GUARD_END
}

int gpemu_model_scalars(const gpemu_model* m, double* out) {
  if (!m || !out) return set_error(GPEMU_VALIDATION, "model_scalars: null argument");
  out[0] = m->neg2;
  out[1] = m->mu;
  out[2] = m->sigma2;
  out[3] = m->jitter;
  return GPEMU_OK;
}

int gpemu_model_destroy(gpemu_model* m) {
  release(m);
  return GPEMU_OK;
}

int gpemu_model_factor(gpemu_model* m, double* L_out, double* log_det) {
  GPEMU_GUARD_BEGIN
  if (!m) return set_error(GPEMU_VALIDATION, "model_factor: null model");
  if (log_det) *log_det = m->log_det;
  if (!L_out) return GPEMU_OK;
  ck(cudaSetDevice(m->ctx->device), "cudaSetDevice");
  cudaStream_t s = m->ctx->stream;
  DevBuf<double> dL;
  own(&m->ctx->stream, dL);
  dL.alloc((size_t)m->n * m->n);
  launch_tiles_to_rowmajor(m->tiles.p, m->n, m->NT, dL.p, s);
  m->ctx->launches += 1;
  ck(cudaGetLastError(), "tiles_to_rowmajor launch");
  d2h_sync(L_out, dL.p, (size_t)m->n * m->n * sizeof(double), s, "D2H L");
  return GPEMU_OK;
  GPEMU_GUARD_END
}

int gpemu_model_alpha(gpemu_model* m, double* alpha_out) {
  GPEMU_GUARD_BEGIN
  if (!m || !alpha_out) return set_error(GPEMU_VALIDATION, "model_alpha: null argument");
  ck(cudaSetDevice(m->ctx->device), "cudaSetDevice");
  d2h_sync(alpha_out, m->alpha.p, (size_t)m->n * sizeof(double), m->ctx->stream, "D2H alpha");
  return GPEMU_OK;
  GPEMU_GUARD_END
}

int gpemu_model_import(gpemu_ctx* ctx, const double* X, size_t n, size_t d, const double* theta,
                       double p, const double* scalars, double log_det, const double* L,
                       const double* alpha, gpemu_model** out) {
  GPEMU_GUARD_BEGIN
  if (!ctx || !X || !theta || !scalars || !L || !alpha || !out)
    return set_error(GPEMU_VALIDATION, "model_import: null argument");
  if (n < 1 || d < 1) return set_error(GPEMU_VALIDATION, "model_import: empty model");
  int rc = validate_params(theta, d, p, 0.0);
  if (rc) return rc;
  rc = validate_unit_cube(X, n, d, "model_import");
  if (rc) return rc;
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t s = ctx->stream;
  auto* m = new gpemu_model();
  m->ctx = ctx;
  m->bind();
  ctx_adopt(ctx);
  try {
    m->n = (int)n;
    m->d = (int)d;
    m->NT = (int)((n + TILE - 1) / TILE);
    const int Npad = m->NT * TILE;
    m->p = p;
    m->neg2 = scalars[0];
    m->mu = scalars[1];
    m->sigma2 = scalars[2];
    m->jitter = scalars[3];
    m->log_det = log_det;
    m->theta.assign(theta, theta + d);
    m->X.alloc(n * d);
    m->theta_d.alloc(d);
    m->alpha.alloc(Npad);
    m->tiles.alloc((size_t)num_tiles(m->NT) * TILE_ELEMS);
    m->u.alloc(Npad);
    m->v.alloc(Npad);
    DevBuf<double> dL, ones, dvtv;
    DevBuf<int> flags, counter, error;
    own(&ctx->stream, dL, ones, dvtv);
    own(&ctx->stream, flags, counter, error);
    dL.alloc(n * n);
    ones.alloc(n);
    dvtv.alloc(1);
    flags.alloc(m->NT);
    counter.alloc(1);
    error.alloc(1);
    const std::vector<double> h1(n, 1.0);
    ck(cudaMemcpyAsync(m->X.p, X, n * d * sizeof(double), cudaMemcpyHostToDevice, s), "H2D X");
    ck(cudaMemcpyAsync(m->theta_d.p, theta, d * sizeof(double), cudaMemcpyHostToDevice, s), "H2D theta");
    ck(cudaMemsetAsync(m->alpha.p, 0, Npad * sizeof(double), s), "memset");
    ck(cudaMemcpyAsync(m->alpha.p, alpha, n * sizeof(double), cudaMemcpyHostToDevice, s), "H2D alpha");
    ck(cudaMemsetAsync(m->u.p, 0, Npad * sizeof(double), s), "memset");
    ck(cudaMemcpyAsync(dL.p, L, n * n * sizeof(double), cudaMemcpyHostToDevice, s), "H2D L");
    ck(cudaMemcpyAsync(ones.p, h1.data(), n * sizeof(double), cudaMemcpyHostToDevice, s), "H2D ones");
    ck(cudaMemsetAsync(flags.p, 0, m->NT * sizeof(int), s), "memset");
    ck(cudaMemsetAsync(error.p, 0, sizeof(int), s), "memset");
    launch_rowmajor_to_tiles(dL.p, (int)n, m->NT, 0.0, m->tiles.p, s);
    // v = L^-1 1 (the kriging MSE's GLS term) and v'v in the reference's dot order
    launch_tile_trsv(m->tiles.p, m->NT, ones.p, nullptr, 0.0, (int)n, m->v.p, 0, flags.p, counter.p, 1,
                     error.p, ctx->num_sms, s);
    launch_dot_seq(m->v.p, m->v.p, (int)n, dvtv.p, s);
    ctx->launches += 3;
    ck(cudaGetLastError(), "model_import launch");
    int err = 0;
    ck(cudaMemcpyAsync(&m->vtv, dvtv.p, sizeof(double), cudaMemcpyDeviceToHost, s), "D2H vtv");
    ck(cudaMemcpyAsync(&err, error.p, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H error");
    ck(cudaStreamSynchronize(s), "model_import");
    if (err) throw CudaError{"tile_trsv: dependency wait timed out (deadlock guard)"};
  } catch (...) {
    release(m);
    throw;
  }
  *out = m;
  return GPEMU_OK;
  GPEMU_GUARD_END
}

int gpemu_predict(gpemu_model* m, const double* Xtest, size_t N, double* yhat, double* mse) {
  GPEMU_GUARD_BEGIN
  NvtxRange range(mse ? "K4 predict + kriging MSE" : "K4 predict");
  if (!m || (!Xtest && N) || (!yhat && N)) return set_error(GPEMU_VALIDATION, "predict: null argument");
  int rc = validate_unit_cube(Xtest, N, m->d, "predict");
  if (rc) return set_error(GPEMU_VALIDATION, "predict: test point outside the unit cube");
  if (N == 0) return GPEMU_OK;
  ck(cudaSetDevice(m->ctx->device), "cudaSetDevice");
  cudaStream_t s = m->ctx->stream;
  DevBuf<double>&dXt = m->pred_xt, &dy = m->pred_y, &dm = m->pred_mse, &dpart = m->pred_part;
  DevBuf<int>& bad = m->pred_bad;
  dXt.reserve(N * m->d);
  dy.reserve(N);
  dpart.reserve((size_t)predict_blocks(m->n) * N);
  bad.reserve(1);
  ck(cudaMemcpyAsync(dXt.p, Xtest, N * m->d * sizeof(double), cudaMemcpyHostToDevice, s), "H2D Xtest");
  ck(cudaMemsetAsync(bad.p, 0, sizeof(int), s), "memset");
  if (m->single) {  // float model: corr_vector<float> + dot_accumulate (predictor.hpp:36-44)
    launch_predict_f32(dXt.p, (int)N, m->X.p, m->n, m->d, m->theta_d.p, m->p, m->mu, m->alpha.p,
                       dy.p, bad.p, s);
    m->ctx->launches += 1;
  }
  if (!mse) {
    if (!m->single) {
      launch_predict(dXt.p, (int)N, m->X.p, m->n, m->d, m->theta_d.p, m->p, m->mu, m->alpha.p,
                     dpart.p, dy.p, bad.p, s);
      m->ctx->launches += 2;
    }
  } else {
    // Cross-correlation tiles r for chunks of test points; yhat = mu + r.alpha from the tiles
    // (predict_kernel's summation order: the same bits as the yhat-only call); then
    // W = L^-1 r as extension rows of the factor (DMMA tiles) and one warp per point: the
    // kriging MSE.
    dm.reserve(N);
    const int NT = m->NT;
    const int chunk_pts = 65536;
    const int rt_cap = (int)std::min<size_t>((N + TILE - 1) / TILE, chunk_pts / TILE);
    if (m->ext_rt_cap < rt_cap) {
      m->ext.alloc((size_t)rt_cap * NT * TILE_ELEMS);
      m->ext_flags.alloc((size_t)rt_cap * NT);
      ck(cudaMemsetAsync(m->ext_flags.p, 0, (size_t)rt_cap * NT * sizeof(int), s), "memset");
      m->ext_slot.alloc(1);
      ck(cudaMemsetAsync(m->ext_slot.p, 0, sizeof(int), s), "memset");
      m->counter.alloc(1);
      m->error.alloc(1);
      ck(cudaMemsetAsync(m->error.p, 0, sizeof(int), s), "memset");
      m->ext_rt_cap = rt_cap;
    }
    for (size_t p0 = 0; p0 < N; p0 += chunk_pts) {
      const int Nc = (int)std::min<size_t>(chunk_pts, N - p0);
      const int RT = (Nc + TILE - 1) / TILE;
      launch_cross_tiles(dXt.p + p0 * m->d, Nc, m->X.p, m->n, m->d, m->theta_d.p, m->p, NT, RT,
                         m->ext.p, bad.p, s);
      if (!m->single) launch_yhat_tiles(m->ext.p, Nc, m->n, NT, m->alpha.p, dpart.p, N, p0, s);
      DagLaunch a;
      a.factors = m->tiles.p;
      a.borders = nullptr;
      a.slot_stride = 0;
      a.n = m->n;
      a.NT = NT;
      a.slots = m->ext_slot.p;
      a.nslots = 1;
      a.counter = m->counter.p;
      a.flags = nullptr;
      a.epoch = ++m->epoch;
      a.status = nullptr;
      a.error = m->error.p;
      a.ext = m->ext.p;
      a.ext_rt = RT;
      a.ext_flags = m->ext_flags.p;
      launch_chol_dag(a, m->ctx->num_sms, s);
      launch_ext_reduce(m->ext.p, Nc, m->n, NT, m->u.p, m->v.p, m->mu, m->sigma2, m->vtv,
                        nullptr, dm.p + p0, s);
      m->ctx->launches += 4;
    }
    if (!m->single) {
      launch_predict_combine(dpart.p, (int)N, m->n, m->mu, dy.p, s);
      m->ctx->launches += 1;
    }
  }
  ck(cudaGetLastError(), "predict launch");
  int hbad = 0;
  ck(cudaMemcpyAsync(yhat, dy.p, N * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H yhat");
  if (mse) ck(cudaMemcpyAsync(mse, dm.p, N * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H mse");
  ck(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H bad");
  ck(cudaStreamSynchronize(s), "predict");
  if (mse && m->error.p) {
    int err = 0;
    d2h_sync(&err, m->error.p, sizeof(int), m->ctx->stream, "D2H error");
    if (err) return set_error(GPEMU_CUDA, "chol_dag (extension): dependency wait timed out");
  }
  if (hbad) return set_error(GPEMU_NONFINITE, "corr_vector: non-finite correlation value");
  return GPEMU_OK;
  GPEMU_GUARD_END
}

// maximin_lhd (experiment.hpp:142-172). The host side draws exactly what the reference draws,
// in the same order, with the reference RNG's engine and output mappings (detail/rng.hpp:12-47:
// splitmix64 seed derivation, std::mt19937_64, uniform01 = (u >> 11) 2^-53, Lemire's
// below(n) = (u * n) >> 64): the random LHD (experiment.hpp:36-50), then (k, a, b) of every swap
// (:155-158) -- the draws do not depend on acceptance. The device scores the swaps
// (kernels_design.cu).
int gpemu_maximin_lhd(gpemu_ctx* ctx, size_t n, size_t d, uint64_t seed, size_t exchange_budget,
                      double* x_out, double* min_dist) {
  GPEMU_GUARD_BEGIN
  if (!ctx || !x_out) return set_error(GPEMU_VALIDATION, "maximin_lhd: null argument");
  if (n < 2) return set_error(GPEMU_VALIDATION, "DesignSpec: n must be at least 2");
  if (d < 1) return set_error(GPEMU_VALIDATION, "DesignSpec: d must be at least 1");
  if (n > (size_t)INT32_MAX / 2 || d > 1000000 || exchange_budget > (size_t)INT32_MAX / 3)
    return set_error(GPEMU_VALIDATION, "maximin_lhd: design too large");
  NvtxRange range("maximin_lhd");
  Rng rng(derive_seed(seed, 0x1d64ull));
  // random_lhd: per column a Fisher-Yates permutation, then one uniform per point
  std::vector<size_t> perm(n);
  for (size_t k = 0; k < d; ++k) {
    for (size_t i = 0; i < n; ++i) perm[i] = i;
    for (size_t i = n - 1; i > 0; --i) std::swap(perm[i], perm[rng.below(i + 1)]);
    for (size_t i = 0; i < n; ++i)
      x_out[i * d + k] = (static_cast<double>(perm[i]) + rng.uniform01()) / static_cast<double>(n);
  }
  if (exchange_budget == 0 || n == 2) {  // nothing to exchange (experiment.hpp:147-149)
    if (min_dist) *min_dist = std::nan("");
    return GPEMU_OK;
  }
  std::vector<int> draws(3 * exchange_budget);
  for (size_t it = 0; it < exchange_budget; ++it) {
    const auto k = rng.below(d);
    const auto a = rng.below(n);
    auto b = rng.below(n - 1);
    if (b >= a) ++b;
    draws[3 * it] = (int)k;
    draws[3 * it + 1] = (int)a;
    draws[3 * it + 2] = (int)b;
  }
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t s = ctx->stream;
  DevBuf<double> dX, dra, drb, res;
  DevBuf<unsigned long long> r0, r1, red;
  DevBuf<int> dD, fl;
  own(&ctx->stream, dX, dra, drb, res, r0, r1, red, dD, fl);
  dX.alloc(n * d);
  dra.alloc(n);
  drb.alloc(n);
  res.alloc(2);
  r0.alloc(n);
  r1.alloc(n);
  red.alloc(9);
  dD.alloc(draws.size());
  fl.alloc(n);
  const unsigned long long inf = 0x7FF0000000000000ull;
  const unsigned long long init[9] = {inf, inf, inf, 0, inf, inf, inf, 0, inf};
  ck(cudaMemcpyAsync(dX.p, x_out, n * d * sizeof(double), cudaMemcpyHostToDevice, s), "H2D design");
  ck(cudaMemcpyAsync(dD.p, draws.data(), draws.size() * sizeof(int), cudaMemcpyHostToDevice, s), "H2D draws");
  ck(cudaMemcpyAsync(red.p, init, sizeof(init), cudaMemcpyHostToDevice, s), "H2D init");
  gpemu_dev::MaximinLaunch L{dX.p, (int)n, (int)d, (int)exchange_budget, dD.p, r0.p, r1.p, dra.p, drb.p, fl.p,
                             red.p, red.p + 8, res.p};
  ck(gpemu_dev::launch_maximin(L, ctx->num_sms, s), "maximin launch");
  ctx->launches += 3;
  double hres[2];
  ck(cudaMemcpyAsync(x_out, dX.p, n * d * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H design");
  ck(cudaMemcpyAsync(hres, res.p, sizeof(hres), cudaMemcpyDeviceToHost, s), "D2H result");
  ck(cudaStreamSynchronize(s), "maximin_lhd");
  if (min_dist) *min_dist = hres[0];
  return GPEMU_OK;
  GPEMU_GUARD_END
}

}  // extern "C"
