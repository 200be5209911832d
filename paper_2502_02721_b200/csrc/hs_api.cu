// C-ABI of the B200 sketched-Hessenberg / sLSLU loop (include/hessketch_b200.h).
//
// The solve (hs_solve) restates _hessenberg_solve (solvers.py:410-539) for the
// sketched solvers: a host loop issues, per iteration, the operator kernel,
// the sketch kernel, the pivot-row forward substitution, ONE fused
// elimination/argmax pass over the basis, the pivot commit and the
// normalisation (twice for the rectangular process), then the cooperative
// projected-solve kernel.  Nothing is copied back per iteration: breakdown and
// all trace scalars live on the device and are read once at the end.
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <array>
#include <atomic>
#include <condition_variable>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/hessketch_b200.h"
#include "hs_build.cuh"
#include "hs_common.cuh"
#include "hs_diag.cuh"
#include "hs_krylov.cuh"
#include "hs_loop.cuh"
#include "hs_ops.cuh"
#include "hs_c2.cuh"
#include "hs_qr.cuh"
#include "hs_shard.cuh"
#include "hs_sketch.cuh"

using namespace hs;

// ---------------------------------------------------------------------------
// errors

static thread_local std::string g_err;

namespace {

struct HsError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  throw HsError{code, buf};
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) fail(HS_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, \
                                cudaGetErrorString(e_));                               \
  } while (0)

static std::atomic<unsigned long long> g_launches{0};  // kernels launched by this library (all streams)
#define CKL()                   \
  do {                          \
    CK(cudaGetLastError());     \
    ++g_launches;               \
  } while (0)

template <class F>
int guarded(F&& f) {
  (void)cudaGetLastError();  // a stale error of an unrelated earlier call is not this call's
  try {
    f();
    return HS_OK;
  } catch (const HsError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HS_ERR_RUNTIME;
  }
}

size_t dsize(int dt) { return dt == HS_F64 ? 8 : (dt == HS_F32 ? 4 : 2); }
long long round_up(long long a, long long b) { return (a + b - 1) / b * b; }

// Stream-ordered allocations.  Every buffer is allocated and freed on the
// main stream of the context active on the calling thread (CtxScope, set by
// each C entry point), from a memory pool that keeps freed blocks (repeated
// solves reuse the 7.5 GB of bases instead of paying cudaMalloc/cudaFree and
// page unmapping each time).  The stream is reference-counted: a context's
// operators, sketches and results keep it alive after hs_ctx_destroy, so a
// late free is still ordered after the work that used the buffer.  Without
// an active context (none of the entry points) the synchronous allocator is
// used.
struct StreamRef {
  cudaStream_t s = nullptr;
  int device = 0;
  ~StreamRef() {
    if (!s) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    cudaSetDevice(cur);
  }
};
static thread_local std::shared_ptr<StreamRef> tl_alloc;

// Guard mode (HS_GUARD=1, read at each allocation; compute-sanitizer is not
// available on the GPU pool): every buffer gets 4 KB guard bands filled with
// 0xA5 on both sides, checked when the buffer is released; a changed byte is
// an out-of-bounds write by some kernel, counted in hs_guard_violations().
constexpr size_t kGuard = 4096;
static std::atomic<unsigned long long> g_guard_violations{0};
static bool guard_mode() {
  const char* e = getenv("HS_GUARD");
  return e && *e && !(e[0] == '0' && e[1] == 0);
}

// device buffer with RAII
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  std::shared_ptr<StreamRef> owner;
  bool guarded = false;
  DBuf() = default;
  explicit DBuf(size_t b, bool zero = true) { alloc(b, zero); }
  void alloc(size_t b, bool zero = true) {
    release();
    bytes = b;
    if (b) {
      owner = tl_alloc;
      guarded = guard_mode();
      const size_t total = guarded ? b + 2 * kGuard : b;
      void* base = nullptr;
      if (owner) {
        CK(cudaMallocAsync(&base, total, owner->s));
      } else {
        CK(cudaMalloc(&base, total));
      }
      p = guarded ? reinterpret_cast<char*>(base) + kGuard : base;
      cudaStream_t s = owner ? owner->s : nullptr;
      if (zero) CK(cudaMemsetAsync(p, 0, b, s));
      if (guarded) {
        CK(cudaMemsetAsync(base, 0xA5, kGuard, s));
        CK(cudaMemsetAsync(reinterpret_cast<char*>(p) + b, 0xA5, kGuard, s));
      }
      // buffers are also filled by pageable-host copies and read by the
      // context's second stream: make the allocation complete now
      CK(cudaStreamSynchronize(s));
    }
  }
  void check_guards() {
    cudaStream_t s = owner ? owner->s : nullptr;
    std::vector<unsigned char> g(2 * kGuard);
    if (cudaStreamSynchronize(s) != cudaSuccess ||
        cudaMemcpy(g.data(), reinterpret_cast<char*>(p) - kGuard, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(g.data() + kGuard, reinterpret_cast<char*>(p) + bytes, kGuard, cudaMemcpyDeviceToHost) !=
            cudaSuccess)
      return;
    size_t bad = 0, first = 0;
    for (size_t i = 0; i < g.size(); ++i)
      if (g[i] != 0xA5 && bad++ == 0) first = i;
    if (bad) {
      ++g_guard_violations;
      fprintf(stderr, "[hessketch guard] %zu bytes changed %s a %zu-byte buffer (first at guard offset %zu)\n", bad,
              first < kGuard ? "before" : "after", bytes, first % kGuard);
    }
  }
  void release() {
    if (p) {
      if (guarded) check_guards();
      void* base = guarded ? reinterpret_cast<char*>(p) - kGuard : p;
      if (owner) cudaFreeAsync(base, owner->s);  // ordered after the owning stream's work
      else cudaFree(base);
    }
    p = nullptr;
    bytes = 0;
    owner.reset();
    guarded = false;
  }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes), owner(std::move(o.owner)), guarded(o.guarded) {
    o.p = nullptr;
    o.bytes = 0;
    o.guarded = false;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    release();
    p = o.p; bytes = o.bytes; owner = std::move(o.owner); guarded = o.guarded;
    o.p = nullptr; o.bytes = 0; o.guarded = false;
    return *this;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

// the context whose main stream owns allocations made on this thread (DBuf)
struct CtxScope {
  std::shared_ptr<StreamRef> prev;
  template <class C>
  explicit CtxScope(const C* c) : prev(tl_alloc) {
    if (c) tl_alloc = c->main;
  }
  ~CtxScope() { tl_alloc = prev; }
};

// experiment switches (tools/ab_spmv.py): set and not "0"/empty
bool env_flag(const char* name) {
  const char* e = getenv(name);
  return e && *e && !(e[0] == '0' && e[1] == 0);
}

// sum of squares of a host vector: eight interleaved partial sums combined in a
// fixed order (|x_true| for the relative errors; one dependent add chain over
// 16.8M entries cost 17 ms of every config-5 solve)
double host_sumsq(const double* v, long long n) {
  double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long i = 0;
  for (; i + 8 <= n; i += 8)
    for (int j = 0; j < 8; ++j) a[j] += v[i + j] * v[i + j];
  for (int j = 0; i < n; ++i, ++j) a[j] += v[i] * v[i];
  return ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

int grid_for(long long work, int block, int cap) {
  long long g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace

// ---------------------------------------------------------------------------
// context

struct KStat {
  long long launches = 0;
  double ms = 0.0;
  double bytes = 0.0;
};

struct hs_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;  // == main->s
  std::shared_ptr<StreamRef> main;
  cudaStream_t aux = nullptr;  // second stream: sketches + projected solve overlap the basis passes
  int num_sms = 148;
  int nranks = 1, rank = 0;
  void* comm = nullptr;  // ncclComm_t when nranks > 1 (hs_dist.inc)
  std::shared_ptr<struct LocalComm> lcomm;  // in-process ranks (hs_comm_init_local), instead of NCCL
  bool force_shard = false;  // run the sharded operator/loop even with one rank (tests)
  bool profiling = false;
  std::map<std::string, KStat> stats;
  // pending event pairs for profiled launches
  struct Pending {
    std::string name;
    cudaEvent_t a, b;
    double bytes;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> free_events;

  cudaEvent_t get_event() {
    if (!free_events.empty()) {
      cudaEvent_t e = free_events.back();
      free_events.pop_back();
      return e;
    }
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
  }
  // per-solve events and pinned scratch, kept across solves: creating and
  // destroying ~600 events and a pinned buffer per solve sporadically cost
  // ~0.25 s of host time (measured, tools/e2e_breakdown.py)
  std::vector<cudaEvent_t> pool_timed, pool_sync;
  std::mutex solve_mu;  // solves on one context are serialised (they share its streams and scratch)
  void* pinned = nullptr;
  size_t pinned_cap = 0;
  std::vector<cudaEvent_t> take_events(size_t n, bool timed) {
    auto& pool = timed ? pool_timed : pool_sync;
    std::vector<cudaEvent_t> out;
    out.reserve(n);
    while (out.size() < n && !pool.empty()) {
      out.push_back(pool.back());
      pool.pop_back();
    }
    while (out.size() < n) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, timed ? cudaEventDefault : cudaEventDisableTiming));
      out.push_back(e);
    }
    return out;
  }
  void give_events(std::vector<cudaEvent_t>& v, bool timed) {
    auto& pool = timed ? pool_timed : pool_sync;
    pool.insert(pool.end(), v.begin(), v.end());
    v.clear();
  }
  void* pinned_buf(size_t bytes) {
    if (bytes > pinned_cap) {
      if (pinned) CK(cudaFreeHost(pinned));
      pinned = nullptr;
      pinned_cap = 0;
      CK(cudaMallocHost(&pinned, bytes));
      pinned_cap = bytes;
    }
    return pinned;
  }
  void harvest() {
    if (pending.empty()) return;
    // pairs recorded on either stream (aux: sketches, projected solves)
    CK(cudaStreamSynchronize(stream));
    CK(cudaStreamSynchronize(aux));
    for (auto& p : pending) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, p.a, p.b));
      auto& s = stats[p.name];
      s.launches += 1;
      s.ms += ms;
      s.bytes += p.bytes;
      free_events.push_back(p.a);
      free_events.push_back(p.b);
    }
    pending.clear();
  }
};

// Experiment (HS_L2PERSIST=1): keep the gathered vector resident in L2 while
// the matrix streams past it (stream access-policy window, persisting hits).
struct L2Window {
  cudaStream_t s = nullptr;
  L2Window(cudaStream_t st, const void* p, size_t bytes) {
    const bool on = env_flag("HS_L2PERSIST");
    if (!on || p == nullptr) return;
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)64 << 20);  // per device, idempotent
    cudaStreamAttrValue a = {};
    a.accessPolicyWindow.base_ptr = const_cast<void*>(p);
    a.accessPolicyWindow.num_bytes = bytes;
    a.accessPolicyWindow.hitRatio = 1.0f;
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a) == cudaSuccess) s = st;
  }
  ~L2Window() {
    if (!s) return;
    cudaStreamAttrValue a = {};
    a.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &a);
  }
};

// scoped profiling bracket around one launch
struct Prof {
  hs_ctx* c;
  const char* name;
  double bytes;
  cudaEvent_t a = nullptr;
  cudaStream_t st;
  Prof(hs_ctx* c_, const char* n, double b, cudaStream_t s_ = nullptr)
      : c(c_), name(n), bytes(b), st(s_ ? s_ : c_->stream) {
    if (c->profiling) {
      a = c->get_event();
      CK(cudaEventRecord(a, st));
    }
  }
  ~Prof() noexcept(false) {
    if (c->profiling) {
      cudaEvent_t b = c->get_event();
      CK(cudaEventRecord(b, st));
      c->pending.push_back({name, a, b, bytes});
      if (c->pending.size() > 4096) c->harvest();
    }
  }
};

// ---------------------------------------------------------------------------
// operators

enum { OP_DENSE = 0, OP_CSR = 1, OP_PSF = 2 };

struct Csr {
  long long rows = 0, cols = 0, nnz = 0;
  DBuf rowptr, col, val;
};

// SELL-32x4 copy of a CSR (hs_ops.cuh: sell_spmv_kernel)
struct Sell {
  long long rows = 0, cols = 0, nnz = 0, slots = 0, nslices = 0;
  DBuf sptr, rlen, col, val;
  DBuf rperm;         // optional slot -> row map (slots are nslices*32; -1 = empty)
  DBuf sorder, sched; // slices longest-first + the dynamic scheduler's two counters
  long long nslots() const { return nslices * 32; }
  bool d16 = false;   // columns stored as int16 deltas (rbase + dcol) instead of col
  DBuf rbase, dcol;
  bool d16v = false;  // d16 + dominant-value flags: val holds only the explicit values (hs_ops.cuh: d16v)
  DBuf fv, vptr;
  long long n_explicit = 0;
  bool c8 = false;    // columns stored as 8-bit transition codes (hs_ops.cuh: C8Geom)
  C8Geom c8g{0, 0};
  DBuf code, xoff, exc;
  long long n_exc = 0;
  // 2-bit step codes on the slices flagged in c2ok (hs_c2.cuh); the rest keep their 16-bit deltas
  bool c2 = false;
  DBuf c2ok, c2tab, c2start, c2esc, c2code;
  long long c2_slices = 0, c2_slots = 0;
  bool t8 = false;    // A^T: 8-bit step codes (hs_c2.cuh: t8) on the flagged slices; shares the c2 buffers
  int t8_bins = 0;
  double index_bytes() const { return c8 ? 1.0 : d16 ? 2.0 : 4.0; }
  double slot_bytes() const { return c8 ? 12.0 : d16v ? 12.0 : d16 ? 8.0 : 4.0; }
  long long stored_values() const { return d16v ? n_explicit : nnz; }  // rlen (+ rbase) (+ escape offset) per slot
};

// Switch a SELL copy to 16-bit column deltas when every in-row step fits.
static bool sell_try_delta16(hs_ctx* ctx, Sell& S) {
  if (S.nslices == 0) return false;
  cudaStream_t s = ctx->stream;
  DBuf mx(sizeof(unsigned int));
  sell_delta_range_kernel<<<grid_for(S.nslices, 8, 1 << 30), 256, 0, s>>>(
      S.nslots(), S.nslices, S.sptr.as<long long>(), S.rlen.as<int>(), S.col.as<int>(), mx.as<unsigned int>());
  CKL();
  unsigned int h = 0;
  CK(cudaMemcpyAsync(&h, mx.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (h > 32767u) return false;
  S.rbase.alloc(std::max<long long>(S.nslots(), 1) * sizeof(int), false);
  S.dcol.alloc(std::max<long long>(S.slots, 4) * sizeof(short), false);
  sell_delta_fill_kernel<<<grid_for(S.nslices, 8, 1 << 30), 256, 0, s>>>(
      S.nslots(), S.nslices, S.sptr.as<long long>(), S.rlen.as<int>(), S.col.as<int>(), S.rbase.as<int>(),
      S.dcol.as<short>());
  CKL();
  CK(cudaStreamSynchronize(s));
  S.col.release();
  S.d16 = true;
  return true;
}

// 2-bit step codes for a tomography A (hs_c2.cuh), on the int32 image-order
// columns before they become deltas.  A slice takes the codes when every row
// of it needs at most two escapes; the others keep their 16-bit deltas, so
// this only pays when sell_try_delta16 succeeds afterwards.  HS_C2=0 disables.
static void sell_try_c2(hs_ctx* ctx, Sell& S, const unsigned char* sflag, int grid) {
  if (S.nslices == 0 || S.col.p == nullptr || S.rperm.p != nullptr) return;
  if (env_int("HS_C2", 1) == 0) return;
  cudaStream_t s = ctx->stream;
  const long long ns = S.nslots();
  DBuf ok(S.nslices, true), tab(S.nslices * sizeof(int4), false), start(ns * sizeof(int), false),
      esc(ns * sizeof(int4), false), code(S.slots / 4 + 96 * S.nslices + 128, true);
  sell_c2_encode_kernel<<<grid_for(S.nslices, 8, 1 << 30), 256, 0, s>>>(
      ns, S.nslices, S.sptr.as<long long>(), S.rlen.as<int>(), S.col.as<int>(), sflag, grid, ok.as<unsigned char>(),
      tab.as<int4>(), start.as<int>(), esc.as<int4>(), code.as<unsigned char>());
  CKL();
  std::vector<unsigned char> hok(S.nslices);
  std::vector<long long> hp(S.nslices + 1);
  CK(cudaMemcpyAsync(hok.data(), ok.p, S.nslices, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hp.data(), S.sptr.p, (S.nslices + 1) * sizeof(long long), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  long long n_ok = 0, slots_ok = 0;
  for (long long i = 0; i < S.nslices; ++i)
    if (hok[i]) {
      ++n_ok;
      slots_ok += hp[i + 1] - hp[i];
    }
  // below half of the stream the mixed kernel is not worth its extra state
  if (2 * slots_ok < S.slots) return;
  S.c2ok = std::move(ok);
  S.c2tab = std::move(tab);
  S.c2start = std::move(start);
  S.c2esc = std::move(esc);
  S.c2code = std::move(code);
  S.c2_slices = n_ok;
  S.c2_slots = slots_ok;
  S.c2 = true;
}

// 8-bit step codes for a tomography A^T (hs_c2.cuh: t8), from the int32
// ray-order columns (before the sinogram layout mapping and the deltas).  The
// caller then maps the columns to SinoBlk{n_bins, 4, 1, n_bins} and builds the
// 16-bit deltas the non-conforming slices keep.  Opt-in (HS_T8=1; HS_T8=2 also
// forces it on operators that take the latency-bound d16 schedules): config
// 4's A^T moves 17% fewer bytes, bit-identical, and runs 3.55 against 3.62 ms
// in isolation but 4.04 against 3.80 ms inside the solve -- A^T is bound by its
// gather round trips (one per chunk per warp), and the table decode adds 14
// instructions per chunk to a kernel that shares the SMs with the aux stream.
static bool sell_try_t8(hs_ctx* ctx, Sell& S, int n_bins) {
  if (S.nslices == 0 || S.col.p == nullptr || n_bins <= 0) return false;
  const int mode = env_int("HS_T8", 0);
  if (mode == 0) return false;
  const bool few = S.nslices < 2LL * ctx->num_sms * 48 && S.slots / (S.nslices * 128) < 256;
  if (few && mode != 2) return false;
  if ((4LL * n_bins + 4 * 63) >= 32767) return false;  // the fallback slices' 16-bit deltas must hold a group step
  cudaStream_t s = ctx->stream;
  const long long ns = S.nslots();
  DBuf ok(S.nslices, true), start(ns * sizeof(int), false), esc(ns * sizeof(int4), false),
      code(std::max<long long>(S.slots, 4) + 128, true);
  sell_t8_encode_kernel<<<grid_for(S.nslices, 8, 1 << 30), 256, 0, s>>>(
      ns, S.nslices, S.sptr.as<long long>(), S.rlen.as<int>(), S.col.as<int>(), n_bins, ok.as<unsigned char>(),
      start.as<int>(), esc.as<int4>(), code.as<unsigned char>());
  CKL();
  std::vector<unsigned char> hok(S.nslices);
  std::vector<long long> hp(S.nslices + 1);
  CK(cudaMemcpyAsync(hok.data(), ok.p, S.nslices, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hp.data(), S.sptr.p, (S.nslices + 1) * sizeof(long long), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  long long n_ok = 0, slots_ok = 0;
  for (long long i = 0; i < S.nslices; ++i)
    if (hok[i]) {
      ++n_ok;
      slots_ok += hp[i + 1] - hp[i];
    }
  if (2 * slots_ok < S.slots) return false;
  S.c2ok = std::move(ok);
  S.c2start = std::move(start);
  S.c2esc = std::move(esc);
  S.c2code = std::move(code);
  S.c2_slices = n_ok;
  S.c2_slots = slots_ok;
  S.t8 = true;
  S.t8_bins = n_bins;
  return true;
}

// Switch a d16 SELL copy to dominant-value flags (hs_ops.cuh: d16v) when at
// least 15% of its values equal their row's most frequent value and every
// delta fits 15 bits.  fp32 values only; operators whose SpMV takes the
// latency-bound schedules (few slices of short rows) keep plain d16.
// Opt-in (HS_D16V=1): config 4's A stream shrinks from 6 to 4.3 B/nonzero
// (59% of values explicit), bit-identical, but the kernel measured 4.41 ms
// against d16's 3.47 -- the per-lane variable-rate value loads (four scalar
// loads and four ballots per chunk) raise the kernel from 44 to 111 warp
// instructions per chunk, moving the limit from HBM to issue.
template <class V>
static bool sell_try_dominant(hs_ctx* ctx, Sell& S) {
  if constexpr (sizeof(V) != 4) {
    return false;
  } else {
    if (!S.d16 || S.nslices == 0 || !env_flag("HS_D16V")) return false;
    const long long avg_chunks = S.slots / (S.nslices * 128);
    if (S.nslices < 2LL * ctx->num_sms * 48 && avg_chunks < 256 && !env_flag("HS_D16V_FORCE")) return false;
    cudaStream_t s = ctx->stream;
    const long long ns = S.nslots();
    DBuf fv(std::max<long long>(ns, 1) * sizeof(V), false), cnt((S.nslices + 1) * sizeof(long long), true),
        mx(sizeof(unsigned int), true);
    const int gb = (int)grid_for(S.nslices, 8, 1 << 30);
    sell_dominant_kernel<V><<<gb, 256, 0, s>>>(ns, S.nslices, S.sptr.as<long long>(), S.rlen.as<int>(),
                                               S.dcol.as<short>(), S.val.as<V>(), fv.as<V>(), cnt.as<long long>(),
                                               mx.as<unsigned int>());
    CKL();
    DBuf vptr((S.nslices + 1) * sizeof(long long), false);
    {
      size_t tmp = 0;
      CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.as<long long>(), vptr.as<long long>(), S.nslices + 1, s));
      DBuf t(tmp, false);
      CK(cub::DeviceScan::ExclusiveSum(t.p, tmp, cnt.as<long long>(), vptr.as<long long>(), S.nslices + 1, s));
    }
    long long nx = 0;
    unsigned int h = 0;
    CK(cudaMemcpyAsync(&nx, vptr.as<long long>() + S.nslices, sizeof(nx), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&h, mx.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (h > 16383u || (double)nx > 0.85 * (double)S.nnz) return false;
    // +128: the kernel's clamped one-chunk-ahead loads may read past the last slice's stream
    DBuf out((nx + 128) * sizeof(V), true);
    sell_d16v_fill_kernel<V><<<gb, 256, 0, s>>>(ns, S.nslices, S.sptr.as<long long>(), S.rlen.as<int>(),
                                                S.dcol.as<short>(), S.val.as<V>(), fv.as<V>(), vptr.as<long long>(),
                                                out.as<V>());
    CKL();
    CK(cudaStreamSynchronize(s));
    S.val = std::move(out);
    S.fv = std::move(fv);
    S.vptr = std::move(vptr);
    S.n_explicit = nx;
    S.d16v = true;
    return true;
  }
}

// Switch a SELL copy of a tomography operator to 8-bit transition codes
// (hs_ops.cuh: C8Geom).  `span` = number of distinct r values (image rows /
// angles), used to bound the gather addresses.  Opt-in (HS_C8=1 for A,
// HS_AT_C8=1 for A^T): inside the solve loop, where the SM clock sits at the
// power cap, the 5 B/nonzero stream measured slower than 16-bit deltas
// (A: 3.94 vs 3.80 ms at 2048^2), though 2% faster in isolation.
static bool sell_try_code8(hs_ctx* ctx, Sell& S, C8Geom g, long long span, const unsigned char* sflag) {
  if (S.nslices == 0) return false;
  if (g.mode == 0 && span * (long long)g.G >= (1LL << 31)) return false;
  if (g.mode == 1 && ((span + 3) / 4) * 4 * (long long)g.G >= (1LL << 30)) return false;
  cudaStream_t s = ctx->stream;
  const long long ns = S.nslots();
  S.code.alloc(std::max<long long>(S.slots, 4), false);
  S.rbase.alloc(std::max<long long>(ns, 1) * sizeof(int), false);
  DBuf cnt((ns + 1) * sizeof(int));
  S.xoff.alloc((ns + 1) * sizeof(int), false);
  const int gb = (int)grid_for(S.nslices, 8, 1 << 30);
  sell_c8_encode_kernel<<<gb, 256, 0, s>>>(S.nslices, S.sptr.as<long long>(), S.rlen.as<int>(), S.col.as<int>(), sflag,
                                           g, 0, S.code.as<unsigned char>(), S.rbase.as<int>(), cnt.as<int>(), nullptr,
                                           nullptr);
  CKL();
  {
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.as<int>(), S.xoff.as<int>(), ns + 1, s));
    DBuf t(tmp, false);
    CK(cub::DeviceScan::ExclusiveSum(t.p, tmp, cnt.as<int>(), S.xoff.as<int>(), ns + 1, s));
  }
  int nx = 0;
  CK(cudaMemcpyAsync(&nx, S.xoff.as<int>() + ns, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  S.n_exc = nx;
  S.exc.alloc(std::max(nx, 1) * sizeof(int), false);
  sell_c8_encode_kernel<<<gb, 256, 0, s>>>(S.nslices, S.sptr.as<long long>(), S.rlen.as<int>(), S.col.as<int>(), sflag,
                                           g, 1, nullptr, nullptr, nullptr, S.xoff.as<int>(), S.exc.as<int>());
  CKL();
  CK(cudaStreamSynchronize(s));
  S.col.release();
  S.c8 = true;
  S.c8g = g;
  return true;
}

// tile_grid > 0: slots follow 8x4 pixel tiles of a tile_grid^2 image (rows = pixels)
template <class V>
static void csr_to_sell(hs_ctx* ctx, const Csr& A, Sell& S, int tile_grid = 0) {
  cudaStream_t s = ctx->stream;
  S.rows = A.rows;
  S.cols = A.cols;
  S.nnz = A.nnz;
  if (tile_grid > 0) {
    const long long rows_img = (A.rows + tile_grid - 1) / tile_grid;  // image rows in this block
    // tile shape tw x (32 / tw): 8 x 4 by default (HS_AT_TILE_W = 4 or 16 for A/B runs)
    int tw = env_int("HS_AT_TILE_W", 8);
    if (tw != 4 && tw != 16) tw = 8;
    const int th = 32 / tw;
    const long long tiles = (long long)((tile_grid + tw - 1) / tw) * ((rows_img + th - 1) / th);
    S.nslices = tiles;
    S.rperm.alloc(S.nslots() * sizeof(int), false);
    tile_perm_block_kernel<<<grid_for(S.nslots(), 256, 1 << 30), 256, 0, s>>>(
        tile_grid, (int)((A.rows + tile_grid - 1) / tile_grid), S.nslots(), S.rperm.as<int>(), tw);
    CKL();
  } else {
    S.nslices = (A.rows + 31) / 32;
  }
  S.rlen.alloc(std::max<long long>(S.nslots(), 1) * sizeof(int), false);
  DBuf slots((S.nslices + 1) * sizeof(long long));
  sell_slice_chunks_kernel<<<grid_for(S.nslices, 8, 1 << 30), 256, 0, s>>>(
      A.rows, S.nslices, A.rowptr.as<long long>(), S.rperm.as<int>(), S.rlen.as<int>(), slots.as<long long>());
  CKL();
  S.sptr.alloc((S.nslices + 1) * sizeof(long long), false);
  size_t tmp = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, slots.as<long long>(), S.sptr.as<long long>(), S.nslices + 1, s));
  DBuf t(tmp, false);
  CK(cub::DeviceScan::ExclusiveSum(t.p, tmp, slots.as<long long>(), S.sptr.as<long long>(), S.nslices + 1, s));
  CK(cudaMemcpyAsync(&S.slots, S.sptr.as<long long>() + S.nslices, sizeof(long long), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  {  // longest-first slice order for the dynamic scheduler
    DBuf sz(S.nslices * sizeof(unsigned int), false), szo(S.nslices * sizeof(unsigned int), false),
        id(S.nslices * sizeof(int), false);
    S.sorder.alloc(S.nslices * sizeof(int), false);
    S.sched.alloc(2 * sizeof(unsigned int), true);
    sell_slice_size_kernel<<<grid_for(S.nslices, 256, 1 << 30), 256, 0, s>>>(S.nslices, S.sptr.as<long long>(),
                                                                             sz.as<unsigned int>(), id.as<int>());
    CKL();
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, sz.as<unsigned int>(), szo.as<unsigned int>(),
                                                 id.as<int>(), S.sorder.as<int>(), (int)S.nslices, 0, 32, s));
    DBuf tt(tb, false);
    CK(cub::DeviceRadixSort::SortPairsDescending(tt.p, tb, sz.as<unsigned int>(), szo.as<unsigned int>(),
                                                 id.as<int>(), S.sorder.as<int>(), (int)S.nslices, 0, 32, s));
    CK(cudaStreamSynchronize(s));
  }
  S.col.alloc(std::max<long long>(S.slots, 4) * sizeof(int), false);
  S.val.alloc(std::max<long long>(S.slots, 4) * sizeof(V), false);
  sell_fill_kernel<V><<<grid_for(S.nslices, 8, 1 << 30), 256, 0, s>>>(
      A.rows, S.nslices, A.rowptr.as<long long>(), S.rperm.as<int>(), A.col.as<int>(), A.val.as<V>(),
      S.sptr.as<long long>(), S.col.as<int>(), S.val.as<V>());
  CKL();
  CK(cudaStreamSynchronize(s));
}

struct hs_op {
  hs_ctx* ctx = nullptr;
  int device = 0;
  int kind = OP_DENSE;
  int vdtype = HS_F64;
  long long m = 0, n = 0;
  // dense: column-major A (m x n) and column-major A^T (n x m)
  DBuf Acm, Atcm;
  // csr (kept for export / small operators) and the SELL-32x4 copies used by the loop
  Csr A, At;
  Sell As, Ats;
  bool csr_kept = true;
  // row sharding (multi-GPU): A rows [m_off, m_off+m_loc), A^T rows [n_off, n_off+n_loc),
  // padded block sizes m_blk / n_blk (the all-gathered vectors are P*blk long)
  bool sharded = false;
  long long m_off = 0, m_loc = 0, m_blk = 0, n_off = 0, n_loc = 0, n_blk = 0;
  // tomography (hs_op_tomo_create): image side, ray tables, and the slices
  // of As whose columns RayGen regenerates (hs_ops.cuh: sell_spmv_imp_kernel)
  long long tomo_grid = 0;
  int tomo_bins = 0;
  DBuf tcos, tsin, toff, imp;
  long long imp_slices = 0, imp_slots = 0;
  RayTab ray_tab() const {
    return RayTab{tcos.as<double>(), tsin.as<double>(), toff.as<double>(), tomo_bins, (int)tomo_grid,
                  sharded ? m_off : 0};
  }
  // tomography: per-slice transposed-layout flags of As and the scratch copy of x
  int img_grid = 0;
  DBuf sflag;
  mutable DBuf xT;
  // tomography: A^T gathers from a blocked copy of the sinogram (hs_ops.cuh: SinoBlk)
  SinoBlk sblk{0, 0, 0, 0};
  long long n_angles = 0;
  mutable DBuf yB;
  // psf
  int H = 0, W = 0, kh = 0, kw = 0;
  DBuf K;
  // sharded psf: this rank's image rows [psf_row0, psf_row0 + psf_rows); window scratch
  long long psf_row0 = 0, psf_rows = 0;
  mutable DBuf psfwin;

  // tomography A^T input staged by the caller in the blocked sinogram layout
  // (the loop's normalize kernel writes it beside d_{k+1}); null if the
  // operator does not gather from a blocked sinogram
  void* blocked_input(size_t elem_bytes) const {
    if (kind != OP_CSR || sblk.n_bins <= 0 || Ats.nslices <= 0) return nullptr;
    const size_t need = (size_t)sblk.size(n_angles) * elem_bytes;
    if (yB.bytes < need) yB.alloc(need, false);
    return yB.p;
  }

  // tomography A input staged by the caller in the transposed image layout
  // (the loop's L-side normalisation writes it beside l_{k+1}); null if the
  // operator has no transposed-layout slices
  void* transposed_input(size_t elem_bytes) const {
    if (kind != OP_CSR || sflag.p == nullptr || img_grid <= 0 || As.nslices <= 0 || sharded) return nullptr;
    const size_t need = (size_t)n * elem_bytes;
    if (xT.bytes < need) xT.alloc(need, false);
    return xT.p;
  }

  template <class V, class Tin, class T>
  void apply_t(const void* x, void* y, bool transpose, bool preblocked = false) const {
    cudaStream_t s = ctx->stream;
    const Tin* xi = reinterpret_cast<const Tin*>(x);
    T* yo = reinterpret_cast<T*>(y);
    if (kind == OP_CSR && (transpose ? Ats.nslices : As.nslices) > 0) {
      const Sell& M = transpose ? Ats : As;
      // blocks per SM of the dynamically scheduled SpMV kernels: the resident count (6 at fp32) rather
      // than a longer grid whose late blocks start only to find the slice counter exhausted
      // (config 4 in the solve: 130.1 -> 130.3 it/s; 12 and 32 per SM: no better)
      const int grid = grid_for(M.nslices, 8, ctx->num_sms * env_int("HS_SPMV_GRID", 6));
      // algorithmic bytes of the stored encoding: values + column indices (4 B, or 2 B deltas)
      // + row lengths (+ row bases) + slice pointers + x once + y
      const bool impl = !transpose && imp_slices > 0 && M.d16 && !M.d16v && !M.c8;
      // few slices of short rows: the d16 kernel's latency-bound schedules win (config 3); HS_C2=2 forces the codes
      const bool few = M.nslices < 2LL * ctx->num_sms * 48 && (M.nslices > 0 ? M.slots / (M.nslices * 128) : 0) < 256;
      const int c2env = M.c2 ? env_int("HS_C2", 1) : 0;
      const bool c2 = !transpose && M.c2 && M.d16 && !M.d16v && !M.c8 && !impl && c2env != 0 && (!few || c2env == 2);
      // c2 slices: a quarter byte of step codes per nonzero instead of the 2-byte delta, 16 B of escapes per row
      const bool t8 = transpose && M.t8 && M.d16 && !M.c8;
      const double c2frac = c2 || t8 ? (double)M.c2_slots / std::max<long long>(M.slots, 1) : 0.0;
      const double bytes = (double)M.stored_values() * sizeof(V) +
                           ((double)M.nnz - (impl ? (double)imp_slots * M.nnz / std::max<long long>(M.slots, 1) : 0.0)) *
                               M.index_bytes() * (1.0 - c2frac) +
                           c2frac * ((double)M.nnz * (t8 ? 1.0 : 0.25) + (double)M.rows * 16.0) +
                           (c2 ? (double)M.c2_slices * 16.0 : 0.0) +
                           (double)M.rows * M.slot_bytes() +
                           (double)M.n_exc * 4 + (double)M.nslices * 8 + (double)M.cols * sizeof(Tin) +
                           (double)M.rows * sizeof(T);
      const bool tflag = !transpose && sflag.p != nullptr;
      if (transpose && sblk.n_bins > 0 && preblocked) {
        xi = yB.as<Tin>();
      } else if (transpose && sblk.n_bins > 0) {
        Prof p(ctx, "y_block", 2.0 * (double)m * sizeof(Tin));
        const size_t need = (size_t)sblk.size(n_angles) * sizeof(Tin);
        if (yB.bytes < need) yB.alloc(need, false);
        sino_block_kernel<Tin><<<grid_for(m, 256, ctx->num_sms * 8), 256, 0, s>>>(m, sblk, xi, yB.as<Tin>());
        CKL();
        xi = yB.as<Tin>();
      }
      if (tflag && preblocked) {
        // the caller wrote the transposed image copy beside x (normalize_transpose_kernel)
      } else if (tflag) {
        // transposed image copy of x for the near-horizontal ray slices
        Prof p(ctx, "x_transpose", 2.0 * (double)n * sizeof(Tin));
        const size_t need = (size_t)n * sizeof(Tin);
        if (xT.bytes < need) xT.alloc(need, false);
        dim3 tg((img_grid + 31) / 32, (img_grid + 31) / 32);
        image_transpose_kernel<Tin><<<tg, 256, 0, s>>>(img_grid, xi, xT.as<Tin>());
        CKL();
      }
      Prof p(ctx, transpose ? "spmv_AT" : "spmv_A", bytes);
      L2Window l2w(s, xi, (size_t)M.cols * sizeof(Tin));
      if (M.c8) {
        // 3-deep ring, 6 blocks of 8 warps per SM (fp32); fp64 values / work fit 3 blocks
        constexpr int MINB = (sizeof(T) == 4 && sizeof(V) == 4) ? 6 : 3;
        auto kern = M.c8g.mode == 0 ? sell_spmv_c8_kernel<V, Tin, T, 0, 3, MINB> : sell_spmv_c8_kernel<V, Tin, T, 1, 3, MINB>;
        const int smem = C8Lane<V, 3>::smem_bytes(256);
        CK(ensure_smem((const void*)kern, smem));
        kern<<<grid, 256, smem, s>>>(M.rows, M.nslices, M.sptr.as<long long>(), M.rlen.as<int>(), M.rbase.as<int>(),
                                  M.code.as<unsigned char>(), M.xoff.as<int>(), M.exc.as<int>(), M.val.as<V>(), xi,
                                  tflag ? xT.as<Tin>() : nullptr, tflag ? sflag.as<unsigned char>() : nullptr, M.c8g.G,
                                  M.rperm.as<int>(), transpose ? nullptr : M.sorder.as<int>(),
                                  M.sched.as<unsigned int>(), yo);
      } else if (M.d16v) {
        if constexpr (sizeof(V) == 4) {
          int gshift = -1;
          if (img_grid > 0 && (img_grid & (img_grid - 1)) == 0) gshift = __builtin_ctz((unsigned)img_grid);
          const bool p2 = gshift >= 0 || !tflag;
          auto kern = p2 ? sell_spmv_d16v_kernel<Tin, T, true> : sell_spmv_d16v_kernel<Tin, T, false>;
          kern<<<grid, 256, 0, s>>>(M.rows, M.nslices, M.sptr.as<long long>(), M.vptr.as<long long>(),
                                    M.rlen.as<int>(), M.rbase.as<int>(), M.dcol.as<short>(), M.val.as<float>(),
                                    M.fv.as<float>(), xi, tflag ? xT.as<Tin>() : nullptr,
                                    tflag ? sflag.as<unsigned char>() : nullptr, img_grid, gshift >= 0 ? gshift : 0,
                                    M.rperm.as<int>(), transpose ? nullptr : M.sorder.as<int>(),
                                    M.sched.as<unsigned int>(), yo);
        } else {
          fail(HS_ERR_RUNTIME, "d16v SELL with non-fp32 values");
        }
      } else if (t8) {
        // 8-bit step codes over the 4-angle interleaved sinogram (hs_c2.cuh), 16-bit deltas elsewhere
        constexpr bool F32 = sizeof(T) == 4 && sizeof(V) == 4;
        constexpr int MINB = F32 ? 6 : 3;
        sell_spmv_t8_kernel<V, Tin, T, MINB><<<grid, 256, 0, s>>>(
            M.rows, M.nslices, M.sptr.as<long long>(), M.rlen.as<int>(), M.rbase.as<int>(), M.dcol.as<short>(),
            M.val.as<V>(), xi, M.c2ok.as<unsigned char>(), M.c2start.as<int>(), M.c2esc.as<int4>(),
            M.c2code.as<unsigned char>(), M.t8_bins, M.rperm.as<int>(), nullptr, M.sched.as<unsigned int>(), yo);
      } else if (c2) {
        // 2-bit step codes on the conforming ray slices (hs_c2.cuh), 16-bit deltas elsewhere
        int gshift = -1;
        if (img_grid > 0 && (img_grid & (img_grid - 1)) == 0) gshift = __builtin_ctz((unsigned)img_grid);
        const bool p2 = gshift >= 0 || !tflag;
        constexpr bool F32 = sizeof(T) == 4 && sizeof(V) == 4;
#ifndef HS_C2_MINB
#define HS_C2_MINB 6
#endif
        constexpr int MINB = F32 ? HS_C2_MINB : 3;
        // (8 blocks per SM, 32 registers with 40 B of spills: 3.17 against 2.78 ms)
        auto kern = p2 ? sell_spmv_c2_kernel<V, Tin, T, true, MINB> : sell_spmv_c2_kernel<V, Tin, T, false, MINB>;
        kern<<<grid, 256, 0, s>>>(M.rows, M.nslices, M.sptr.as<long long>(), M.rlen.as<int>(), M.rbase.as<int>(),
                                  M.dcol.as<short>(), M.val.as<V>(), xi, tflag ? xT.as<Tin>() : nullptr,
                                  tflag ? sflag.as<unsigned char>() : nullptr, M.c2ok.as<unsigned char>(),
                                  M.c2tab.as<int4>(), M.c2start.as<int>(), M.c2esc.as<int4>(),
                                  M.c2code.as<unsigned short>(), img_grid, gshift >= 0 ? gshift : 0,
                                  M.sorder.as<int>(), M.sched.as<unsigned int>(), yo);
      } else if (impl) {
        // implicit columns on the verified ray slices (RayGen), 16-bit deltas elsewhere
        int gshift = -1;
        if (img_grid > 0 && (img_grid & (img_grid - 1)) == 0) gshift = __builtin_ctz((unsigned)img_grid);
        const bool p2 = gshift >= 0 || !tflag;
        // resident blocks per SM: 6 caps registers at 40 (RayGen state spills to the stack), 4 allows 64
        constexpr bool F32 = sizeof(T) == 4 && sizeof(V) == 4;
        const bool b6 = F32 && env_flag("HS_IMP_MINB6");
        auto kern = b6 ? (p2 ? sell_spmv_imp_kernel<V, Tin, T, true, F32 ? 6 : 3>
                             : sell_spmv_imp_kernel<V, Tin, T, false, F32 ? 6 : 3>)
                       : (p2 ? sell_spmv_imp_kernel<V, Tin, T, true, F32 ? 4 : 2>
                             : sell_spmv_imp_kernel<V, Tin, T, false, F32 ? 4 : 2>);
        kern<<<grid, 256, 0, s>>>(M.rows, M.nslices, M.sptr.as<long long>(), M.rlen.as<int>(), M.rbase.as<int>(),
                                  M.dcol.as<short>(), M.val.as<V>(), xi, tflag ? xT.as<Tin>() : nullptr,
                                  tflag ? sflag.as<unsigned char>() : nullptr, imp.as<unsigned char>(), ray_tab(),
                                  gshift >= 0 ? gshift : 0, M.sorder.as<int>(), M.sched.as<unsigned int>(), yo);
      } else if (M.d16) {
        int gshift = -1;
        if (img_grid > 0 && (img_grid & (img_grid - 1)) == 0) gshift = __builtin_ctz((unsigned)img_grid);
        // few slices (< 2 per resident warp): the walk is latency-bound, use the deeper pipeline
        // -- but not for long rows (one rank's share of config 4 on 8 GPUs: 8.1k
        // slices of ~460 chunks; depth 0 at full occupancy 0.52 ms, depth 1 0.68 ms,
        // tools/ab_rank_share.py)
        const long long avg_chunks = M.nslices > 0 ? M.slots / (M.nslices * 128) : 0;
        const bool deep = env_flag("HS_D16_DEEP") ||
                          (M.nslices < 2LL * ctx->num_sms * 48 && avg_chunks < 256 && !env_flag("HS_D16_SHALLOW"));
        const bool p2 = gshift >= 0 || !tflag;
        // pipeline depth in chunks per gather step (HS_D16_PIPE overrides for A/B runs)
        // (fewer slices than ~32 per SM, e.g. config 3's A: 4,078 slices of 460-entry rays: depth 2,
        // 0.157 -> 0.107 ms; its A^T, 8,192 shorter slices, stays at depth 1: 0.091 vs 0.106 ms)
        // between 32 and 96 slices per SM (config 3's A^T: 8,192 slices of 57 chunks) the
        // stream goes through the per-lane cp.async ring: 0.090 -> 0.080 ms (depth 1)
        // (3: the full-occupancy kernel with unconditional, alternating-buffer prefetch;
        // config 4 A 3.54 -> 3.47 ms, A^T 3.72 -> 3.64 ms against depth 0)
        int depth = deep ? (M.nslices < 32LL * ctx->num_sms ? 2 : 8) : 3;
        if (const char* e = getenv("HS_D16_PIPE")) depth = atoi(e);
        auto pick = [&](auto p2c) {
          constexpr bool P2 = decltype(p2c)::value;
          return depth >= 4 ? sell_spmv_d16_kernel<V, Tin, T, P2, 4>
               : depth == 3 ? sell_spmv_d16_kernel<V, Tin, T, P2, 3>
               : depth == 2 ? sell_spmv_d16_kernel<V, Tin, T, P2, 2>
               : depth == 1 ? sell_spmv_d16_kernel<V, Tin, T, P2, 1>
                            : sell_spmv_d16_kernel<V, Tin, T, P2, 0>;
        };
        if (depth == 8) {
          // per-lane cp.async ring (hs_ops.cuh: sell_spmv_d16_ring_kernel)
          constexpr bool F32 = sizeof(T) == 4 && sizeof(V) == 4;
          constexpr int NS = 8, MINB = F32 ? 4 : 2;
          auto rk = p2 ? sell_spmv_d16_ring_kernel<V, Tin, T, true, NS, MINB>
                       : sell_spmv_d16_ring_kernel<V, Tin, T, false, NS, MINB>;
          const int smem = D16Ring<V, NS>::smem_bytes(256);
          CK(ensure_smem((const void*)rk, smem));
          rk<<<grid, 256, smem, s>>>(M.rows, M.nslices, M.sptr.as<long long>(), M.rlen.as<int>(), M.rbase.as<int>(),
                                     M.dcol.as<short>(), M.val.as<V>(), xi, tflag ? xT.as<Tin>() : nullptr,
                                     tflag ? sflag.as<unsigned char>() : nullptr, img_grid, gshift >= 0 ? gshift : 0,
                                     M.rperm.as<int>(), transpose ? nullptr : M.sorder.as<int>(),
                                     M.sched.as<unsigned int>(), yo);
          CKL();
          return;
        }
        auto kern = p2 ? pick(std::true_type{}) : pick(std::false_type{});
        kern<<<grid, 256, 0, s>>>(M.rows, M.nslices, M.sptr.as<long long>(), M.rlen.as<int>(), M.rbase.as<int>(),
                                  M.dcol.as<short>(), M.val.as<V>(), xi, tflag ? xT.as<Tin>() : nullptr,
                                  tflag ? sflag.as<unsigned char>() : nullptr, img_grid, gshift >= 0 ? gshift : 0,
                                  M.rperm.as<int>(),
                                  transpose ? nullptr : M.sorder.as<int>(),
                                  M.sched.as<unsigned int>(), yo);
      } else {
        sell_spmv_kernel<V, Tin, T><<<grid, 256, 0, s>>>(M.rows, M.nslices, M.sptr.as<long long>(), M.rlen.as<int>(),
                                                        M.col.as<int>(), M.val.as<V>(), xi,
                                                        tflag ? xT.as<Tin>() : nullptr,
                                                        tflag ? sflag.as<unsigned char>() : nullptr,
                                                        M.rperm.as<int>(), yo);
      }
      CKL();
    } else if (kind == OP_CSR) {
      const Csr& M = transpose ? At : A;
      constexpr int WARPS = sizeof(T) == 8 ? 4 : 8, CH = 32;
      const long long tiles = (M.rows + 31) / 32;
      const int grid = grid_for(tiles, WARPS, ctx->num_sms * 64);
      const double bytes = (double)M.nnz * (sizeof(V) + 4) + (double)(M.rows + 1) * 8 + (double)M.cols * sizeof(Tin) +
                           (double)M.rows * sizeof(T);
      Prof p(ctx, transpose ? "spmv_AT" : "spmv_A", bytes);
      csr_seq_spmv_kernel<V, Tin, T, WARPS, CH><<<grid, WARPS * 32, 0, s>>>(
          M.rows, M.rowptr.as<long long>(), M.col.as<int>(), M.val.as<V>(), xi, yo);
      CKL();
    } else if (kind == OP_DENSE) {
      const long long rows = transpose ? n : m, cols = transpose ? m : n;
      const V* Mcm = (transpose ? Atcm : Acm).as<V>();
      Prof p(ctx, "dense_gemv", (double)rows * cols * sizeof(V));
      if (env_flag("HS_DENSE_SIMPLE")) {
        dense_seq_gemv_kernel<V, Tin, T><<<grid_for(rows, 256, 1 << 30), 256, 1024 * sizeof(T), s>>>(rows, cols, Mcm,
                                                                                                     xi, yo);
      } else {
        const bool rb32 = env_flag("HS_DENSE_RB32");
        const int RB = rb32 ? 32 : 8;
        const size_t smem = rb32 ? dense_tile_smem(sizeof(T), 32, 256) : dense_tile_smem(sizeof(T), 8, 1024);
        auto kern = rb32 ? dense_tile_gemv_kernel<V, Tin, T, 32, 256> : dense_tile_gemv_kernel<V, Tin, T, 8, 1024>;
        CK(ensure_smem((const void*)kern, smem));
        kern<<<(int)((rows + RB - 1) / RB), 256, smem, s>>>(rows, cols, Mcm, xi, yo);
      }
      CKL();
    } else if (kind == OP_PSF && sharded) {
      // x is the full image (all ranks' rows): cut this rank's window (own
      // rows + kh/2 halo rows each side, zero outside the image)
      const int ry = kh / 2;
      const long long win_rows = psf_rows + 2LL * ry;
      const size_t need = (size_t)win_rows * W * sizeof(Tin);
      if (psfwin.bytes < need) psfwin.alloc(need, false);
      CK(cudaMemsetAsync(psfwin.p, 0, need, s));
      const long long g0 = std::max<long long>(0, psf_row0 - ry), g1 = std::min<long long>(H, psf_row0 + psf_rows + ry);
      CK(cudaMemcpyAsync(psfwin.as<Tin>() + (g0 - (psf_row0 - ry)) * W, xi + g0 * W, (size_t)(g1 - g0) * W * sizeof(Tin),
                         cudaMemcpyDeviceToDevice, s));
      psf_launch<V, Tin, T>(psfwin.as<Tin>(), (int)win_rows, ry, (int)psf_rows, yo, transpose);
    } else {
      psf_launch<V, Tin, T>(xi, H, 0, H, yo, transpose);
    }
  }

  // PSF stencil on an x of `rows` image rows (width W), output rows
  // [out_row0, out_row0 + out_rows) into y (row out_row0 first)
  template <class V, class Tin, class T>
  void psf_launch(const Tin* xi, int rows, int out_row0, int out_rows, T* yo, bool transpose) const {
    cudaStream_t s = ctx->stream;
    Prof p(ctx, "psf_stencil", (double)out_rows * W * (sizeof(Tin) + sizeof(T)));
    // register-blocked tiles (128 x 16 outputs) when they fill the GPU; small
    // images (config 2: 256^2 -> 32 tiles) keep the 32 x 8 tiles of the simple kernel
    const long long rb_tiles = (long long)((W + 127) / 128) * ((out_rows + 15) / 16);
    if ((kw == 15 || kw == 31) && !env_flag("HS_PSF_SIMPLE") &&
        (rb_tiles >= 2LL * ctx->num_sms || env_flag("HS_PSF_RB"))) {
      auto launch = [&](auto kwc) {
        constexpr int KWc = decltype(kwc)::value;
        using G = PsfRb<T, KWc>;
        const dim3 grid((W + G::TILE_X - 1) / G::TILE_X, (out_rows + G::TY - 1) / G::TY);
        const size_t smem = G::smem(kh);
        auto kern = transpose ? psf_stencil_rb_kernel<V, Tin, T, KWc, G::R, G::TXT, G::TY, true>
                              : psf_stencil_rb_kernel<V, Tin, T, KWc, G::R, G::TXT, G::TY, false>;
        CK(ensure_smem((const void*)kern, smem));
        kern<<<grid, G::TXT * G::TY, smem, s>>>(rows, W, kh, K.as<V>(), xi, yo, out_row0, out_rows);
        CKL();
      };
      if (kw == 15) launch(std::integral_constant<int, 15>());
      else launch(std::integral_constant<int, 31>());
    } else {
      constexpr int TX = 32, TY = 8;
      dim3 grid((W + TX - 1) / TX, (out_rows + TY - 1) / TY);
      const size_t smem = ((size_t)(TX + 2 * (kw / 2)) * (TY + 2 * (kh / 2)) + (size_t)kh * kw) * sizeof(T);
      // 15-wide rows unrolled (config 2: 19 -> see DESIGN.md); other widths generic
      auto kern = kw == 15 && !env_flag("HS_PSF_GENERIC") ? psf_stencil_kernel<V, Tin, T, TX, TY, 15>
                                                          : psf_stencil_kernel<V, Tin, T, TX, TY, 0>;
      CK(ensure_smem((const void*)kern, smem));
      kern<<<grid, TX * TY, smem, s>>>(rows, W, kh, kw, K.as<V>(), xi, yo, transpose ? 1 : 0, out_row0, out_rows);
      CKL();
    }
  }

  // sharded PSF: stencil of this rank's rows from a prepared window (own rows
  // + halos, `win_rows` = psf_rows + 2 * (kh / 2) rows, type xdt) into y (wdt)
  void apply_psf_window(const void* win, int xdt, void* y, int wdt, bool transpose) const {
    const int ry = kh / 2;
    auto go = [&](auto vt, auto it, auto ot) {
      using V = decltype(vt);
      using Tin = decltype(it);
      using T = decltype(ot);
      psf_launch<V, Tin, T>(reinterpret_cast<const Tin*>(win), (int)(psf_rows + 2 * ry), ry, (int)psf_rows,
                            reinterpret_cast<T*>(y), transpose);
    };
    if (wdt == HS_F64) {
      if (xdt != HS_F64) fail(HS_ERR_TYPE, "fp64 work needs fp64 input vectors");
      if (vdtype == HS_F64) go(double{}, double{}, double{});
      else go(float{}, double{}, double{});
    } else if (xdt == HS_F32) {
      if (vdtype == HS_F64) go(double{}, float{}, float{});
      else go(float{}, float{}, float{});
    } else {
      if (vdtype == HS_F64) go(double{}, __nv_bfloat16{}, float{});
      else go(float{}, __nv_bfloat16{}, float{});
    }
  }

  // x: type xdt; y: type T (wdt)
  void apply(const void* x, int xdt, void* y, int wdt, bool transpose, bool preblocked = false) const {
    const bool pb = preblocked;
    if (wdt == HS_F64) {
      if (xdt != HS_F64) fail(HS_ERR_TYPE, "fp64 work needs fp64 input vectors");
      if (vdtype == HS_F64) apply_t<double, double, double>(x, y, transpose, pb);
      else apply_t<float, double, double>(x, y, transpose, pb);
    } else if (wdt == HS_F32) {
      if (xdt == HS_F32) {
        if (vdtype == HS_F64) apply_t<double, float, float>(x, y, transpose, pb);
        else apply_t<float, float, float>(x, y, transpose, pb);
      } else if (xdt == HS_BF16) {
        if (vdtype == HS_F64) apply_t<double, __nv_bfloat16, float>(x, y, transpose, pb);
        else apply_t<float, __nv_bfloat16, float>(x, y, transpose, pb);
      } else {
        fail(HS_ERR_TYPE, "fp32 work needs fp32/bf16 input vectors");
      }
    } else {
      fail(HS_ERR_TYPE, "work dtype must be fp64 or fp32");
    }
  }

  // Shard granule of the range (side 0, length m) / domain (side 1, length
  // n) vectors: row shards are whole granules (rays in power-of-two blocks;
  // 8 image rows), and the sketches of these vectors sum their partials
  // granule by granule (hs_sketch.cuh), so solves give the same bits for any
  // number of ranks.  Operators that never shard: one granule.
  long long granule(int side) const {
    if (kind == OP_CSR && tomo_grid > 0) return side == 0 ? std::max<long long>(64, shard_granule(m)) : 8LL * tomo_grid;
    if (kind == OP_PSF) return 8LL * W;
    return side == 0 ? m : n;
  }

  long long nnz_total() const { return kind == OP_CSR ? A.nnz : (kind == OP_DENSE ? m * n : 0); }
};

// Mark the slices of a tomography A (SELL copy with int32 columns, natural
// row order) whose every row RayGen reproduces exactly; those slices then
// stream values only (hs_ops.cuh: sell_spmv_imp_kernel).  Opt-in
// (HS_IMPLICIT=1): bit-identical, and 4 instead of 6 B per nonzero, but the
// per-image-row fp64 range update runs in divergent lanes almost every entry
// for steep rays; config 4's A apply measured 10.7 ms against 3.6 ms for the
// 16-bit deltas.
static void tomo_enable_implicit(hs_ctx* ctx, hs_op* op) {
  Sell& S = op->As;
  if (S.nslices == 0 || S.col.p == nullptr || S.rperm.p != nullptr || !env_flag("HS_IMPLICIT")) return;
  cudaStream_t s = ctx->stream;
  DBuf bad(S.nslices, true);
  tomo_implicit_check_kernel<<<grid_for(S.nslots(), 128, 1 << 30), 128, 0, s>>>(
      S.rows, S.nslices, S.sptr.as<long long>(), S.rlen.as<int>(), S.col.as<int>(), op->ray_tab(),
      bad.as<unsigned char>());
  CKL();
  std::vector<unsigned char> hb(S.nslices);
  std::vector<long long> hp(S.nslices + 1);
  CK(cudaMemcpyAsync(hb.data(), bad.p, S.nslices, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hp.data(), S.sptr.p, (S.nslices + 1) * sizeof(long long), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::vector<unsigned char> ok(S.nslices);
  long long ns = 0, nslot = 0;
  for (long long i = 0; i < S.nslices; ++i) {
    ok[i] = hb[i] ? 0 : 1;
    if (ok[i]) {
      ++ns;
      nslot += hp[i + 1] - hp[i];
    }
  }
  if (ns == 0) return;
  op->imp.alloc(S.nslices, false);
  CK(cudaMemcpyAsync(op->imp.p, ok.data(), S.nslices, cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  op->imp_slices = ns;
  op->imp_slots = nslot;
}

// build the transpose of a row-sorted CSR (rows x cols) on device: output rows
// are the columns [cb, ce), each sorted by the original row index
// (scipy M.T.tocsr() order).  `row_offset` is added to the stored keys.
template <class V>
static void csr_transpose(hs_ctx* ctx, const Csr& src, long long row_offset, long long cb, long long ce, Csr& dst) {
  cudaStream_t s = ctx->stream;
  const long long nr = ce - cb;
  dst.rows = nr;
  dst.cols = src.rows;  // caller fixes if row_offset != 0
  DBuf cnt((nr + 1) * sizeof(unsigned int));
  const int wpb = 8;
  if (src.rows > 0) {
    csr_colcount_kernel<<<grid_for(src.rows, wpb, 1 << 30), wpb * 32, 0, s>>>(
        src.rows, src.rowptr.as<long long>(), src.col.as<int>(), cb, ce, cnt.as<unsigned int>());
    CKL();
  }
  DBuf cnt64((nr + 1) * sizeof(long long));
  u32_to_i64_kernel<<<grid_for(nr + 1, 256, 1 << 30), 256, 0, s>>>(nr + 1, cnt.as<unsigned int>(), cnt64.as<long long>());
  CKL();
  dst.rowptr.alloc((nr + 1) * sizeof(long long));
  {
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt64.as<long long>(), dst.rowptr.as<long long>(), nr + 1, s));
    DBuf t(tmp, false);
    CK(cub::DeviceScan::ExclusiveSum(t.p, tmp, cnt64.as<long long>(), dst.rowptr.as<long long>(), nr + 1, s));
  }
  long long nnz = 0;
  CK(cudaMemcpyAsync(&nnz, dst.rowptr.as<long long>() + nr, sizeof(long long), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  dst.nnz = nnz;
  cnt.release();
  cnt64.release();
  DBuf cursor(nr * sizeof(unsigned long long), false);
  i64_to_u64_kernel<<<grid_for(nr, 256, 1 << 30), 256, 0, s>>>(nr, dst.rowptr.as<long long>(),
                                                               cursor.as<unsigned long long>());
  CKL();
  DBuf keys((size_t)std::max<long long>(nnz, 1) * sizeof(int), false);
  DBuf vals((size_t)std::max<long long>(nnz, 1) * sizeof(V), false);
  if (src.rows > 0) {
    csr_scatter_kernel<V><<<grid_for(src.rows, wpb, 1 << 30), wpb * 32, 0, s>>>(
        src.rows, row_offset, src.rowptr.as<long long>(), src.col.as<int>(), src.val.as<V>(), cb, ce,
        cursor.as<unsigned long long>(), keys.as<int>(), vals.as<V>());
    CKL();
  }
  cursor.release();
  // sort each output row by key, in batches of rows with < 2^30 items
  dst.col.alloc((size_t)std::max<long long>(nnz, 1) * sizeof(int), false);
  dst.val.alloc((size_t)std::max<long long>(nnz, 1) * sizeof(V), false);
  std::vector<long long> hptr(nr + 1);
  CK(cudaMemcpyAsync(hptr.data(), dst.rowptr.p, (nr + 1) * sizeof(long long), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const long long kBatch = 1LL << 30;
  long long r0 = 0;
  while (r0 < nr) {
    long long r1 = r0 + 1;
    while (r1 < nr && hptr[r1 + 1] - hptr[r0] <= kBatch) ++r1;
    const long long base = hptr[r0];
    const long long items = hptr[r1] - base;
    const int nseg = (int)(r1 - r0);
    if (items > 0) {
      // offsets relative to the batch base, as int
      std::vector<int> off(nseg + 1);
      for (int i = 0; i <= nseg; ++i) off[i] = (int)(hptr[r0 + i] - base);
      DBuf doff((nseg + 1) * sizeof(int), false);
      CK(cudaMemcpyAsync(doff.p, off.data(), (nseg + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
      size_t tmp = 0;
      CK(cub::DeviceSegmentedSort::SortPairs(nullptr, tmp, keys.as<int>() + base, dst.col.as<int>() + base,
                                             vals.as<V>() + base, dst.val.as<V>() + base, (int)items, nseg,
                                             doff.as<int>(), doff.as<int>() + 1, s));
      DBuf t(tmp, false);
      CK(cub::DeviceSegmentedSort::SortPairs(t.p, tmp, keys.as<int>() + base, dst.col.as<int>() + base,
                                             vals.as<V>() + base, dst.val.as<V>() + base, (int)items, nseg,
                                             doff.as<int>(), doff.as<int>() + 1, s));
      CK(cudaStreamSynchronize(s));
    }
    r0 = r1;
  }
}

// ---------------------------------------------------------------------------
// sketches

struct hs_sketch {
  hs_ctx* ctx = nullptr;
  int device = 0;
  int kind = HS_SKETCH_DENSE;
  long long ell = 0, m = 0;
  unsigned long long seed = 0;
  int zeta = 0;
  DBuf S;                 // dense row-major fp64
  DBuf rowptr, scol;      // CSR kind: rows, cols
  DBuf cval;              // CSR kind: fp64 values
  long long tile = 0;     // columns per partial tile (power of two; sparse sign: at most)
  // sparse sign: the tile layouts (hs_sketch.cuh: sketch_sparse_gather_kernel),
  // one per tile size in use, built on first use from the regenerated entries
  struct SparseLayout {
    long long tc = 0, ntiles = 0, nent = 0;
    int nsl = 0;
    DBuf tbase, soff, perm, ent;
  };
  mutable std::map<long long, std::unique_ptr<SparseLayout>> layouts;
  mutable std::mutex lay_mu;
  const SparseLayout& sparse_layout(long long tc) const;
  // tile size used with granule G: sparse-sign tiles must divide G
  long long tile_for(long long G) const {
    if (kind != HS_SKETCH_SPARSE_SIGN || G >= m) return tile;  // one granule: no alignment needed
    const long long low = G & -G;
    return std::min(tile, low);
  }
  uint2 key() const { return make_uint2((unsigned)seed, (unsigned)(seed >> 32)); }
  bool tiled() const { return kind != HS_SKETCH_CSR; }
  double scale() const {
    return kind == HS_SKETCH_GAUSSIAN ? 1.0 / std::sqrt((double)ell)
         : kind == HS_SKETCH_SPARSE_SIGN ? 1.0 / std::sqrt((double)zeta) : 1.0;
  }
  int tpg(long long G) const { return (int)((G + tile_for(G) - 1) / tile_for(G)); }
  // partial slots for `cols` input entries cut in granules of G
  long long slots(long long cols, long long G) const { return tiled() ? ((cols + G - 1) / G) * tpg(G) : 0; }
  // scratch (doubles) for the partials of nv vectors over `cols` input entries
  long long scratch_elems(int nv, long long cols, long long G) const { return (long long)nv * slots(cols, G) * ell; }

  // partials of nv vectors (column stride ldv) over the local entries
  // [0, loc) = global input entries [off, off + loc), off a multiple of the
  // granule G: part[(w * tstride + slot) * ell + i]
  template <class Tin>
  void partials_t(const Tin* v, long long ldv, int nv, long long off, long long loc, long long G, double* part,
                  long long tstride, cudaStream_t s) const {
    if (off % G != 0) fail(HS_ERR_VALUE, "sketch block offset %lld is not a multiple of the granule (%lld)", off, G);
    const TileMap tm{G, tile_for(G), loc, tpg(G)};
    if (kind == HS_SKETCH_GAUSSIAN) {
      CK(cudaGetLastError());
      g_launches += gauss_partials<Tin>(s, (int)ell, tm, off, key(), v, ldv, nv, part, tstride);
      CK(cudaGetLastError());
      return;
    }
    const long long nt = tm.slots();
    for (int w = 0; w < nv; ++w) {
      const Tin* vw = v + (long long)w * ldv;
      double* pw = part + (long long)w * tstride * ell;
      if (nt == 0) continue;
      if (kind == HS_SKETCH_DENSE) {
        sketch_dense_tile_kernel<Tin><<<dim3((unsigned)nt, (unsigned)((ell + 7) / 8)), 256, 0, s>>>((int)ell, tm, off,
                                                                                                  S.as<double>(), m, vw,
                                                                                                  pw);
        CKL();
      } else if (kind == HS_SKETCH_SPARSE_SIGN) {
        const SparseLayout& L = sparse_layout(tm.tc);
        sparse_partials<Tin>(s, (int)ell, tm, off, L.tbase.as<long long>(), L.soff.as<int>(),
                             L.perm.as<unsigned short>(), L.ent.as<unsigned short>(), vw, pw);
        CKL();
      } else {
        fail(HS_ERR_NOTIMPL, "explicit CSR sketches have no tile partials");
      }
    }
  }
  void partials(const void* v, int vdt, long long ldv, int nv, long long off, long long loc, long long G, double* part,
                long long tstride, cudaStream_t s) const {
    if (vdt == HS_F64) partials_t<double>(reinterpret_cast<const double*>(v), ldv, nv, off, loc, G, part, tstride, s);
    else if (vdt == HS_F32) partials_t<float>(reinterpret_cast<const float*>(v), ldv, nv, off, loc, G, part, tstride, s);
    else partials_t<__nv_bfloat16>(reinterpret_cast<const __nv_bfloat16*>(v), ldv, nv, off, loc, G, part, tstride, s);
  }
  // z[w * ldz + i] = scale * the ordered sum of all partials of the m inputs,
  // laid out as blocks of gpr granules ([block][w][slot][i])
  void reduce(const double* part, int nv, long long G, long long gpr, double* z, long long ldz, cudaStream_t s) const {
    sketch_tile_reduce_kernel<<<dim3((unsigned)((ell + RROWS - 1) / RROWS), nv), RROWS * RPH, 0, s>>>(
        (int)ell, m, G, tile_for(G), tpg(G), gpr, nv, part, scale(), z, ldz);
    CKL();
  }
  const char* prof_name() const {
    return kind == HS_SKETCH_GAUSSIAN ? "sketch_gauss" : kind == HS_SKETCH_SPARSE_SIGN ? "sketch_sparse"
         : kind == HS_SKETCH_DENSE ? "sketch_dense" : "sketch_csr";
  }
  // algorithmic bytes of one sketch of nv vectors of element size es
  double prof_bytes(int nv, size_t es, long long G) const {
    const double pbytes = 2.0 * nv * (double)slots(m, G) * ell * 8;  // partials written + read
    if (kind == HS_SKETCH_SPARSE_SIGN) {
      double eb = 2.0 * m * zeta;
      {
        std::lock_guard<std::mutex> g(lay_mu);
        const auto it = layouts.find(tile_for(G));
        if (it != layouts.end()) eb = 2.0 * it->second->nent;
      }
      return nv * (eb + (double)m * es) + pbytes;
    }
    if (kind == HS_SKETCH_DENSE) return nv * ((double)ell * m * 8 + (double)m * es) + pbytes;
    if (kind == HS_SKETCH_GAUSSIAN) return nv * (double)m * es + pbytes;
    return 0.0;
  }

  // z[:, w] = S v_w for nv vectors (column stride ldv; z column stride ldz)
  // over the whole input cut in granules of G (the operator's shard granule;
  // G = m: one granule), with `scratch` >= scratch_elems(nv, m, G) doubles.
  // The Gaussian kind generates S once for the whole batch; per vector the
  // result equals a single apply.
  void apply_many(const void* v, int vdt, long long ldv, int nv, double* z, long long ldz, double* scratch,
                  long long G, cudaStream_t st = nullptr) const {
    cudaStream_t s = st ? st : ctx->stream;
    if (nv <= 0) return;
    Prof p(ctx, prof_name(), prof_bytes(nv, dsize(vdt), G), s);
    if (kind == HS_SKETCH_CSR) {
      const size_t es = dsize(vdt);
      for (int w = 0; w < nv; ++w) {
        const void* vw = reinterpret_cast<const char*>(v) + (size_t)w * ldv * es;
        double* zw = z + (long long)w * ldz;
        auto go = [&](auto tag) {
          using Tin = decltype(tag);
          sketch_csr_kernel<Tin><<<(int)ell, 256, 0, s>>>((int)ell, rowptr.as<long long>(), scol.as<int>(),
                                                          cval.as<double>(), reinterpret_cast<const Tin*>(vw), zw);
        };
        if (vdt == HS_F64) go(double{});
        else if (vdt == HS_F32) go(float{});
        else go(__nv_bfloat16{});
        CKL();
      }
      return;
    }
    if (!scratch) fail(HS_ERR_RUNTIME, "sketch apply without partial scratch");
    const long long gpr = (m + G - 1) / G;
    partials(v, vdt, ldv, nv, 0, m, G, scratch, slots(m, G), s);
    reduce(scratch, nv, G, gpr, z, ldz, s);
  }
  void apply(const void* v, int vdt, double* z, double* scratch, long long G, cudaStream_t st = nullptr) const {
    apply_many(v, vdt, 0, 1, z, 0, scratch, G, st);
  }
};

// Sparse-sign tile layout for tile size tc (hs_sketch.cuh:
// sketch_sparse_gather_kernel): the entries (rows and signs from Philox,
// sparse_sign_gen_kernel) are regenerated on the device and bucketed on the
// host, per absolute tile of tc columns, by sketch row (columns ascending);
// rows sorted by entry count (descending, ties by row), slices of 32 rows,
// each slice padded to a multiple of 8 entries per lane and chunk-interleaved.
const hs_sketch::SparseLayout& hs_sketch::sparse_layout(long long tc) const {
  std::lock_guard<std::mutex> g(lay_mu);
  auto it = layouts.find(tc);
  if (it != layouts.end()) return *it->second;
  if (tc > 8192 || tc < 1) fail(HS_ERR_VALUE, "sparse-sign tile %lld out of range", tc);
  // entry = column offset (14 bits, the padding offset tc included) | sign bit 15
  cudaStream_t s = ctx->stream;
  const long long nnz = m * (long long)zeta;
  std::vector<int> rows(nnz), scol(nnz);
  {
    DBuf dr(nnz * sizeof(int), false), ds(nnz * sizeof(int), false);
    sparse_sign_gen_kernel<<<grid_for(m, 128, 1 << 30), 128, 0, s>>>(m, (int)ell, zeta, key(), dr.as<int>(),
                                                                    ds.as<int>());
    CKL();
    CK(cudaMemcpyAsync(rows.data(), dr.p, nnz * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(scol.data(), ds.p, nnz * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  auto L = std::make_unique<SparseLayout>();
  L->tc = tc;
  L->ntiles = (m + tc - 1) / tc;
  L->nsl = (int)((ell + 31) / 32);
  const int nsl = L->nsl;
  std::vector<long long> tbase(L->ntiles + 1, 0);
  std::vector<int> soff((size_t)L->ntiles * (nsl + 1), 0);
  std::vector<unsigned short> perm((size_t)L->ntiles * nsl * 32, 0xFFFF);
  std::vector<unsigned short> ent;
  ent.reserve((size_t)(nnz * 1.2) + 256);
  std::vector<int> cnt(ell), order(ell), pos(ell), fill(ell);
  for (long long k = 0; k < L->ntiles; ++k) {
    const long long c0 = k * tc, c1 = std::min(m, c0 + tc);
    std::fill(cnt.begin(), cnt.end(), 0);
    for (long long c = c0; c < c1; ++c)
      for (int j = 0; j < zeta; ++j) ++cnt[rows[c * zeta + j]];
    for (int r = 0; r < ell; ++r) order[r] = r;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cnt[a] > cnt[b]; });
    for (int p = 0; p < (int)ell; ++p) pos[order[p]] = p;
    tbase[k] = (long long)ent.size();
    int* so = soff.data() + (size_t)k * (nsl + 1);
    int off = 0;
    for (int sl = 0; sl < nsl; ++sl) {
      so[sl] = off;
      const int first = sl * 32;
      const int len = first < ell ? cnt[order[first]] : 0;  // longest row of the slice
      off += ((len + 7) / 8) * 256;
      for (int l = 0; l < 32 && first + l < ell; ++l) perm[((size_t)k * nsl + sl) * 32 + l] = (unsigned short)order[first + l];
    }
    so[nsl] = off;
    ent.resize(ent.size() + (size_t)off, (unsigned short)tc);  // padding reads the zero after the tile
    std::fill(fill.begin(), fill.end(), 0);
    for (long long c = c0; c < c1; ++c)
      for (int j = 0; j < zeta; ++j) {
        const int r = rows[c * zeta + j];
        const int p = pos[r], sl = p / 32, lane = p % 32, e = fill[r]++;
        const size_t idx = (size_t)tbase[k] + so[sl] + (size_t)(e / 8) * 256 + lane * 8 + e % 8;
        ent[idx] = (unsigned short)((c - c0) | (scol[c * zeta + j] < 0 ? 0x8000 : 0));
      }
  }
  tbase[L->ntiles] = (long long)ent.size();
  L->nent = (long long)ent.size();
  L->tbase.alloc(tbase.size() * sizeof(long long), false);
  L->soff.alloc(soff.size() * sizeof(int), false);
  L->perm.alloc(perm.size() * sizeof(unsigned short), false);
  L->ent.alloc(std::max<size_t>(ent.size(), 8) * sizeof(unsigned short), false);
  CK(cudaMemcpyAsync(L->tbase.p, tbase.data(), tbase.size() * sizeof(long long), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(L->soff.p, soff.data(), soff.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(L->perm.p, perm.data(), perm.size() * sizeof(unsigned short), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(L->ent.p, ent.data(), ent.size() * sizeof(unsigned short), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  auto& ref = *L;
  layouts.emplace(tc, std::move(L));
  return ref;
}

// ---------------------------------------------------------------------------
// result

struct hs_result {
  int n_records = 0, termination = HS_TERM_MAXITER, k = 0, bd_side = -1;
  int n_basis_data = 0, n_basis_sol = 0;
  bool square = true;
  long long m = 0, n = 0, ell = 0;
  int basis_dtype = HS_F64;
  std::vector<double> x, sres, proj, relerr, wall_ms, H, W, Z, sr0, y, resnorm, kappa_basis, kappa_dbar, eps_embed;
  std::vector<int> rankfb;
  std::vector<long long> matvecs, tmatvecs, dots, sketches, t, g;
  double loop_ms = 0.0;
  // device-resident bases kept for on-demand export
  std::shared_ptr<DBuf> Lb, Db;
  // final iterate on the device (n doubles), when the solver keeps it there instead of in x
  std::shared_ptr<DBuf> xdev;
  long long ldn = 0, ldm = 0;
  hs_ctx* ctx = nullptr;
  int device = 0;
  // sharded solves keep only this rank's rows of the bases
  bool sharded = false;
  long long n_loc = 0, m_loc = 0;
};

// ---------------------------------------------------------------------------
// the solver

namespace {

// Incremental QR (classical Gram-Schmidt, one reorthogonalisation) of a
// growing set of device columns, for the condition-number diagnostics
// (hs_diag.cuh).  Q and R in fp64.
struct DiagQR {
  hs_ctx* ctx = nullptr;
  long long len = 0, ld = 0;
  int cap = 0, cnt = 0;
  DBuf Q, R, v, rtmp, part, sq;
  void init(hs_ctx* c, long long n, int capacity) {
    ctx = c;
    len = n;
    ld = (n + 63) / 64 * 64;
    cap = capacity;
    cnt = 0;
    Q.alloc((size_t)cap * ld * sizeof(double));
    R.alloc((size_t)cap * cap * sizeof(double));
    v.alloc(ld * sizeof(double));
    rtmp.alloc((cap + 1) * sizeof(double));
    part.alloc((size_t)c->num_sms * 2 * (cap + 1) * sizeof(double));
    sq.alloc(2 * sizeof(double));
  }
  template <class X>
  void append(const X* col) {
    if (cnt >= cap) fail(HS_ERR_RUNTIME, "diagnostic QR capacity exceeded");
    cudaStream_t s = ctx->stream;
    const int NB = ctx->num_sms * 2, G = ctx->num_sms * 8;
    double* vq = v.as<double>();
    to_f64_kernel<X><<<grid_for(len, 256, G), 256, 0, s>>>(len, col, vq);
    CKL();
    double* rc = R.as<double>() + (long long)cnt * cap;
    const double* Qp = Q.as<double>();
    for (int pass = 0; pass < 2 && cnt > 0; ++pass) {
      double* coef = pass == 0 ? rc : rtmp.as<double>();
      mdot_kernel<double><<<NB, 256, 0, s>>>(len, Qp, ld, cnt, vq, part.as<double>());
      CKL();
      mdot_finish_kernel<<<(cnt + 127) / 128, 128, 0, s>>>(NB, cnt, part.as<double>(), coef, 0);
      CKL();
      maxpy_kernel<double><<<grid_for(len, 256, G), 256, (size_t)cnt * sizeof(double), s>>>(len, Qp, ld, cnt, coef, vq);
      CKL();
      if (pass == 1) {
        add_into_kernel<<<(cnt + 127) / 128, 128, 0, s>>>(cnt, rc, rtmp.as<double>());
        CKL();
      }
    }
    mdot_kernel<double><<<NB, 256, 0, s>>>(len, vq, 0, 1, vq, part.as<double>());
    CKL();
    mdot_finish_kernel<<<1, 32, 0, s>>>(NB, 1, part.as<double>(), sq.as<double>(), 0);
    CKL();
    qr_col_finish_kernel<<<1, 1, 0, s>>>(cnt, sq.as<double>(), rc, sq.as<double>() + 1);
    CKL();
    double* qn = Q.as<double>() + (long long)cnt * ld;
    CK(cudaMemcpyAsync(qn, vq, len * sizeof(double), cudaMemcpyDeviceToDevice, s));
    scale_inv_kernel<<<grid_for(len, 256, G), 256, 0, s>>>(len, qn, sq.as<double>() + 1);
    CKL();
    ++cnt;
  }
  // singular values of the leading kk columns (R[:kk, :kk]) into sv
  void singular_values(int kk, double* sv, DBuf& work) {
    cudaStream_t s = ctx->stream;
    if (work.bytes < (size_t)kk * kk * sizeof(double)) work.alloc((size_t)cap * cap * sizeof(double));
    r_block_kernel<<<(kk * kk + 255) / 256, 256, 0, s>>>(kk, R.as<double>(), cap, work.as<double>());
    CKL();
    jacobi_sv_kernel<<<1, 1024, 0, s>>>(kk, kk, work.as<double>(), kk, sv, 40);
    CKL();
  }
};

template <class T, class B>
struct Solver {
  static constexpr int VEC = 16 / sizeof(B);
  hs_ctx* ctx;
  hs_op* op;
  const hs_config cfg;
  hs_sketch* S2;
  hs_sketch* S1;
  int wdt, bdt;

  Solver(hs_ctx* c, hs_op* o, const hs_config& cf, hs_sketch* s2, hs_sketch* s1, int w, int b)
      : ctx(c), op(o), cfg(cf), S2(s2), S1(s1), wdt(w), bdt(b) {}

  void fsub(const T* u, const long long* pos, const T* P, int ldp, int k, int iter, int side, T* c,
            double* hcol) {
    if (k == 0) return;
    cudaStream_t s = ctx->stream;
    launch_fsub<T>(s, u, pos, P, ldp, k, st, iter, side, c, hcol);
    CKL();
  }

  LoopState* st = nullptr;

  void run(const double* b_h, const double* x0_h, const double* xt_h, hs_result* res) {
    cudaStream_t s = ctx->stream;
    const bool timing = getenv("HS_TIMING") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
      return std::chrono::duration<double, std::milli>(b - a).count();
    };
    const auto t_start = now();
    const bool square = cfg.square != 0;
    const int K = cfg.maxiter;
    const long long m = op->m, n = op->n;
    // unsketched cmrh / lslu (solvers.py:542-559): the projected matrix is H
    // itself ((K+1) rows), rhs beta e1, penalty columns e_j (N = I)
    const bool skd = cfg.sketched != 0;
    const long long ell = skd ? S2->ell : (long long)K + 1;
    const bool lamon = cfg.lam > 0.0;
    const bool sb = cfg.sketch_basis != 0;
    // sketch granules: S2 sketches range vectors, S1 domain vectors
    const long long G2 = op->granule(0), G1 = op->granule(1);
    const bool printed = cfg.printed_f != 0 && !square && lamon && skd;  // slslu_tikhonov(printed_f_columns=True)
    const long long ldm = round_up(m, 64), ldn = round_up(n, 64);
    const int ldp = K + 2;
    const int Ls = (int)(lamon ? 2 * ell : ell);
    const int ldq = (int)round_up(Ls, 32);
    const int SMS = ctx->num_sms;

    // ---- buffers
    auto Lb = std::make_shared<DBuf>((size_t)(K + 1) * ldn * sizeof(B));
    std::shared_ptr<DBuf> Db;
    if (!square) Db = std::make_shared<DBuf>((size_t)(K + 2) * ldm * sizeof(B));
    DBuf u(ldm * sizeof(T)), q(ldn * sizeof(T)), r0(ldm * sizeof(T)), bT(ldm * sizeof(T));
    DBuf bd(m * sizeof(double), false), x0d, xtd;
    // x stays on the device with the result; hs_result_x copies it straight
    // into the caller's array (no host staging vector)
    auto xdp = std::make_shared<DBuf>(n * sizeof(double));
    DBuf& xd = *xdp;
    DBuf Hb((size_t)(K + 1) * K * sizeof(double)), Wb((size_t)(K + 2) * (K + 1) * sizeof(double));
    DBuf PD((size_t)ldp * ldp * sizeof(T)), PL((size_t)ldp * ldp * sizeof(T));
    DBuf tpos(ldp * sizeof(long long)), gpos(ldp * sizeof(long long));
    DBuf cvec(ldp * sizeof(T)), pv(2 * sizeof(T));
    DBuf Zb((size_t)ell * K * sizeof(double)), Fb((size_t)ell * (K + 1) * sizeof(double)),
        Gb((size_t)ell * (K + 2) * sizeof(double)), sr0(ell * sizeof(double));
    DBuf Qb((size_t)ldq * K * sizeof(double)), Rinv((size_t)K * K * sizeof(double)), Rdiag(K * sizeof(double)),
        yb(K * sizeof(double)), Yh((size_t)K * K * sizeof(double));
    const int NB = qr_blocks(Ls);
    DBuf part((size_t)4 * NB * (K + 2) * sizeof(double));
    DBuf sresb(K * sizeof(double)), projb(K * sizeof(double)), rfb(K * sizeof(int)), rel2((K + 1) * sizeof(double));
    const int CAND_CAP = (int)std::min<long long>(1LL << 20, std::max<long long>(4096, (std::max(ldm, ldn) / VEC + 255) / 256));
    DBuf candp((size_t)CAND_CAP * sizeof(Cand)), xpart((size_t)CAND_CAP * sizeof(double));
    DBuf stb(sizeof(LoopState));
    st = stb.as<LoopState>();
    LoopState hst;
    const bool diag = cfg.diagnostics != 0;
    DBuf xk(diag ? n * sizeof(double) : 0), xkT(diag ? ldn * sizeof(T) : 0), axk(diag ? ldm * sizeof(T) : 0),
        resn2(diag ? (K + 1) * sizeof(double) : 0), rpart(diag ? SMS * 2 * sizeof(double) : 0);
    // condition numbers / embedding distortion (solvers.py:526-532): incremental
    // QR of the data basis (qB, rectangular), the solution basis (qL) and
    // [r0, A l_1, ...] (qW); Jacobi SVDs of the small factors (hs_diag.cuh)
    DiagQR qB, qL, qW;
    DBuf svA, svB, djac, Xw, Mw, kbuf;
    const bool diag_eps = diag && skd && !sb;
    if (diag) {
      qL.init(ctx, n, K + 2);
      if (!square) qB.init(ctx, m, K + 2);
      if (diag_eps) {
        qW.init(ctx, m, K + 2);
        Xw.alloc((size_t)ell * (K + 2) * sizeof(double));
        Mw.alloc((size_t)ell * (K + 2) * sizeof(double));
      }
      svA.alloc((K + 2) * sizeof(double));
      svB.alloc((K + 2) * sizeof(double));
      kbuf.alloc((size_t)3 * (K + 1) * sizeof(double));
    }

    // sampled pivoting (hessenberg.py:93-129): host-drawn positions per
    // selection slot, device copies of the permutations t / g and inverses
    const int ps = cfg.pivot_sample;
    DBuf posd, permT, whereT, permG, whereG;
    if (ps > 0) {
      const int nslots = square ? K + 1 : 2 * K + 2;
      posd.alloc((size_t)nslots * ps * sizeof(long long), false);
      CK(cudaMemcpyAsync(posd.p, cfg.pivot_positions, (size_t)nslots * ps * sizeof(long long), cudaMemcpyHostToDevice, s));
      const long long dt = square ? n : m;
      for (DBuf* b : {&permT, &whereT}) {
        b->alloc(dt * sizeof(long long), false);
        iota_kernel<<<grid_for(dt, 256, 1 << 30), 256, 0, s>>>(b->as<long long>(), (int)dt);
        CKL();
      }
      if (!square) {
        for (DBuf* b : {&permG, &whereG}) {
          b->alloc(n * sizeof(long long), false);
          iota_kernel<<<grid_for(n, 256, 1 << 30), 256, 0, s>>>(b->as<long long>(), (int)n);
          CKL();
        }
      }
    }
    // the sampled pick after the full-scan winner is in st (no draw when the
    // admissible population dim - used is <= the sample size)
    auto sample = [&](const T* v, long long dim, long long used, int slot, int side, int iter) {
      if (ps <= 0 || used >= dim || (long long)ps >= dim - used) return;
      sample_pick_kernel<T><<<1, 256, 0, s>>>(v, (side == 0 ? permT : permG).template as<long long>(), used,
                                              posd.as<long long>() + (long long)slot * ps, ps, st, side, iter);
      CKL();
    };
    auto swap_perm = [&](int side, long long used) {
      if (ps <= 0) return;
      perm_swap_kernel<<<1, 1, 0, s>>>((side == 0 ? permT : permG).template as<long long>(),
                                       (side == 0 ? whereT : whereG).template as<long long>(), used, st, side);
      CKL();
    };

    if (timing) CK(cudaStreamSynchronize(s));
    const auto t_alloc = now();
    CK(cudaMemcpyAsync(bd.p, b_h, m * sizeof(double), cudaMemcpyHostToDevice, s));
    if (x0_h) {
      x0d.alloc(n * sizeof(double), false);
      CK(cudaMemcpyAsync(x0d.p, x0_h, n * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    double xt_norm = 0.0;
    if (xt_h) {
      xtd.alloc(n * sizeof(double), false);
      CK(cudaMemcpyAsync(xtd.p, xt_h, n * sizeof(double), cudaMemcpyHostToDevice, s));
      xt_norm = std::sqrt(host_sumsq(xt_h, n));
      if (xt_norm == 0.0) fail(HS_ERR_VALUE, "x_true must be nonzero for relative errors");
    }
    convert_kernel<T, double><<<grid_for(m, 256, SMS * 16), 256, 0, s>>>(m, bd.as<double>(), bT.as<T>());
    CKL();

    B* L = Lb->template as<B>();
    B* D = square ? nullptr : Db->template as<B>();
    auto Lcol = [&](int j) { return L + (long long)j * ldn; };
    auto Dcol = [&](int j) { return D + (long long)j * ldm; };
    double* H = Hb.as<double>();
    double* Wm = Wb.as<double>();
    auto Hcol = [&](int j) { return H + (long long)j * (K + 1); };
    auto Wcol = [&](int j) { return Wm + (long long)j * (K + 2); };

    // ---- r0 = b (or b - A x0), hessenberg.py:163-168 / 281-288
    int matvec0 = 0;
    if (x0_h) {
      DBuf x0T(ldn * sizeof(T));
      convert_kernel<T, double><<<grid_for(n, 256, SMS * 16), 256, 0, s>>>(n, x0d.as<double>(), x0T.as<T>());
      CKL();
      op->apply(x0T.p, wdt, r0.p, wdt, false);
      sub_kernel<T><<<grid_for(m, 256, SMS * 16), 256, 0, s>>>(m, bT.as<T>(), r0.as<T>());
      CKL();
      CK(cudaStreamSynchronize(s));
      matvec0 = 1;
    } else {
      CK(cudaMemcpyAsync(r0.p, bT.p, m * sizeof(T), cudaMemcpyDeviceToDevice, s));
    }

    auto trivial = [&]() {
      res->termination = HS_TERM_TRIVIAL;
      res->n_records = 0;
      res->x.assign(n, 0.0);
      if (x0_h) std::copy(x0_h, x0_h + n, res->x.begin());
    };
    auto argmax_host = [&](const T* v, long long len, int side, double& val, long long& idx) {
      const int g = grid_for(len, 256, SMS * 4);
      argmax_kernel<T><<<g, 256, 0, s>>>(len, 0, v, candp.as<Cand>(), st, side);
      CKL();
      sample(v, len, 0, side, side, 0);
      CK(cudaMemcpyAsync(&hst, st, sizeof(LoopState), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      val = hst.piv_val[side];
      idx = hst.piv_idx[side];
    };
    auto set_pivot = [&](T* pvslot, double val) {
      T tv = (T)val;
      CK(cudaMemcpyAsync(pvslot, &tv, sizeof(T), cudaMemcpyHostToDevice, s));
    };
    auto set_pos_and_unit = [&](long long* pos, T* P, long long idx) {
      T one = T(1);
      CK(cudaMemcpyAsync(pos, &idx, sizeof(long long), cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(P, &one, sizeof(T), cudaMemcpyHostToDevice, s));
      CK(cudaStreamSynchronize(s));
    };
    const int NORM_G = SMS * env_int("HS_NORM_BLOCKS", 8);

    int tmat0 = 0, sk0 = 0;
    double beta, alpha = 0.0;
    long long idx;
    argmax_host(r0.as<T>(), m, 0, beta, idx);
    if (beta == 0.0) {
      trivial();
      return;
    }
    B* first_basis;  // d1 (rect) or l1 (square)
    swap_perm(0, 0);
    if (square) {
      set_pos_and_unit(tpos.as<long long>(), PL.as<T>(), idx);
      set_pivot(pv.as<T>(), beta);
      normalize_kernel<T, B><<<grid_for(ldn, 256, NORM_G), 256, 0, s>>>(n, ldn, r0.as<T>(), pv.as<T>(), Lcol(0), st, 0, 0);
      CKL();
      first_basis = Lcol(0);
    } else {
      set_pos_and_unit(tpos.as<long long>(), PD.as<T>(), idx);
      set_pivot(pv.as<T>(), beta);
      normalize_kernel<T, B><<<grid_for(ldm, 256, NORM_G), 256, 0, s>>>(m, ldm, r0.as<T>(), pv.as<T>(), Dcol(0), st, 0, 0);
      CKL();
      first_basis = Dcol(0);
      // v0 = A^T r0
      op->apply(r0.p, wdt, q.p, wdt, true);
      tmat0++;
      long long idx2;
      argmax_host(q.as<T>(), n, 1, alpha, idx2);
      if (alpha == 0.0) {
        trivial();
        return;
      }
      swap_perm(1, 0);
      set_pos_and_unit(gpos.as<long long>(), PL.as<T>(), idx2);
      set_pivot(pv.as<T>() + 1, alpha);
      normalize_kernel<T, B><<<grid_for(ldn, 256, NORM_G), 256, 0, s>>>(n, ldn, q.as<T>(), pv.as<T>() + 1, Lcol(0), st, 1, 0);
      CKL();
      // r = A^T d1, W(1,1) = r[g0]
      op->apply(Dcol(0), bdt, q.p, wdt, true);
      tmat0++;
      T w00;
      CK(cudaMemcpyAsync(&w00, q.as<T>() + idx2, sizeof(T), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      double w00d = (double)w00;
      CK(cudaMemcpyAsync(Wcol(0), &w00d, sizeof(double), cudaMemcpyHostToDevice, s));
    }
    // sketch setup (solvers.py:454-463)
    DBuf skinit;
    if (skd) {
      skinit.alloc((size_t)std::max<long long>({1LL, S2->scratch_elems(1, S2->m, G2), lamon && S1 ? S1->scratch_elems(1, S1->m, G1) : 0LL}) *
                       sizeof(double),
                   false);
      S2->apply(r0.p, wdt, sr0.as<double>(), skinit.as<double>(), G2);
      sk0++;
      if (sb) {
        S2->apply(first_basis, bdt, Gb.as<double>(), skinit.as<double>(), G2);
        sk0++;
      }
      if (lamon) {
        // printed variant: the unreduced r = A^T d1 still in q (solvers.py:460-461)
        if (printed) S1->apply(q.p, wdt, Fb.as<double>(), skinit.as<double>(), G1);
        else S1->apply(Lcol(0), bdt, Fb.as<double>(), skinit.as<double>(), G1);
        sk0++;
      }
    } else {
      // rhs = beta e1 (solvers.py:502-504); N = I_k (506-508) as columns e_j
      CK(cudaMemcpyAsync(sr0.p, &beta, sizeof(double), cudaMemcpyHostToDevice, s));
      if (lamon) {
        std::vector<double> eye((size_t)ell * (K + 1), 0.0);
        for (int j = 0; j <= K && j < ell; ++j) eye[(size_t)j * ell + j] = 1.0;
        CK(cudaMemcpyAsync(Fb.p, eye.data(), eye.size() * sizeof(double), cudaMemcpyHostToDevice, s));
      }
      CK(cudaStreamSynchronize(s));
    }
    (void)first_basis;

    if (diag) {
      if (square) {
        qL.append(Lcol(0));
      } else {
        qB.append(Dcol(0));
        qL.append(Lcol(0));
      }
      if (diag_eps) qW.append(r0.as<T>());
    }
    if (timing) CK(cudaStreamSynchronize(s));
    const auto t_init = now();
    // ---- the loop (solvers.py:468-538)
    std::vector<cudaEvent_t> ev = ctx->take_events(K + 2, true);  // ev[K + 1]: end of loop
    std::vector<cudaEvent_t> sev = ctx->take_events(4, false);
    std::vector<cudaEvent_t> flag_ev, ev_skb, ev_qrb;
    struct Lease {  // events go back to the context pool on every exit path
      hs_ctx* c;
      std::vector<std::vector<cudaEvent_t>*> timed, sync;
      ~Lease() {
        for (auto* v : timed) c->give_events(*v, true);
        for (auto* v : sync) c->give_events(*v, false);
      }
    } lease{ctx, {&ev}, {&sev, &flag_ev, &ev_skb, &ev_qrb}};
    QrArgs qa;
    qa.ell = (int)ell; qa.Ls = Ls; qa.ldq = ldq; qa.kmax = K; qa.lam = cfg.lam;
    qa.Z = Zb.as<double>(); qa.F = lamon ? Fb.as<double>() : nullptr; qa.sr0 = sr0.as<double>();
    qa.Q = Qb.as<double>(); qa.Rinv = Rinv.as<double>(); qa.Rdiag = Rdiag.as<double>(); qa.y = yb.as<double>();
    qa.Yhist = Yh.as<double>(); qa.part = part.as<double>(); qa.sres = sresb.as<double>(); qa.proj = projb.as<double>();
    qa.rankfb = rfb.as<int>(); qa.st = st;
    DBuf Nnull((size_t)K * K * sizeof(double)), ndrop(sizeof(int));
    qa.Nnull = Nnull.as<double>(); qa.ndrop = ndrop.as<int>();
    DBuf qdone(sizeof(unsigned int));  // zeroed; the reducing block resets it
    qa.qdone = qdone.as<unsigned int>();
    const size_t qr_smem = qr_smem_bytes(Ls, NB, K);
    CK(prepare_qr_step(qr_smem));
    const bool rec_x = cfg.record_x && xt_h;
    const size_t elim_smem_base = 16;
    auto elim = [&](T* vec, long long len, long long ldv, const B* basis, int k, int side, int iter, int kx,
                    const double* yx, double* relerr_slot, T* vout) {
      // short vectors (configs 1-3): one element per thread, so the pass spreads
      // over every SM and each thread keeps 16 basis loads in flight
      const bool v1 = (len + VEC - 1) / VEC < 2LL * ctx->num_sms * 256 && !env_flag("HS_ELIM_VEC");
      const long long nvec = v1 ? len : (len + VEC - 1) / VEC;
      const int g = grid_for(nvec, 256, CAND_CAP);
      const size_t smem = ((k * sizeof(T) + 15) / 16) * 16 + (size_t)kx * sizeof(double) + elim_smem_base;
      const double bytes = (double)std::max(k, kx) * len * sizeof(B) + 2.0 * len * sizeof(T) +
                           (kx ? (double)len * 8 : 0.0);
      Prof p(ctx, side == 0 && !square ? "elim_D" : "elim_L", bytes);
      auto kern = v1 ? (kx ? elim_pass_kernel<T, B, 1, true> : elim_pass_kernel<T, B, 1, false>)
                     : (kx ? elim_pass_kernel<T, B, VEC, true> : elim_pass_kernel<T, B, VEC, false>);
      CK(ensure_smem((const void*)kern, smem));
      (void)ldv;
      kern<<<g, 256, smem, s>>>(
          len, 0, basis, square || side == 1 ? ldn : ldm, nullptr, k, cvec.as<T>(), vec, kx, yx, nullptr,
          x0_h ? x0d.as<double>() : nullptr, kx ? xtd.as<double>() : nullptr, xpart.as<double>(), relerr_slot,
          candp.as<Cand>(), st, side, iter, 1, vout);
      CKL();
    };

    // Short vectors (configs 1-3): the whole basis step -- forward substitution,
    // elimination pass, commit, normalisation -- as ONE cooperative kernel
    // (hs_loop.cuh: basis_step_kernel) instead of four latency-bound launches.
    // Not with sampled pivoting (its pick runs between the pass and the commit).
    // Measured (tools/run_configs.py, loop it/s without per-kernel events): config 1 (n = 1024) 17.2k ->
    // 20.3k, config 2 (n = 65,536) 14.6k -> 15.1k; config 3 (n = 262,144: 2.92k -> 2.84k) keeps the
    // separate kernels -- there the pass wants more blocks than a cooperative grid holds, and the step
    // is bound by the dependent chains inside the phases, not by the launches.
    const long long step_fuse_max = env_int("HS_STEP_FUSE_MAX", 65536);
    auto step_fusable = [&](long long len) {
      return ps <= 0 && !env_flag("HS_NO_STEP_FUSE") && len <= step_fuse_max && !env_flag("HS_ELIM_VEC");
    };
    auto step_fused = [&](const T* uin, T* P, double* hcol, long long len, long long ldv, const B* basis, T* uout,
                          int k, int side, int iter, int kx, const double* yx, double* relerr_slot, long long dim,
                          long long* pos, T* pivval, bool do_norm, B* dst, SinoBlk blk, B* yb) {
      StepArgs<T, B> a;
      a.u = uin; a.P = P; a.Pw = P; a.ldp = ldp; a.k = k; a.c = cvec.as<T>(); a.hcol = hcol;
      a.n = len; a.ld = ldv; a.basis = basis; a.uo = uout; a.kx = kx; a.yx = yx;
      a.x0 = x0_h ? x0d.as<double>() : nullptr; a.xt = kx ? xtd.as<double>() : nullptr;
      a.xpart = xpart.as<double>(); a.relerr_out = relerr_slot; a.cand = candp.as<Cand>();
      a.dim = dim; a.pos = pos; a.pivval = pivval;
      a.do_norm = do_norm ? 1 : 0; a.n_pad = ldv; a.dst = dst; a.blk = blk; a.yb = yb;
      a.st = st; a.side = side; a.iter = iter;
      const size_t smem = basis_step_smem(k, kx, sizeof(T));
      auto kern = kx ? basis_step_kernel<T, B, true> : basis_step_kernel<T, B, false>;
      // (the kernel's ~1 KB of static shared memory counts against the 48 KB default too)
      CK(ensure_smem((const void*)kern, smem > 40 * 1024 ? std::max<size_t>(smem, 64 * 1024) : smem));
      // two blocks per SM at most: the projected solve's cooperative grid runs beside this one
      int per_sm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)kern, 256, smem));
      if (per_sm < 1) fail(HS_ERR_RUNTIME, "basis step kernel does not fit an SM (%zu B of shared memory)", smem);
      const int g = (int)std::min<long long>((len + 255) / 256, std::min(std::min(2, per_sm) * SMS, CAND_CAP));
      const double bytes = (double)std::max(k, kx) * len * sizeof(B) + 4.0 * len * sizeof(T) +
                           (kx ? (double)len * 8 : 0.0);
      Prof p(ctx, side == 0 && !square ? "step_D" : "step_L", bytes);
      void* args[] = {(void*)&a};
      CK(cudaLaunchCooperativeKernel((void*)kern, dim3(g), dim3(256), args, smem, s));
      ++g_launches;
    };

    // Two streams (column sketching): the sketch of u = A l_k and the projected
    // solve of iteration k run on ctx->aux while the main stream does the
    // basis work; u is not overwritten by the elimination (it writes u2), the
    // next A-apply waits for the sketch to have read u, and the fused iterate
    // of iteration k+1 waits for y^{(k)}.
    const bool ovl = skd && !sb && !diag && !env_flag("HS_NO_OVERLAP");  // knob: serialise for A/B
    cudaStream_t s2 = ovl ? ctx->aux : s;
    DBuf u2(ovl ? ldm * sizeof(T) : 0);
    T* uel = ovl ? u2.as<T>() : u.as<T>();  // elimination output on the side that is sketched
    cudaEvent_t ev_u = sev[0], ev_sk = sev[1], ev_qr = sev[2], ev_l = sev[3];
    if (ovl) {  // the aux stream starts after the init work (sr0, F col 0) on the main stream
      CK(cudaEventRecord(ev_l, s));
      CK(cudaStreamWaitEvent(s2, ev_l, 0));
    }
    // Batched Gaussian sketches.  Nothing in the basis recurrence reads a
    // sketch (pivots, H, W and the bases depend on A and b only), so the
    // columns z_k = S2 A l_k (and f_k = S1 l_{k+1}) can be formed SB at a
    // time: the operator writes u_k into a ring of 2*SB slots, and every SB
    // iterations the aux stream sketches the SB slots with ONE pass of the
    // counter-based generator (hs_sketch.cuh) and runs the SB projected solves.
    // Each z_k is bit-identical to the per-iteration sketch; only the fused
    // iterate lags (x_j rides on the basis pass of iteration j + 2*SB - 1,
    // the last ones are formed after the loop).
    const bool sk_main = skd && S2 && S2->kind == HS_SKETCH_SPARSE_SIGN && !env_flag("HS_SK_AUX");
    const bool gauss_any = ovl && ((S2 && S2->kind == HS_SKETCH_GAUSSIAN) ||
                                   (lamon && S1 && S1->kind == HS_SKETCH_GAUSSIAN));
    int SB = 1;
    if (gauss_any) {
      const char* e = getenv("HS_SKETCH_BATCH");
      SB = e && *e ? atoi(e) : GAUSS_NV_MAX;
      SB = std::max(1, std::min(SB, std::max(1, K)));
    }
    const int xlag = SB > 1 ? 2 * SB - 1 : 1;
    DBuf uring(SB > 1 ? (size_t)2 * SB * ldm * sizeof(T) : 0);
    const int nbatch = (K + SB - 1) / SB;
    // sketch partial scratch: one per stream the sketches run on (hs_sketch::apply_many)
    auto skelems = [&](int nv) {
      long long e = 0;
      if (skd) e = std::max(e, S2->scratch_elems(nv, S2->m, G2));
      if (skd && lamon && S1) e = std::max(e, S1->scratch_elems(nv, S1->m, G1));
      return (size_t)std::max<long long>(e, 1);
    };
    DBuf skaux(skelems(SB) * sizeof(double), false), skmain(skelems(1) * sizeof(double), false);
    double* const skA = skaux.as<double>();
    double* const skM = skmain.as<double>();
    ev_skb = ctx->take_events(SB > 1 ? nbatch : 0, false);
    ev_qrb = ctx->take_events(SB > 1 ? nbatch : 0, false);
    // (measured: the batched sketches on a third stream, so the generator pass of batch b + 1
    // overlaps the SB projected solves of batch b, leave config 2 at 15.1k it/s and config 5 at
    // 292 -- the basis stream, not the aux stream, is the longer one there)
    struct AuxJoin {  // an exception leaves no aux-stream kernel reading buffers about to be released
      hs_ctx* c;
      int n0 = std::uncaught_exceptions();
      ~AuxJoin() {
        if (std::uncaught_exceptions() > n0) cudaStreamSynchronize(c->aux);
      }
    } aux_join{ctx};
    std::vector<int> fused_at(K + 2, 0);  // iteration whose basis pass formed x_j
    int flushed = 0;                       // iterations whose sketches / projected solves are queued
    // sketch + projected solves of iterations flushed+1 .. kend_b on the aux stream
    auto flush_batch = [&](int kend_b) {
      if (kend_b <= flushed) return;
      const int kb0 = flushed + 1, nb = kend_b - flushed;
      const int bidx = (kb0 - 1) / SB;
      CK(cudaEventRecord(ev_l, s));
      CK(cudaStreamWaitEvent(s2, ev_l, 0));
      const long long slot0 = (long long)((kb0 - 1) % (2 * SB));
      S2->apply_many(uring.as<T>() + slot0 * ldm, wdt, ldm, nb, Zb.as<double>() + (long long)(kb0 - 1) * ell, ell, skA, G2, s2);
      CK(cudaEventRecord(ev_skb[bidx], s2));
      if (lamon && !printed) S1->apply_many(Lcol(kb0), bdt, ldn, nb, Fb.as<double>() + (long long)kb0 * ell, ell, skA, G1, s2);
      for (int kk = kb0; kk <= kend_b; ++kk) {
        qa.zcol = Zb.as<double>() + (long long)(kk - 1) * ell;
        qa.fcol = lamon ? Fb.as<double>() + (long long)(kk - 1) * ell : nullptr;
        Prof p(ctx, "qr_step", 0.0, s2);
        int k1 = kk, it = kk;
        CK(launch_qr_step(qa, k1, it, NB, qr_smem, s2));
        ++g_launches;
      }
      CK(cudaEventRecord(ev_qrb[bidx], s2));
      flushed = kend_b;
    };

    // host-side breakdown polling (pinned flag copied at the end of each iteration)
    // pinned scratch: breakdown flags, then the staging area for x
    const size_t flag_bytes = round_up(sizeof(int) * (K + 1), 4096);
    char* pin = reinterpret_cast<char*>(ctx->pinned_buf(flag_bytes + (size_t)n * sizeof(double)));
    int* hflag = reinterpret_cast<int*>(pin);
    double* xstage = reinterpret_cast<double*>(pin + flag_bytes);
    for (int i = 0; i <= K; ++i) hflag[i] = 0;
    flag_ev = ctx->take_events(K + 1, false);

    // rectangular tomography: the L-side normalisation also writes the
    // transposed image copy the next A apply gathers from (not with the
    // diagnostics, whose extra forward applies reuse the operator's copy)
    B* const lT = (!square && !diag && !env_flag("HS_NO_XT_FUSE"))
                      ? reinterpret_cast<B*>(op->transposed_input(sizeof(B)))
                      : nullptr;
    bool lT_ready = false;
    CK(cudaEventRecord(ev[0], s));
    int k_last = 0;
    int bd_at = 0;
    for (int k = 1; k <= K; ++k) {
      // stop launching once a breakdown two iterations back is visible
      if (k >= 3) {
        CK(cudaEventSynchronize(flag_ev[k - 2]));
        if (hflag[k - 2] != 0) break;
      }
      k_last = k;
      const int kx = (rec_x && k - xlag >= 1) ? k - xlag : 0;
      const double* yprev = kx ? Yh.as<double>() + (long long)(kx - 1) * K : nullptr;
      double* relslot = kx ? rel2.as<double>() + (kx - 1) : nullptr;
      if (kx) fused_at[kx] = k;
      T* const ucur = SB > 1 ? uring.as<T>() + (long long)((k - 1) % (2 * SB)) * ldm : u.as<T>();
      if (SB > 1) {
        // this half of the ring was last read by the sketch of batch bidx - 2
        const int bidx = (k - 1) / SB;
        if ((k - 1) % SB == 0 && bidx >= 2) CK(cudaStreamWaitEvent(s, ev_skb[bidx - 2], 0));
      } else if (ovl && k > 1) {
        // u is free once the previous iteration's sketch has read it
        CK(cudaStreamWaitEvent(s, ev_sk, 0));
      }
      op->apply(Lcol(k - 1), bdt, ucur, wdt, false, lT_ready);
      if (diag_eps) qW.append(u.as<T>());  // the unreduced A l_k (solvers.py:480-481)
      // rectangular: the sketch of u (and the projected solve after it) starts
      // once the data side is normalised, so the aux stream overlaps the long
      // A^T apply instead of competing with the D elimination pass for the SMs
      const bool defer_sk = ovl && SB == 1 && !square && !env_flag("HS_SK_EARLY");
      auto sketch_u = [&] {
        if (sk_main) {
          // a sparse-sign sketch is a ~10 us HBM stream: run it in order on
          // the main stream rather than beside the A^T apply, whose L1-bound
          // gathers lose when the sketch's 96 KB shared-memory blocks share
          // their SMs
          S2->apply(u.p, wdt, Zb.as<double>() + (long long)(k - 1) * ell, skM, G2);
          CK(cudaEventRecord(ev_u, s));
          CK(cudaStreamWaitEvent(s2, ev_u, 0));
          CK(cudaEventRecord(ev_sk, s));
          return;
        }
        CK(cudaEventRecord(ev_u, s));
        CK(cudaStreamWaitEvent(s2, ev_u, 0));
        S2->apply(u.p, wdt, Zb.as<double>() + (long long)(k - 1) * ell, skA, G2, s2);
        CK(cudaEventRecord(ev_sk, s2));
      };
      if (SB > 1) {
        // sketched in batches (flush_batch)
      } else if (defer_sk) {
        // launched after normalize (below)
      } else if (ovl) {
        CK(cudaEventRecord(ev_u, s));
        CK(cudaStreamWaitEvent(s2, ev_u, 0));
        S2->apply(u.p, wdt, Zb.as<double>() + (long long)(k - 1) * ell, skA, G2, s2);
        CK(cudaEventRecord(ev_sk, s2));
      } else if (skd && !sb && !square) {  // serialised (diagnostics): sketch before the in-place elimination
        S2->apply(u.p, wdt, Zb.as<double>() + (long long)(k - 1) * ell, skM, G2);
      }
      // the fused iterate x_{k-1} needs y^{(k-1)} from the aux stream
      auto wait_y = [&] {
        if (ovl && kx) CK(cudaStreamWaitEvent(s, SB > 1 ? ev_qrb[(kx - 1) / SB] : ev_qr, 0));
      };
      if (!square) {
        // d_{k+1}, and the same values in the blocked sinogram layout A^T gathers from
        B* ybk = reinterpret_cast<B*>(op->blocked_input(sizeof(B)));
        if (env_flag("HS_NO_YB_FUSE")) ybk = nullptr;
        if (step_fusable(m)) {
          step_fused(ucur, PD.as<T>(), Hcol(k - 1), m, ldm, D, uel, k, 0, k, 0, nullptr, nullptr, m,
                     tpos.as<long long>(), pv.as<T>(), true, Dcol(k), op->sblk, ybk);
          if (!skd)
            CK(cudaMemcpyAsync(Zb.as<double>() + (long long)(k - 1) * ell, Hcol(k - 1),
                               (size_t)(k + 1) * sizeof(double), cudaMemcpyDeviceToDevice, s));
        } else {
        fsub(ucur, tpos.as<long long>(), PD.as<T>(), ldp, k, k, 0, cvec.as<T>(), Hcol(k - 1));
        elim(ucur, m, ldm, D, k, 0, k, 0, nullptr, nullptr, uel);
        sample(uel, m, k, 2 * k, 0, k);
        pivot_commit_kernel<T, B><<<1, 256, 0, s>>>(k, m, Hcol(k - 1), tpos.as<long long>(), PD.as<T>(), ldp, D, ldm,
                                                    0, m, st, 0, k, pv.as<T>());
        CKL();
        swap_perm(0, k);
        if (!skd)
          CK(cudaMemcpyAsync(Zb.as<double>() + (long long)(k - 1) * ell, Hcol(k - 1), (size_t)(k + 1) * sizeof(double),
                             cudaMemcpyDeviceToDevice, s));
        normalize_kernel<T, B><<<grid_for(ldm, 256, NORM_G), 256, 0, s>>>(m, ldm, uel, pv.as<T>(), Dcol(k), st, 0, k,
                                                                          op->sblk, ybk);
        CKL();
        }
        if (defer_sk) sketch_u();
        if (sb) S2->apply(Dcol(k), bdt, Gb.as<double>() + (long long)k * ell, skM, G2);
        op->apply(Dcol(k), bdt, q.p, wdt, true, ybk != nullptr);
        // printed variant: F column k = S1 q before the elimination (solvers.py:488-490)
        if (printed) S1->apply(q.p, wdt, Fb.as<double>() + (long long)k * ell, skM, G1);
        const bool fuse_l = step_fusable(n);
        if (fuse_l) {
          wait_y();
          step_fused(q.as<T>(), PL.as<T>(), Wcol(k), n, ldn, L, q.as<T>(), k, 1, k, kx, yprev, relslot, n,
                     gpos.as<long long>(), pv.as<T>() + 1, lT == nullptr, Lcol(k), SinoBlk{0, 0, 0, 0}, nullptr);
        } else {
        fsub(q.as<T>(), gpos.as<long long>(), PL.as<T>(), ldp, k, k, 1, cvec.as<T>(), Wcol(k));
        wait_y();
        elim(q.as<T>(), n, ldn, L, k, 1, k, kx, yprev, relslot, q.as<T>());
        sample(q.as<T>(), n, k, 2 * k + 1, 1, k);
        pivot_commit_kernel<T, B><<<1, 256, 0, s>>>(k, n, Wcol(k), gpos.as<long long>(), PL.as<T>(), ldp, L, ldn, 0,
                                                    n, st, 1, k, pv.as<T>() + 1);
        CKL();
        swap_perm(1, k);
        }
        if (fuse_l && !lT) {
          // normalised inside the step kernel
        } else if (lT) {
          const dim3 tg((op->img_grid + 31) / 32, (op->img_grid + 31) / 32);
          normalize_transpose_kernel<T, B><<<tg, 256, 0, s>>>(op->img_grid, ldn, q.as<T>(), pv.as<T>() + 1, Lcol(k),
                                                              lT, st, k);
        } else {
          normalize_kernel<T, B><<<grid_for(ldn, 256, NORM_G), 256, 0, s>>>(n, ldn, q.as<T>(), pv.as<T>() + 1, Lcol(k),
                                                                            st, 1, k);
        }
        CKL();
        lT_ready = lT != nullptr;
      } else {
        if (skd && !ovl && !sb) S2->apply(u.p, wdt, Zb.as<double>() + (long long)(k - 1) * ell, skM, G2);
        if (step_fusable(n)) {
          wait_y();
          step_fused(ucur, PL.as<T>(), Hcol(k - 1), n, ldn, L, uel, k, 0, k, kx, yprev, relslot, n,
                     tpos.as<long long>(), pv.as<T>(), true, Lcol(k), SinoBlk{0, 0, 0, 0}, nullptr);
          if (!skd)
            CK(cudaMemcpyAsync(Zb.as<double>() + (long long)(k - 1) * ell, Hcol(k - 1),
                               (size_t)(k + 1) * sizeof(double), cudaMemcpyDeviceToDevice, s));
        } else {
        fsub(ucur, tpos.as<long long>(), PL.as<T>(), ldp, k, k, 0, cvec.as<T>(), Hcol(k - 1));
        wait_y();
        elim(ucur, n, ldn, L, k, 0, k, kx, yprev, relslot, uel);
        sample(uel, n, k, k, 0, k);
        pivot_commit_kernel<T, B><<<1, 256, 0, s>>>(k, n, Hcol(k - 1), tpos.as<long long>(), PL.as<T>(), ldp, L, ldn,
                                                    0, n, st, 0, k, pv.as<T>());
        CKL();
        swap_perm(0, k);
        if (!skd)
          CK(cudaMemcpyAsync(Zb.as<double>() + (long long)(k - 1) * ell, Hcol(k - 1), (size_t)(k + 1) * sizeof(double),
                             cudaMemcpyDeviceToDevice, s));
        normalize_kernel<T, B><<<grid_for(ldn, 256, NORM_G), 256, 0, s>>>(n, ldn, uel, pv.as<T>(), Lcol(k), st, 0, k);
        CKL();
        }
        if (sb) S2->apply(Lcol(k), bdt, Gb.as<double>() + (long long)k * ell, skM, G2);
      }
      if (sb) {
        // M column k-1 = G[:, :k+1] @ H[:k+1, k-1]  (zero columns/entries past a breakdown)
        gemv_small_kernel<<<grid_for(ell, 128, 1 << 30), 128, 0, s>>>((int)ell, k + 1, Gb.as<double>(), Hcol(k - 1),
                                                                       Zb.as<double>() + (long long)(k - 1) * ell);
        CKL();
      }
      qa.zcol = Zb.as<double>() + (long long)(k - 1) * ell;
      qa.fcol = lamon ? Fb.as<double>() + (long long)(k - 1) * ell : nullptr;
      if (SB == 1) {
        Prof p(ctx, "qr_step", 0.0, s2);
        int kk = k, it = k;
        CK(launch_qr_step(qa, kk, it, NB, qr_smem, s2));
        ++g_launches;
      }
      if (ovl && SB == 1) CK(cudaEventRecord(ev_qr, s2));
      if (diag) {  // compute_diagnostics: x_k and |b - A x_k| (raw forward, uncounted; solvers.py:523-525)
        if (ovl) CK(cudaStreamWaitEvent(s, ev_qr, 0));
        xpass_kernel<B><<<grid_for(n, 256, SMS * 8), 256, (size_t)k * sizeof(double), s>>>(
            n, L, ldn, k, Yh.as<double>() + (long long)(k - 1) * K, x0_h ? x0d.as<double>() : nullptr, nullptr,
            xk.as<double>(), xpart.as<double>(), nullptr, st);
        CKL();
        convert_kernel<T, double><<<grid_for(n, 256, SMS * 8), 256, 0, s>>>(n, xk.as<double>(), xkT.as<T>());
        CKL();
        op->apply(xkT.p, wdt, axk.p, wdt, false);
        resid_part_kernel<T><<<SMS * 2, 256, 0, s>>>(m, bd.as<double>(), axk.as<T>(), rpart.as<double>());
        CKL();
        mdot_finish_kernel<<<1, 32, 0, s>>>(SMS * 2, 1, rpart.as<double>(), resn2.as<double>() + (k - 1), 0);
        CKL();
        // which bases grew this iteration (hessenberg.py:219-224, 356-389)
        CK(cudaMemcpyAsync(&hst, st, sizeof(LoopState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const bool bd_now = hst.bd_iter == k;
        if (square) {
          if (!bd_now) qL.append(Lcol(k));
        } else {
          if (!(bd_now && hst.bd_side == 0)) qB.append(Dcol(k));
          if (!bd_now) qL.append(Lcol(k));
        }
        DiagQR& qb = square ? qL : qB;
        double* kb = kbuf.as<double>();
        qb.singular_values(qb.cnt, svA.as<double>(), djac);
        kappa_kernel<<<1, 1, 0, s>>>(qb.cnt, svA.as<double>(), 0, nullptr, 0, kb + (k - 1));
        CKL();
        if (lamon) {  // kappa_dbar = cond of [basis, L_k] (union of singular values)
          qL.singular_values(k, svB.as<double>(), djac);
          kappa_kernel<<<1, 1, 0, s>>>(qb.cnt, svA.as<double>(), k, svB.as<double>(), 0, kb + (K + 1) + (k - 1));
          CKL();
        }
        if (diag_eps) {  // eps of S2 on span[r0, A l_1..A l_k]: S Q = [S r0, Z] R_W^{-1}
          CK(cudaMemcpyAsync(Xw.p, sr0.p, ell * sizeof(double), cudaMemcpyDeviceToDevice, s));
          CK(cudaMemcpyAsync(Xw.as<double>() + ell, Zb.p, (size_t)ell * k * sizeof(double), cudaMemcpyDeviceToDevice, s));
          trsm_right_kernel<<<(int)((ell + 127) / 128), 128, 0, s>>>((int)ell, k + 1, Xw.as<double>(), (int)ell,
                                                                     qW.R.as<double>(), qW.cap, Mw.as<double>());
          CKL();
          jacobi_sv_kernel<<<1, 1024, 0, s>>>((int)ell, k + 1, Mw.as<double>(), (int)ell, svB.as<double>(), 40);
          CKL();
          kappa_kernel<<<1, 1, 0, s>>>(k + 1, svB.as<double>(), 0, nullptr, 1, kb + 2 * (K + 1) + (k - 1));
          CKL();
        }
      }
      if (SB > 1) {
        if (k % SB == 0) flush_batch(k);
      } else if (lamon && !printed) {
        // F column k = S1 l_{k+1} (used by the projected solve of iteration k+1)
        if (ovl) {
          CK(cudaEventRecord(ev_l, s));
          CK(cudaStreamWaitEvent(s2, ev_l, 0));
        }
        if (skd) S1->apply(Lcol(k), bdt, Fb.as<double>() + (long long)k * ell, skA, G1, s2);
      }
      CK(cudaEventRecord(ev[k], s));
      CK(cudaMemcpyAsync(hflag + k, &st->bd_iter, sizeof(int), cudaMemcpyDeviceToHost, s));
      CK(cudaEventRecord(flag_ev[k], s));
    }
    if (SB > 1) flush_batch(k_last);
    // join the aux stream (last sketch / projected solve) before timing and readback
    cudaEvent_t ev_end = ev[K + 1];
    if (ovl) {
      CK(cudaEventRecord(ev_sk, s2));
      CK(cudaStreamWaitEvent(s, ev_sk, 0));
    }
    CK(cudaEventRecord(ev_end, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaMemcpy(&hst, st, sizeof(LoopState), cudaMemcpyDeviceToHost));
    bd_at = hst.bd_iter;
    const int kend = bd_at ? bd_at : k_last;
    res->k = kend;
    res->n_records = kend;
    res->termination = bd_at ? HS_TERM_BREAKDOWN : HS_TERM_MAXITER;
    res->bd_side = bd_at ? hst.bd_side : -1;

    const auto t_loop = now();
    // ---- final iterate(s): x_kend, and x_{kend-1} when the fused pass skipped it
    auto xpass = [&](int kx, double* xout, double* relslot) {
      const int g = grid_for(n, 256, SMS * 8);
      Prof p(ctx, "xpass", (double)kx * n * sizeof(B) + 16.0 * n);
      xpass_kernel<B><<<g, 256, (size_t)kx * sizeof(double), s>>>(n, L, ldn, kx, Yh.as<double>() + (long long)(kx - 1) * K,
                                                                  x0_h ? x0d.as<double>() : nullptr,
                                                                  xt_h ? xtd.as<double>() : nullptr, xout,
                                                                  xpart.as<double>(), relslot, st);
      CKL();
    };
    xpass(kend, xd.as<double>(), xt_h ? rel2.as<double>() + (kend - 1) : nullptr);
    const bool data_bd = bd_at && !square && hst.bd_side == 0;
    // iterates whose fused pass did not run (lagged past the end, or on the
    // solution-side pass of an iteration whose data side broke down)
    if (rec_x)
      for (int j = 1; j < kend; ++j) {
        const int f = fused_at[j];
        if (!(f && (f < kend || (f == kend && !data_bd)))) xpass(j, nullptr, rel2.as<double>() + (j - 1));
      }
    CK(cudaStreamSynchronize(s));
    const auto t_xpass = now();
    float lms = 0;
    CK(cudaEventElapsedTime(&lms, ev[0], kend == k_last ? ev_end : ev[kend]));
    res->loop_ms = lms;
    res->wall_ms.resize(kend);
    for (int k = 1; k <= kend; ++k) {
      float w = 0;
      CK(cudaEventElapsedTime(&w, ev[k - 1], (k == kend && kend == k_last) ? ev_end : ev[k]));
      res->wall_ms[k - 1] = w;
    }
    const auto t_events = now();

    // ---- copy back
    CK(cudaStreamSynchronize(s));
    (void)xstage;
    res->xdev = xdp;
    const auto t_xcopy = now();
    res->sres.resize(kend);
    res->proj.resize(kend);
    res->rankfb.resize(kend);
    CK(cudaMemcpy(res->sres.data(), sresb.p, kend * sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(res->proj.data(), projb.p, kend * sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(res->rankfb.data(), rfb.p, kend * sizeof(int), cudaMemcpyDeviceToHost));
    res->relerr.assign(kend, NAN);
    if (diag) {
      std::vector<double> r2(kend);
      CK(cudaMemcpy(r2.data(), resn2.p, kend * sizeof(double), cudaMemcpyDeviceToHost));
      res->resnorm.resize(kend);
      for (int k = 0; k < kend; ++k) res->resnorm[k] = std::sqrt(r2[k]);
      std::vector<double> kb((size_t)3 * (K + 1));
      CK(cudaMemcpy(kb.data(), kbuf.p, kb.size() * sizeof(double), cudaMemcpyDeviceToHost));
      res->kappa_basis.assign(kb.begin(), kb.begin() + kend);
      res->kappa_dbar.assign(kend, NAN);
      res->eps_embed.assign(kend, NAN);
      if (lamon) std::copy(kb.begin() + (K + 1), kb.begin() + (K + 1) + kend, res->kappa_dbar.begin());
      if (diag_eps) std::copy(kb.begin() + 2 * (K + 1), kb.begin() + 2 * (K + 1) + kend, res->eps_embed.begin());
    }
    if (xt_h) {
      std::vector<double> r2(K + 1);
      CK(cudaMemcpy(r2.data(), rel2.p, (K + 1) * sizeof(double), cudaMemcpyDeviceToHost));
      for (int k = 1; k <= kend; ++k)
        if (rec_x || k == kend) res->relerr[k - 1] = std::sqrt(r2[k - 1]) / xt_norm;
    }
    // H (k+1) x k, W
    res->H.assign((size_t)(kend + 1) * kend, 0.0);
    {
      std::vector<double> hb((size_t)(K + 1) * K);
      CK(cudaMemcpy(hb.data(), Hb.p, hb.size() * sizeof(double), cudaMemcpyDeviceToHost));
      for (int j = 0; j < kend; ++j)
        for (int i = 0; i <= j + 1 && i <= kend; ++i) res->H[(size_t)j * (kend + 1) + i] = hb[(size_t)j * (K + 1) + i];
    }
    // basis sizes (hessenberg.py: D grows unless the data side broke down, L unless any side did)
    const int grew_last_D = (bd_at && (square || hst.bd_side == 0)) ? 0 : 1;
    const int grew_last_L = bd_at ? 0 : 1;
    if (square) {
      res->n_basis_sol = 1 + (kend - 1) + grew_last_L;
      res->n_basis_data = res->n_basis_sol;
    } else {
      res->n_basis_data = 1 + (kend - 1) + grew_last_D;
      res->n_basis_sol = 1 + (kend - 1) + grew_last_L;
      const int nw = res->n_basis_data;  // W has one column per D column
      res->W.assign((size_t)nw * nw, 0.0);
      std::vector<double> wb((size_t)(K + 2) * (K + 1));
      CK(cudaMemcpy(wb.data(), Wb.p, wb.size() * sizeof(double), cudaMemcpyDeviceToHost));
      for (int j = 0; j < nw; ++j)
        for (int i = 0; i <= j; ++i) res->W[(size_t)j * nw + i] = wb[(size_t)j * (K + 2) + i];
    }
    {
      std::vector<long long> tp(ldp), gp(ldp);
      CK(cudaMemcpy(tp.data(), tpos.p, ldp * sizeof(long long), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(gp.data(), gpos.p, ldp * sizeof(long long), cudaMemcpyDeviceToHost));
      if (square) {
        res->t.assign(tp.begin(), tp.begin() + res->n_basis_sol);
      } else {
        res->t.assign(tp.begin(), tp.begin() + res->n_basis_data);
        res->g.assign(gp.begin(), gp.begin() + res->n_basis_sol);
      }
    }
    res->Z.resize((size_t)ell * kend);
    CK(cudaMemcpy(res->Z.data(), Zb.p, res->Z.size() * sizeof(double), cudaMemcpyDeviceToHost));
    res->sr0.resize(ell);
    CK(cudaMemcpy(res->sr0.data(), sr0.p, ell * sizeof(double), cudaMemcpyDeviceToHost));
    res->y.resize(kend);
    CK(cudaMemcpy(res->y.data(), Yh.as<double>() + (long long)(kend - 1) * K, kend * sizeof(double),
                  cudaMemcpyDeviceToHost));
    // counters (linops.py:53-68 semantics, per record)
    res->matvecs.resize(kend);
    res->tmatvecs.resize(kend);
    res->dots.assign(kend, 0);
    res->sketches.resize(kend);
    long long tm = tmat0, sk = sk0;
    for (int k = 1; k <= kend; ++k) {
      const bool last = (k == kend);
      const bool grewD = !(last && bd_at && (square || hst.bd_side == 0));
      const bool grewL = !(last && bd_at);
      if (!square && grewD) tm += 1;              // q = A^T d_{k+1}
      if (skd) {
        sk += sb ? (grewD ? 1 : 0) : 1;           // G or Z column
        if (lamon && (printed ? grewD : grewL)) sk += 1;  // F column
      }
      res->matvecs[k - 1] = matvec0 + k;
      res->tmatvecs[k - 1] = tm;
      res->sketches[k - 1] = sk;
    }
    res->Lb = Lb;
    res->Db = Db;
    res->ldn = ldn;
    res->ldm = ldm;
    if (timing) {
      const auto t_end = now();
      fprintf(stderr, "[hs_solve] alloc %.1f ms, init %.1f ms, loop %.1f ms (device %.1f), finalize %.1f ms "
              "(xpass %.1f, events %.1f, x copy %.1f, rest %.1f)\n",
              ms(t_start, t_alloc), ms(t_alloc, t_init), ms(t_init, t_loop), res->loop_ms, ms(t_loop, t_end),
              ms(t_loop, t_xpass), ms(t_xpass, t_events), ms(t_events, t_xcopy), ms(t_xcopy, t_end));
    }
  }

};

}  // namespace

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

const char* hs_last_error(void) { return g_err.c_str(); }
unsigned long long hs_launch_count(void) { return g_launches; }
unsigned long long hs_guard_violations(void) { return g_guard_violations; }
const char* hs_version(void) { return "hessketch_b200 0.1.0 (sm_100a)"; }

int hs_ctx_create(int device, hs_ctx** out) {
  return guarded([&] {
    if (!out) fail(HS_ERR_VALUE, "null output handle");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) fail(HS_ERR_VALUE, "device %d out of range (have %d)", device, ndev);
    CK(cudaSetDevice(device));
    auto* c = new hs_ctx();
    c->device = device;
    // the main stream carries the basis recurrence (the critical path); the aux
    // stream (sketches, projected solves) gets the lower priority, so its blocks
    // only take SM slots the main stream's pending kernels do not claim
    int prio_lo = 0, prio_hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    if (env_flag("HS_FLAT_PRIO")) prio_lo = prio_hi = 0;
    c->main = std::make_shared<StreamRef>();
    c->main->device = device;
    CK(cudaStreamCreateWithPriority(&c->main->s, cudaStreamNonBlocking, prio_hi));
    c->stream = c->main->s;
    CK(cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, prio_lo));
    {
      // keep freed blocks in the device pool (no release back to the driver)
      cudaMemPool_t pool;
      CK(cudaDeviceGetDefaultMemPool(&pool, device));
      unsigned long long thr = ~0ULL;
      CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    }
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    *out = c;
  });
}

int hs_ctx_destroy(hs_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaStreamSynchronize(ctx->stream);
    for (auto& p : ctx->pending) {
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
    for (auto e : ctx->free_events) cudaEventDestroy(e);
    for (auto e : ctx->pool_timed) cudaEventDestroy(e);
    for (auto e : ctx->pool_sync) cudaEventDestroy(e);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    cudaStreamSynchronize(ctx->aux);
    cudaStreamDestroy(ctx->aux);
    // the main stream lives on while operators / sketches / results of this
    // context still hold buffers allocated on it (StreamRef)
    ctx->main.reset();
    delete ctx;
  });
}

int hs_ctx_synchronize(hs_ctx* ctx) { return guarded([&] { CK(cudaStreamSynchronize(ctx->stream)); }); }

}  // extern "C"

#include "hs_krylov.inc"
#include "hs_dist.inc"
#include "hs_stepper.inc"

#include "hs_abi.inc"
