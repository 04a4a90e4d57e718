// C ABI + native controllers for the B200 sparse FFT (see include/sfft2d_b200.h).
//
// Controllers (host C++, stream-ordered, one host sync per data-dependent
// decision):
//   run_sfft  — Algorithm 1, engine.py:256-284
//   run_ats   — Algorithm 2, tuner.py:142-282 (tuning loop, confirmation
//               passes, vote budget, fallback, estimation)
// Kernels live in the .cuh files next to this one.
#include "../../include/sfft2d_b200.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <tuple>
#include <string_view>
#include <unordered_map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"
#include "estimate.cuh"
#include "fft.cuh"
#include "fft_launch.cuh"
#include "fold.cuh"
#include "generate.cuh"
#include "host.cuh"
#include "npyrng.h"
#include "select.cuh"
#include "vote.cuh"
#include "passconv.cuh"

using namespace sfft;

// numpy's bounded-integer routine (numpy/random/lib/libnpyrandom.a, the code
// behind Generator.integers): drawing through it on the caller's own bitgen_t
// reproduces draw_permutation's stream consumption exactly (hashing.py:72-80).
extern "C" void random_bounded_uint64_fill(void* bitgen_state, uint64_t off, uint64_t rng,
                                           intptr_t cnt, bool use_masked, uint64_t* out);

namespace {

template <typename T> constexpr int prec_of();
template <> constexpr int prec_of<float>() { return SFFT2D_FP32; }
template <> constexpr int prec_of<double>() { return SFFT2D_FP64; }

struct DevTables {
  int n = 0, lgn = 0;
  double dpass = 0, dstop = 0;
  void* space[2] = {nullptr, nullptr};
  void* freq[2] = {nullptr, nullptr};
  void* tw[2] = {nullptr, nullptr};
  std::vector<int> support;  // samples per axis with nonzero window weight, per log2(B)
  std::vector<std::vector<int>> nz;   // those samples' indices, per log2(B)
  // per log2(B): R when the window is untruncated (support N) and its DC-
  // normalised response F vanishes (|F| <= 1e-14) beyond |d| = R <= 4, else 0
  // (k_estimate_conv)
  std::vector<int> conv_r;
};

}  // namespace

struct sfft2d_ctx {
  int device = 0;
  std::string err;
  std::vector<DevTables> tables;
  // named workspace buffers (names are string literals: views stay valid)
  // (three sets: a tuner pass's private buffers live in set slot % 3, so the
  // post-fold work of pass t on the side stream never shares a buffer with
  // the folds of passes t + 1 and t + 2 on the main stream)
  std::unordered_map<std::string_view, std::pair<void*, size_t>> bufs[3];
  int ws_set = 0;
  // workspace source: the context's own memory pool (default; a private pool
  // so the process-wide default pool keeps its attributes), or a caller-owned
  // device arena (sfft2d_ctx_set_workspace) sub-allocated first-fit
  cudaMemPool_t pool = nullptr;
  char* arena = nullptr;
  size_t arena_bytes = 0;
  std::map<size_t, size_t> arena_free;   // offset -> size of free blocks
  size_t ws_in_use = 0, ws_peak = 0;
  unsigned* pinned = nullptr;  // small host scratch for counts
  Perm* perm_pinned = nullptr; // pinned ring staging permutation uploads
  int perm_pos = 0;             // next free ring entry
  cudaEvent_t ev_perm = nullptr;   // after the latest upload from the ring
  // last results
  long long res_count = 0;
  int res_prec = SFFT2D_FP64;
  bool has_res = false;
  long long votes_count = 0;
  bool has_votes = false;
  int launches = 0;
  double sync_us = 0;   // host time blocked in stream synchronisation (diagnostic)
  // zero-copy count publication (tuner passes) and the side stream for votes
  unsigned* mapped_h = nullptr;
  void* host_out_buf = nullptr;   // mapped pinned results (grow-only)
  size_t host_out_cap = 0;
  int64_t* out_ij_h = nullptr;
  void* out_v_h = nullptr;
  unsigned* mapped_d = nullptr;
  unsigned* done_d = nullptr;
  unsigned seq = 0;
  cudaStream_t vote_st = nullptr;
  cudaEvent_t ev_lmax = nullptr;
  cudaEvent_t ev_pass[4] = {nullptr, nullptr, nullptr, nullptr};   // per tuner pass: list complete
  cudaEvent_t ev_fold[4] = {nullptr, nullptr, nullptr, nullptr};   // per tuner pass: fold complete
  cudaEvent_t ev_fork_votes = nullptr;
  cudaEvent_t ev_vote[2] = {nullptr, nullptr};
  // optional per-launch profiling (CUDA events on the launching stream)
  bool profiling = false;
  bool prof_open = false;
  struct ProfRec {
    const char* name;
    double bytes;
    cudaEvent_t a, b;
  };
  std::vector<ProfRec> prof;
  cudaStream_t ws_st = nullptr;     // stream of the running call: workspace grows stream-ordered on it
  std::chrono::steady_clock::time_point t_entry, t_sync_end;   // host-latency tracing
  double first_launch_us = 0;
  cudaEvent_t ev_ws = nullptr;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
};

namespace sfft {

// Power-of-two capacities: buffers sized by data-dependent counts (candidates,
// maxima) settle after a few calls instead of reallocating -- a cudaFree /
// cudaFreeHost synchronises the whole device, stalling every other stream.
size_t pow2_cap(size_t bytes) {
  size_t cap = 4096;
  while (cap < bytes) cap <<= 1;
  return cap;
}

static void arena_release(sfft2d_ctx* c, void* p, size_t bytes) {
  size_t off = (size_t)((char*)p - c->arena);
  auto it = c->arena_free.emplace(off, bytes).first;
  auto nx = std::next(it);   // coalesce with the following free block
  if (nx != c->arena_free.end() && it->first + it->second == nx->first) {
    it->second += nx->second;
    c->arena_free.erase(nx);
  }
  if (it != c->arena_free.begin()) {   // and with the preceding one
    auto pv = std::prev(it);
    if (pv->first + pv->second == it->first) {
      pv->second += it->second;
      c->arena_free.erase(it);
    }
  }
}

static void* arena_take(sfft2d_ctx* c, size_t bytes) {
  for (auto it = c->arena_free.begin(); it != c->arena_free.end(); ++it) {
    if (it->second < bytes) continue;
    const size_t off = it->first, rest = it->second - bytes;
    c->arena_free.erase(it);
    if (rest) c->arena_free.emplace(off + bytes, rest);
    return c->arena + off;
  }
  return nullptr;
}

void* ws(sfft2d_ctx* c, const char* name, size_t bytes) {
  auto& e = c->bufs[c->ws_set][name];
  if (bytes == 0) bytes = 16;
  if (e.second < bytes) {
    // Stream-ordered growth: cudaMalloc / cudaFree would synchronise the
    // whole device and stall every other in-flight transform.  The side
    // (vote) stream may still read the old buffer, so its release is ordered
    // after that stream's pending work (and, in arena mode, reuse of the
    // released range happens only in work enqueued later on this stream).
    cudaStream_t s = c->ws_st;
    if (e.first) {
      ck(cudaEventRecord(c->ev_ws, c->vote_st), "cudaEventRecord");
      ck(cudaStreamWaitEvent(s, c->ev_ws, 0), "cudaStreamWaitEvent");
      if (c->arena) arena_release(c, e.first, e.second);
      else ck(cudaFreeAsync(e.first, s), "cudaFreeAsync");
      c->ws_in_use -= e.second;
    }
    e.first = nullptr;
    e.second = 0;
    const size_t cap = pow2_cap(bytes);
    if (getenv("SFFT2D_TRACE_ALLOC"))
      fprintf(stderr, "[sfft2d] ctx %p workspace '%s' -> %zu bytes\n", (void*)c, name, cap);
    if (c->arena) {
      e.first = arena_take(c, cap);
      if (!e.first)
        fail(SFFT2D_ERR_NOMEM, std::string("caller workspace exhausted: '") + name + "' needs " +
                                   std::to_string(cap) + " more bytes (" +
                                   std::to_string(c->ws_in_use) + " in use of " +
                                   std::to_string(c->arena_bytes) + ")");
    } else if (cudaMallocFromPoolAsync(&e.first, cap, c->pool, s) != cudaSuccess) {
      cudaGetLastError();
      e.first = nullptr;
      fail(SFFT2D_ERR_NOMEM, std::string("cannot allocate workspace '") + name + "' of " +
                                 std::to_string(cap) + " bytes");
    }
    e.second = cap;
    c->ws_in_use += cap;
    c->ws_peak = std::max(c->ws_peak, c->ws_in_use);
  }
  return e.first;
}

static cudaEvent_t next_event(sfft2d_ctx* c) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "cudaEventCreate");
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_used++];
}

// pre/post bracket every kernel launch: count it, check the launch, and when
// profiling record an event pair on the launching stream with the launch's
// algorithmic bytes (SURVEY.md §8(d) accounting).
void pre(sfft2d_ctx* c, cudaStream_t st) {
  if (!c->profiling) return;
  cudaEvent_t a = next_event(c);
  ck(cudaEventRecord(a, st), "cudaEventRecord");
  c->prof.push_back({nullptr, 0.0, a, nullptr});
  c->prof_open = true;
}

void post(sfft2d_ctx* c, const char* what, cudaStream_t st, double bytes) {
  if (++c->launches == 1)
    c->first_launch_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - c->t_entry).count();
  ck(cudaGetLastError(), what);
  if (!c->profiling || !c->prof_open) return;
  cudaEvent_t b = next_event(c);
  ck(cudaEventRecord(b, st), "cudaEventRecord");
  c->prof.back().name = what;
  c->prof.back().bytes = bytes;
  c->prof.back().b = b;
  c->prof_open = false;
}

void allow_smem_ptr(const void* kernel) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, bool> done;
  int dev = 0;
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_pair(dev, kernel);
  if (done.count(key)) return;
  ck(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDynSmem),
     "cudaFuncSetAttribute");
  done[key] = true;
}

int ctas_per_sm_ptr(const void* kernel, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int, size_t>, int> cache;
  int dev = 0;
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  const auto key = std::make_tuple(dev, kernel, threads, smem);
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int n = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem),
     "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  n = std::max(n, 1);
  cache[key] = n;
  return n;
}

}  // namespace sfft

namespace {

const DevTables& find_tables(sfft2d_ctx* c, int n, double dpass, double dstop) {
  for (auto& t : c->tables)
    if (t.n == n && t.dpass == dpass && t.dstop == dstop) return t;
  fail(SFFT2D_ERR_STATE, "no tables registered for n=" + std::to_string(n) +
                             " (call sfft2d_ctx_set_tables)");
}

const DevTables& find_twiddles(sfft2d_ctx* c, int n) {
  for (auto& t : c->tables)
    if (t.n == n) return t;
  fail(SFFT2D_ERR_STATE, "no twiddle table registered for n=" + std::to_string(n));
}

constexpr int kPermPinned = 4096;

// `count` pinned ring entries that are free to write now: uploads are
// stream-ordered, so the ring wraps only after the latest upload completed
// (one event wait every ~kPermPinned / count calls, instead of a stream
// synchronisation per upload)
Perm* perm_stage(sfft2d_ctx* c, int count) {
  if (count > kPermPinned) fail(SFFT2D_ERR_UNSUPPORTED, "too many permutations");
  if (c->perm_pos + count > kPermPinned) {
    ck(cudaEventSynchronize(c->ev_perm), "cudaEventSynchronize");
    c->perm_pos = 0;
  }
  Perm* p = c->perm_pinned + c->perm_pos;
  c->perm_pos += count;
  return p;
}

// draw_permutation (hashing.py:72-80) on a numpy bitgen_t: the reference's
// four Generator.integers calls in order, with numpy's bounded routine
Perm draw_perm_bitgen(void* bitgen, int n) {
  uint64_t v[4] = {0, 0, 0, 0};
  if (n > 1) {
    random_bounded_uint64_fill(bitgen, 0, (uint64_t)(n / 2 - 1), 1, false, &v[0]);
    random_bounded_uint64_fill(bitgen, 0, (uint64_t)(n / 2 - 1), 1, false, &v[1]);
  }
  random_bounded_uint64_fill(bitgen, 0, (uint64_t)(n - 1), 1, false, &v[2]);
  random_bounded_uint64_fill(bitgen, 0, (uint64_t)(n - 1), 1, false, &v[3]);
  const uint32_t mask = (uint32_t)n - 1u;
  Perm q;
  q.s1 = n > 1 ? (uint32_t)(2 * v[0] + 1) : 1u;
  q.s2 = n > 1 ? (uint32_t)(2 * v[1] + 1) : 1u;
  q.t1 = (uint32_t)v[2];
  q.t2 = (uint32_t)v[3];
  uint32_t a = q.s1, b = q.s2;   // inverses mod 2^k by Newton iteration
  for (int i = 0; i < 5; ++i) { a *= 2u - q.s1 * a; b *= 2u - q.s2 * b; }
  q.s1i = a & mask;
  q.s2i = b & mask;
  return q;
}

// Algorithm 1's stream derivation (engine.py:266-280): 2L child seeds
// rng.integers(2**63) from the caller's stream, each child
// np.random.default_rng(seed) (npyrng.h), one draw_permutation per child
void sfft_child_perms(void* bitgen, int n, int loops, sfft2d_perm* out) {
  std::vector<uint64_t> seeds(2 * loops);
  for (auto& sd : seeds) random_bounded_uint64_fill(bitgen, 0, (1ULL << 63) - 1, 1, false, &sd);
  for (int i = 0; i < 2 * loops; ++i) {
    npyrng::Pcg64 st;
    npyrng::default_rng(seeds[i], &st);
    npyrng::bitgen_t bg;
    npyrng::bind(&bg, &st);
    const Perm q = draw_perm_bitgen(&bg, n);
    out[i] = sfft2d_perm{q.s1, q.s2, q.t1, q.t2, q.s1i, q.s2i};
  }
}

Perm to_perm(const sfft2d_perm& p, int n) {
  const long long m = n;
  auto md = [m](long long v) { return (uint32_t)(((v % m) + m) % m); };
  Perm q;
  q.s1 = md(p.sigma1);
  q.s2 = md(p.sigma2);
  q.t1 = md(p.tau1);
  q.t2 = md(p.tau2);
  q.s1i = md(p.sigma1_inv);
  q.s2i = md(p.sigma2_inv);
  return q;
}

uint32_t inv_pow2(uint32_t s, uint32_t mask) {  // s odd: s^-1 mod 2^k by Newton iteration
  uint32_t x = s;
  for (int i = 0; i < 5; ++i) x *= 2u - s * x;
  return x & mask;
}

// Permutations for a transform: from a caller array, or drawn on demand from a
// numpy bitgen_t*.  Drawn permutations are staged in pinned memory and copied
// to the device array in stream order.
struct PermSource {
  const sfft2d_perm* arr = nullptr;
  int n_arr = 0;
  void* bitgen = nullptr;
  int n = 0;
  std::vector<Perm> hp;
  Perm* pinned = nullptr;
  Perm* dev = nullptr;
  int cap = 0;

  const Perm& get(int i, cudaStream_t st) {
    if (i >= cap) fail(SFFT2D_ERR_VALUE, "permutation list exhausted");
    while ((int)hp.size() <= i) {
      Perm q;
      const int k = (int)hp.size();
      if (bitgen) {
        q = draw_perm_bitgen(bitgen, n);
      } else {
        if (k >= n_arr) fail(SFFT2D_ERR_VALUE, "permutation list exhausted");
        q = to_perm(arr[k], n);
      }
      hp.push_back(q);
      pinned[k] = q;
    }
    return hp[i];
  }
  // device copies are only needed by the estimation loops: one copy for them
  void upload(int from, int count, cudaStream_t st, cudaEvent_t done) {
    ck(cudaMemcpyAsync(dev + from, pinned + from, (size_t)count * sizeof(Perm),
                       cudaMemcpyHostToDevice, st),
       "H2D perms");
    ck(cudaEventRecord(done, st), "cudaEventRecord");
  }
  int used() const { return (int)hp.size(); }
};

unsigned read_u32(sfft2d_ctx* c, const unsigned* dev, cudaStream_t st) {
  ck(cudaMemcpyAsync(c->pinned, dev, sizeof(unsigned), cudaMemcpyDeviceToHost, st), "D2H");
  const auto t0 = std::chrono::steady_clock::now();
  ck(cudaStreamSynchronize(st), "sync");
  c->t_sync_end = std::chrono::steady_clock::now();
  c->sync_us += std::chrono::duration<double, std::micro>(c->t_sync_end - t0).count();
  return c->pinned[0];
}

void raise_if_nonfinite(sfft2d_ctx* c) {   // after a synchronisation of the stream
  if (c->pinned[1]) fail(SFFT2D_ERR_VALUE, "matrix contains NaN or Inf");
}

// Mapped pinned host buffer for results (grow-only).
void* host_out(sfft2d_ctx* c, size_t bytes) {
  if (c->host_out_cap < bytes) {
    if (c->host_out_buf) {
      ck(cudaDeviceSynchronize(), "sync");
      cudaFreeHost(c->host_out_buf);
    }
    c->host_out_buf = nullptr;
    c->host_out_cap = 0;
    // pinned allocation synchronises the device: start at 32 MB (1M results)
    const size_t cap = pow2_cap(std::max<size_t>(bytes, 32u << 20));
    if (getenv("SFFT2D_TRACE_ALLOC"))
      fprintf(stderr, "[sfft2d] ctx %p host_out -> %zu bytes\n", (void*)c, cap);
    ck(cudaHostAlloc(&c->host_out_buf, cap, cudaHostAllocMapped), "cudaHostAlloc");
    c->host_out_cap = cap;
  }
  return c->host_out_buf;
}

// Prepare a count publication for a launch of `grid` CTAs.
// One 16-byte mapped slot per publication sequence number (a ring of
// kPubSlots): a pass enqueued speculatively behind the one being waited for
// publishes into its own slot instead of overwriting the word the host spins on.
constexpr unsigned kPubSlots = 256;

volatile unsigned* pub_slot_h(sfft2d_ctx* c, unsigned seq) { return c->mapped_h + 4 * (seq % kPubSlots); }

// Each publication has its own CTA ticket counter (one per seq slot, reset by
// the last CTA), so publishing kernels on different streams may overlap.
Publish make_publish(sfft2d_ctx* c, unsigned grid) {
  Publish p;
  p.seq = ++c->seq;
  p.done = c->done_d + (p.seq % kPubSlots);
  p.target = grid;
  p.slot = c->mapped_d + 4 * (p.seq % kPubSlots);
  return p;
}

// Spin on the mapped slot until the launch published `seq`; returns the count.
unsigned wait_published(sfft2d_ctx* c, unsigned seq, cudaStream_t st) {
  const auto t0 = std::chrono::steady_clock::now();
  volatile unsigned* h = pub_slot_h(c, seq);
  volatile unsigned long long* h64 = reinterpret_cast<volatile unsigned long long*>(h);
  for (unsigned long spin = 0;; ++spin) {
    const unsigned long long word = *h64;   // (count << 32) | seq, one device store
    if ((unsigned)word == seq) {
      std::atomic_thread_fence(std::memory_order_acquire);
      const unsigned v = (unsigned)(word >> 32);
      c->sync_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
      return v;
    }
#if defined(__x86_64__)
    __builtin_ia32_pause();   // spin politely (sibling hyperthread, power)
#endif
    // error / lost-publication check: a driver call (it takes the context lock
    // that every other in-flight transform's launches need), so only after
    // ~65K spins (tens of us) and then every ~65K spins
    if ((spin & 65535) == 65535) {
      const cudaError_t e = cudaStreamQuery(st);
      if (e != cudaErrorNotReady && e != cudaSuccess) ck(e, "tuner pass");
      if (e == cudaSuccess && h[0] != seq) fail(SFFT2D_ERR_CUDA, "count publication lost");
    }
  }
}

// ------------------------------------------------------------------ pieces
template <typename Tin>
__global__ void k_check_finite(const Tin* __restrict__ x, long n, unsigned* flag) {
  pdl_wait();
  bool bad = false;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    const Tin v = x[i];
    bad |= !isfinite(v.x) || !isfinite(v.y);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

__global__ void k_sel_init(SelState* st, int nseg, long long num, long long seglen) {
  pdl_wait();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nseg) {
    st[s].prefix = 0;
    st[s].mask = 0;
    st[s].need = num;
    st[s].take_all = num >= seglen ? 1 : 0;
  }
}

__global__ void k_iota_segments(int32_t* out, long seglen, int nseg) {
  pdl_wait();
  const long total = seglen * nseg;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x)
    out[e] = (int32_t)(e % seglen);
}

// One fold launch for g <= 8 loops; returns where the result lives:
// natural-order partials [Z][g][B][B] (Z > 1) or the permuted grids (Z == 1).
struct FoldOut {
  void* data;
  int Z;
};

PermPack identity_pack(int g) {
  PermPack pp;
  std::memset(&pp, 0, sizeof(pp));
  for (int i = 0; i < g; ++i) pp.p[i] = Perm{1, 1, 0, 0, 1, 1};
  return pp;
}

// ATSFFT estimation at B < N with an untruncated window from the dense
// spectrum (k_estimate_conv; SFFT2D_NO_CONV=1: folds + FFTs, for A/B runs)
bool conv_on() {
  static const bool on = getenv("SFFT2D_NO_CONV") == nullptr;
  return on;
}

// multi-loop folds for B < 512 go through k_fold_ml (SFFT2D_OLD_MLFOLD=1:
// k_fold, for A/B runs)
bool ml_fold_on() {
  static const bool on = getenv("SFFT2D_OLD_MLFOLD") == nullptr;
  return on;
}

template <typename T, typename Tin>
FoldOut fold_launch(sfft2d_ctx* c, const Tin* x, int lgN, int lgB, const DevTables& tb,
                    const Perm* hp, int g, void* y_direct, cudaStream_t st,
                    unsigned long long* zero_peak = nullptr, bool natural = false,
                    const Perm* spec_q = nullptr, void* spec_y = nullptr, int* spec_z = nullptr,
                    bool spec_same = false, unsigned* nonfinite = nullptr) {
  using C = cplx<T>;
  const int B = 1 << lgB;
  const size_t BB = (size_t)B * B;
  const T* space = (const T*)tb.space[prec_of<T>()] + ((size_t)lgB << lgN);
  PermPack pp;
  std::memset(&pp, 0, sizeof(pp));
  for (int i = 0; i < g; ++i) pp.p[i] = hp[i];
  const int cpt = (g == 1) ? 2 : 1;
  FoldGeom gm = fold_geometry(lgN, lgB, cpt);
  const int threads = gm.TW / cpt;
  const dim3 grid(gm.ktiles, B, gm.Z);
  const int nlt = (g == 1) ? 1 : kMaxFoldLoops;
  size_t dyn = (B < gm.TW) ? (size_t)nlt * gm.TW * sizeof(C) : 0;
  if (((size_t)sizeof(T) << lgN) <= 32 * 1024) {   // window table staged in smem
    gm.tab = (int)dyn;
    dyn += (size_t)sizeof(T) << lgN;
  }
  const double sup = (double)tb.support[lgB];
  // window weights are gathered from the window table inside the fold
  // kernels; `natural` places bucket (rho, kappa) at row rho, column kappa
  const int seg_cols0 = kRingSegBytes / (int)sizeof(Tin);
  if (spec_q && B < 512) {
    // TMA ring fold of pass t at B and of the next pass at 2B <= 512 (or, for
    // the first two tuner passes, at the same B), one read
    if (!(g == 1 && (spec_same || 2 * B <= 512) && gm.TW == 512 && (1 << lgN) >= seg_cols0 &&
          y_direct && spec_y && spec_z && (natural || spec_same)))
      fail(SFFT2D_ERR_STATE, "speculative ring fold outside its geometry");
    const T* space2 = (const T*)tb.space[prec_of<T>()] + ((size_t)(lgB + (spec_same ? 0 : 1)) << lgN);
    const int nslot = 3;
    FoldGeom gr = gm;
    const int aliases = (1 << lgN) >> lgB;
    const int Z = (int)std::max(1L, std::min<long>(aliases, 2L * kNumSMs / B));
    int rpc = (aliases + Z - 1) / Z;
    if (rpc > kFoldMaxRows) rpc = kFoldMaxRows;
    gr.rpc = rpc;
    gr.Z = (aliases + rpc - 1) / rpc;
    gr.ktiles = 1;
    C* dstr = (gr.Z == 1) ? (C*)y_direct : (C*)ws(c, "fold_part", (size_t)gr.Z * BB * sizeof(C));
    const size_t dynr = (size_t)nslot * kRingSegBytes + 3 * 512 * sizeof(C);
    pre(c, st);
    if (spec_same)
      kl(k_fold_ring2<Tin, T, true>, dim3(1, B, gr.Z), 256, dynr, st, x, space, space2, pp.p[0],
         *spec_q, gr, nslot, dstr, (C*)spec_y, zero_peak);
    else
      kl(k_fold_ring2<Tin, T>, dim3(1, B, gr.Z), 256, dynr, st, x, space, space2, pp.p[0], *spec_q,
         gr, nslot, dstr, (C*)spec_y, zero_peak);
    post(c, "k_fold_ring2", st, sup * sup * sizeof(Tin) + 5.0 * gr.Z * BB * sizeof(C));
    if (spec_same && gr.Z == 1) fail(SFFT2D_ERR_STATE, "same-B speculative fold needs partials");
    *spec_z = gr.Z;
    return FoldOut{dstr, gr.Z};
  }
  if (spec_q) {
    // pass t's fold at B plus the next pass's fold at 2B from one read
    if (spec_z) *spec_z = 1;
    if (!(g == 1 && B >= 512 && lgN - lgB <= 5 && lgN - lgB >= 2 && y_direct && spec_y && natural))
      fail(SFFT2D_ERR_STATE, "speculative fold outside its geometry");
    const T* space2 = (const T*)tb.space[prec_of<T>()] + ((size_t)(lgB + 1) << lgN);
    const double by = sup * sup * sizeof(Tin) + 5.0 * (double)BB * sizeof(C);
    pre(c, st);
    kl(k_fold_wide2<Tin, T>, dim3(B / 256, B), 128, 0, st, x, space, space2, pp.p[0], *spec_q, lgN,
       lgB, (C*)y_direct, (C*)spec_y, zero_peak);
    post(c, "k_fold_wide2", st, by);
    return FoldOut{y_direct, 1};
  }
  if (g == 1 && B >= 512 && lgN - lgB <= 5 && y_direct) {
    // wide single-loop fold, grid written directly
    const double by = sup * sup * sizeof(Tin) + (double)BB * sizeof(C);
    // RH=2 (two bucket rows per CTA) in fp32; fp64 accumulators would need 128
    // registers (2 CTAs/SM), so fp64 keeps RH=1
    const int rh = (B >= 1024 && sizeof(T) == 4) ? 2 : 1;
    const dim3 grid_w(B / 512, B / rh);
    pre(c, st);
    if (rh == 2)
      kl(k_fold_wide<Tin, T, 2>, grid_w, 256, 0, st, x, space, pp.p[0], lgN, lgB, natural, (C*)y_direct, zero_peak);
    else
      kl(k_fold_wide<Tin, T, 1>, grid_w, 256, 0, st, x, space, pp.p[0], lgN, lgB, natural, (C*)y_direct, zero_peak);
    post(c, "k_fold_wide", st, by);
    return FoldOut{y_direct, 1};
  }
  const int seg_cols = kRingSegBytes / (int)sizeof(Tin);
  if (g == 1 && B < 512 && gm.TW == 512 && (1 << lgN) >= seg_cols) {
    // TMA ring fold, 3 x 32 KB slots (2 CTAs per SM), row aliases chunked so
    // that ~2 CTAs per SM stream rows (measured best of slots 3-6 x 1-4 CTAs
    // per SM on c3)
    const int nslot = 3;
    // one wave: at most 2 CTAs per SM (floor, not ceil — a 384-CTA grid
    // over 296 slots left a 30% tail; c3 B = 128/256: 28.5 -> 26.2 us, and
    // B >= 256 writes its grid directly, no partials)
    const long target = 2L * kNumSMs;
    FoldGeom gr = gm;
    const int aliases = (1 << lgN) >> lgB;
    int Z = (int)std::max(1L, std::min<long>(aliases, target / B));
    int rpc = (aliases + Z - 1) / Z;
    if (rpc > kFoldMaxRows) rpc = kFoldMaxRows;
    gr.rpc = rpc;
    gr.Z = (aliases + rpc - 1) / rpc;
    gr.ktiles = 1;
    C* dstr = (gr.Z == 1) ? (C*)y_direct : (C*)ws(c, "fold_part", (size_t)gr.Z * BB * sizeof(C));
    const size_t dynr = (size_t)nslot * kRingSegBytes + 512 * sizeof(C);
    pre(c, st);
    kl(k_fold_ring<Tin, T>, dim3(1, B, gr.Z), 256, dynr, st, x, space, pp.p[0], gr, natural, nslot,
       dstr, zero_peak);
    post(c, "k_fold_ring", st, sup * sup * sizeof(Tin) + (double)gr.Z * BB * sizeof(C));
    return FoldOut{dstr, gr.Z};
  }
  if (g > 1 && B < 512 && ml_fold_on()) {
    // multi-loop fold: column tiles x bucket rows x row chunks, UNR 16-byte
    // loads in flight per thread
    const int N = 1 << lgN;
    const int twc = std::min(N, 512);
    const int tiles = N / twc;
    const int aliases = N >> lgB;
    int zr = (aliases + kFoldMaxRows - 1) / kFoldMaxRows;
    const long ctas = (long)tiles * B;
    if (ctas < 2L * kNumSMs) zr = std::max<long>(zr, std::min<long>(aliases, (2L * kNumSMs + ctas - 1) / ctas));
    const int rpc = (aliases + zr - 1) / zr;
    zr = (aliases + rpc - 1) / rpc;
    // the column tiles of one bucket row are summed inside a thread-block
    // cluster (DSMEM), so c3 (8 tiles) writes its grid directly
    const int csz = std::min(tiles, 8);
    const int zp = (tiles / csz) * zr;
    C* dstm = (zp == 1) ? (C*)y_direct : (C*)ws(c, "fold_part", (size_t)zp * g * BB * sizeof(C));
    const size_t dynm = (size_t)kMaxFoldLoops * (twc + B) * sizeof(C);
    pre(c, st);
    if constexpr (sizeof(T) == 4)
      klc(k_fold_ml<Tin, T, kMaxFoldLoops, 8>, dim3(tiles, B, zr), 256, dynm, st, csz, x, space, pp, g,
          lgN, lgB, twc, rpc, natural, zp, dstm, nonfinite);
    else
      klc(k_fold_ml<Tin, T, kMaxFoldLoops, 4>, dim3(tiles, B, zr), 256, dynm, st, csz, x, space, pp, g,
          lgN, lgB, twc, rpc, natural, zp, dstm, nonfinite);
    post(c, "k_fold_ml", st, sup * sup * sizeof(Tin) + (double)zp * g * BB * sizeof(C));
    return FoldOut{dstm, zp};
  }
  C* dst = (gm.Z == 1) ? (C*)y_direct : (C*)ws(c, "fold_part", (size_t)gm.Z * g * BB * sizeof(C));
  const double fold_bytes = sup * sup * sizeof(Tin) + (double)gm.Z * g * BB * sizeof(C);
  pre(c, st);
  if (g == 1 && ((1 << lgN) / std::max(B, gm.TW)) >= 4)
    kl(k_fold<Tin, T, 1, 2, 4>, grid, threads, dyn, st, x, space, pp, g, gm, natural, dst, zero_peak);
  else if (g == 1)
    kl(k_fold<Tin, T, 1, 2>, grid, threads, dyn, st, x, space, pp, g, gm, natural, dst, zero_peak);
  else
    kl(k_fold<Tin, T, kMaxFoldLoops, 1>, grid, threads, dyn, st, x, space, pp, g, gm, natural, dst, zero_peak);
  post(c, "k_fold", st, fold_bytes);
  return FoldOut{dst, gm.Z};
}

// Fold (+window, +permutation) and bucket FFT for `nloops` permutations.
// spec (optional): complex spectra [nloops][B][B]; mags/peaks (optional):
// |Z| [nloops][B][B] and per-loop peak keys (zeroed here).
template <typename T, typename Tin>
void fold_spectrum(sfft2d_ctx* c, const Tin* x, int lgN, int lgB, const DevTables& tb,
                   const Perm* hp, int nloops, cplx<T>* spec, T* mags, unsigned long long* peaks,
                   cudaStream_t st, bool natural = false, cplx<T>* prefolded = nullptr,
                   const Perm* spec_q = nullptr, cplx<T>* spec_y = nullptr, int pre_z = 1,
                   int* spec_z = nullptr, unsigned* nonfinite = nullptr,
                   cudaStream_t post_st = nullptr, cudaEvent_t handoff = nullptr) {
  using C = cplx<T>;
  const int B = 1 << lgB;
  const int P = prec_of<T>();
  const T* space = (const T*)tb.space[P] + ((size_t)lgB << lgN);
  const C* tw = (const C*)tb.tw[P];
  const size_t BB = (size_t)B * B;
  const bool small = BB * sizeof(C) <= (size_t)kSmall2DBytes;
  // one loop: the fold kernel zeroes the peak slot (no separate memset)
  if (peaks && nloops > 1)
    ck(cudaMemsetAsync(peaks, 0, (size_t)nloops * sizeof(unsigned long long), st), "memset");
  for (int g0 = 0; g0 < nloops; g0 += kMaxFoldLoops) {
    const int g = std::min(kMaxFoldLoops, nloops - g0);
    PermPack pp;
    std::memset(&pp, 0, sizeof(pp));
    for (int i = 0; i < g; ++i) pp.p[i] = hp[g0 + i];
    if (natural) pp = identity_pack(g);     // output placement only (see fold_launch)
    C* sp = spec ? spec + (size_t)g0 * BB : nullptr;
    T* mg = mags ? mags + (size_t)g0 * BB : nullptr;
    unsigned long long* pk = peaks ? peaks + g0 : nullptr;
    // bucket grid y (permuted fold) for this group
    C* y = (small && sp) ? sp : (C*)ws(c, "fold_y", (size_t)g * BB * sizeof(C));
    FoldOut fo{y, 1};
    if (prefolded) {   // the previous pass's speculative fold is this pass's grid (or partials)
      if (nloops != 1 || small) fail(SFFT2D_ERR_STATE, "prefolded grid for a multi-loop pass");
      if (pre_z == 1) y = prefolded;
      fo = FoldOut{prefolded, pre_z};
      if (pk) ck(cudaMemsetAsync(pk, 0, sizeof(unsigned long long), st), "memset");
    } else {
      fo = fold_launch<T, Tin>(c, x, lgN, lgB, tb, hp + g0, g, y, st, (nloops == 1) ? pk : nullptr,
                               natural, spec_q, spec_y, spec_z, false, nonfinite);
    }
    C* dst = (C*)fo.data;
    struct { int Z; } gm{fo.Z};
    // post-fold work (partial sums, FFT, |Z|) on post_st once the fold is done
    // (tuner passes: the next pass's fold proceeds on st meanwhile)
    const cudaStream_t main_st = st;
    const cudaStream_t ws_saved = c->ws_st;
    if (post_st) {
      ck(cudaEventRecord(handoff, main_st), "cudaEventRecord");
      ck(cudaStreamWaitEvent(post_st, handoff, 0), "cudaStreamWaitEvent");
      st = post_st;
      c->ws_st = post_st;
    }
    if (small) {
      if (gm.Z == 1) {
        fft2d_grids<T>(c, y, lgB, g, tw, lgN, sp, mg, pk, st);
      } else {
        pre(c, st);
        kl(k_fold_reduce_fft_small<T>, g, 1024, small_fft_smem<T>(lgB), st, dst, gm.Z, g, lgB, pp, tw,
           lgN, y);
        post(c, "k_fold_reduce_fft_small", st, (double)(gm.Z + 1) * g * BB * sizeof(C));
        if (sp && sp != y)
          ck(cudaMemcpyAsync(sp, y, (size_t)g * BB * sizeof(C), cudaMemcpyDeviceToDevice, st), "copy");
        if (mg) mags_of<T>(c, y, (long)BB, g, mg, pk, st);
      }
    } else {
      if (gm.Z != 1) {
        pre(c, st);
        kl(k_fold_reduce<T>, grid_for((long long)BB * g), 256, 0, st, dst, gm.Z, g, lgB, pp, y);
        post(c, "k_fold_reduce", st, (double)(gm.Z + 1) * g * BB * sizeof(C));
      }
      fft2d_grids<T>(c, y, lgB, g, tw, lgN, sp, mg, pk, st);
    }
    st = main_st;
    c->ws_st = ws_saved;
  }
}

// Compact the set bits of `nseg` segments (bits/counts from a *_bits kernel).
void compact(sfft2d_ctx* c, const uint32_t* bits, const unsigned* cnts, long seglen, int nseg,
             int32_t* out, long out_stride, unsigned* total_dev, cudaStream_t st) {
  const int nblk = blocks_for(seglen);
  unsigned* offs = (unsigned*)ws(c, "cmp_off", (size_t)nblk * nseg * sizeof(unsigned));
  pre(c, st);
  kl(k_scan_blocks, nseg, 1024, 0, st, cnts, nblk, offs, total_dev);
  post(c, "k_scan_blocks", st, 0);
  pre(c, st);
  kl(k_compact_bits, dim3(nblk, nseg), kCmpThreads, 0, st, bits, seglen, offs, out, out_stride);
  post(c, "k_compact_bits", st, 0);
}

// Local maxima of one B x B magnitude grid (seen through the permutation
// (s1, s2) when perm) -> row-major flat list; returns the count (host sync).
template <typename T>
unsigned local_maxima_dev(sfft2d_ctx* c, const T* mags, int lgB, const unsigned long long* peak,
                          double floor_rel, int32_t* out, cudaStream_t st, bool perm = false,
                          unsigned s1 = 1, unsigned s2 = 1) {
  const long BB = 1L << (2 * lgB);
  const int B = 1 << lgB;
  const int nblk = blocks_for(BB);
  uint32_t* bits = (uint32_t*)ws(c, "lm_bits", words_for(BB) * 4);
  unsigned* cnts = (unsigned*)ws(c, "lm_cnt", (size_t)nblk * 4);
  unsigned* tot = (unsigned*)ws(c, "lm_tot", 16);
  if (B >= 32) {
    // tile = rb output rows (+2 halo rows staged in smem); ~B/128 rows so that
    // small grids still spread over many SMs, capped by shared memory
    const int smem_rows = (int)((96 * 1024) / ((size_t)B * sizeof(T)));
    int rb = std::max(1, std::min(B / 128, smem_rows - 2));
    while (B % rb) --rb;
    const size_t sm = (size_t)(rb + 2) * B * sizeof(T);
    if (sm > kMaxDynSmem) fail(SFFT2D_ERR_UNSUPPORTED, "grid too large for the local-maximum tile");
    ck(cudaMemsetAsync(cnts, 0, (size_t)nblk * 4, st), "memset");
    pre(c, st);
    if (perm)
      kl(k_lmax_rows<T, true>, B / rb, 512, sm, st, mags, lgB, s1, s2, rb, peak, floor_rel, bits, cnts, (int32_t*)nullptr, (unsigned*)nullptr, Publish{nullptr, 0, nullptr, 0});
    else
      kl(k_lmax_rows<T, false>, B / rb, 512, sm, st, mags, lgB, 1, 1, rb, peak, floor_rel, bits, cnts, (int32_t*)nullptr, (unsigned*)nullptr, Publish{nullptr, 0, nullptr, 0});
    post(c, "k_lmax_rows", st, (double)BB * sizeof(T) + BB / 8.0);
  } else {
    if (perm) fail(SFFT2D_ERR_UNSUPPORTED, "permuted local maxima need B >= 32");
    pre(c, st);
    kl(k_lmax_bits<T>, dim3(nblk, 1), kCmpThreads, 0, st, mags, lgB, 0, peak, floor_rel, bits, cnts);
    post(c, "k_lmax_bits", st, (double)BB * sizeof(T) + BB / 8.0);
  }
  compact(c, bits, cnts, BB, 1, out, 0, tot, st);
  return read_u32(c, tot, st);
}

// Tuner local maxima: unordered list + device count (no host sync).
constexpr int kLmaxStreamMinB = 512;

template <typename T>
unsigned lmax_tuner(sfft2d_ctx* c, const T* mags, int lgB, const unsigned long long* peak,
                    double floor_rel, int32_t* list, unsigned* count, cudaStream_t st, bool perm,
                    unsigned s1, unsigned s2, unsigned s2inv, int32_t* cand = nullptr,
                    unsigned* cand_count = nullptr, bool* emitted = nullptr,
                    bool live_most = false, bool count64 = false) {
  if (emitted) *emitted = false;
  const int B = 1 << lgB;
  const double by = (double)B * B * sizeof(T);
  const size_t row = (size_t)B * sizeof(T);
  const size_t wb = 16 * kWarpBuf * sizeof(int32_t);
  if ((B >= kLmaxStreamMinB || (live_most && !cand && B >= 128)) && 4 * row + wb <= kMaxDynSmem) {
    // streaming bands: ~2 CTAs per SM, a ring of row buffers per CTA
    int nslot = (int)std::max<size_t>(4, std::min<size_t>(8, (96 * 1024 - wb) / row));
    if (nslot * row + wb > kMaxDynSmem) nslot = (int)((kMaxDynSmem - wb) / row);
    // ~2 CTAs per SM, or fewer when the kernel's registers / shared memory
    // allow fewer (fp64 register windows of k_lmax_win: one CTA per SM at 512
    // threads): the bands are sized for one wave of resident CTAs
    const bool win = live_most && !cand && B <= 4096;
    const int thr = 512;
    const size_t sm = nslot * row + wb;
    // count64: `count` is the low word of an 8-byte slot whose high word is
    // free for the CTA tickets (k_lmax_win2; SFFT2D_OLD_LMAX_WIN=1: k_lmax_win)
    static const bool win2_on = getenv("SFFT2D_OLD_LMAX_WIN") == nullptr;
    if (win && count64 && win2_on) {
      const int groups = B / 32;
      const int gpw = std::max(1, groups / 16);
      const int tw2 = 32 * (groups / gpw);
      auto go = [&](auto G) {
        constexpr int GPW = decltype(G)::value;
        const int resident = ctas_per_sm(k_lmax_win2<T, GPW>, tw2, sm);
        const int cps = std::max(1, std::min(2, resident));
        const int band = (B + cps * kNumSMs - 1) / (cps * kNumSMs);
        const int grid = (B + band - 1) / band;
        const Publish pub = make_publish(c, (unsigned)grid);
        pre(c, st);
        kl(k_lmax_win2<T, GPW>, grid, tw2, sm, st, mags, lgB, perm ? s1 : 1u, perm ? s2 : 1u, band,
           nslot, peak, floor_rel, list, reinterpret_cast<unsigned long long*>(count),
           (unsigned)grid, pub.slot, pub.seq);
        post(c, "k_lmax_win", st, by);
        return pub.seq;
      };
      switch (gpw) {
        case 1: return go(std::integral_constant<int, 1>{});
        case 2: return go(std::integral_constant<int, 2>{});
        case 4: return go(std::integral_constant<int, 4>{});
        default: return go(std::integral_constant<int, 8>{});
      }
    }
    const int tw_win = std::min(512, B / 4);
    const int resident = win ? ((B / 128 > 16) ? ctas_per_sm(k_lmax_win<T, 2>, tw_win, sm)
                                               : ctas_per_sm(k_lmax_win<T, 1>, tw_win, sm))
                             : ctas_per_sm(k_lmax_stream<T>, thr, sm);
    const int cps = std::max(1, std::min(2, resident));
    const int band = (B + cps * kNumSMs - 1) / (cps * kNumSMs);
    const int grid = (B + band - 1) / band;
    const Publish pub = make_publish(c, (unsigned)grid);
    pre(c, st);
    if (win) {
      // most bins pass the floor: register neighbourhood windows, one warp per
      // 128-column group (fewer threads for narrow grids)
      const int tw = tw_win;
      if (B / 128 > 16)
        kl(k_lmax_win<T, 2>, grid, tw, sm, st, mags, lgB, perm ? s1 : 1u, perm ? s2 : 1u,
           perm ? s2inv : 1u, band, nslot, peak, floor_rel, list, count, pub);
      else
        kl(k_lmax_win<T, 1>, grid, tw, sm, st, mags, lgB, perm ? s1 : 1u, perm ? s2 : 1u,
           perm ? s2inv : 1u, band, nslot, peak, floor_rel, list, count, pub);
      post(c, "k_lmax_win", st, by);
      return pub.seq;
    }
    kl(k_lmax_stream<T>, grid, thr, sm, st, mags, lgB, perm ? s1 : 1u, perm ? s2 : 1u,
       perm ? s2inv : 1u, band, nslot, peak, floor_rel, list, count, pub, cand, cand_count);
    if (emitted) *emitted = cand != nullptr;
    post(c, "k_lmax_stream", st, by);
    return pub.seq;
  }
  const int smem_rows = (int)((96 * 1024) / ((size_t)B * sizeof(T)));
  int rb = std::max(1, std::min(B / 128, smem_rows - 2));
  while (B % rb) --rb;
  const size_t sm = (size_t)(rb + 2) * B * sizeof(T) + (size_t)rb * B / 32 * sizeof(unsigned);
  static const bool tri_on = getenv("SFFT2D_NO_LMAX_TRI") == nullptr;
  if (perm && !live_most && B >= 8192 && 3 * row <= kMaxDynSmem && tri_on) {
    // a B = N view too wide for the ring but three rows fit shared memory:
    // each row tested against its two neighbour rows staged by TMA
    const unsigned grid = (unsigned)std::min(B, kNumSMs);
    const Publish pub = make_publish(c, grid);
    pre(c, st);
    kl(k_lmax_tri<T>, grid, 512, 3 * row, st, mags, lgB, s1, s2, inv_pow2(s1, (uint32_t)B - 1u), s2inv,
       peak, floor_rel, list, count, pub, cand, cand_count);
    if (emitted) *emitted = cand != nullptr;
    post(c, "k_lmax_tri", st, by);
    return pub.seq;
  }
  if (sm > kMaxDynSmem || (perm && !live_most && B >= 8192)) {
    // rows too long to stage (fp64 at B = 16384), or a B = N view too wide for
    // the ring (fp32 16384: one 3-row tile per SM): test straight from global
    // memory — below-floor bins (almost all at B = N) cost one coalesced read
    if (!perm) fail(SFFT2D_ERR_UNSUPPORTED, "grid too large for the local-maximum tile");
    const unsigned grid = kNumSMs * 8;
    const Publish pub = make_publish(c, grid);
    pre(c, st);
    kl(k_lmax_direct<T>, grid, 256, 0, st, mags, lgB, s1, s2, inv_pow2(s1, (uint32_t)B - 1u), s2inv, peak,
       floor_rel, list, count, pub, cand, cand_count);
    if (emitted) *emitted = cand != nullptr;
    post(c, "k_lmax_direct", st, by);
    return pub.seq;
  }
  const Publish pub = make_publish(c, (unsigned)(B / rb));
  pre(c, st);
  if (perm)
    kl(k_lmax_rows<T, true, true>, B / rb, 512, sm, st, mags, lgB, s1, s2, rb, peak, floor_rel,
                                                        nullptr, nullptr, list, count, pub);
  else
    kl(k_lmax_rows<T, false, true>, B / rb, 512, sm, st, mags, lgB, 1, 1, rb, peak, floor_rel,
                                                         nullptr, nullptr, list, count, pub);
  post(c, "k_lmax_rows", st, by);
  return pub.seq;
}

// Exact top-`num` selection bitmask per segment (ties -> lowest index).
template <typename T>
void topk_bits(sfft2d_ctx* c, const T* vals, long seglen, int nseg, long long num, uint32_t* bits,
               unsigned* cnts, cudaStream_t st) {
  SelState* sst = (SelState*)ws(c, "sel_state", (size_t)nseg * sizeof(SelState));
  unsigned* hist = (unsigned*)ws(c, "sel_hist", (size_t)nseg * 256 * sizeof(unsigned));
  ck(cudaMemsetAsync(hist, 0, (size_t)nseg * 256 * sizeof(unsigned), st), "memset");
  pre(c, st);
  kl(k_sel_init, (nseg + 127) / 128, 128, 0, st, sst, nseg, num, seglen);
  post(c, "k_sel_init", st, 0);
  const int nblk = blocks_for(seglen);
  if (num < seglen && seglen <= kSelSegMax) {
    pre(c, st);
    kl(k_radix_select_seg<T>, nseg, 1024, 0, st, vals, seglen, sst);
    post(c, "k_radix_select_seg", st, (double)seglen * nseg * sizeof(T) * 8);
  } else if (num < seglen) {
    unsigned hb = (unsigned)std::max<long long>(1, std::min<long long>(256, (seglen + 4095) / 4096));
    for (int shift = 56; shift >= 0; shift -= 8) {
      pre(c, st);
      kl(k_radix_hist<T>, dim3(hb, nseg), 256, 0, st, vals, seglen, sst, shift, hist);
      post(c, "k_radix_hist", st, 0);
      pre(c, st);
      kl(k_radix_pick, (nseg + 31) / 32, 32, 0, st, sst, hist, shift, nseg);
      post(c, "k_radix_pick", st, 0);
    }
  }
  unsigned* tie_blk = (unsigned*)ws(c, "sel_tie", (size_t)nblk * nseg * sizeof(unsigned));
  unsigned* tie_off = (unsigned*)ws(c, "sel_tieoff", (size_t)nblk * nseg * sizeof(unsigned));
  pre(c, st);
  kl(k_tie_counts<T>, dim3(nblk, nseg), kCmpThreads, 0, st, vals, seglen, sst, tie_blk);
  post(c, "k_tie_counts", st, 0);
  pre(c, st);
  kl(k_scan_blocks, nseg, 1024, 0, st, tie_blk, nblk, tie_off, nullptr);
  post(c, "k_scan_blocks", st, 0);
  pre(c, st);
  kl(k_select_bits<T>, dim3(nblk, nseg), kCmpThreads, 0, st, vals, seglen, sst, tie_off, bits, cnts);
  post(c, "k_select_bits", st, 0);
}

size_t hist_bytes(long nkeys, int mode) {
  if (mode == kVoteAdd32) return (size_t)nkeys * 4;
  return (size_t)((nkeys + 31) / 32) * 32;  // bytes, padded to whole 32-key groups
}

// keys (ascending) of histogram entries >= thr; returns the count (synchronises).
unsigned hist_compact(sfft2d_ctx* c, const uint32_t* hist, long nkeys, int mode, unsigned thr,
                      int32_t* keys, unsigned* total_dev, cudaStream_t st) {
  const int nblk = blocks_for(nkeys);
  uint32_t* bits = (uint32_t*)ws(c, "hc_bits", words_for(nkeys) * 4);
  unsigned* cnts = (unsigned*)ws(c, "hc_cnt", (size_t)nblk * 4);
  pre(c, st);
  kl(k_hist_bits, nblk, kCmpThreads, 0, st, hist, nkeys, mode, thr, bits, cnts);
  post(c, "k_hist_bits", st, (double)hist_bytes(nkeys, mode) + nkeys / 8.0);
  compact(c, bits, cnts, nkeys, 1, keys, 0, total_dev, st);
  return read_u32(c, total_dev, st);
}


template <typename T, typename Tin>
void dense_xhat(sfft2d_ctx* c, const Tin* x, int lgN, const DevTables& tb, cplx<T>* xhat, T* mags,
                unsigned long long* peak, cudaStream_t st, unsigned* nonfinite = nullptr) {
  // (peak: zeroed by the caller — run_ats's per-call scratch)
  dense_fft<T, Tin>(c, x, xhat, mags, peak, lgN, (const cplx<T>*)tb.tw[prec_of<T>()], st,
                    nonfinite);
}

// K7 tail shared by every estimation path (engine.py:228-253): from the
// per-coordinate medians `med`, |med| `mags`, `alive` flags and the peak key,
// the exact top-k cut (when more than k are alive), the prune against
// prune_rel * max |med|, the ordered compaction and the gather of the
// results into mapped host memory (one synchronisation).
template <typename T>
void finish_select(sfft2d_ctx* c, int lgN, const int32_t* keys, unsigned m, long long k,
                   double prune_rel, cplx<T>* med, T* mags, uint8_t* alive,
                   unsigned long long* peak, long long n_alive, cudaStream_t st,
                   sfft2d_result* res, const unsigned* alive_cnt_dev = nullptr) {
  using C = cplx<T>;
  res->n_candidates = m;
  if (n_alive == 0) {
    res->count = 0;
    res->ordered_by_magnitude = 0;
    c->res_count = 0;
    return;
  }
  // n_alive < 0: the alive count is still on the device (alive_cnt_dev) and
  // m > k.  The exact top-k selection runs regardless: dead coordinates carry
  // magnitude -1, so with alive <= k every alive coordinate is selected and
  // k_final_bits drops the dead ones — the kept set is the one the reference
  // keeps without a cut.  Only the order flag needs the count, and it is read
  // with the final synchronisation (one host round trip less).
  const bool deferred = n_alive < 0;
  // up to kTopkCtaMax candidates: the whole tail in one CTA (k_finish_cut_small),
  // count and alive count through the publication slot (SFFT2D_NO_FUSED_CUT=1:
  // the general kernels below)
  static const bool fused_cut_on = getenv("SFFT2D_NO_FUSED_CUT") == nullptr;
  if (fused_cut_on && m <= (unsigned)kTopkCtaMax) {
    const size_t cap = (size_t)m;
    char* outh = (char*)host_out(c, cap * (16 + sizeof(C)) + 64);
    int64_t* oij_h = (int64_t*)outh;
    C* ov_h = (C*)(outh + cap * 16);
    int64_t* oij_d;
    ck(cudaHostGetDevicePointer((void**)&oij_d, oij_h, 0), "cudaHostGetDevicePointer");
    C* ov_d = (C*)((char*)oij_d + cap * 16);
    const Publish pub = make_publish(c, 1);
    pre(c, st);
    kl(k_finish_cut_small<T>, 1, 1024, 0, st, (const C*)med, (const T*)mags, (const uint8_t*)alive,
       (int)m, k, prune_rel, (const unsigned long long*)peak, deferred ? -1LL : n_alive,
       alive_cnt_dev, keys, lgN, oij_d, ov_d, pub.slot, pub.seq);
    post(c, "k_finish_cut_small", st, 0);
    const unsigned count = wait_published(c, pub.seq, st);
    const long long na = deferred ? (long long)pub_slot_h(c, pub.seq)[2] : n_alive;
    c->out_ij_h = oij_h;
    c->out_v_h = ov_h;
    res->count = count;
    res->ordered_by_magnitude = na > k ? 1 : 0;
    c->res_count = count;
    return;
  }
  const bool cut = deferred ? (long long)m > k : n_alive > k;
  const int nblk = blocks_for(m);
  uint32_t* sel = nullptr;
  if (cut) {
    sel = (uint32_t*)ws(c, "fsel_bits", words_for(m) * 4);
    unsigned* scnt = (unsigned*)ws(c, "fsel_cnt", (size_t)nblk * 4);
    topk_bits<T>(c, mags, (long)m, 1, k, sel, scnt, st);
  }
  uint32_t* fb = (uint32_t*)ws(c, "fin_bits", words_for(m) * 4);
  unsigned* fc = (unsigned*)ws(c, "fin_cnt", (size_t)nblk * 4);
  pre(c, st);
  kl(k_final_bits<T>, nblk, kCmpThreads, 0, st, mags, alive, sel, (long)m, peak, prune_rel, fb, fc);
  post(c, "k_final_bits", st, 0);
  int32_t* pos = (int32_t*)ws(c, "fin_pos", (size_t)m * 4);
  unsigned* tot = (unsigned*)ws(c, "fin_tot", 16);
  compact(c, fb, fc, (long)m, 1, pos, 0, tot, st);
  // gather straight into mapped (zero-copy) host memory sized for the m
  // candidates, then ONE synchronisation yields the count and the results
  const size_t cap = (size_t)m;
  char* outh = (char*)host_out(c, cap * (16 + sizeof(C)) + 64);
  int64_t* oij_h = (int64_t*)outh;
  C* ov_h = (C*)(outh + cap * 16);
  int64_t* oij_d;
  ck(cudaHostGetDevicePointer((void**)&oij_d, oij_h, 0), "cudaHostGetDevicePointer");
  C* ov_d = (C*)((char*)oij_d + cap * 16);
  pre(c, st);
  kl(k_gather_out<T>, grid_for(m), 256, 0, st, pos, tot, keys, med, lgN, oij_d, ov_d);
  post(c, "k_gather_out", st, 0);
  bool ordered = cut;
  if (deferred) {
    ck(cudaMemcpyAsync(c->pinned + 2, alive_cnt_dev, sizeof(unsigned), cudaMemcpyDeviceToHost, st), "D2H");
  }
  const unsigned count = read_u32(c, tot, st);
  if (deferred) ordered = (long long)c->pinned[2] > k;
  c->out_ij_h = oij_h;
  c->out_v_h = ov_h;
  res->count = count;
  res->ordered_by_magnitude = ordered ? 1 : 0;
  c->res_count = count;
}


// Per-call scratch of small counters, zeroed by ONE memset at the start of a
// tuner run (each cudaMemsetAsync is a stream op of its own): the NaN flag,
// the estimation scalars, the candidate count, the dense peak, one peak per
// tuner slot and one count per tuner slot.
constexpr size_t kScrFinite = 0, kScrEst = 16, kScrCand = 48, kScrXpeak = 64, kScrPeaks = 80;
constexpr size_t kScrCounts = kScrPeaks + 8 * 2 * SFFT2D_MAX_HISTORY;
constexpr size_t kScrBytes = kScrCounts + 8 * 2 * SFFT2D_MAX_HISTORY;
unsigned char* call_scratch(sfft2d_ctx* c) {
  const int saved = c->ws_set;
  c->ws_set = 0;
  unsigned char* p = (unsigned char*)ws(c, "call_scratch", kScrBytes);
  c->ws_set = saved;
  return p;
}
unsigned long long* est_scalars(sfft2d_ctx* c) {
  return (unsigned long long*)(call_scratch(c) + kScrEst);
}
void zero_est_scalars(sfft2d_ctx* c, cudaStream_t st) {
  ck(cudaMemsetAsync(est_scalars(c), 0, 32, st), "memset");
}

// K6 + K7 + output compaction, shared by both algorithms.
template <typename T, typename Tin>
void estimate_and_select(sfft2d_ctx* c, const Tin* x, int lgN, int lgB, const DevTables& tb,
                         const Perm* hp, const Perm* dp, int L, const int32_t* keys, unsigned m,
                         const unsigned* m_dev, long long k, double gain_floor, double prune_rel,
                         bool dense, const cplx<T>* xhat, cudaStream_t st, sfft2d_result* res,
                         const cplx<T>* dscratch = nullptr, const cplx<T>* xconv = nullptr,
                         int conv_r = 0, cplx<T>* pre_grids = nullptr,
                         cudaEvent_t pre_ready = nullptr) {
  using C = cplx<T>;
  const int P = prec_of<T>();
  C* med = (C*)ws(c, "med", (size_t)m * sizeof(C));
  T* mags = (T*)ws(c, "emag", (size_t)m * sizeof(T));
  uint8_t* alive = (uint8_t*)ws(c, "alive", (size_t)m);
  // [peak key, alive count], zeroed by zero_est_scalars before the
  // candidate-count synchronisation (one memset off the critical path)
  unsigned long long* peak = est_scalars(c);
  unsigned* alive_cnt = (unsigned*)(peak + 1);
  long long n_alive;
  if (dense) {
    // gain = freq[0]^2 = 1 for the all-pass window (hashing.py:228-246)
    const bool usable_all = 1.0 >= gain_floor;
    pre(c, st);
    if (dscratch) {   // x_hat never stored: L2-point DFTs of the four-step scratch
      int lgL1 = 0, lgL2 = 0;
      dense_split(lgN, P, &lgL1, &lgL2);
      kl(k_estimate_dense_fs<T>, grid_for((long long)m * 32, 256), 256, 0, st, dscratch, lgN, lgL1,
         lgL2, (const C*)tb.tw[P], keys, m_dev, usable_all, med, mags, alive, peak);
      post(c, "k_estimate_dense_fs", st, (double)m * (1 << lgL2) * sizeof(C));
    } else {
      kl(k_estimate_dense<T>, grid_for(m), 256, 0, st, xhat, keys, m_dev, usable_all, med, mags,
         alive, peak);
      post(c, "k_estimate_dense", st, 0);
    }
    n_alive = usable_all ? (long long)m : 0;
  } else {
    if (L > kMaxLoops) fail(SFFT2D_ERR_UNSUPPORTED, "more than 64 estimation loops");
    const int B = 1 << lgB;
    const size_t BB = (size_t)B * B;
    C* vals = (C*)ws(c, "vals", (size_t)L * m * sizeof(C));
    uint8_t* usable = (uint8_t*)ws(c, "usable", (size_t)L * m);
    const T* freq = (const T*)tb.freq[P] + ((size_t)lgB << lgN);
    if (xconv) {
      // untruncated window: (2R+1)^2 gathers of the dense spectrum per
      // (candidate, loop) replace the L folds and B x B FFTs
      pre(c, st);
      auto go = [&](auto RC) {
        constexpr int R = decltype(RC)::value;
        kl(k_estimate_conv<T, R>, grid_for((long long)m * L), 256, 0, st, xconv, L, keys, m_dev, dp, lgN,
           lgB, freq, (const C*)tb.tw[P], gain_floor, vals, usable, (long)m);
      };
      switch (conv_r) {
        case 1: go(std::integral_constant<int, 1>{}); break;
        case 2: go(std::integral_constant<int, 2>{}); break;
        case 3: go(std::integral_constant<int, 3>{}); break;
        case 4: go(std::integral_constant<int, 4>{}); break;
        default: fail(SFFT2D_ERR_STATE, "convolution estimate outside its tap range");
      }
      const double taps = (double)(2 * conv_r + 1) * (2 * conv_r + 1);
      post(c, "k_estimate_conv", st, (double)m * L * taps * sizeof(C));
    } else {
      C* grids = pre_grids;
      if (pre_grids) {
        // folded + transformed on the side stream beside the location phase
        ck(cudaStreamWaitEvent(st, pre_ready, 0), "cudaStreamWaitEvent");
      } else {
        grids = (C*)ws(c, "est_grids", (size_t)L * BB * sizeof(C));
        // natural-order folds (coalesced writes; k_estimate reads the permuted view)
        fold_spectrum<T, Tin>(c, x, lgN, lgB, tb, hp, L, grids, (T*)nullptr, nullptr, st, true);
      }
      pre(c, st);
      kl(k_estimate<T>, grid_for((long long)m * L), 256, 0, st, grids, L, keys, m_dev, dp, lgN, lgB, freq, (const C*)tb.tw[P], gain_floor, vals, usable,
          (long)m, true);
      post(c, "k_estimate", st, 0);
    }
    pre(c, st);
    kl(k_median<T>, grid_for(m, 128), 128, 0, st, vals, usable, L, (long)m, m_dev, med, mags,
                                                   alive, alive_cnt, peak);
    post(c, "k_median", st, 0);
    // the alive count decides whether a top-k cut is needed (alive > k); with
    // m <= k candidates no cut is possible, so the count is not read (one
    // host synchronisation less; an all-dead result still compacts to 0)
    // (m > k: the count only decides the output order flag; finish_select
    // reads it with its final synchronisation; SFFT2D_SYNC_ALIVE=1: read it now)
    static const bool sync_alive = getenv("SFFT2D_SYNC_ALIVE") != nullptr;
    n_alive = ((long long)m <= k) ? (long long)m
                                  : (sync_alive ? (long long)read_u32(c, alive_cnt, st) : -1LL);
  }
  finish_select<T>(c, lgN, keys, m, k, prune_rel, med, mags, alive, peak, n_alive, st, res,
                   alive_cnt);
}

// ------------------------------------------------------------------ ATSFFT
int nearest_pow2(double v) {
  long long lo = 1;
  if (v >= 1) {
    int e = (int)std::floor(std::log2(v));
    if (e < 0) e = 0;
    lo = 1LL << e;
  }
  const long long hi = lo * 2;
  return (int)((v - lo) <= (hi - v) ? lo : hi);
}

int default_bins(int n, long long k) {
  if (k < 1) k = 1;
  const int b = nearest_pow2(std::sqrt((double)(std::min(n, 256)) * (double)k));
  return std::max(4, std::min(b, n));
}

int update_bins(int b, double r, const sfft2d_tuner_config& cf, int n) {
  double v;
  if (r < cf.delta1) v = b * cf.eps1;
  else if (r < cf.delta2) v = (double)b;
  else v = b * (1.0 + cf.eps2);
  return std::max(4, std::min(nearest_pow2(v), n));
}

template <typename T, typename Tin>
void run_ats(sfft2d_ctx* c, const Tin* x, int n, const sfft2d_tuner_config& cf, int est_loops,
             const sfft2d_perm* perms, int n_perms, void* bitgen, cudaStream_t st, bool do_estimate,
             sfft2d_result* res, sfft2d_tuner_state* S) {
  using C = cplx<T>;
  const int lgN = ilog2(n);
  const DevTables& tb = find_tables(c, n, cf.window_delta_pass, cf.window_delta_stop);
  const int max_iters = cf.max_tuning_iters >= 0 ? cf.max_tuning_iters : 2 * std::max(lgN, 1);
  if (max_iters + 2 > SFFT2D_MAX_HISTORY)
    fail(SFFT2D_ERR_UNSUPPORTED, "max_tuning_iters too large for the history buffer");
  if (!is_pow2(cf.b0)) fail(SFFT2D_ERR_CONFIG, "b0 is not a power of 2");
  const int L = std::max(est_loops, 1);
  PermSource ps;
  ps.arr = perms;
  ps.n_arr = n_perms;
  ps.bitgen = bitgen;
  ps.n = n;
  ps.cap = max_iters + 2 + L;
  ps.hp.reserve(ps.cap);
  ps.pinned = perm_stage(c, ps.cap);
  ps.dev = (Perm*)ws(c, "perms", (size_t)ps.cap * sizeof(Perm));
  Perm* dp = ps.dev;
  const long nkeys = (long)n * n;
  const long long budget = std::max((long long)n * n / 8, 1LL << 16);   // tuner.py:165
  const int mode = (4 * (max_iters + 2) <= 255) ? kVoteAdd8 : kVoteAdd32;
  uint32_t* hist = (uint32_t*)ws(c, "hist", hist_bytes(nkeys, mode));
  // deferred votes (k_vote_lazy): byte tallies, N >= 128; the histogram is
  // only materialised (zeroed here) when a pass must vote with atomics
  const bool lazy = mode == kVoteAdd8 && lgN >= 7;
  bool hist_zeroed = false;
  auto zero_hist = [&](cudaStream_t s2) {
    if (hist_zeroed) return;
    ck(cudaMemsetAsync(hist, 0, hist_bytes(nkeys, mode), s2), "memset hist");
    hist_zeroed = true;
  };
  if (!lazy) zero_hist(st);
  LazyPasses lp;
  std::memset(&lp, 0, sizeof(lp));
  lp.lgBmax = 2;
  long long arch_cap = kLazyScan;   // entries per archived pass, bounded by the vote budget
  for (int lb = 2; lb <= std::min(9, lgN); ++lb) {
    const long long w = n >> lb, len = (w == 1) ? 3 : w + 2;
    arch_cap = std::max(arch_cap, std::min((long long)1 << (2 * lb), budget / (len * len)));
  }
  int32_t* arch = lazy ? (int32_t*)ws(c, "vote_arch", (size_t)arch_cap * kLazyMax * 4) : nullptr;
  long long arch_used = 0;
  // bitmap archive: the passes' bitmaps built by k_vote_bitmap, then one
  // staging bitmap per tuner slot that k_small_pass writes itself (B <= 64)
  const long long small_base = (long long)lazy_bm_words(std::min(9, lgN)) * kLazyMax;
  const int small_words = lazy_bm_words(6);
  uint32_t* bmarch = lazy ? (uint32_t*)ws(c, "vote_bm", (size_t)(small_base + 2LL * SFFT2D_MAX_HISTORY * small_words) * 4)
                          : nullptr;
  long long bm_used = 0;
  int bm_smem_used = 0;   // words of k_vote_lazy2's shared copy of the bitmap passes
  bool hist_used = false;
  // NaN/Inf check (as_complex_matrix, corefft.py:49-50): fused into the dense
  // FFT's row pass when the trajectory reaches B = N, else one pass at the end
  unsigned char* scr = call_scratch(c);
  ck(cudaMemsetAsync(scr, 0, kScrBytes, st), "memset scratch");
  unsigned* finite = (unsigned*)(scr + kScrFinite);
  bool finite_scanned = false;
  // whatever path leaves run_ats, later work on st is ordered after the side
  // stream's (post-fold work of speculative passes, votes)
  struct JoinSide {
    sfft2d_ctx* c;
    cudaStream_t st;
    ~JoinSide() {
      cudaEventRecord(c->ev_lmax, c->vote_st);
      cudaStreamWaitEvent(st, c->ev_lmax, 0);
    }
  } join_side{c, st};

  std::memset(S, 0, sizeof(*S));
  int b = std::max(4, std::min(cf.b0, n));
  bool xhat_ready = false;
  C* xhat = nullptr;
  T* M = nullptr;
  unsigned long long* peakM = nullptr;
  int32_t* maxlist = (int32_t*)ws(c, "maxlist", (size_t)(nkeys / 4 + 64) * 4);
  int pidx = 0;
  bool have_votes = false;
  int vote_passes = 0;
  bool last_valid = false;
  int last_b = 0, last_pi = 0;
  cudaEvent_t last_ready = nullptr;
  long long last_count = 0;
  long long last_bm_off = -1;

  // sides >= 2048: the dense FFT stops after four-step pass A (x_hat is never
  // stored), pass B writes |x_hat| only when a B = N tuner pass needs it
  // ... unless the B = N/2 passes can come from the stored spectrum (k_pass_conv,
  // N <= 4096): two passes of fold + three FFT passes cost more than the
  // complex128 x_hat write the factored form saves (SFFT2D_FP64_FACTORED=1: as before)
  static const bool fp64_factored_always = getenv("SFFT2D_FP64_FACTORED") != nullptr;
  static const bool passconv_env_on = getenv("SFFT2D_NO_PASSCONV") == nullptr;
  const bool conv_possible = passconv_env_on && !fp64_factored_always && n >= 1024 && n <= 4096 &&
                             tb.conv_r[lgN - 1] == 2 && (size_t)3 * n * sizeof(C) <= 200 * 1024;
  const bool factored = dense_factored(lgN, prec_of<T>()) && !conv_possible;
  C* dscratch = nullptr;
  auto ensure_xhat = [&](bool need_mags) {
    if (factored) {
      const C* tw = (const C*)tb.tw[prec_of<T>()];
      if (!dscratch) {
        dscratch = dense_fft_front<T, Tin>(c, x, lgN, tw, st, finite);   // + NaN check
        finite_scanned = true;
      }
      if (need_mags && !M) {
        M = (T*)ws(c, "xmag", (size_t)nkeys * sizeof(T));
        peakM = (unsigned long long*)(scr + kScrXpeak);   // zeroed with the scratch
        dense_fft_mags<T>(c, M, peakM, lgN, tw, st);
      }
      return;
    }
    if (!xhat_ready) {
      xhat = (C*)ws(c, "xhat", (size_t)nkeys * sizeof(C));
      if (need_mags) {
        M = (T*)ws(c, "xmag", (size_t)nkeys * sizeof(T));
        peakM = (unsigned long long*)(scr + kScrXpeak);
      }
      dense_xhat<T, Tin>(c, x, lgN, tb, xhat, M, peakM, st, finite);   // |x_hat|, peak, NaN check
      finite_scanned = true;
      xhat_ready = true;
    }
    if (need_mags && !M) {
      M = (T*)ws(c, "xmag", (size_t)nkeys * sizeof(T));
      peakM = (unsigned long long*)(scr + kScrXpeak);
      mags_of<T>(c, xhat, nkeys, 1, M, peakM, st);
    }
  };

  // the complex dense spectrum in natural order (k_estimate_conv): stored by
  // the unfactored dense FFT; the factored one runs pass B once more with a
  // complex output
  C* xfull = nullptr;
  auto dense_xhat_complex = [&]() -> const C* {
    if (!factored) {
      ensure_xhat(false);
      return xhat;
    }
    if (!xfull) {
      ensure_xhat(false);
      xfull = (C*)ws(c, "xhat_full", (size_t)nkeys * sizeof(C));
      dense_fft_xhat<T>(c, xfull, lgN, (const C*)tb.tw[prec_of<T>()], st);
    }
    return xfull;
  };

  // per-pass count slots (zeroed once), double-buffered maxima lists: the
  // vote of pass k runs on the side stream while pass k+1 proceeds
  unsigned* cnt_slots = (unsigned*)(scr + kScrCounts);   // zeroed with the scratch
  int32_t* maxlists[2] = {maxlist, (int32_t*)ws(c, "maxlist2", (size_t)(nkeys / 4 + 64) * 4)};
  bool vote_pending[2] = {false, false};
  int npass = 0;
  int last_slot = 0;
  // the vote of a pass is issued once the host has read its count (passes over
  // the budget cast nothing): in deferred mode the pass's maxima list is
  // archived for k_vote_lazy (bitmap passes B <= 512, short list passes), else
  // one atomic per preimage coordinate into the histogram on the side stream
  auto vote_list = [&](const Perm& pv, int lgb, int slot, long long count, cudaEvent_t list_ready,
                       long long prebuilt_off) {
    if (count <= 0) return;
    const int w = n >> lgb;
    const long long len = (w == 1) ? 3 : std::min<long long>(w + 2, n);
    if (lazy && (lgb <= 9 || count <= kLazyScan) && lp.n < kLazyMax && count <= arch_cap) {
      LazyPass& P = lp.v[lp.n++];
      P.p = pv;
      P.lgB = lgb;
      P.count = (int)count;
      P.off = arch_used;
      if (lgb <= 9) {
        // bitmap pass: B x B maxima bitmap + row flags, built on the side
        // stream (off the tuner's critical path; joined before k_vote_lazy)
        lp.lgBmax = std::max(lp.lgBmax, lgb);
        const int words = lazy_bm_words(lgb);
        P.soff = bm_smem_used;
        bm_smem_used += words;
        if (prebuilt_off >= 0) {   // written by the pass's own k_small_pass
          P.off = prebuilt_off;
          return;
        }
        P.off = bm_used;
        cudaStream_t vs = c->profiling ? st : c->vote_st;
        ck(cudaStreamWaitEvent(vs, list_ready, 0), "cudaStreamWaitEvent");
        ck(cudaMemsetAsync(bmarch + bm_used, 0, (size_t)words * 4, vs), "memset bitmap");
        pre(c, vs);
        kl(k_vote_bitmap, grid_for(count, 256, kNumSMs), 256, 0, vs,
           (const int32_t*)maxlists[slot & 1], (const unsigned*)(cnt_slots + 2 * slot), lgb,
           bmarch + bm_used);
        post(c, "k_vote_bitmap", vs, (double)count * 4.0);
        ck(cudaEventRecord(c->ev_vote[slot & 1], vs), "cudaEventRecord");
        vote_pending[slot & 1] = true;   // the list slot is reused two passes later
        bm_used += words;
        return;
      }
      // (stream order: a speculative pass enqueued after this list's pass
      // writes the other list buffer)
      ck(cudaStreamWaitEvent(st, list_ready, 0), "cudaStreamWaitEvent");
      ck(cudaMemcpyAsync(arch + arch_used, maxlists[slot & 1], (size_t)count * 4,
                         cudaMemcpyDeviceToDevice, st), "archive maxima");
      arch_used += count;
      return;
    }
    // profiling serialises the votes onto the main stream so every launch's
    // event pair times that kernel alone
    cudaStream_t vs = c->profiling ? st : c->vote_st;
    ck(cudaStreamWaitEvent(vs, list_ready, 0), "cudaStreamWaitEvent");
    zero_hist(vs);
    hist_used = true;
    const long long total = count * len * len;
    pre(c, vs);
    kl(k_vote, grid_for(total, 256, kNumSMs * 2), 256, 0, vs, maxlists[slot & 1], 0,
       cnt_slots + 2 * slot, 0, nullptr, lgN, lgb, 1, mode, 0, hist, 0LL, pv);
    post(c, "k_vote", vs, (double)total * 4.0);
    ck(cudaEventRecord(c->ev_vote[slot & 1], vs), "cudaEventRecord");
    vote_pending[slot & 1] = true;
  };

  // deferred-vote tallies of the archived passes in `lp` (tile by tile in
  // shared memory), seeded from the histogram when it holds votes already;
  // thresholded into the compaction bitmask (bits) or written to hist_out
  auto launch_lazy = [&](cudaStream_t s2, unsigned thr_, uint32_t* bits, unsigned* cnts,
                         uint32_t* hist_out) {
    int lgG = 13;
    while (lgG < 15 && ((long long)1 << (lgG + 1)) * (2 * kNumSMs) <= nkeys) ++lgG;
    // every bitmap pass staged at once when they fit beside the tallies
    // (k_vote_lazy2, no per-pass barriers); else one at a time
    static const bool v2_on = getenv("SFFT2D_OLD_VOTE_LAZY") == nullptr;
    const size_t smem2 = ((size_t)1 << lgG) + (size_t)bm_smem_used * 4;
    pre(c, s2);
    if (v2_on && smem2 <= kMaxDynSmem) {
      kl(k_vote_lazy2, (unsigned)(nkeys >> lgG), 256, smem2, s2, (const int32_t*)arch,
         (const uint32_t*)bmarch, (int)bm_used, lp, lgN, lgG,
         (const uint32_t*)(hist_used ? hist : nullptr), hist_out, thr_, bits, cnts);
    } else {
      const size_t smem = vote_lazy_smem(lgN, lgG, lp.lgBmax);
      kl(k_vote_lazy, (unsigned)(nkeys >> lgG), 256, smem, s2, (const int32_t*)arch,
         (const uint32_t*)bmarch, lp, lgN, lgG,
         (const uint32_t*)(hist_used ? hist : nullptr), hist_out, thr_, bits, cnts);
    }
    post(c, "k_vote_lazy", s2, (double)nkeys / 8.0 + (hist_used ? (double)nkeys : 0.0) +
                                   (hist_out ? (double)nkeys : 0.0));
  };
  // Once the trajectory reaches B = N only short passes follow: the passes
  // archived so far are tallied into the histogram on the side stream while
  // they run, and the final tally adds only the later passes
  // (SFFT2D_NO_EARLY_VOTES=1: one tally at the end)
  static const bool early_votes_on = getenv("SFFT2D_NO_EARLY_VOTES") == nullptr;
  bool early_voted = false;
  auto early_votes = [&]() {
    if (!lazy || early_voted || lp.n == 0 || c->profiling || !early_votes_on) return;
    early_voted = true;
    cudaStream_t vs = c->vote_st;
    // list-pass archives are copied on the main stream
    ck(cudaEventRecord(c->ev_fork_votes, st), "cudaEventRecord");
    ck(cudaStreamWaitEvent(vs, c->ev_fork_votes, 0), "cudaStreamWaitEvent");
    const cudaStream_t ws_saved = c->ws_st;
    c->ws_st = vs;
    launch_lazy(vs, 0u, nullptr, nullptr, hist);
    c->ws_st = ws_saved;
    hist_used = true;      // the histogram now seeds every later tally
    hist_zeroed = true;    // (and must not be cleared by a later atomic vote)
    lp.n = 0;              // tallied; later passes are archived from scratch
    bm_smem_used = 0;
  };

  // B = N views after the first one test only the above-floor bins of |x_hat|
  // that the first B = N pass listed (while they are few)
  int32_t* cand = nullptr;
  unsigned* cand_cnt = nullptr;
  bool cand_pending = false, cand_ready = false;
  long long cand_n = 0;

  // speculative next-pass grid (k_fold_wide2), valid for permutation index spec_pi at spec_b
  static const bool spec_on = getenv("SFFT2D_NO_SPEC") == nullptr;
  int spec_pi = -1, spec_b = 0, spec_z = 1;
  C* spec_grid = nullptr;
  // A tuner pass is enqueued (fold / FFT / local maxima, count published to
  // its own mapped slot) and finished later (host reads the count, casts the
  // vote).  While the host waits for pass t, the predicted pass t + 1 is
  // already in the stream (pass 1 repeats pass 0's B; afterwards the tuner
  // doubles B until the counts settle): the permutation of pass t + 1 is the
  // next draw whatever its B, so a hit is exactly the pass the reference runs
  // and hides one host round trip; a miss is discarded (its slot, list and
  // publication are never read) and the real pass is enqueued behind it.
  struct Ticket {
    int pi = -1, slot = -1, bb = 0;
    unsigned seq = 0;
    bool emitted = false;   // first B = N pass: above-floor candidates listed
    Perm p;
    cudaEvent_t ready = nullptr;   // the pass's maxima list is complete
    cudaStream_t lst = nullptr;     // the stream that publishes the count
    long long bm_off = -1;          // vote bitmap written by the pass itself (k_small_pass)
  };
  static const bool pipe_on = getenv("SFFT2D_NO_PIPELINE") == nullptr;
  static const bool pass_pipe_on = getenv("SFFT2D_NO_PASS_PIPE") == nullptr;
  static const bool small_bm_on = getenv("SFFT2D_NO_SMALL_BITMAP") == nullptr;
  // the B = N/2 pass from the dense spectrum: x_hat stored (not factored),
  // untruncated 5-tap window, 512 <= B <= 2048 (SFFT2D_NO_PASSCONV=1: fold + FFT)
  static const bool passconv_on = getenv("SFFT2D_NO_PASSCONV") == nullptr;
  const bool passconv_ok = passconv_on && !factored && n >= 1024 && n <= 4096 &&
                           tb.conv_r[lgN - 1] == 2 && (size_t)3 * n * sizeof(C) <= 200 * 1024;
  int ev_next = 0;
  auto enqueue_pass = [&](int bb, int pi) -> Ticket {
    Ticket tk;
    tk.pi = pi;
    tk.bb = bb;
    const Perm p = ps.get(pi, st);
    tk.p = p;
    const int lgb = ilog2(bb);
    const size_t BB = (size_t)bb * bb;
    const int slot = npass++;
    tk.slot = slot;
    if (slot >= 2 * SFFT2D_MAX_HISTORY) fail(SFFT2D_ERR_UNSUPPORTED, "too many tuner passes");
    int32_t* ml = maxlists[slot & 1];
    unsigned* cnt = cnt_slots + 2 * slot;   // 8-byte slots: count, CTA tickets (k_lmax_win2)
    // the vote two passes back still reads this list: a list written on the
    // main stream waits for it; the side stream runs votes and lists in order
    auto wait_list_free = [&]() {
      if (vote_pending[slot & 1])
        ck(cudaStreamWaitEvent(st, c->ev_vote[slot & 1], 0), "cudaStreamWaitEvent");
    };
    // post-fold work of passes at B < N (reduce, FFT, |Z|, local maxima) goes
    // to the side stream, so the next (speculated) pass's fold runs beside it;
    // the pass's private workspace is set slot % 3 (SFFT2D_NO_PASS_PIPE=1: one stream)
    const bool side = pass_pipe_on && !c->profiling;
    cudaStream_t lst = st;   // the stream that writes this pass's maxima list
    unsigned seq;
    if (bb == n) {
      wait_list_free();
      // B = N: |Z_p[k1, k2]| = |x_hat[s1i k1, s2i k2]| — one dense FFT serves every pass
      ensure_xhat(true);
      const bool listed = cand_ready || cand_pending;   // the device count is exact either way
      if (listed && (!cand_ready || cand_n <= nkeys / 32)) {
        const unsigned grid = cand_ready ? grid_for(std::max<long long>(cand_n, 1), 256, kNumSMs * 8)
                                         : (unsigned)(kNumSMs * 2);
        const Publish pub = make_publish(c, grid);
        seq = pub.seq;
        pre(c, st);
        kl(k_lmax_cand<T>, grid, 256, 0, st, (const T*)M, lgb, p.s1i, p.s2i, p.s1, p.s2,
           (const int32_t*)cand, (const unsigned*)cand_cnt, ml, cnt, pub);
        post(c, "k_lmax_cand", st, (double)(cand_ready ? cand_n : nkeys / 32) * 9 * sizeof(T));
      } else if (!listed) {
        cand = (int32_t*)ws(c, "cand", (size_t)nkeys * 4);
        cand_cnt = (unsigned*)(scr + kScrCand);   // zeroed with the scratch
        bool emitted = false;
        seq = lmax_tuner<T>(c, M, lgb, peakM, cf.mag_floor, ml, cnt, st, true, p.s1i, p.s2i, p.s2,
                            cand, cand_cnt, &emitted);
        cand_pending = emitted;
        tk.emitted = emitted;
      } else {
        seq = lmax_tuner<T>(c, M, lgb, peakM, cf.mag_floor, ml, cnt, st, true, p.s1i, p.s2i, p.s2);
      }
    } else if (2 * bb == n && passconv_ok) {
      // B = N/2 from the dense spectrum (k_pass_conv): the dense FFT is
      // computed here, one pass early, and serves the B = N passes after it
      wait_list_free();
      ensure_xhat(true);
      // a buffer of its own: this pass runs on the main stream in the default
      // workspace set (0), and "grid_mag" of set 0 also belongs to the
      // side-stream passes with slot % 3 == 0 — a speculated B = N/2 pass
      // enqueued behind such a pass would overwrite the |Z| grid its local
      // maxima are still being counted from (found by the large-N fuzz)
      T* mg = (T*)ws(c, "grid_mag_conv", BB * sizeof(T));
      // this slot's peak, zeroed with the scratch
      unsigned long long* pk = (unsigned long long*)(scr + kScrPeaks) + slot;
      const T* freq = (const T*)tb.freq[prec_of<T>()] + ((size_t)lgb << lgN);
      const C* tw = (const C*)tb.tw[prec_of<T>()];
      constexpr int RB = sizeof(T) == 4 ? 4 : 2;
      const size_t sm = (size_t)3 * n * sizeof(C);
      pre(c, st);
      // taps |d| <= R: R = 2 in fp64; in fp32 the |d| = 2 taps (|F| = 2.5e-9)
      // are below float resolution
      constexpr int RT = sizeof(T) == 4 ? 1 : 2;
      static const bool band_on = getenv("SFFT2D_OLD_PASSCONV") == nullptr;
      if (band_on) {
        // bands of output rows sized for one wave of resident CTAs (at least
        // the RB rows of the fixed-tile kernel, to bound the halo re-reads)
        auto go = [&](auto CP) {
          constexpr int CPT = decltype(CP)::value;
          const int cps = std::max(1, ctas_per_sm(k_pass_conv_band<T, CPT, 3, RT>, 256, sm));
          const int nb = std::max(RB, (bb + cps * kNumSMs - 1) / (cps * kNumSMs));
          kl(k_pass_conv_band<T, CPT, 3, RT>, (bb + nb - 1) / nb, 256, sm, st, (const C*)xhat, lgN, p,
             freq, tw, nb, mg, pk);
        };
        if (bb == 2048) go(std::integral_constant<int, 8>{});
        else if (bb == 1024) go(std::integral_constant<int, 4>{});
        else go(std::integral_constant<int, 2>{});
      } else if (bb == 2048)
        kl(k_pass_conv<T, 8, RB, 3, RT>, bb / RB, 256, sm, st, (const C*)xhat, lgN, p, freq, tw, mg, pk);
      else if (bb == 1024)
        kl(k_pass_conv<T, 4, RB, 3, RT>, bb / RB, 256, sm, st, (const C*)xhat, lgN, p, freq, tw, mg, pk);
      else
        kl(k_pass_conv<T, 2, RB, 3, RT>, bb / RB, 256, sm, st, (const C*)xhat, lgN, p, freq, tw, mg, pk);
      // algorithmic bytes: x_hat once + |Z| (the band halo rows re-read,
      // (2 RB + 2 RT - 1) / (2 RB) of x_hat, are the kernel's own overhead)
      post(c, "k_pass_conv", st, (double)n * n * sizeof(C) + (double)BB * sizeof(T));
      seq = lmax_tuner<T>(c, mg, lgb, pk, cf.mag_floor, ml, cnt, st, true, 1u, 1u, 1u, nullptr, nullptr,
                          nullptr, true, true);
    } else if (BB * sizeof(C) <= (size_t)kSmall2DBytes) {
      if (!side) wait_list_free();
      c->ws_set = side ? slot % 3 : 0;
      C* y = (C*)ws(c, "fold_y", BB * sizeof(C));
      FoldOut fo{y, 1};
      if (spec_pi == pi && spec_b == bb) {
        fo = FoldOut{spec_grid, spec_z};   // folded with pass 0 (same B, one read)
        spec_pi = -1;
      } else {
        spec_pi = -1;
        // the first two tuner passes share B (no ratio after pass 0) and pass 1
        // always follows when max_iters >= 2: fold both from one read
        const long zs = std::min<long>(n / bb, 2L * kNumSMs / bb);
        static const bool spec0_on = getenv("SFFT2D_NO_SPEC0") == nullptr;
        // (an explicit permutation list must hold pass 1's permutation: the
        // reference may never draw it, and the library must not overrun)
        if (spec_on && spec0_on && pi == 0 && max_iters >= 2 && (size_t)n * sizeof(Tin) >= kRingSegBytes &&
            bb < 512 && zs > 1 && (ps.bitgen || ps.n_arr > 1)) {
          const Perm* sq = &ps.get(1, st);
          spec_grid = (C*)ws(c, "spec_small", (size_t)zs * BB * sizeof(C));
          spec_pi = 1;
          spec_b = bb;
          fo = fold_launch<T, Tin>(c, x, lgN, lgb, tb, &p, 1, y, st, nullptr, false, sq, spec_grid,
                                   &spec_z, true);
        } else {
          fo = fold_launch<T, Tin>(c, x, lgN, lgb, tb, &p, 1, y, st);
        }
      }
      const Publish pub = make_publish(c, 1);
      seq = pub.seq;
      if (side) {
        ck(cudaEventRecord(c->ev_fold[ev_next], st), "cudaEventRecord");
        ck(cudaStreamWaitEvent(c->vote_st, c->ev_fold[ev_next], 0), "cudaStreamWaitEvent");
        lst = c->vote_st;
      }
      pre(c, lst);
      if (BB > 4 * 1024) fail(SFFT2D_ERR_UNSUPPORTED, "small pass holds at most 4 bins per thread");
      const size_t sps = (size_t)bb * (bb + 1) * sizeof(C) + BB * sizeof(T) + bb * sizeof(C);
      // the pass writes its own vote bitmap (used if it votes): no bitmap
      // kernel / memset later
      uint32_t* sbm = nullptr;
      if (lazy && lgb <= 6 && small_bm_on) {
        tk.bm_off = small_base + (long long)slot * small_words;
        sbm = bmarch + tk.bm_off;
      }
      if (BB <= 1024)   // one (bin, partial-slice) slot per thread
        kl(k_small_pass<T, 1>, 1, 1024, sps, lst, (const C*)fo.data, fo.Z, fo.Z == 1, lgb, p,
           (const C*)tb.tw[prec_of<T>()], lgN, cf.mag_floor, ml, cnt, pub, sbm);
      else
        kl(k_small_pass<T, 4>, 1, 1024, sps, lst, (const C*)fo.data, fo.Z, fo.Z == 1, lgb, p,
           (const C*)tb.tw[prec_of<T>()], lgN, cf.mag_floor, ml, cnt, pub, sbm);
      post(c, "k_small_pass", lst, (double)(fo.Z + 1) * BB * sizeof(C));
      c->ws_set = 0;
    } else {
      if (!side) wait_list_free();
      c->ws_set = side ? slot % 3 : 0;
      T* mg = (T*)ws(c, "grid_mag", BB * sizeof(T));
      unsigned long long* pk = (unsigned long long*)ws(c, "gpeak", 16);
      // |Z[k1,k2]| = |Y^[s1i k1, s2i k2]| for the natural-order fold Y
      // (Z[a,b] = Y[s1 a + t1, s2 b + t2]; the tau shifts are a phase):
      // fold without the bucket scatter, FFT Y, and test the permuted view
      // speculation: B >= 128 folds also produce the next pass's grid at 2B
      // (its permutation is the next draw whatever the next pass is; with
      // estimation loops to follow that draw is always made, so drawing it
      // early leaves the caller's Generator exactly where the reference does)
      C* pre_y = (spec_pi == pi && spec_b == bb) ? spec_grid : nullptr;
      const int pre_z = spec_z;
      spec_pi = -1;
      const Perm* sq = nullptr;
      C* sy = nullptr;
      // ring pair (128 <= B <= 256, full-support rows) or wide pair (B >= 512)
      const bool ring_pair = bb >= 128 && 2 * bb <= 512 && (size_t)n * sizeof(Tin) >= kRingSegBytes;
      const bool wide_pair = bb >= 512 && lgN - lgb <= 5 && lgN - lgb >= 2;
      if (!pre_y && spec_on && do_estimate && 2 * bb < n && (ring_pair || wide_pair) &&
          (ps.bitgen || pi + 1 < ps.n_arr)) {
        sq = &ps.get(pi + 1, st);
        const int zmax = ring_pair ? std::max(1, (int)(2L * kNumSMs / bb)) : 1;
        sy = spec_grid = (C*)ws(c, "spec_y", (size_t)zmax * 4 * BB * sizeof(C));
        spec_pi = pi + 1;
        spec_b = 2 * bb;
      }
      if (side) lst = c->vote_st;
      fold_spectrum<T, Tin>(c, x, lgN, lgb, tb, &p, 1, (C*)nullptr, mg, pk, st, true, pre_y, sq, sy,
                            pre_z, &spec_z, nullptr, side ? lst : nullptr, c->ev_fold[ev_next]);
      const unsigned mb = (unsigned)bb - 1u;
      // B < N: the fold aliases the noise floor into most buckets
      const cudaStream_t ws_saved = c->ws_st;
      c->ws_st = lst;
      seq = lmax_tuner<T>(c, mg, lgb, pk, cf.mag_floor, ml, cnt, lst, true, p.s1i & mb, p.s2i & mb,
                          p.s2 & mb, nullptr, nullptr, nullptr, true, true);
      c->ws_st = ws_saved;
      c->ws_set = 0;
    }
    tk.seq = seq;
    tk.ready = c->ev_pass[ev_next];
    ev_next = (ev_next + 1) % 4;
    ck(cudaEventRecord(tk.ready, lst), "cudaEventRecord");   // the maxima list is complete
    tk.lst = lst;
    return tk;
  };
  // a speculative pass that the tuner did not take: nothing of it is read;
  // its fold speculation (if any) is dropped and a candidate listing it
  // started is redone by the next B = N pass
  auto discard_pass = [&](const Ticket& tk) {
    spec_pi = -1;
    if (tk.emitted) cand_pending = false;
  };
  auto finish_pass = [&](const Ticket& tk) -> long long {
    const long long count = wait_published(c, tk.seq, tk.lst ? tk.lst : st);
    if (tk.emitted) {   // the candidate count rides along with the maxima count
      cand_n = pub_slot_h(c, tk.seq)[2];
      cand_pending = false;
      cand_ready = true;
    }
    pidx = tk.pi + 1;
    last_valid = true;
    last_b = tk.bb;
    last_pi = tk.pi;
    last_count = count;
    last_slot = tk.slot;
    last_ready = tk.ready;
    last_bm_off = tk.bm_off;
    const int lgb = ilog2(tk.bb);
    const long long w = n / tk.bb;
    const long long len = (w == 1) ? 3 : std::min<long long>(w + 2, n);
    if (count > 0 && count * len * len <= budget) {   // tuner.py:165,175
      vote_list(tk.p, lgb, tk.slot, count, tk.ready, tk.bm_off);
      ++vote_passes;
      have_votes = true;
    }
    return count;
  };

  auto t_pass = std::chrono::steady_clock::now();
  auto push = [&](int bb, long long cnt, double r, bool has) {
    const int i = S->passes++;
    const auto now = std::chrono::steady_clock::now();
    S->hist_us[i] = std::chrono::duration<double, std::micro>(now - t_pass).count();
    t_pass = now;
    S->hist_bins[i] = bb;
    S->hist_count[i] = cnt;
    S->hist_ratio[i] = has ? r : NAN;
    S->hist_has_ratio[i] = has ? 1 : 0;
  };

  std::map<std::pair<int, long long>, int> seen;
  bool moved = false;
  bool converged = false;
  long long prev = -1;
  Ticket cur;
  if (max_iters > 0) cur = enqueue_pass(b, pidx);
  for (int it = 0; it < max_iters; ++it) {
    // the predicted next pass goes into the stream before this pass's count
    // is read (pass 1: same B; later: B doubled, capped at n)
    Ticket spec;
    bool have_spec = false;
    if (pipe_on && it + 1 < max_iters && (ps.bitgen || cur.pi + 1 < ps.n_arr)) {
      spec = enqueue_pass(it == 0 ? b : std::min(2 * b, n), cur.pi + 1);
      have_spec = true;
    }
    const long long cnt = finish_pass(cur);
    if (cur.bb == n) early_votes();
    bool has = false;
    bool stop = false;
    double r = 0.0;
    if (prev < 0) {
      has = false;
    } else if (prev == 0 && cnt == 0) {
      push(b, cnt, 0.0, true);
      converged = true;
      stop = true;
    } else {
      has = true;
      r = (prev == 0) ? INFINITY : std::fabs(1.0 - (double)cnt / (double)prev);
    }
    if (!stop) {
      push(b, cnt, r, has);
      if (has && cf.delta1 <= r && r < cf.delta2) {
        converged = true;
        stop = true;
      }
    }
    if (!stop) {
      int& sc = seen[std::make_pair(b, cnt)];
      ++sc;
      if (sc >= 3 && moved) {
        converged = true;
        stop = true;
      }
    }
    if (stop) {
      if (have_spec) discard_pass(spec);
      break;
    }
    prev = cnt;
    if (has) {
      const int nb = update_bins(b, r, cf, n);
      moved = moved || nb != b;
      b = nb;
    }
    if (it + 1 >= max_iters) break;
    if (have_spec && spec.bb == b) {
      cur = spec;
    } else {
      if (have_spec) discard_pass(spec);
      cur = enqueue_pass(b, pidx);
    }
  }
  long long maxc = 0;
  int btop = 0;
  for (int i = 0; i < S->passes; ++i) {
    maxc = std::max(maxc, (long long)S->hist_count[i]);
    btop = std::max(btop, S->hist_bins[i]);
  }
  if (S->passes > 0 && maxc > 0) {
    // confirmation passes at 2 b_top and 4 b_top (tuner.py:209-226): both
    // are certain now, so both are enqueued before either count is read
    Ticket conf[2];
    int nconf = 0;
    for (int mult = 2; mult <= 4; mult *= 2) {
      const long long bc = (long long)mult * btop;
      if (bc <= n) {
        conf[nconf] = enqueue_pass((int)bc, pidx + nconf);
        ++nconf;
      }
    }
    for (int i = 0; i < nconf; ++i) {
      const long long cnt = finish_pass(conf[i]);
      push(conf[i].bb, cnt, NAN, false);
      maxc = std::max(maxc, cnt);
    }
  }
  int bdet = b;
  if (S->passes > 0) {
    bdet = 0;
    for (int i = 0; i < S->passes; ++i) bdet = std::max(bdet, S->hist_bins[i]);
  }
  if (!finite_scanned) {
    pre(c, st);
    kl(k_check_finite<Tin>, grid_for(nkeys, 256, kNumSMs * 8), 256, 0, st, x, nkeys, finite);
    post(c, "k_check_finite", st, (double)nkeys * sizeof(Tin));
  }
  // the NaN/Inf flag rides along with the next synchronisation (the fused
  // tail publishes it itself and never enqueues this copy)
  bool finite_fetched = false;
  auto fetch_finite = [&]() {
    if (finite_fetched) return;
    finite_fetched = true;
    ck(cudaMemcpyAsync(c->pinned + 1, finite, sizeof(unsigned), cudaMemcpyDeviceToHost, st), "D2H");
  };
  auto nan_check = [&](bool need_sync) {
    if (need_sync) fetch_finite();
    if (need_sync) ck(cudaStreamSynchronize(st), "sync");
    if (c->pinned[1]) {
      std::memset(S, 0, sizeof(*S));
      fail(SFFT2D_ERR_VALUE, "matrix contains NaN or Inf");
    }
  };
  S->converged = converged ? 1 : 0;
  S->detected_k = maxc;
  S->b_detect = bdet;
  S->b_estimate = default_bins(n, maxc);
  if (!have_votes && last_valid && maxc > 0) {
    // every pass exceeded the vote budget: fall back to the final pass (tuner.py:228-234)
    if (last_count > 0) {
      // its list and count slot are intact (later passes were discarded
      // speculation writing the other list buffer)
      vote_list(ps.hp[last_pi], ilog2(last_b), last_slot, last_count, last_ready, last_bm_off);
      have_votes = true;
    }
    vote_passes = 1;
  }
  S->vote_passes = vote_passes;
  // the histogram is complete once the side-stream votes are
  ck(cudaEventRecord(c->ev_lmax, c->vote_st), "cudaEventRecord");
  ck(cudaStreamWaitEvent(st, c->ev_lmax, 0), "cudaStreamWaitEvent");
  int32_t* keys = (int32_t*)ws(c, "keys", (size_t)nkeys * 4);
  unsigned* kt = (unsigned*)ws(c, "keys_tot", 16);
  // deferred votes: tallies of every archived pass, tile by tile in shared
  // memory; either thresholded into the compaction bitmask (bits != nullptr)
  // or written out as the histogram (the detect_sparsity API's tallies)
  auto lazy_votes = [&](unsigned thr_, uint32_t* bits, unsigned* cnts, uint32_t* hist_out) {
    launch_lazy(st, thr_, bits, cnts, hist_out);
  };


  if (!do_estimate) {
    unsigned nv = 0;
    if (have_votes) {
      if (lazy) lazy_votes(0u, nullptr, nullptr, hist);
      fetch_finite();
      nv = hist_compact(c, hist, nkeys, mode, 1u, keys, kt, st);
      nan_check(false);
      int32_t* tal = (int32_t*)ws(c, "tallies", (size_t)std::max(nv, 1u) * 4);
      pre(c, st);
      kl(k_gather_tallies, grid_for(nv), 256, 0, st, hist, mode, keys, kt, tal);
      post(c, "k_gather_tallies", st, 0);
    } else {
      nan_check(true);
    }
    S->n_votes = nv;
    S->perms_used = pidx;
    S->perms_drawn = (int32_t)ps.used();
    c->votes_count = nv;
    c->has_votes = true;
    return;
  }

  res->count = 0;
  res->ordered_by_magnitude = 0;
  res->n_candidates = 0;
  c->res_count = 0;
  if (maxc == 0 || !have_votes) {
    nan_check(true);
    S->perms_used = pidx;
    S->perms_drawn = (int32_t)ps.used();
    res->perms_used = pidx;
    return;
  }
  const unsigned thr = (unsigned)((std::max(vote_passes, 1) + 1) / 2);
  unsigned m;   // (the estimation scalars were zeroed with the scratch)
  if (lazy) {
    uint32_t* bits = (uint32_t*)ws(c, "hc_bits", words_for(nkeys) * 4);
    unsigned* cnts = (unsigned*)ws(c, "hc_cnt", (size_t)blocks_for(nkeys) * 4);
    lazy_votes(thr, bits, cnts, nullptr);
    // Dense estimate (b_estimate = N, x_hat stored) of what is almost always a
    // small candidate set: the fused tail kernel is launched before the host
    // knows m (it reads m on the device) and publishes m, the NaN flag, the
    // results and their count to mapped memory — one host round trip instead
    // of two and one launch instead of five.  It only reports m when
    // m > limit (limit <= k: no top-k cut can be needed below it); the
    // general path then runs with that m.  SFFT2D_NO_FUSED_TAIL=1: general path.
    static const bool fused_tail_on = getenv("SFFT2D_NO_FUSED_TAIL") == nullptr;
    const long long lim = std::min<long long>(maxc, (long long)finish_small_max<T>());
    const int best0 = S->b_estimate;
    bool m_known = false;
    if (fused_tail_on && best0 == n && !factored && lim >= 1 &&
        std::max(1LL, 2 * maxc) <= (long long)best0 * best0 &&
        (ps.bitgen || pidx + L <= ps.n_arr)) {
      // compaction without the scan launch; the tail kernel sums the block
      // counts itself (and stores m for the general path)
      pre(c, st);
      kl(k_compact_bits_self, blocks_for(nkeys), kCmpThreads, 0, st, (const uint32_t*)bits, nkeys,
         (const unsigned*)cnts, keys);
      post(c, "k_compact_bits", st, 0);
      ensure_xhat(false);
      const size_t cap = (size_t)lim;
      char* outh = (char*)host_out(c, cap * (16 + sizeof(C)) + 64);
      int64_t* oij_h = (int64_t*)outh;
      C* ov_h = (C*)(outh + cap * 16);
      int64_t* oij_d;
      ck(cudaHostGetDevicePointer((void**)&oij_d, oij_h, 0), "cudaHostGetDevicePointer");
      C* ov_d = (C*)((char*)oij_d + cap * 16);
      const Publish pub = make_publish(c, 1);
      pre(c, st);
      kl(k_finish_dense_small<T>, 1, 1024, (size_t)lim * sizeof(C), st, (const C*)xhat, (const int32_t*)keys,
         (const unsigned*)cnts, blocks_for(nkeys), kt, (unsigned)lim, 1.0 >= cf.gain_floor, cf.prune_rel,
         (const unsigned*)finite, lgN, oij_d, ov_d, pub.slot, pub.seq);
      post(c, "k_finish_dense_small", st, 0);
      const unsigned count = wait_published(c, pub.seq, st);
      volatile unsigned* sl = pub_slot_h(c, pub.seq);
      m = sl[2];
      m_known = true;
      if (sl[3]) {
        std::memset(S, 0, sizeof(*S));
        fail(SFFT2D_ERR_VALUE, "matrix contains NaN or Inf");
      }
      if (count != kFinishFallback) {
        S->n_candidates = m;
        res->n_candidates = m;
        if (m > 0) {
          for (int i = 0; i < L; ++i) ps.get(pidx + i, st);   // drawn as the reference draws them
          pidx += L;
          c->out_ij_h = oij_h;
          c->out_v_h = ov_h;
          res->count = count;
          c->res_count = count;
        }
        S->perms_used = pidx;
        S->perms_drawn = (int32_t)ps.used();
        res->perms_used = pidx;
        return;
      }
    }
    if (!m_known) {
      compact(c, bits, cnts, nkeys, 1, keys, 0, kt, st);
      fetch_finite();
      m = read_u32(c, kt, st);
      nan_check(false);
    }
  } else {
    fetch_finite();
    m = hist_compact(c, hist, nkeys, mode, thr, keys, kt, st);
    nan_check(false);
  }
  S->n_candidates = m;
  if (m == 0) {
    S->perms_used = pidx;
    S->perms_drawn = (int32_t)ps.used();
    res->perms_used = pidx;
    return;
  }
  const long long k = maxc;
  const int best = S->b_estimate;
  if (std::max(1LL, 2 * k) > (long long)best * best) {
    S->perms_used = pidx;
    S->perms_drawn = (int32_t)ps.used();
    fail(SFFT2D_ERR_CONFIG, "d_factor*k = " + std::to_string(std::max(1LL, 2 * k)) +
                                " exceeds the " + std::to_string(best) + "x" +
                                std::to_string(best) + " bin budget");
  }
  for (int i = 0; i < L; ++i) ps.get(pidx + i, st);   // drawn as the reference draws them
  const bool dense = (best == n);
  if (!dense) ps.upload(pidx, L, st, c->ev_perm);   // the dense estimate reads x_hat only
  if (dense) ensure_xhat(false);
  // B < N with an untruncated window: estimate from the dense spectrum when
  // it is already (partly) computed, or when B >= N/4 (a dense FFT is then
  // cheaper than L folds + L B x B FFTs)
  const int lgbest = ilog2(best);
  const cplx<T>* xconv = nullptr;
  const int conv_r = tb.conv_r[lgbest];
  if (!dense && conv_r > 0 && conv_on() &&
      (xhat_ready || dscratch || (long long)best * 4 >= (long long)n)) {
    xconv = dense_xhat_complex();
  }
  estimate_and_select<T, Tin>(c, x, lgN, lgbest, tb, ps.hp.data() + pidx, dp + pidx, L, keys, m,
                              kt, k, cf.gain_floor, cf.prune_rel, dense, xhat, st, res,
                              dense ? dscratch : nullptr, xconv, conv_r);
  pidx += L;
  S->perms_used = pidx;
  S->perms_drawn = (int32_t)ps.used();
  res->perms_used = pidx;
}

// ------------------------------------------------------------------ SFFT
// SFFT location phase (engine.py:130-160) for `nloc` loops: fold all loops
// from one read of x, top-num bins per loop, unhash with per-loop dedup.
// Output: a byte histogram — OR of loop bits (mode kVoteOrBit, nloc <= 8 and
// !want_counts) or per-coordinate loop counts (mode kVoteAdd8).  Returns the mode.
template <typename T, typename Tin>
int sfft_location(sfft2d_ctx* c, const Tin* x, const sfft2d_sfft_config& cf, const DevTables& tb,
                  const Perm* hp, const Perm* dp, int nloc, bool want_counts, uint32_t* out,
                  cudaStream_t st, unsigned* nonfinite = nullptr, cudaEvent_t after_fold = nullptr) {
  const int n = cf.n, lgN = ilog2(n), b = cf.b_bins, lgb = ilog2(b);
  const long BB = (long)b * b;
  const long nkeys = (long)n * n;
  const long long num = std::max(1LL, (long long)cf.d_factor * cf.k);
  T* mags = (T*)ws(c, "loc_mags", (size_t)nloc * BB * sizeof(T));
  fold_spectrum<T, Tin>(c, x, lgN, lgb, tb, hp, nloc, (cplx<T>*)nullptr, mags, nullptr, st, false,
                        nullptr, nullptr, nullptr, 1, nullptr, nonfinite);
  if (after_fold) ck(cudaEventRecord(after_fold, st), "cudaEventRecord");
  int32_t* bins = (int32_t*)ws(c, "loc_bins", (size_t)nloc * num * 4);
  if (num >= BB) {
    pre(c, st);
    kl(k_iota_segments, grid_for(BB * nloc), 256, 0, st, bins, BB, nloc);
    post(c, "k_iota_segments", st, 0);
  } else {
    static const bool topk_list_on = getenv("SFFT2D_NO_TOPK_LIST") == nullptr;
    if (topk_list_on && BB <= (long)kTopkCtaMax) {
      // one CTA per loop: radix threshold, tie ranks and the ascending bin list
      pre(c, st);
      kl(k_topk_list_seg<T>, nloc, 1024, 0, st, (const T*)mags, (int)BB, num, bins, (long)num);
      post(c, "k_topk_list_seg", st, (double)BB * nloc * sizeof(T));
    } else {
    const int nblk = blocks_for(BB);
    uint32_t* sb = (uint32_t*)ws(c, "loc_selbits", (size_t)nloc * words_for(BB) * 4);
    unsigned* sc = (unsigned*)ws(c, "loc_selcnt", (size_t)nloc * nblk * 4);
    topk_bits<T>(c, mags, BB, nloc, num, sb, sc, st);
    unsigned* tots = (unsigned*)ws(c, "loc_tot", (size_t)nloc * 4 + 16);
    compact(c, sb, sc, BB, nloc, bins, (long)num, tots, st);
    }
  }
  const size_t hb = hist_bytes(nkeys, kVoteAdd8);
  const int w = n / b;
  const long long len = (w == 1) ? 3 : std::min<long long>(w + 2, n);
  const long long per = num * len * len;
  const bool direct = nloc <= 8 && !want_counts;
  uint32_t* masks = direct ? out : (uint32_t*)ws(c, "hist_masks", hb);
  ck(cudaMemsetAsync(masks, 0, hb, st), "memset hist");
  if (!direct) ck(cudaMemsetAsync(out, 0, hb, st), "memset counts");
  const long nw = (long)(hb / 4);
  for (int g0 = 0; g0 < nloc; g0 += 8) {
    const int g = std::min(8, nloc - g0);
    pre(c, st);
    kl(k_vote, dim3(grid_for(per, 256, kNumSMs * 8), g), 256, 0, st, bins + (size_t)g0 * num, (long)num, nullptr, (long)num, dp + g0, lgN, lgb, 1, kVoteOrBit,
        0, masks, 0LL, Perm{0, 0, 0, 0, 0, 0});
    post(c, "k_vote", st, (double)per * g * 4.0);
    if (!direct) {
      pre(c, st);
      kl(k_mask_to_counts, grid_for(nw, 256, kNumSMs * 8), 256, 0, st, masks, out, nw);
      post(c, "k_mask_to_counts", st, 3.0 * nw * 4);
    }
  }
  return direct ? kVoteOrBit : kVoteAdd8;
}

// SFFT vote threshold + estimation (engine.py:148-160, 163-284) from a
// histogram in `mode`; results go to the context's result buffers.
template <typename T, typename Tin>
void sfft_from_hist(sfft2d_ctx* c, const Tin* x, const sfft2d_sfft_config& cf, const DevTables& tb,
                    const uint32_t* hist, int mode, const Perm* hp_est, const Perm* dp_est,
                    cudaStream_t st, sfft2d_result* res, bool nan_pending = false,
                    cplx<T>* pre_grids = nullptr, cudaEvent_t pre_ready = nullptr) {
  const int n = cf.n, lgN = ilog2(n), lgb = ilog2(cf.b_bins);
  const long nkeys = (long)n * n;
  int32_t* keys = (int32_t*)ws(c, "keys", (size_t)nkeys * 4);
  unsigned* kt = (unsigned*)ws(c, "keys_tot", 16);
  zero_est_scalars(c, st);
  const unsigned m = hist_compact(c, hist, nkeys, mode, (unsigned)cf.vote_threshold, keys, kt, st);
  if (nan_pending) raise_if_nonfinite(c);   // the scan's flag came with that synchronisation
  res->count = 0;
  res->ordered_by_magnitude = 0;
  res->n_candidates = m;
  c->res_count = 0;
  if (m == 0) return;
  estimate_and_select<T, Tin>(c, x, lgN, lgb, tb, hp_est, dp_est, cf.loops, keys, m, kt, cf.k,
                              cf.gain_floor, cf.prune_rel, false, (const cplx<T>*)nullptr, st, res,
                              nullptr, nullptr, 0, pre_grids, pre_ready);
}

void check_sfft_cfg(const sfft2d_sfft_config& cf) {
  const int n = cf.n, b = cf.b_bins, L = cf.loops;
  if (!is_pow2(b) || b > n || n % b) fail(SFFT2D_ERR_CONFIG, "bin count must be a power of 2 dividing n");
  if (L < 1) fail(SFFT2D_ERR_CONFIG, "loops must be >= 1");
  if (cf.vote_threshold < 1 || cf.vote_threshold > L) fail(SFFT2D_ERR_CONFIG, "vote_threshold out of range");
  if (L > kMaxLoops) fail(SFFT2D_ERR_UNSUPPORTED, "more than 64 loops");
  const long long num = std::max(1LL, (long long)cf.d_factor * cf.k);
  if (num > (long long)b * b) fail(SFFT2D_ERR_CONFIG, "d_factor*k exceeds the bin budget");
}

// NaN/Inf scan of x (as_complex_matrix, corefft.py:49-50) whose flag lands in
// pinned[1] with the next synchronisation of `st` (no sync of its own)
template <typename Tin>
void check_finite_async(sfft2d_ctx* c, const Tin* x, long nkeys, cudaStream_t st) {
  unsigned* finite = (unsigned*)ws(c, "finite", 16);
  ck(cudaMemsetAsync(finite, 0, 16, st), "memset");
  pre(c, st);
  kl(k_check_finite<Tin>, grid_for(nkeys, 256, kNumSMs * 8), 256, 0, st, x, nkeys, finite);
  post(c, "k_check_finite", st, (double)nkeys * sizeof(Tin));
  ck(cudaMemcpyAsync(c->pinned + 1, finite, sizeof(unsigned), cudaMemcpyDeviceToHost, st), "D2H");
}

// True when the location fold of these loops goes through k_fold_ml (which
// then checks every sample it reads) and the loops' row windows together
// cover all n rows, so that fold reads every sample of x.  The converted
// value is checked, so a c128 input folded in fp32 keeps the separate scan
// (a finite double can overflow float).
template <typename T, typename Tin>
bool fold_reads_all(const DevTables& tb, int lgb, const Perm* hp, int loops, int n) {
  if (loops < 2 || (1 << lgb) >= 512 || !ml_fold_on()) return false;
  if (sizeof(Tin) == 16 && sizeof(T) == 4) return false;
  std::vector<unsigned char> cov((size_t)n, 0);
  const unsigned maskN = (unsigned)n - 1u;
  for (int l = 0; l < loops; ++l)
    for (int u : tb.nz[lgb]) cov[(hp[l].s1 * (unsigned)u + hp[l].t1) & maskN] = 1;
  for (int r = 0; r < n; ++r)
    if (!cov[r]) return false;
  return true;
}

template <typename Tin>
void check_finite_now(sfft2d_ctx* c, const Tin* x, long nkeys, cudaStream_t st) {
  check_finite_async<Tin>(c, x, nkeys, st);
  ck(cudaStreamSynchronize(st), "sync");
  raise_if_nonfinite(c);
}

// Upload `count` permutations to a named device array; returns (host, device).
std::pair<std::vector<Perm>, Perm*> upload_perms(sfft2d_ctx* c, const char* name,
                                                 const sfft2d_perm* perms, int count, int n,
                                                 cudaStream_t st) {
  std::vector<Perm> hp(std::max(count, 1));
  for (int i = 0; i < count; ++i) hp[i] = to_perm(perms[i], n);
  Perm* dp = (Perm*)ws(c, name, hp.size() * sizeof(Perm));
  Perm* stage = perm_stage(c, std::max(count, 1));
  for (int i = 0; i < count; ++i) stage[i] = hp[i];
  ck(cudaMemcpyAsync(dp, stage, (size_t)count * sizeof(Perm), cudaMemcpyHostToDevice, st),
     "H2D perms");
  ck(cudaEventRecord(c->ev_perm, st), "cudaEventRecord");   // the ring slot is in flight
  return {hp, dp};
}

template <typename T, typename Tin>
void run_sfft(sfft2d_ctx* c, const Tin* x, const sfft2d_sfft_config& cf, const sfft2d_perm* perms,
              cudaStream_t st, sfft2d_result* res) {
  check_sfft_cfg(cf);
  const int L = cf.loops;
  const DevTables& tb = find_tables(c, cf.n, cf.window_delta_pass, cf.window_delta_stop);
  auto up = upload_perms(c, "perms", perms, 2 * L, cf.n, st);
  // the NaN/Inf verdict is read at the first synchronisation (the candidate
  // count); nothing before it leaves the device.  When the location loops'
  // windows together cover every row, the multi-loop fold reads every sample
  // and checks them as it goes; otherwise one k_check_finite pass.
  unsigned* fin = nullptr;
  if (fold_reads_all<T, Tin>(tb, ilog2(cf.b_bins), up.first.data(), L, cf.n)) {
    fin = (unsigned*)ws(c, "finite", 16);
    ck(cudaMemsetAsync(fin, 0, 16, st), "memset");
  } else {
    check_finite_async<Tin>(c, x, (long)cf.n * cf.n, st);
  }
  uint32_t* hist = (uint32_t*)ws(c, "hist", hist_bytes((long)cf.n * cf.n, kVoteAdd8));
  // The estimation loops' permutations are known up front (engine.py:267), so
  // their folds + bucket FFTs do not wait for the candidates: they run on the
  // side stream right after the location fold (both folds are HBM-bound reads
  // of x; back to back they do not share the bandwidth), beside the location
  // phase's latency-bound selection / vote kernels and the candidate-count
  // round trip.  Same grids as the reference's lazy order; they are wasted
  // only when no candidate survives the vote.  SFFT2D_NO_EARLY_EST=1: folded
  // after the candidate count, on the main stream.
  static const bool early_est_on = getenv("SFFT2D_NO_EARLY_EST") == nullptr;
  const bool early_est = early_est_on && !c->profiling;
  struct JoinSide {   // later work on st is ordered after the side stream's, whatever the exit
    sfft2d_ctx* c;
    cudaStream_t st;
    bool on;
    ~JoinSide() {
      if (!on) return;
      cudaEventRecord(c->ev_lmax, c->vote_st);
      cudaStreamWaitEvent(st, c->ev_lmax, 0);
    }
  } join_side{c, st, early_est};
  const int mode = sfft_location<T, Tin>(c, x, cf, tb, up.first.data(), up.second, L, false, hist, st,
                                         fin, early_est ? c->ev_fold[0] : nullptr);
  cplx<T>* pre_grids = nullptr;
  if (early_est) {
    const cudaStream_t side = c->vote_st;
    const size_t BB = (size_t)cf.b_bins * cf.b_bins;
    ck(cudaStreamWaitEvent(side, c->ev_fold[0], 0), "cudaStreamWaitEvent");
    const cudaStream_t ws_saved = c->ws_st;
    c->ws_st = side;
    c->ws_set = 1;   // private workspace: the location phase's buffers stay in set 0
    pre_grids = (cplx<T>*)ws(c, "est_grids", (size_t)L * BB * sizeof(cplx<T>));
    fold_spectrum<T, Tin>(c, x, ilog2(cf.n), ilog2(cf.b_bins), tb, up.first.data() + L, L, pre_grids,
                          (T*)nullptr, nullptr, side, true);
    c->ws_set = 0;
    c->ws_st = ws_saved;
    ck(cudaEventRecord(c->ev_fold[1], side), "cudaEventRecord");
  }
  if (fin)
    ck(cudaMemcpyAsync(c->pinned + 1, fin, sizeof(unsigned), cudaMemcpyDeviceToHost, st), "D2H");
  res->perms_used = 2 * L;
  sfft_from_hist<T, Tin>(c, x, cf, tb, hist, mode, up.first.data() + L, up.second + L, st, res, true,
                         pre_grids, c->ev_fold[1]);
}

template <typename F>
void dispatch(int x_dtype, int prec, F&& f) {
  if (x_dtype != SFFT2D_C64 && x_dtype != SFFT2D_C128) fail(SFFT2D_ERR_VALUE, "unknown x_dtype");
  if (prec != SFFT2D_FP32 && prec != SFFT2D_FP64) fail(SFFT2D_ERR_VALUE, "unknown precision");
  if (prec == SFFT2D_FP64) {
    if (x_dtype == SFFT2D_C64) f(double(), float2());
    else f(double(), double2());
  } else {
    if (x_dtype == SFFT2D_C64) f(float(), float2());
    else f(float(), double2());
  }
}

template <typename F>
void dispatch_prec(int prec, F&& f) {
  if (prec == SFFT2D_FP64) f(double());
  else if (prec == SFFT2D_FP32) f(float());
  else fail(SFFT2D_ERR_VALUE, "unknown precision");
}

const void* stage_input(sfft2d_ctx* c, const void* x, int x_dtype, int x_on_host, int n,
                        cudaStream_t st) {
  if (!x_on_host) return x;
  const size_t bytes = (size_t)n * n * (x_dtype == SFFT2D_C64 ? 8 : 16);
  void* d = ws(c, "x_in", bytes);
  ck(cudaMemcpyAsync(d, x, bytes, cudaMemcpyHostToDevice, st), "H2D x");
  return d;
}

template <typename Fn>
int guarded(sfft2d_ctx* c, Fn&& fn) {
  if (!c) return SFFT2D_ERR_STATE;
  try {
    c->err.clear();
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    fn();
    return SFFT2D_OK;
  } catch (const SfftError& e) {
    c->err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    c->err = e.what();
    return SFFT2D_ERR_CUDA;
  }
}

void check_side(int n) {
  if (!is_pow2(n)) fail(SFFT2D_ERR_VALUE, "side " + std::to_string(n) + " is not a power of 2");
  if (n < 4) fail(SFFT2D_ERR_UNSUPPORTED, "side must be >= 4");
  if ((long long)n * n > (1LL << 30)) fail(SFFT2D_ERR_UNSUPPORTED, "side too large");
}

}  // namespace

// ====================================================================== ABI
extern "C" {

int sfft2d_abi_version(void) { return SFFT2D_ABI_VERSION; }

double sfft2d_ctx_sync_us(const sfft2d_ctx* c) { return c ? c->sync_us : 0.0; }

int sfft2d_ctx_create(int device, sfft2d_ctx** out) {
  if (!out) return SFFT2D_ERR_VALUE;
  *out = nullptr;
  sfft2d_ctx* c = new sfft2d_ctx();
  c->device = device;
  int rc = guarded(c, [&] {
    ck(cudaMallocHost(&c->pinned, 4096), "cudaMallocHost");
    ck(cudaMallocHost(&c->perm_pinned, kPermPinned * sizeof(Perm)), "cudaMallocHost");
    ck(cudaHostAlloc((void**)&c->mapped_h, 16 * kPubSlots, cudaHostAllocMapped), "cudaHostAlloc");
    std::memset(c->mapped_h, 0, 16 * kPubSlots);
    ck(cudaHostGetDevicePointer((void**)&c->mapped_d, c->mapped_h, 0), "cudaHostGetDevicePointer");
    ck(cudaMalloc(&c->done_d, 4 * kPubSlots), "cudaMalloc");
    ck(cudaMemset(c->done_d, 0, 4 * kPubSlots), "cudaMemset");
    ck(cudaStreamCreateWithFlags(&c->vote_st, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreateWithFlags(&c->ev_lmax, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventCreateWithFlags(&c->ev_ws, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventCreateWithFlags(&c->ev_perm, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventCreateWithFlags(&c->ev_fork_votes, cudaEventDisableTiming), "cudaEventCreate");
    for (int i = 0; i < 4; ++i) {
      ck(cudaEventCreateWithFlags(&c->ev_pass[i], cudaEventDisableTiming), "cudaEventCreate");
      ck(cudaEventCreateWithFlags(&c->ev_fold[i], cudaEventDisableTiming), "cudaEventCreate");
    }
    ck(cudaEventRecord(c->ev_perm, 0), "cudaEventRecord");
    // the context's own memory pool, keeping freed workspace (no release at
    // sync points); the device's default pool is left untouched
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    ck(cudaMemPoolCreate(&c->pool, &props), "cudaMemPoolCreate");
    uint64_t keep = UINT64_MAX;
    ck(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep), "cudaMemPoolSetAttribute");
    for (int i = 0; i < 2; ++i)
      ck(cudaEventCreateWithFlags(&c->ev_vote[i], cudaEventDisableTiming), "cudaEventCreate");
  });
  if (rc != SFFT2D_OK) {
    fprintf(stderr, "sfft2d_ctx_create: %s\n", c->err.c_str());
    delete c;
    return rc;
  }
  *out = c;
  return SFFT2D_OK;
}

void sfft2d_ctx_destroy(sfft2d_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  if (!c->arena)
    for (auto& set : c->bufs)
      for (auto& kv : set)
        if (kv.second.first) cudaFreeAsync(kv.second.first, 0);
  cudaDeviceSynchronize();
  if (c->pool) cudaMemPoolDestroy(c->pool);
  for (auto& t : c->tables)
    for (int p = 0; p < 2; ++p) {
      cudaFree(t.space[p]);
      cudaFree(t.freq[p]);
      cudaFree(t.tw[p]);
    }
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->perm_pinned) cudaFreeHost(c->perm_pinned);
  if (c->mapped_h) cudaFreeHost(c->mapped_h);
  if (c->host_out_buf) cudaFreeHost(c->host_out_buf);
  if (c->done_d) cudaFree(c->done_d);
  if (c->vote_st) cudaStreamDestroy(c->vote_st);
  if (c->ev_lmax) cudaEventDestroy(c->ev_lmax);
  if (c->ev_ws) cudaEventDestroy(c->ev_ws);
  if (c->ev_perm) cudaEventDestroy(c->ev_perm);
  if (c->ev_fork_votes) cudaEventDestroy(c->ev_fork_votes);
  for (int i = 0; i < 4; ++i) {
    if (c->ev_pass[i]) cudaEventDestroy(c->ev_pass[i]);
    if (c->ev_fold[i]) cudaEventDestroy(c->ev_fold[i]);
  }
  for (int i = 0; i < 2; ++i)
    if (c->ev_vote[i]) cudaEventDestroy(c->ev_vote[i]);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  delete c;
}

const char* sfft2d_ctx_last_error(const sfft2d_ctx* c) { return c ? c->err.c_str() : "null context"; }

int sfft2d_ctx_set_tables(sfft2d_ctx* c, int n, double dpass, double dstop, const double* space,
                          const double* freq, const double* twiddle) {
  return guarded(c, [&] {
    check_side(n);
    if (!space || !freq || !twiddle) fail(SFFT2D_ERR_VALUE, "null table");
    for (auto& t : c->tables)
      if (t.n == n && t.dpass == dpass && t.dstop == dstop) return;  // already registered
    DevTables t;
    t.n = n;
    t.lgn = ilog2(n);
    t.dpass = dpass;
    t.dstop = dstop;
    const size_t rows = (size_t)(t.lgn + 1) * n;
    std::vector<float> f32(std::max(rows, (size_t)2 * n));
    auto up = [&](const double* src, size_t cnt, void** d64, void** d32) {
      ck(cudaMalloc(d64, cnt * 8), "cudaMalloc");
      ck(cudaMemcpy(*d64, src, cnt * 8, cudaMemcpyHostToDevice), "H2D table");
      for (size_t i = 0; i < cnt; ++i) f32[i] = (float)src[i];
      ck(cudaMalloc(d32, cnt * 4), "cudaMalloc");
      ck(cudaMemcpy(*d32, f32.data(), cnt * 4, cudaMemcpyHostToDevice), "H2D table");
    };
    up(space, rows, &t.space[SFFT2D_FP64], &t.space[SFFT2D_FP32]);
    up(freq, rows, &t.freq[SFFT2D_FP64], &t.freq[SFFT2D_FP32]);
    up(twiddle, (size_t)2 * n, &t.tw[SFFT2D_FP64], &t.tw[SFFT2D_FP32]);
    t.support.assign(t.lgn + 1, n);
    t.nz.assign(t.lgn + 1, {});
    for (int lb = 0; lb <= t.lgn; ++lb) {
      for (int i = 0; i < n; ++i)
        if (space[(size_t)lb * n + i] != 0.0) t.nz[lb].push_back(i);
      t.support[lb] = (int)t.nz[lb].size();
    }
    t.conv_r.assign(t.lgn + 1, 0);
    for (int lb = 1; lb < t.lgn; ++lb) {
      if (t.support[lb] != n) continue;
      const double* f = freq + (size_t)lb * n;
      int r = 0;
      for (int d = 1; d <= n / 2; ++d)
        if (std::fabs(f[d]) > 1e-14 * std::fabs(f[0]) || std::fabs(f[n - d]) > 1e-14 * std::fabs(f[0])) r = d;
      t.conv_r[lb] = (r >= 1 && r <= 4) ? r : 0;
    }
    c->tables.push_back(t);
  });
}

int sfft2d_ctx_set_profiling(sfft2d_ctx* c, int enable) {
  return guarded(c, [&] {
    c->profiling = enable != 0;
    c->prof.clear();
    c->ev_used = 0;
    c->prof_open = false;
  });
}

int64_t sfft2d_ctx_profile_report(sfft2d_ctx* c, char* buf, int64_t buflen) {
  std::string out;
  int rc = guarded(c, [&] {
    ck(cudaDeviceSynchronize(), "sync");
    std::map<std::string, std::pair<long long, std::pair<double, double>>> agg;
    for (auto& r : c->prof) {
      if (!r.name || !r.b) continue;
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, r.a, r.b), "cudaEventElapsedTime");
      auto& e = agg[r.name];
      e.first += 1;
      e.second.first += ms;
      e.second.second += r.bytes;
    }
    for (auto& kv : agg) {
      char line[256];
      snprintf(line, sizeof(line), "%s %lld %.6f %.0f\n", kv.first.c_str(), kv.second.first,
               kv.second.second.first, kv.second.second.second);
      out += line;
    }
    c->prof.clear();
    c->ev_used = 0;
    c->prof_open = false;
  });
  if (rc != SFFT2D_OK) return rc;
  if (buf && buflen > 0) {
    const size_t n = std::min<size_t>(out.size(), (size_t)buflen - 1);
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return (int64_t)out.size();
}

int sfft2d_sfft(sfft2d_ctx* c, const void* x, int x_dtype, int x_on_host,
                const sfft2d_sfft_config* cfg, const sfft2d_perm* perms, int precision,
                void* stream, sfft2d_result* res) {
  return guarded(c, [&] {
    if (!cfg || !perms || !res || !x) fail(SFFT2D_ERR_VALUE, "null argument");
    check_side(cfg->n);
    cudaStream_t st = (cudaStream_t)stream;
    c->ws_st = st;
    std::memset(res, 0, sizeof(*res));
    c->launches = 0;
    c->has_res = false;
    const void* xd = stage_input(c, x, x_dtype, x_on_host, cfg->n, st);
    dispatch(x_dtype, precision, [&](auto t, auto tin) {
      using T = decltype(t);
      using Tin = decltype(tin);
      run_sfft<T, Tin>(c, (const Tin*)xd, *cfg, perms, st, res);
    });
    res->precision = precision;
    res->gpu_launches = c->launches;
    c->res_prec = precision;
    c->has_res = true;
  });
}

int sfft2d_sfft_draw_perms(void* numpy_bitgen, int n, int loops, sfft2d_perm* out) {
  if (!numpy_bitgen || !out || loops < 1 || !is_pow2(n)) return SFFT2D_ERR_VALUE;
  try {
    sfft_child_perms(numpy_bitgen, n, loops, out);
  } catch (...) {
    return SFFT2D_ERR_VALUE;
  }
  return SFFT2D_OK;
}

int sfft2d_sfft_bitgen(sfft2d_ctx* c, const void* x, int x_dtype, int x_on_host,
                       const sfft2d_sfft_config* cfg, void* numpy_bitgen, int precision,
                       void* stream, sfft2d_result* res) {
  if (!cfg || !numpy_bitgen || cfg->loops < 1 || cfg->loops > kMaxLoops) return SFFT2D_ERR_VALUE;
  std::vector<sfft2d_perm> perms(2 * cfg->loops);
  if (is_pow2(cfg->n)) sfft_child_perms(numpy_bitgen, cfg->n, cfg->loops, perms.data());
  return sfft2d_sfft(c, x, x_dtype, x_on_host, cfg, perms.data(), precision, stream, res);
}

static int atsfft_impl(sfft2d_ctx* c, const void* x, int x_dtype, int x_on_host, int n,
                       const sfft2d_tuner_config* cfg, int est_loops, const sfft2d_perm* perms,
                       int n_perms, void* bitgen, int precision, void* stream, sfft2d_result* res,
                       sfft2d_tuner_state* state) {
  return guarded(c, [&] {
    c->t_entry = std::chrono::steady_clock::now();
    if (!cfg || !res || !state || !x || (n_perms > 0 && !perms)) fail(SFFT2D_ERR_VALUE, "null argument");
    check_side(n);
    cudaStream_t st = (cudaStream_t)stream;
    c->ws_st = st;
    std::memset(res, 0, sizeof(*res));
    c->launches = 0;
    c->sync_us = 0;
    c->has_res = false;
    const void* xd = stage_input(c, x, x_dtype, x_on_host, n, st);
    dispatch(x_dtype, precision, [&](auto t, auto tin) {
      using T = decltype(t);
      using Tin = decltype(tin);
      run_ats<T, Tin>(c, (const Tin*)xd, n, *cfg, est_loops, perms, n_perms, bitgen, st, true, res,
                      state);
    });
    res->precision = precision;
    res->gpu_launches = c->launches;
    c->res_prec = precision;
    c->has_res = true;
    if (getenv("SFFT2D_TRACE_HOST")) {
      const auto now = std::chrono::steady_clock::now();
      fprintf(stderr, "[sfft2d] entry->first launch %.1f us, last sync->return %.1f us, total %.1f us\n",
              c->first_launch_us,
              std::chrono::duration<double, std::micro>(now - c->t_sync_end).count(),
              std::chrono::duration<double, std::micro>(now - c->t_entry).count());
    }
  });
}

static int detect_impl(sfft2d_ctx* c, const void* x, int x_dtype, int x_on_host, int n,
                       const sfft2d_tuner_config* cfg, const sfft2d_perm* perms, int n_perms,
                       void* bitgen, int precision, void* stream, sfft2d_tuner_state* state) {
  return guarded(c, [&] {
    if (!cfg || !state || !x || (n_perms > 0 && !perms)) fail(SFFT2D_ERR_VALUE, "null argument");
    check_side(n);
    cudaStream_t st = (cudaStream_t)stream;
    c->ws_st = st;
    c->launches = 0;
    c->has_votes = false;
    const void* xd = stage_input(c, x, x_dtype, x_on_host, n, st);
    sfft2d_result dummy;
    std::memset(&dummy, 0, sizeof(dummy));
    dispatch(x_dtype, precision, [&](auto t, auto tin) {
      using T = decltype(t);
      using Tin = decltype(tin);
      run_ats<T, Tin>(c, (const Tin*)xd, n, *cfg, 0, perms, n_perms, bitgen, st, false, &dummy,
                      state);
    });
  });
}

int sfft2d_sfft_votes(sfft2d_ctx* c, const void* x, int x_dtype, int x_on_host,
                      const sfft2d_sfft_config* cfg, const sfft2d_perm* perms, int nloops,
                      int precision, void* stream, void* counts) {
  return guarded(c, [&] {
    if (!cfg || !perms || !x || !counts || nloops < 1) fail(SFFT2D_ERR_VALUE, "bad arguments");
    check_side(cfg->n);
    check_sfft_cfg(*cfg);
    if (nloops > cfg->loops) fail(SFFT2D_ERR_VALUE, "more loops than the configuration");
    cudaStream_t st = (cudaStream_t)stream;
    c->ws_st = st;
    c->launches = 0;
    const void* xd = stage_input(c, x, x_dtype, x_on_host, cfg->n, st);
    const DevTables& tb = find_tables(c, cfg->n, cfg->window_delta_pass, cfg->window_delta_stop);
    auto up = upload_perms(c, "perms", perms, nloops, cfg->n, st);
    dispatch(x_dtype, precision, [&](auto t, auto tin) {
      using T = decltype(t);
      using Tin = decltype(tin);
      check_finite_now<Tin>(c, (const Tin*)xd, (long)cfg->n * cfg->n, st);
      sfft_location<T, Tin>(c, (const Tin*)xd, *cfg, tb, up.first.data(), up.second, nloops, true,
                            (uint32_t*)counts, st);
    });
  });
}

int sfft2d_sfft_from_votes(sfft2d_ctx* c, const void* x, int x_dtype, int x_on_host,
                           const sfft2d_sfft_config* cfg, const void* counts,
                           const sfft2d_perm* est_perms, int precision, void* stream,
                           sfft2d_result* res) {
  return guarded(c, [&] {
    if (!cfg || !est_perms || !x || !counts || !res) fail(SFFT2D_ERR_VALUE, "bad arguments");
    check_side(cfg->n);
    check_sfft_cfg(*cfg);
    cudaStream_t st = (cudaStream_t)stream;
    c->ws_st = st;
    std::memset(res, 0, sizeof(*res));
    c->launches = 0;
    c->has_res = false;
    const void* xd = stage_input(c, x, x_dtype, x_on_host, cfg->n, st);
    const DevTables& tb = find_tables(c, cfg->n, cfg->window_delta_pass, cfg->window_delta_stop);
    auto up = upload_perms(c, "perms_est", est_perms, cfg->loops, cfg->n, st);
    dispatch(x_dtype, precision, [&](auto t, auto tin) {
      using T = decltype(t);
      using Tin = decltype(tin);
      sfft_from_hist<T, Tin>(c, (const Tin*)xd, *cfg, tb, (const uint32_t*)counts, kVoteAdd8,
                             up.first.data(), up.second, st, res);
    });
    res->precision = precision;
    res->gpu_launches = c->launches;
    c->res_prec = precision;
    c->has_res = true;
  });
}

// Estimation loops for caller-given candidates, and the median/selection over
// gathered per-loop estimates: the two halves of engine.py:163-253 as separate
// entry points, so ranks can split the estimation loops (distributed.py).
int sfft2d_estimate_loops(sfft2d_ctx* c, const void* x, int x_dtype, int x_on_host, int n, int b,
                          double delta_pass, double delta_stop, double gain_floor,
                          const int32_t* keys, int64_t m, const sfft2d_perm* perms, int nloops,
                          int precision, void* stream, void* vals, uint8_t* usable) {
  return guarded(c, [&] {
    if (!x || !keys || !perms || !vals || !usable || m < 0 || nloops < 1)
      fail(SFFT2D_ERR_VALUE, "bad arguments");
    check_side(n);
    if (!is_pow2(b) || b > n || n % b) fail(SFFT2D_ERR_CONFIG, "bin count must be a power of 2 dividing n");
    if (nloops > kMaxFoldLoops * 8) fail(SFFT2D_ERR_UNSUPPORTED, "too many estimation loops");
    if (m == 0) return;
    cudaStream_t st = (cudaStream_t)stream;
    c->ws_st = st;
    c->launches = 0;
    const void* xd = stage_input(c, x, x_dtype, x_on_host, n, st);
    const DevTables& tb = find_tables(c, n, delta_pass, delta_stop);
    auto up = upload_perms(c, "perms_estl", perms, nloops, n, st);
    unsigned* m_dev = (unsigned*)ws(c, "estl_m", 16);
    const unsigned m32 = (unsigned)m;
    ck(cudaMemcpyAsync(m_dev, &m32, 4, cudaMemcpyHostToDevice, st), "H2D m");
    const int lgN = ilog2(n), lgB = ilog2(b);
    dispatch(x_dtype, precision, [&](auto t, auto tin) {
      using T = decltype(t);
      using Tin = decltype(tin);
      using C = cplx<T>;
      const int P = prec_of<T>();
      const size_t BB = (size_t)b * b;
      C* grids = (C*)ws(c, "est_grids", (size_t)nloops * BB * sizeof(C));
      fold_spectrum<T, Tin>(c, (const Tin*)xd, lgN, lgB, tb, up.first.data(), nloops, grids,
                            (T*)nullptr, nullptr, st, true);
      const T* freq = (const T*)tb.freq[P] + ((size_t)lgB << lgN);
      pre(c, st);
      kl(k_estimate<T>, grid_for((long long)m * nloops), 256, 0, st, (const C*)grids, nloops, keys,
         (const unsigned*)m_dev, (const Perm*)up.second, lgN, lgB, freq, (const C*)tb.tw[P],
         gain_floor, (C*)vals, usable, (long)m, true);
      post(c, "k_estimate", st, 0);
    });
    ck(cudaStreamSynchronize(st), "sync");
  });
}

int sfft2d_median_select(sfft2d_ctx* c, int n, const int32_t* keys, int64_t m, const void* vals,
                         const uint8_t* usable, int nloops, int64_t k, double prune_rel,
                         int precision, void* stream, sfft2d_result* res) {
  return guarded(c, [&] {
    if (!keys || !vals || !usable || !res || m < 0 || nloops < 1) fail(SFFT2D_ERR_VALUE, "bad arguments");
    if (nloops > kMaxLoops) fail(SFFT2D_ERR_UNSUPPORTED, "more than 64 estimation loops");
    check_side(n);
    cudaStream_t st = (cudaStream_t)stream;
    c->ws_st = st;
    std::memset(res, 0, sizeof(*res));
    c->launches = 0;
    c->has_res = false;
    c->res_count = 0;
    if (m > 0) {
      unsigned* m_dev = (unsigned*)ws(c, "msel_m", 16);
      const unsigned m32 = (unsigned)m;
      ck(cudaMemcpyAsync(m_dev, &m32, 4, cudaMemcpyHostToDevice, st), "H2D m");
      dispatch_prec(precision, [&](auto t) {
        using T = decltype(t);
        using C = cplx<T>;
        C* med = (C*)ws(c, "med", (size_t)m * sizeof(C));
        T* mags = (T*)ws(c, "emag", (size_t)m * sizeof(T));
        uint8_t* alive = (uint8_t*)ws(c, "alive", (size_t)m);
        unsigned long long* peak = (unsigned long long*)ws(c, "epeak", 16);
        unsigned* alive_cnt = (unsigned*)ws(c, "ealive", 16);
        ck(cudaMemsetAsync(peak, 0, 16, st), "memset");
        ck(cudaMemsetAsync(alive_cnt, 0, 16, st), "memset");
        pre(c, st);
        kl(k_median<T>, grid_for(m, 128), 128, 0, st, (const C*)vals, usable, nloops, (long)m,
           (const unsigned*)m_dev, med, mags, alive, alive_cnt, peak);
        post(c, "k_median", st, 0);
        const long long n_alive = read_u32(c, alive_cnt, st);
        res->n_candidates = m;
        finish_select<T>(c, ilog2(n), keys, (unsigned)m, k, prune_rel, med, mags, alive, peak,
                         n_alive, st, res);
      });
    }
    res->precision = precision;
    res->gpu_launches = c->launches;
    c->res_prec = precision;
    c->has_res = true;
  });
}

int sfft2d_atsfft(sfft2d_ctx* c, const void* x, int x_dtype, int x_on_host, int n,
                  const sfft2d_tuner_config* cfg, int est_loops, const sfft2d_perm* perms,
                  int n_perms, int precision, void* stream, sfft2d_result* res,
                  sfft2d_tuner_state* state) {
  return atsfft_impl(c, x, x_dtype, x_on_host, n, cfg, est_loops, perms, n_perms, nullptr,
                     precision, stream, res, state);
}

int sfft2d_atsfft_bitgen(sfft2d_ctx* c, const void* x, int x_dtype, int x_on_host, int n,
                         const sfft2d_tuner_config* cfg, int est_loops, void* numpy_bitgen,
                         int precision, void* stream, sfft2d_result* res,
                         sfft2d_tuner_state* state) {
  if (!numpy_bitgen) return SFFT2D_ERR_VALUE;
  return atsfft_impl(c, x, x_dtype, x_on_host, n, cfg, est_loops, nullptr, 0, numpy_bitgen,
                     precision, stream, res, state);
}

int sfft2d_detect_sparsity(sfft2d_ctx* c, const void* x, int x_dtype, int x_on_host, int n,
                           const sfft2d_tuner_config* cfg, const sfft2d_perm* perms, int n_perms,
                           int precision, void* stream, sfft2d_tuner_state* state) {
  return detect_impl(c, x, x_dtype, x_on_host, n, cfg, perms, n_perms, nullptr, precision, stream,
                     state);
}

int sfft2d_detect_sparsity_bitgen(sfft2d_ctx* c, const void* x, int x_dtype, int x_on_host, int n,
                                  const sfft2d_tuner_config* cfg, void* numpy_bitgen,
                                  int precision, void* stream, sfft2d_tuner_state* state) {
  if (!numpy_bitgen) return SFFT2D_ERR_VALUE;
  return detect_impl(c, x, x_dtype, x_on_host, n, cfg, nullptr, 0, numpy_bitgen, precision, stream,
                     state);
}

int sfft2d_fetch_result(sfft2d_ctx* c, int64_t* ij, void* values, int dst_on_host, void* stream) {
  return guarded(c, [&] {
    if (!c->has_res) fail(SFFT2D_ERR_STATE, "no transform result to fetch");
    cudaStream_t st = (cudaStream_t)stream;
    c->ws_st = st;
    const size_t n = (size_t)c->res_count;
    if (n == 0) return;
    const size_t vb = n * (c->res_prec == SFFT2D_FP64 ? 16 : 8);
    // results already sit in mapped host memory (written by k_gather_out)
    if (dst_on_host) {
      if (ij) std::memcpy(ij, c->out_ij_h, n * 16);
      if (values) std::memcpy(values, c->out_v_h, vb);
    } else {
      if (ij) ck(cudaMemcpyAsync(ij, c->out_ij_h, n * 16, cudaMemcpyDefault, st), "copy ij");
      if (values) ck(cudaMemcpyAsync(values, c->out_v_h, vb, cudaMemcpyDefault, st), "copy v");
    }
  });
}

int sfft2d_fetch_votes(sfft2d_ctx* c, int32_t* keys, int32_t* tallies, int dst_on_host,
                       void* stream) {
  return guarded(c, [&] {
    if (!c->has_votes) fail(SFFT2D_ERR_STATE, "no detection votes to fetch");
    cudaStream_t st = (cudaStream_t)stream;
    c->ws_st = st;
    const size_t n = (size_t)c->votes_count;
    if (n == 0) return;
    if (keys) ck(cudaMemcpyAsync(keys, ws(c, "keys", n * 4), n * 4, cudaMemcpyDefault, st), "copy keys");
    if (tallies)
      ck(cudaMemcpyAsync(tallies, ws(c, "tallies", n * 4), n * 4, cudaMemcpyDefault, st), "copy tallies");
    if (dst_on_host) ck(cudaStreamSynchronize(st), "sync");
  });
}

int sfft2d_binned_spectrum(sfft2d_ctx* c, const void* x, int x_dtype, int n, int b,
                           const sfft2d_perm* perms, int nloops, double dpass, double dstop,
                           int precision, void* out, void* stream) {
  return guarded(c, [&] {
    check_side(n);
    if (!is_pow2(b) || b > n || b < 4) fail(SFFT2D_ERR_VALUE, "bin count must be a power of 2 in [4, n]");
    if (nloops < 1 || !perms || !x || !out) fail(SFFT2D_ERR_VALUE, "bad arguments");
    const DevTables& tb = find_tables(c, n, dpass, dstop);
    std::vector<Perm> hp(nloops);
    for (int i = 0; i < nloops; ++i) hp[i] = to_perm(perms[i], n);
    cudaStream_t st = (cudaStream_t)stream;
    c->ws_st = st;
    c->launches = 0;
    dispatch(x_dtype, precision, [&](auto t, auto tin) {
      using T = decltype(t);
      using Tin = decltype(tin);
      fold_spectrum<T, Tin>(c, (const Tin*)x, ilog2(n), ilog2(b), tb, hp.data(), nloops,
                            (cplx<T>*)out, (T*)nullptr, nullptr, st);
    });
  });
}

int sfft2d_fft2d(sfft2d_ctx* c, void* grids, int b, int count, int n_table, int precision,
                 void* stream) {
  return guarded(c, [&] {
    if (!is_pow2(b) || b < 2 || b > n_table) fail(SFFT2D_ERR_VALUE, "bad grid side");
    const DevTables& tb = find_twiddles(c, n_table);
    cudaStream_t st = (cudaStream_t)stream;
    c->ws_st = st;
    dispatch_prec(precision, [&](auto t) {
      using T = decltype(t);
      fft2d_grids<T>(c, (cplx<T>*)grids, ilog2(b), count, (const cplx<T>*)tb.tw[prec_of<T>()],
                     tb.lgn, (cplx<T>*)grids, (T*)nullptr, nullptr, st);
    });
  });
}

int sfft2d_local_maxima(sfft2d_ctx* c, const void* grid, int b, double mag_floor, int precision,
                        int64_t* count, int32_t* out_flat, int64_t capacity, void* stream) {
  return guarded(c, [&] {
    if (b < 4 || b > 65536) fail(SFFT2D_ERR_VALUE, "bin grid must be at least 4x4");
    cudaStream_t st = (cudaStream_t)stream;
    c->ws_st = st;
    dispatch_prec(precision, [&](auto t) {
      using T = decltype(t);
      const long BB = (long)b * b;
      T* mg = (T*)ws(c, "api_mag", BB * sizeof(T));
      unsigned long long* pk = (unsigned long long*)ws(c, "api_peak", 16);
      ck(cudaMemsetAsync(pk, 0, 16, st), "memset");
      pre(c, st);
      kl(k_mags<T>, dim3(grid_for(BB, 256, 1024), 1), 256, 0, st, (const cplx<T>*)grid, BB, mg, pk);
      post(c, "k_mags", st, 0);
      int32_t* tmp = (int32_t*)ws(c, "api_lm", (size_t)(BB / 4 + 64) * 4);
      long long cnt;
      if (is_pow2(b)) {
        cnt = local_maxima_dev<T>(c, mg, ilog2(b), pk, mag_floor, tmp, st);
      } else {
        // any square grid (tuner.py:97-118 accepts every side >= 4)
        const int nblk = blocks_for(BB);
        uint32_t* bits = (uint32_t*)ws(c, "lm_bits", words_for(BB) * 4);
        unsigned* cnts = (unsigned*)ws(c, "lm_cnt", (size_t)nblk * 4);
        unsigned* tot = (unsigned*)ws(c, "lm_tot", 16);
        pre(c, st);
        kl(k_lmax_bits_any<T>, dim3(nblk, 1), kCmpThreads, 0, st, (const T*)mg, b, (const unsigned long long*)pk,
           mag_floor, bits, cnts);
        post(c, "k_lmax_bits_any", st, (double)BB * sizeof(T) + BB / 8.0);
        compact(c, bits, cnts, BB, 1, tmp, 0, tot, st);
        cnt = read_u32(c, tot, st);
      }
      if (count) *count = cnt;
      const long long cp = std::min<long long>(cnt, capacity);
      if (out_flat && cp > 0)
        ck(cudaMemcpyAsync(out_flat, tmp, (size_t)cp * 4, cudaMemcpyDefault, st), "copy");
    });
  });
}

int sfft2d_top_bins(sfft2d_ctx* c, const void* grids, int b, int nseg, int64_t num, int precision,
                    int32_t* out_flat, void* stream) {
  return guarded(c, [&] {
    if (!is_pow2(b) || b < 1 || nseg < 1 || num < 1 || !out_flat) fail(SFFT2D_ERR_VALUE, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    c->ws_st = st;
    dispatch_prec(precision, [&](auto t) {
      using T = decltype(t);
      const long BB = (long)b * b;
      if (num > BB) fail(SFFT2D_ERR_VALUE, "num exceeds the number of bins");
      T* mg = (T*)ws(c, "api_mag", (size_t)nseg * BB * sizeof(T));
      pre(c, st);
      kl(k_mags<T>, dim3(grid_for(BB, 256, 1024), nseg), 256, 0, st, (const cplx<T>*)grids, BB, mg,
                                                                     nullptr);
      post(c, "k_mags", st, 0);
      if (num >= BB) {
        pre(c, st);
        kl(k_iota_segments, grid_for(BB * nseg), 256, 0, st, out_flat, BB, nseg);
        post(c, "k_iota_segments", st, 0);
        return;
      }
      const int nblk = blocks_for(BB);
      uint32_t* sb = (uint32_t*)ws(c, "api_selbits", (size_t)nseg * words_for(BB) * 4);
      unsigned* sc = (unsigned*)ws(c, "api_selcnt", (size_t)nseg * nblk * 4);
      topk_bits<T>(c, mg, BB, nseg, num, sb, sc, st);
      unsigned* tots = (unsigned*)ws(c, "api_tot", (size_t)nseg * 4 + 16);
      compact(c, sb, sc, BB, nseg, out_flat, (long)num, tots, st);
    });
  });
}

int sfft2d_ctx_set_workspace(sfft2d_ctx* c, void* base, int64_t bytes) {
  return guarded(c, [&] {
    if (bytes < 0 || (bytes > 0 && !base)) fail(SFFT2D_ERR_VALUE, "bad workspace");
    ck(cudaDeviceSynchronize(), "sync");   // nothing may still use the old buffers
    for (auto& set : c->bufs)
      for (auto& kv : set)
        if (kv.second.first && !c->arena) ck(cudaFreeAsync(kv.second.first, 0), "cudaFreeAsync");
    ck(cudaDeviceSynchronize(), "sync");
    for (auto& set : c->bufs) set.clear();
    c->arena_free.clear();
    c->ws_in_use = 0;
    c->ws_peak = 0;
    c->arena = (char*)base;
    c->arena_bytes = base ? (size_t)bytes : 0;
    if (c->arena) {
      // 256-byte aligned start (every named buffer is a multiple of 4 KiB)
      const size_t skew = (256 - ((uintptr_t)c->arena & 255)) & 255;
      if (c->arena_bytes > skew) c->arena_free.emplace(skew, c->arena_bytes - skew);
    }
  });
}

int sfft2d_ctx_workspace_size(const sfft2d_ctx* c, int64_t* in_use, int64_t* peak) {
  if (!c) return SFFT2D_ERR_STATE;
  if (in_use) *in_use = (int64_t)c->ws_in_use;
  if (peak) *peak = (int64_t)c->ws_peak;
  return SFFT2D_OK;
}

int sfft2d_generate(sfft2d_ctx* c, int n, int64_t k, const int64_t* rows, const int64_t* cols,
                    const double* coeffs, double noise_sd, uint64_t noise_seed, int out_dtype,
                    void* out, void* stream) {
  return guarded(c, [&] {
    check_side(n);
    if (!out || k < 0 || (k > 0 && (!rows || !cols || !coeffs)) || (long long)k > (long long)n * n)
      fail(SFFT2D_ERR_VALUE, "bad arguments");
    if (!(noise_sd >= 0.0) || !std::isfinite(noise_sd)) fail(SFFT2D_ERR_VALUE, "noise sd must be finite and >= 0");
    for (int64_t i = 0; i < k; ++i)
      if (rows[i] < 0 || rows[i] >= n || cols[i] < 0 || cols[i] >= n)
        fail(SFFT2D_ERR_VALUE, "coefficient position outside the image");
    const DevTables& tb = find_twiddles(c, n);
    cudaStream_t st = (cudaStream_t)stream;
    c->ws_st = st;
    c->launches = 0;
    const int lgN = ilog2(n);
    const long total = (long)n * n;
    auto run = [&](auto t) {
      using T = decltype(t);
      using C = cplx<T>;
      C* g = (C*)out;
      ck(cudaMemsetAsync(g, 0, (size_t)total * sizeof(C), st), "memset");
      if (k > 0) {
        char* buf = (char*)ws(c, "gen_coef", (size_t)k * 32);
        ck(cudaMemcpyAsync(buf, rows, (size_t)k * 8, cudaMemcpyHostToDevice, st), "H2D rows");
        ck(cudaMemcpyAsync(buf + (size_t)k * 8, cols, (size_t)k * 8, cudaMemcpyHostToDevice, st), "H2D cols");
        ck(cudaMemcpyAsync(buf + (size_t)k * 16, coeffs, (size_t)k * 16, cudaMemcpyHostToDevice, st),
           "H2D coeffs");
        pre(c, st);
        kl(k_gen_scatter<T>, (unsigned)((k + 255) / 256), 256, 0, st, g, lgN, (const int64_t*)buf,
           (const int64_t*)(buf + (size_t)k * 8), (const double2*)(buf + (size_t)k * 16), (int)k);
        post(c, "k_gen_scatter", st, (double)k * 32);
        fft2d_grids<T>(c, g, lgN, 1, (const C*)tb.tw[prec_of<T>()], tb.lgn, g, (T*)nullptr, nullptr, st);
      }
      pre(c, st);
      kl(k_gen_finish<T>, grid_for(total, 256, kNumSMs * 8), 256, 0, st, g, total,
         1.0 / ((double)n * (double)n), noise_sd, (uint32_t)noise_seed, (uint32_t)(noise_seed >> 32));
      post(c, "k_gen_finish", st, 2.0 * total * sizeof(C));
    };
    if (out_dtype == SFFT2D_C64) run(float());
    else if (out_dtype == SFFT2D_C128) run(double());
    else fail(SFFT2D_ERR_VALUE, "unknown out_dtype");
  });
}

}  // extern "C"
