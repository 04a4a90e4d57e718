// K3 / K4 — bin selection.
//
//  * magnitudes |Z| (np.abs == hypot) with a per-segment peak (atomicMax on an
//    order-preserving integer key — exact, order independent);
//  * K4 local maxima (count_local_maxima, tuner.py:97-118): strict ">" against
//    the 8 toroidal neighbours and ">= mag_floor * peak", peak > 0;
//  * ordered stream compaction (bitmask + per-block counts + scan + scatter)
//    so every emitted list is in ascending flat (row-major) order, like
//    np.argwhere / np.unique;
//  * K3 exact top-`num` selection (engine.py:122-127 stable argsort): MSB-first
//    radix select on the magnitude key finds the threshold key T and how many
//    ties at T to keep; ties are kept lowest-index first.
//
// Everything is segmented: `nseg` independent equal-length segments (e.g. the
// L location loops' grids) are processed by one launch (gridDim.y = segment).
#pragma once
#include "common.cuh"
#include "mags.cuh"

namespace sfft {

constexpr int kCmpThreads = 256;                 // threads per compaction block
constexpr int kCmpWords = kCmpThreads;           // one 32-bit word per thread
constexpr int kCmpElems = kCmpWords * 32;        // 8192 elements per block

__host__ __device__ inline long words_for(long n) { return (n + 31) / 32; }
__host__ __device__ inline int blocks_for(long n) { return (int)((words_for(n) + kCmpWords - 1) / kCmpWords); }

// ---------------------------------------------------------------- local maxima
template <typename T>
__global__ void k_lmax_bits(const T* __restrict__ mags, int lgB, int nseg_stride_log /*unused*/,
                            const unsigned long long* __restrict__ peak, double floor_rel,
                            uint32_t* __restrict__ bits, unsigned* __restrict__ blk_counts) {
  pdl_wait();
  const int seg = blockIdx.y;
  const int B = 1 << lgB;
  const long BB = (long)B * B;
  const T* m = mags + (size_t)seg * BB;
  const long wps = words_for(BB);
  uint32_t* sb = bits + (size_t)seg * wps;
  const double pk = fkey_inv(peak[seg]);
  const bool live = pk > 0.0;
  const double fl = floor_rel * pk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long w0 = (long)blockIdx.x * kCmpWords + warp * 32;
  unsigned cnt = 0;
  const unsigned maskB = (unsigned)B - 1u;
  for (int i = 0; i < 32; ++i) {
    const long w = w0 + i;
    const long e = w * 32 + lane;
    bool f = false;
    if (live && e < BB) {
      const unsigned r = (unsigned)(e >> lgB), c = (unsigned)(e & maskB);
      const T v = m[e];
      if ((double)v >= fl) {
        const unsigned rm = (r - 1u) & maskB, rp = (r + 1u) & maskB;
        const unsigned cm = (c - 1u) & maskB, cp = (c + 1u) & maskB;
        f = v > m[(rm << lgB) | cm] && v > m[(rm << lgB) | c] && v > m[(rm << lgB) | cp] &&
            v > m[(r << lgB) | cm] && v > m[(r << lgB) | cp] && v > m[(rp << lgB) | cm] &&
            v > m[(rp << lgB) | c] && v > m[(rp << lgB) | cp];
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0 && w < wps) sb[w] = bal;
    cnt += __popc(bal);
  }
  __shared__ unsigned s_cnt[kCmpThreads / 32];
  if (lane == 0) s_cnt[warp] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int i = 0; i < kCmpThreads / 32; ++i) t += s_cnt[i];
    blk_counts[(size_t)seg * gridDim.x + blockIdx.x] = t;
  }
}

// Local maxima of a B x B grid of ANY side B >= 4 (the public
// count_local_maxima accepts every square grid, tuner.py:97-118; the tuner's
// own grids are powers of two and use the kernels above/below).  Same bit /
// block-count layout as k_lmax_bits, toroidal neighbours by modulo.
template <typename T>
__global__ void k_lmax_bits_any(const T* __restrict__ m, int B,
                                const unsigned long long* __restrict__ peak, double floor_rel,
                                uint32_t* __restrict__ bits, unsigned* __restrict__ blk_counts) {
  pdl_wait();
  const long BB = (long)B * B;
  const long wps = words_for(BB);
  const double pk = fkey_inv(peak[0]);
  const bool live = pk > 0.0;
  const double fl = floor_rel * pk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long w0 = (long)blockIdx.x * kCmpWords + warp * 32;
  unsigned cnt = 0;
  for (int i = 0; i < 32; ++i) {
    const long w = w0 + i;
    const long e = w * 32 + lane;
    bool f = false;
    if (live && e < BB) {
      const long r = e / B, c = e - r * B;
      const T v = m[e];
      if ((double)v >= fl) {
        const long rm = (r + B - 1) % B * B, r0 = r * B, rp = (r + 1) % B * B;
        const long cm = (c + B - 1) % B, cp = (c + 1) % B;
        f = v > m[rm + cm] && v > m[rm + c] && v > m[rm + cp] && v > m[r0 + cm] &&
            v > m[r0 + cp] && v > m[rp + cm] && v > m[rp + c] && v > m[rp + cp];
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0 && w < wps) bits[w] = bal;
    cnt += __popc(bal);
  }
  __shared__ unsigned s_cnt[kCmpThreads / 32];
  if (lane == 0) s_cnt[warp] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int i = 0; i < kCmpThreads / 32; ++i) t += s_cnt[i];
    blk_counts[blockIdx.x] = t;
  }
}

// Tiled local maxima: CTA = `rb` output rows of the B x B magnitude grid
//   G[r][c] = M[(s1*r) mod B][(s2*c) mod B]      (s1 = s2 = 1 for a plain grid)
// The rb + 2 SOURCE rows it needs (one halo row each side, toroidal) are
// staged whole in shared memory with coalesced loads; the column permutation
// and the 8 neighbour reads are served from shared memory.  At B = N this is
// a tuner pass seen through the permutation (|Z_p[k1,k2]| = |x_hat[s1i k1,
// s2i k2]|, SURVEY.md §7 hard part 2) without materialising the permuted
// grid.  Output: one bit per bin (row-major) and a count per 8192-bin block.
//
// UNORDERED (tuner passes): instead of bits + block counts, maxima are
// appended to `list` through one warp-aggregated atomicAdd on `count` per
// 32-bin word — the tuner only feeds them to the vote histogram, where order
// does not matter, and the count is order independent.
template <typename T, bool PERM, bool UNORDERED = false>
__global__ void __launch_bounds__(512)
k_lmax_rows(const T* __restrict__ M, int lgB, unsigned s1, unsigned s2, int rb,
            const unsigned long long* __restrict__ peak, double floor_rel,
            uint32_t* __restrict__ bits, unsigned* __restrict__ blk_counts,
            int32_t* __restrict__ list = nullptr, unsigned* __restrict__ count = nullptr,
            Publish pub = Publish{nullptr, 0, nullptr, 0}) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);
  __shared__ unsigned s_cnt[32];
  const int B = 1 << lgB;
  unsigned* s_words = reinterpret_cast<unsigned*>(S + ((size_t)(rb + 2) << lgB));  // UNORDERED only
  const unsigned mask = (unsigned)B - 1u;
  const int r0 = blockIdx.x * rb;
  for (int i = threadIdx.x; i < 32; i += blockDim.x) s_cnt[i] = 0;
  const int nrow = rb + 2;
  constexpr int V = 16 / sizeof(T);            // elements per 16-byte chunk
  const int ch_lg = lgB - (sizeof(T) == 4 ? 2 : 1);
  const int chunks = 1 << ch_lg;
  for (int e = threadIdx.x; e < (nrow << ch_lg); e += blockDim.x) {
    const int i = e >> ch_lg, q = e & (chunks - 1);
    const unsigned r = (unsigned)(r0 - 1 + i) & mask;
    const unsigned sr = PERM ? (s1 * r) & mask : r;
    cp_async16(S + ((size_t)i << lgB) + q * V, M + ((size_t)sr << lgB) + q * V);
  }
  cp_async_wait_all();
  __syncthreads();
  const double pk = fkey_inv(*peak);
  const bool live = pk > 0.0;
  const double fl = floor_rel * pk;
  // v >= fl (float64, tuner.py:111) <=> v >= fl rounded up to T, for T-valued v
  const T flT = sizeof(T) == 4 ? (T)__double2float_ru(fl) : (T)fl;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int wpr_lg = lgB - 5;                              // 32-bin words per row (B >= 32)
  const int wtot = rb << wpr_lg;
  const size_t word0 = ((size_t)r0 << lgB) >> 5;
  const int blk_first = (int)((word0 * 32) / kCmpElems);
  // A warp owns a 32-column strip and walks down the tile's rows keeping the
  // strip's own values of 3 rows in registers.  Per row it loads one value per
  // lane and votes on the floor test; only if some lane passes are the
  // horizontal neighbours fetched (lane shuffles, lanes 0/31 load the outside
  // neighbour) — at B = N nearly every bin fails the floor, so a 32-bin word
  // costs a handful of instructions.
  for (int strip = warp; strip < (1 << wpr_lg); strip += nwarps) {
    const unsigned c = ((unsigned)strip << 5) + lane;
    const unsigned cm = (c - 1u) & mask, cp = (c + 1u) & mask;
    const unsigned q1 = PERM ? (s2 * c) & mask : c;
    const unsigned q0 = PERM ? (s2 * cm) & mask : cm;
    const unsigned q2 = PERM ? (s2 * cp) & mask : cp;
    T um = S[q1];
    T mm = S[B + q1];
    for (int i = 1; i <= rb; ++i) {
      const T* dnrow = S + ((i + 1) << lgB);
      const T dm = dnrow[q1];
      const bool cand = live & (mm >= flT);
      unsigned bal = 0;
      if (__any_sync(0xffffffffu, cand)) {
        const T* uprow = dnrow - 2 * B;
        const T* mdrow = dnrow - B;
        T ul = __shfl_up_sync(0xffffffffu, um, 1), ur = __shfl_down_sync(0xffffffffu, um, 1);
        T ml = __shfl_up_sync(0xffffffffu, mm, 1), mr = __shfl_down_sync(0xffffffffu, mm, 1);
        T dl = __shfl_up_sync(0xffffffffu, dm, 1), dr = __shfl_down_sync(0xffffffffu, dm, 1);
        if (lane == 0) { ul = uprow[q0]; ml = mdrow[q0]; dl = dnrow[q0]; }
        if (lane == 31) { ur = uprow[q2]; mr = mdrow[q2]; dr = dnrow[q2]; }
        const bool f = cand & (mm > ul) & (mm > um) & (mm > ur) & (mm > ml) & (mm > mr) &
                       (mm > dl) & (mm > dm) & (mm > dr);
        bal = __ballot_sync(0xffffffffu, f);
      }
      const int w = ((i - 1) << wpr_lg) + strip;
      if (UNORDERED) {
        if (lane == 0) s_words[w] = bal;
      } else if (lane == 0) {
        bits[word0 + w] = bal;
        if (bal)
          atomicAdd(&s_cnt[(int)(((word0 + w) * 32) / kCmpElems) - blk_first], (unsigned)__popc(bal));
      }
      um = mm;
      mm = dm;
    }
  }
  if (UNORDERED) {
    // CTA-level aggregation: scan the tile's ballot words, ONE global atomic
    __syncthreads();
    const int per = (wtot + blockDim.x - 1) / blockDim.x;
    const int w0 = threadIdx.x * per, w1 = min(w0 + per, wtot);
    unsigned mine = 0;
    for (int w = w0; w < w1; ++w) mine += __popc(s_words[w]);
    __shared__ unsigned s_wsum[32];
    __shared__ unsigned s_base;
    unsigned inc = warp_incl_scan(mine);
    if (lane == 31) s_wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      unsigned t = lane < nwarps ? s_wsum[lane] : 0u;
      t = warp_incl_scan(t);
      s_wsum[lane] = t;
      if (lane == 31) s_base = t ? atomicAdd(count, t) : 0u;
    }
    __syncthreads();
    unsigned pos = s_base + inc - mine + (warp ? s_wsum[warp - 1] : 0u);
    for (int w = w0; w < w1; ++w) {
      unsigned b = s_words[w];
      while (b) {
        const int k = __ffs(b) - 1;
        b &= b - 1u;
        list[pos++] = (int32_t)((word0 + w) * 32 + k);
      }
    }
    if (pub.slot && threadIdx.x == 0) publish_count(count, pub.done, pub.target, pub.slot, pub.seq);
    return;
  }
  __syncthreads();
  // per-8192-bin block counts (blk_counts zeroed by the caller; a tile may
  // cover part of a block or several blocks)
  const size_t first = ((size_t)r0 << lgB), last = first + ((size_t)rb << lgB) - 1;
  const int nblk = (int)(last / kCmpElems - first / kCmpElems + 1);
  for (int i = threadIdx.x; i < nblk; i += blockDim.x)
    if (s_cnt[i]) atomicAdd(&blk_counts[first / kCmpElems + i], s_cnt[i]);
}

// cp.async group wait with a runtime depth (the PTX operand is an immediate)
__device__ __forceinline__ void cp_async_wait_upto(int n) {
  switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;\n" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;\n" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;\n" ::: "memory"); break;
    case 3: asm volatile("cp.async.wait_group 3;\n" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 4;\n" ::: "memory"); break;
  }
}

// Streaming local-maximum scan of a large tuner grid (B >= 512), unordered
// list output — same predicate and output as k_lmax_rows<T, PERM, true>.
// Each CTA owns a contiguous band of view rows and streams the rows it needs
// through a ring of `nslot` shared-memory row buffers with cp.async, up to
// nslot - 3 rows ahead of the row being tested, so HBM reads overlap the test
// and only the two halo rows of a band are read twice.  View row r is row
// s1*r of M.  The test walks NATURAL columns C of the staged rows, four per
// lane with one 16-byte (two for fp64) shared load: view column c = s2i*C and
// its view neighbours c -+ 1 are natural columns C -+ s2, so the floor test
// of 128 bins costs a handful of warp instructions, and only bins passing it
// fetch their 8 neighbours.  Maxima are appended to a per-warp shared buffer
// flushed with one global atomicAdd per kWarpBuf entries.
constexpr int kWarpBuf = 256;

template <typename T>
__device__ __forceinline__ void lds4(const T* p, T v[4]) {
  if constexpr (sizeof(T) == 4) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  } else {
    const double2 a = *reinterpret_cast<const double2*>(p);
    const double2 b = *reinterpret_cast<const double2*>(p + 2);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
}

template <typename T>
__global__ void __launch_bounds__(512)
k_lmax_stream(const T* __restrict__ M, int lgB, unsigned s1, unsigned s2, unsigned s2i, int band,
              int nslot, const unsigned long long* __restrict__ peak, double floor_rel,
              int32_t* __restrict__ list, unsigned* __restrict__ count, Publish pub,
              int32_t* __restrict__ cand = nullptr, unsigned* __restrict__ cand_count = nullptr) {
  pdl_wait();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long s_bar[8];
  T* ring = reinterpret_cast<T*>(smem_raw);
  const int B = 1 << lgB;
  const unsigned mask = (unsigned)B - 1u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  int32_t* wbuf = reinterpret_cast<int32_t*>(ring + ((size_t)nslot << lgB)) + warp * kWarpBuf;
  const int r0 = blockIdx.x * band;
  const int nrow = min(band, B - r0);
  const int nload = nrow + 2;                  // view rows r0-1 .. r0+nrow
  const unsigned row_bytes = (unsigned)(sizeof(T) << lgB);
  // rows arrive by TMA bulk copies issued by thread 0, one mbarrier per slot
  auto issue = [&](int t) {                    // load t = view row r0 - 1 + t
    const int slot = t % nslot;
    const unsigned r = (unsigned)(r0 - 1 + t) & mask;
    mbar_expect_tx(&s_bar[slot], row_bytes);
    bulk_g2s(ring + ((size_t)slot << lgB), M + ((size_t)((s1 * r) & mask) << lgB), row_bytes,
             &s_bar[slot]);
  };
  if (threadIdx.x < nslot) mbar_init(&s_bar[threadIdx.x], 1);
  mbar_fence_init();
  __syncthreads();
  if (threadIdx.x == 0)
    for (int t = 0; t < min(nslot, nload); ++t) issue(t);
  // floor test in T: v >= fl (float64, tuner.py:111) <=> v >= fl rounded up
  // to T; a zero peak (no live bins) becomes an unreachable threshold
  const double pk = fkey_inv(*peak);
  const double fl = floor_rel * pk;
  T flT = sizeof(T) == 4 ? (T)__double2float_ru(fl) : (T)fl;
  if (!(pk > 0.0))
    flT = sizeof(T) == 4 ? (T)__int_as_float(0x7f800000) : (T)__longlong_as_double(0x7ff0000000000000ll);
  int nbuf = 0;
  auto flush = [&]() {
    unsigned base = 0;
    if (lane == 0 && nbuf) base = atomicAdd(count, (unsigned)nbuf);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int e = lane; e < nbuf; e += 32) list[base + e] = wbuf[e];
    __syncwarp();
    nbuf = 0;
  };
  // slot of a load = load index mod nslot, tracked incrementally (no integer
  // division per row); one phase bit per slot
  unsigned phase = 0;
  auto wait_slot = [&](int slot) {
    mbar_wait(&s_bar[slot], (phase >> slot) & 1u);
    phase ^= 1u << slot;
  };
  auto next = [&](int slot) { return slot + 1 == nslot ? 0 : slot + 1; };
  const int groups = B >> 7;                   // 128 natural columns per warp step
  int su = 0, sm = next(0), sd = next(sm);     // slots of loads s, s+1, s+2
  wait_slot(su);
  wait_slot(sm);
  for (int s = 0; s < nrow; ++s) {
    wait_slot(sd);                             // loads s and s+1 were waited for earlier
    const T* up = ring + ((size_t)su << lgB);
    const T* md = ring + ((size_t)sm << lgB);
    const T* dn = ring + ((size_t)sd << lgB);
    const unsigned rowbase = (unsigned)(r0 + s) << lgB;
    for (int g = warp; g < groups; g += nwarps) {
      const unsigned C0 = ((unsigned)g << 7) + ((unsigned)lane << 2);
      T m[4];
      lds4(md + C0, m);
      const T hi = fmax(fmax(m[0], m[1]), fmax(m[2], m[3]));
      if (!__any_sync(0xffffffffu, hi >= flT)) continue;
      // the group holds a live bin: test it with lanes on consecutive columns
      // (sub-group j = columns g*128 + j*32 + lane), so every neighbour load
      // at C, C -+ s2 is one conflict-free 32-word wavefront
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const unsigned C = ((unsigned)g << 7) + ((unsigned)j << 5) + (unsigned)lane;
        const T v = md[C];
        bool f = v >= flT;
        if (cand) {   // every above-floor bin, natural index (later views test only these)
          const unsigned cb = __ballot_sync(0xffffffffu, f);
          if (cb) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(cand_count, (unsigned)__popc(cb));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (f) cand[base + __popc(cb & ((1u << lane) - 1u))] =
                (int32_t)((((s1 * (unsigned)(r0 + s)) & mask) << lgB) | C);
          }
        }
        if (f) {
          const unsigned Cl = (C - s2) & mask, Cr = (C + s2) & mask;
          f = (v > up[Cl]) & (v > up[C]) & (v > up[Cr]) & (v > md[Cl]) & (v > md[Cr]) &
              (v > dn[Cl]) & (v > dn[C]) & (v > dn[Cr]);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (!bal) continue;
        const int n = __popc(bal);
        if (nbuf + n > kWarpBuf) flush();
        if (f) wbuf[nbuf + __popc(bal & ((1u << lane) - 1u))] = (int32_t)(rowbase | ((s2i * C) & mask));
        nbuf += n;
      }
    }
    __syncthreads();                           // every thread is done with load s
    if (threadIdx.x == 0 && s + nslot < nload) issue(s + nslot);
    su = sm;
    sm = sd;
    sd = next(sd);
  }
  __syncwarp();
  flush();
  if (pub.slot) {
    __syncthreads();
    if (threadIdx.x == 0) publish_count(count, pub.done, pub.target, pub.slot, pub.seq, cand_count);
  }
}

// k_lmax_stream for grids where most bins pass the floor (tuner passes at
// B < N: the fold aliases the noise into every bucket).  Each warp owns fixed
// column groups (128 natural columns, lanes on consecutive columns) for the
// whole band and keeps, per tested column C, the 3 x 3 neighbourhood
// {C - s2, C, C + s2} of the previous two view rows in registers: each new
// view row costs 3 conflict-free shared loads per bin instead of 9, and the
// strict 8-neighbour test runs on registers.  Same ring, floor, list and
// publication as k_lmax_stream.  GPW = column groups per warp.
template <typename T, int GPW>
__global__ void __launch_bounds__(512)
k_lmax_win(const T* __restrict__ M, int lgB, unsigned s1, unsigned s2, unsigned s2i, int band,
           int nslot, const unsigned long long* __restrict__ peak, double floor_rel,
           int32_t* __restrict__ list, unsigned* __restrict__ count, Publish pub) {
  pdl_wait();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long s_bar[8];
  T* ring = reinterpret_cast<T*>(smem_raw);
  const int B = 1 << lgB;
  const unsigned mask = (unsigned)B - 1u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  int32_t* wbuf = reinterpret_cast<int32_t*>(ring + ((size_t)nslot << lgB)) + warp * kWarpBuf;
  const int r0 = blockIdx.x * band;
  const int nrow = min(band, B - r0);
  const int nload = nrow + 2;
  const unsigned row_bytes = (unsigned)(sizeof(T) << lgB);
  auto issue = [&](int t) {
    const int slot = t % nslot;
    const unsigned r = (unsigned)(r0 - 1 + t) & mask;
    mbar_expect_tx(&s_bar[slot], row_bytes);
    bulk_g2s(ring + ((size_t)slot << lgB), M + ((size_t)((s1 * r) & mask) << lgB), row_bytes,
             &s_bar[slot]);
  };
  if (threadIdx.x < nslot) mbar_init(&s_bar[threadIdx.x], 1);
  mbar_fence_init();
  __syncthreads();
  if (threadIdx.x == 0)
    for (int t = 0; t < min(nslot, nload); ++t) issue(t);
  const double pk = fkey_inv(*peak);
  const double fl = floor_rel * pk;
  T flT = sizeof(T) == 4 ? (T)__double2float_ru(fl) : (T)fl;
  if (!(pk > 0.0))
    flT = sizeof(T) == 4 ? (T)__int_as_float(0x7f800000) : (T)__longlong_as_double(0x7ff0000000000000ll);
  int nbuf = 0;
  auto flush = [&]() {
    unsigned base = 0;
    if (lane == 0 && nbuf) base = atomicAdd(count, (unsigned)nbuf);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int e = lane; e < nbuf; e += 32) list[base + e] = wbuf[e];
    __syncwarp();
    nbuf = 0;
  };
  unsigned phase = 0;
  auto wait_slot = [&](int slot) {
    mbar_wait(&s_bar[slot], (phase >> slot) & 1u);
    phase ^= 1u << slot;
  };
  auto next = [&](int slot) { return slot + 1 == nslot ? 0 : slot + 1; };
  const int groups = B >> 7;
  T wu[GPW][4][3], wm[GPW][4][3];
  int su = 0, sm = next(0), sd = next(sm);
  wait_slot(su);
  wait_slot(sm);
  {
    const T* up = ring + ((size_t)su << lgB);
    const T* md = ring + ((size_t)sm << lgB);
#pragma unroll
    for (int q = 0; q < GPW; ++q) {
      const int g = warp + q * nwarps;
      if (g >= groups) break;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const unsigned C = ((unsigned)g << 7) + ((unsigned)j << 5) + (unsigned)lane;
        const unsigned Cl = (C - s2) & mask, Cr = (C + s2) & mask;
        wu[q][j][0] = up[Cl]; wu[q][j][1] = up[C]; wu[q][j][2] = up[Cr];
        wm[q][j][0] = md[Cl]; wm[q][j][1] = md[C]; wm[q][j][2] = md[Cr];
      }
    }
  }
  for (int s = 0; s < nrow; ++s) {
    wait_slot(sd);
    const T* dn = ring + ((size_t)sd << lgB);
    const unsigned rowbase = (unsigned)(r0 + s) << lgB;
#pragma unroll
    for (int q = 0; q < GPW; ++q) {
      const int g = warp + q * nwarps;
      if (g >= groups) break;
      // the four column sub-groups are tested first (a 4-bit mask per lane),
      // then emitted with one warp scan: one ballot/scan per 128 bins
      unsigned fm = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const unsigned C = ((unsigned)g << 7) + ((unsigned)j << 5) + (unsigned)lane;
        const unsigned Cl = (C - s2) & mask, Cr = (C + s2) & mask;
        const T d0 = dn[Cl], d1 = dn[C], d2 = dn[Cr];
        const T v = wm[q][j][1];
        const T nb = fmax(fmax(fmax(wu[q][j][0], wu[q][j][1]), fmax(wu[q][j][2], wm[q][j][0])),
                          fmax(fmax(wm[q][j][2], d0), fmax(d1, d2)));
        fm |= ((v >= flT) & (v > nb)) ? (1u << j) : 0u;
        wu[q][j][0] = wm[q][j][0]; wu[q][j][1] = wm[q][j][1]; wu[q][j][2] = wm[q][j][2];
        wm[q][j][0] = d0; wm[q][j][1] = d1; wm[q][j][2] = d2;
      }
      if (!__any_sync(0xffffffffu, fm != 0u)) continue;
      const unsigned cntl = (unsigned)__popc(fm);
      const unsigned incl = warp_incl_scan(cntl);
      const int n = (int)__shfl_sync(0xffffffffu, incl, 31);
      if (nbuf + n > kWarpBuf) flush();
      int pos = nbuf + (int)(incl - cntl);
      while (fm) {
        const int j = __ffs(fm) - 1;
        fm &= fm - 1u;
        const unsigned C = ((unsigned)g << 7) + ((unsigned)j << 5) + (unsigned)lane;
        wbuf[pos++] = (int32_t)(rowbase | ((s2i * C) & mask));
      }
      __syncwarp();
      nbuf += n;
    }
    __syncthreads();                           // every thread is done with load s
    if (threadIdx.x == 0 && s + nslot < nload) issue(s + nslot);
    su = sm;
    sm = sd;
    sd = next(sd);
  }
  __syncwarp();
  flush();
  if (pub.slot) {
    __syncthreads();
    if (threadIdx.x == 0) publish_count(count, pub.done, pub.target, pub.slot, pub.seq);
  }
}

// k_lmax_win with the lanes of a warp on 32 CONSECUTIVE VIEW COLUMNS
// c = 32 g + lane (natural column s2 * c: an odd stride, so every shared load
// is conflict-free).  Each lane keeps the last two view rows of its own
// column in registers and loads ONE value per bin and row; the vertical
// 3-maxima of the left / right neighbour columns come from the neighbour
// lanes by shuffle (lanes 0 and 31 keep the column just outside the group in
// a second register window, loaded by one more instruction per group and
// row), so a bin costs 2 shared loads, 4 max and 2 shuffles instead of 3 loads
// and 7 max, and a group's maxima are one ballot: keys rowbase | c, no scan.
// The CTA's maxima are appended with ONE 64-bit atomic on `cd`, which holds
// the count in its low word (read by later kernels as the list length) and
// the CTA tickets in its high word: the CTA taking the last ticket knows the
// final count from the same atomic and publishes (count, seq) to the mapped
// slot — one L2 round trip per CTA instead of count atomics per warp + fence
// + ticket + count read-back.  Same predicate, list (as a set) and
// publication as k_lmax_win.  GPW = 32-column groups per warp
// (blockDim.x = 32 * (B / 32 / GPW)).
template <typename T, int GPW>
__global__ void __launch_bounds__(512)
k_lmax_win2(const T* __restrict__ M, int lgB, unsigned s1, unsigned s2, int band, int nslot,
            const unsigned long long* __restrict__ peak, double floor_rel,
            int32_t* __restrict__ list, unsigned long long* __restrict__ cd, unsigned target,
            volatile unsigned* slot, unsigned seq) {
  pdl_wait();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long s_bar[8];
  __shared__ unsigned s_n[17];
  T* ring = reinterpret_cast<T*>(smem_raw);
  const int B = 1 << lgB;
  const unsigned mask = (unsigned)B - 1u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  int32_t* wbuf = reinterpret_cast<int32_t*>(ring + ((size_t)nslot << lgB)) + warp * kWarpBuf;
  const int r0 = blockIdx.x * band;
  const int nrow = min(band, B - r0);
  const int nload = nrow + 2;
  const unsigned row_bytes = (unsigned)(sizeof(T) << lgB);
  auto issue = [&](int t) {
    const int sl = t % nslot;
    const unsigned r = (unsigned)(r0 - 1 + t) & mask;
    mbar_expect_tx(&s_bar[sl], row_bytes);
    bulk_g2s(ring + ((size_t)sl << lgB), M + ((size_t)((s1 * r) & mask) << lgB), row_bytes,
             &s_bar[sl]);
  };
  if (threadIdx.x < nslot) mbar_init(&s_bar[threadIdx.x], 1);
  mbar_fence_init();
  __syncthreads();
  if (threadIdx.x == 0)
    for (int t = 0; t < min(nslot, nload); ++t) issue(t);
  const double pk = fkey_inv(*peak);
  const double fl = floor_rel * pk;
  T flT = sizeof(T) == 4 ? (T)__double2float_ru(fl) : (T)fl;
  if (!(pk > 0.0))
    flT = sizeof(T) == 4 ? (T)__int_as_float(0x7f800000) : (T)__longlong_as_double(0x7ff0000000000000ll);
  int nbuf = 0;
  auto flush = [&]() {   // a warp buffer that filled up before the end of the band
    __syncwarp();
    unsigned base = 0;
    if (lane == 0 && nbuf) base = (unsigned)atomicAdd(cd, (unsigned long long)nbuf);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int e = lane; e < nbuf; e += 32) list[base + e] = wbuf[e];
    __syncwarp();
    nbuf = 0;
  };
  unsigned phase = 0;
  auto wait_slot = [&](int sl) {
    mbar_wait(&s_bar[sl], (phase >> sl) & 1u);
    phase ^= 1u << sl;
  };
  auto next = [&](int sl) { return sl + 1 == nslot ? 0 : sl + 1; };
  unsigned oc[GPW], oe[GPW];          // natural columns of the lane's own / edge view column
  T up[GPW], md[GPW], eu[GPW], em[GPW];
  int su = 0, sm = next(0), sd = next(sm);
  wait_slot(su);
  wait_slot(sm);
  {
    const T* ru = ring + ((size_t)su << lgB);
    const T* rm = ring + ((size_t)sm << lgB);
#pragma unroll
    for (int q = 0; q < GPW; ++q) {
      const unsigned c = ((unsigned)(warp + q * nwarps) << 5) + (unsigned)lane;
      oc[q] = (s2 * c) & mask;
      oe[q] = (s2 * (lane < 16 ? c - 1u : c + 1u)) & mask;
      up[q] = ru[oc[q]]; md[q] = rm[oc[q]];
      eu[q] = ru[oe[q]]; em[q] = rm[oe[q]];
    }
  }
  const unsigned lt = (1u << lane) - 1u;
  for (int s = 0; s < nrow; ++s) {
    wait_slot(sd);
    const T* rd = ring + ((size_t)sd << lgB);
    const unsigned rowbase = (unsigned)(r0 + s) << lgB;
#pragma unroll
    for (int q = 0; q < GPW; ++q) {
      const T dn = rd[oc[q]], ed = rd[oe[q]];
      const T vm = fmax(fmax(up[q], md[q]), dn);      // vertical 3-max of the own column
      const T ve = fmax(fmax(eu[q], em[q]), ed);      // ... of the column outside the group
      T vl = __shfl_up_sync(0xffffffffu, vm, 1);
      T vr = __shfl_down_sync(0xffffffffu, vm, 1);
      if (lane == 0) vl = ve;
      if (lane == 31) vr = ve;
      const T nb = fmax(fmax(vl, vr), fmax(up[q], dn));
      const T v = md[q];
      const bool f = (v >= flT) & (v > nb);
      up[q] = v; md[q] = dn; eu[q] = em[q]; em[q] = ed;
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (bal) {
        const int n = __popc(bal);
        if (nbuf + n > kWarpBuf) flush();
        if (f) wbuf[nbuf + __popc(bal & lt)] =
            (int32_t)(rowbase | (((unsigned)(warp + q * nwarps) << 5) + (unsigned)lane));
        nbuf += n;
      }
    }
    __syncthreads();                           // every thread is done with load s
    if (threadIdx.x == 0 && s + nslot < nload) issue(s + nslot);
    su = sm;
    sm = sd;
    sd = next(sd);
  }
  // the CTA's buffered maxima: one atomic for the positions and the ticket
  if (lane == 0) s_n[warp] = (unsigned)nbuf;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < nwarps; ++w) {
      const unsigned a = s_n[w];
      s_n[w] = t;
      t += a;
    }
    const unsigned long long old = atomicAdd(cd, (1ull << 32) | (unsigned long long)t);
    s_n[16] = (unsigned)old;
    if ((unsigned)(old >> 32) + 1u == target && slot)
      *reinterpret_cast<volatile unsigned long long*>(slot) =
          ((unsigned long long)((unsigned)old + t) << 32) | (unsigned long long)seq;
  }
  __syncthreads();
  const unsigned base = s_n[16] + s_n[warp];
  for (int e = lane; e < nbuf; e += 32) list[base + e] = wbuf[e];
}

// Local maxima of a permuted view of |x_hat| at B = N tested only at the
// above-floor bins `cand` (natural indices R*N + C, from the first B = N
// pass): view (r, c) = (s1i^-1 R, s2i^-1 C) has its view neighbours at the
// natural bins (R +- s1, C +- s2) (s1, s2 = the view multipliers).  Bins below
// the floor can never be counted, so the count equals k_lmax_stream's.
// Append the flagged keys of the whole block to `list` with ONE global atomic
// per call (block scan for the positions): every thread of the block calls it
// (block-uniform loops).  `s_tmp` holds 33 unsigneds of shared memory.
__device__ __forceinline__ void block_emit(bool f, int32_t key, int32_t* __restrict__ list,
                                           unsigned* __restrict__ count, unsigned* s_tmp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, f);
  if (lane == 0) s_tmp[warp] = (unsigned)__popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < nwarps; ++w) {
      const unsigned a = s_tmp[w];
      s_tmp[w] = t;
      t += a;
    }
    s_tmp[32] = t ? atomicAdd(count, t) : 0u;
  }
  __syncthreads();
  if (f) list[s_tmp[32] + s_tmp[warp] + __popc(bal & ((1u << lane) - 1u))] = key;
  __syncthreads();   // s_tmp is reused by the next call
}

template <typename T>
__global__ void k_lmax_cand(const T* __restrict__ M, int lgB, unsigned s1, unsigned s2,
                            unsigned s1inv, unsigned s2inv, const int32_t* __restrict__ cand,
                            const unsigned* __restrict__ cand_count,
                            int32_t* __restrict__ list, unsigned* __restrict__ count, Publish pub) {
  pdl_wait();
  const unsigned mask = (1u << lgB) - 1u;
  const unsigned n = *cand_count;
  __shared__ unsigned s_tmp[33];
  // a single CTA needs no atomics: positions from a running total, the count
  // stored and published directly (three L2 round trips less on the tuner's
  // critical path: count atomic, ticket, count read-back)
  const bool solo = gridDim.x == 1;
  unsigned run = 0;
  for (unsigned e0 = blockIdx.x * blockDim.x; e0 < n; e0 += gridDim.x * blockDim.x) {
    const unsigned e = e0 + threadIdx.x;
    bool f = false;
    unsigned key = 0;
    if (e < n) {
      const unsigned q = (unsigned)cand[e];
      const unsigned R = q >> lgB, C = q & mask;
      const unsigned Ru = (R - s1) & mask, Rd = (R + s1) & mask;
      const unsigned Cl = (C - s2) & mask, Cr = (C + s2) & mask;
      const T v = M[q];
      const T* up = M + ((size_t)Ru << lgB);
      const T* md = M + ((size_t)R << lgB);
      const T* dn = M + ((size_t)Rd << lgB);
      f = (v > up[Cl]) & (v > up[C]) & (v > up[Cr]) & (v > md[Cl]) & (v > md[Cr]) &
          (v > dn[Cl]) & (v > dn[C]) & (v > dn[Cr]);
      key = (((s1inv * R) & mask) << lgB) | ((s2inv * C) & mask);
    }
    if (solo) {
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (lane == 0) s_tmp[warp] = (unsigned)__popc(bal);
      __syncthreads();
      unsigned before = 0, total = 0;
      for (int w = 0; w < nwarps; ++w) {
        const unsigned a = s_tmp[w];
        before += w < warp ? a : 0u;
        total += a;
      }
      if (f) list[run + before + __popc(bal & ((1u << lane) - 1u))] = (int32_t)key;
      run += total;
      __syncthreads();   // s_tmp is reused by the next iteration
    } else {
      block_emit(f, (int32_t)key, list, count, s_tmp);
    }
  }
  if (solo) {
    if (threadIdx.x == 0) {
      *count = run;
      if (pub.slot)
        *reinterpret_cast<volatile unsigned long long*>(pub.slot) =
            ((unsigned long long)run << 32) | (unsigned long long)pub.seq;
    }
    return;
  }
  if (pub.slot) {
    __syncthreads();
    if (threadIdx.x == 0) publish_count(count, pub.done, pub.target, pub.slot, pub.seq);
  }
}

// Local maxima of a permuted view straight from global memory, for grids whose
// rows do not fit the shared-memory ring (fp64 at B = 16384: 128 KB rows).
// Every natural bin (R, C) above the floor is tested against its view
// neighbours at the natural bins (R -+ s1, C -+ s2) (as k_lmax_cand), and is
// optionally listed as a candidate for the later B = N views.
template <typename T>
__global__ void k_lmax_direct(const T* __restrict__ M, int lgB, unsigned s1, unsigned s2,
                              unsigned s1inv, unsigned s2inv,
                              const unsigned long long* __restrict__ peak, double floor_rel,
                              int32_t* __restrict__ list, unsigned* __restrict__ count, Publish pub,
                              int32_t* __restrict__ cand, unsigned* __restrict__ cand_count) {
  pdl_wait();
  const unsigned mask = (1u << lgB) - 1u;
  const size_t n = (size_t)1 << (2 * lgB);
  const double pk = fkey_inv(*peak);
  const double fl = floor_rel * pk;
  T flT = sizeof(T) == 4 ? (T)__double2float_ru(fl) : (T)fl;
  if (!(pk > 0.0))
    flT = sizeof(T) == 4 ? (T)__int_as_float(0x7f800000) : (T)__longlong_as_double(0x7ff0000000000000ll);
  __shared__ unsigned s_tmp[33];
  for (size_t e0 = (size_t)blockIdx.x * blockDim.x; e0 < n; e0 += (size_t)gridDim.x * blockDim.x) {
    const size_t e = e0 + threadIdx.x;
    const T v = e < n ? M[e] : (T)0;
    const bool live = e < n && v >= flT;
    // (block-uniform: one global atomic per block and list per iteration)
    if (!__syncthreads_or(live)) continue;
    if (cand) block_emit(live, (int32_t)e, cand, cand_count, s_tmp);
    bool f = false;
    unsigned key = 0;
    if (live) {
      const unsigned R = (unsigned)(e >> lgB), C = (unsigned)e & mask;
      const unsigned Ru = (R - s1) & mask, Rd = (R + s1) & mask;
      const unsigned Cl = (C - s2) & mask, Cr = (C + s2) & mask;
      const T* up = M + ((size_t)Ru << lgB);
      const T* md = M + ((size_t)R << lgB);
      const T* dn = M + ((size_t)Rd << lgB);
      f = (v > up[Cl]) & (v > up[C]) & (v > up[Cr]) & (v > md[Cl]) & (v > md[Cr]) &
          (v > dn[Cl]) & (v > dn[C]) & (v > dn[Cr]);
      key = (((s1inv * R) & mask) << lgB) | ((s2inv * C) & mask);
    }
    block_emit(f, (int32_t)key, list, count, s_tmp);
  }
  if (pub.slot) {
    __syncthreads();
    if (threadIdx.x == 0) publish_count(count, pub.done, pub.target, pub.slot, pub.seq, cand_count);
  }
}

// G[r][c] = M[s1i*r mod N][s2i*c mod N]: the |Z| grid of a B == N pass seen
// through the permutation (SURVEY.md §7 hard part 2: tuner passes at B = N are
// permuted views of |x_hat|).  CTA per output row; the source row is staged in
// shared memory so both the read and the write are coalesced.
// B = N view whose rows are too long for the ring of k_lmax_stream (fp32
// B = 16384, fp64 B = 8192: 64 KB rows) but of which THREE rows fit shared
// memory: the view neighbours of natural bin (R, C) are the natural bins
// (R -+ s1, C -+ s2) (as in k_lmax_direct), so a CTA stages the natural rows
// R - s1, R, R + s1 with TMA bulk copies (one mbarrier) and tests row R with
// every neighbour from shared memory — 3 coalesced row reads per row instead
// of 8 scattered 4-byte reads per above-floor bin (c5 k = 4096: most bins
// are above the floor).  Persistent over rows; same outputs as k_lmax_direct
// (unordered list of view keys, count, optional above-floor candidate list).
template <typename T>
__global__ void __launch_bounds__(512)
k_lmax_tri(const T* __restrict__ M, int lgB, unsigned s1, unsigned s2, unsigned s1inv,
           unsigned s2inv, const unsigned long long* __restrict__ peak, double floor_rel,
           int32_t* __restrict__ list, unsigned* __restrict__ count, Publish pub,
           int32_t* __restrict__ cand, unsigned* __restrict__ cand_count) {
  pdl_wait();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long s_bar;
  __shared__ unsigned s_wf[16], s_wc[16], s_base[2];
  const int B = 1 << lgB;
  const unsigned mask = (unsigned)B - 1u;
  T* up = reinterpret_cast<T*>(smem_raw);
  T* md = up + B;
  T* dn = md + B;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int per = B / blockDim.x;   // columns per thread (<= 32: one bit each)
  const double pk = fkey_inv(*peak);
  const double fl = floor_rel * pk;
  T flT = sizeof(T) == 4 ? (T)__double2float_ru(fl) : (T)fl;
  if (!(pk > 0.0))
    flT = sizeof(T) == 4 ? (T)__int_as_float(0x7f800000) : (T)__longlong_as_double(0x7ff0000000000000ll);
  const unsigned row_bytes = (unsigned)(sizeof(T) << lgB);
  if (threadIdx.x == 0) mbar_init(&s_bar, 1);
  mbar_fence_init();
  __syncthreads();
  unsigned phase = 0;
  for (unsigned R = blockIdx.x; R < (unsigned)B; R += gridDim.x) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(&s_bar, 3u * row_bytes);
      bulk_g2s(up, M + ((size_t)((R - s1) & mask) << lgB), row_bytes, &s_bar);
      bulk_g2s(md, M + ((size_t)R << lgB), row_bytes, &s_bar);
      bulk_g2s(dn, M + ((size_t)((R + s1) & mask) << lgB), row_bytes, &s_bar);
    }
    mbar_wait(&s_bar, phase);
    phase ^= 1u;
    // test the row: bit q of fm / cm = column q * blockDim + tid is a maximum /
    // above the floor
    unsigned fm = 0u, cm = 0u;
    for (int q = 0; q < per; ++q) {
      const unsigned C = (unsigned)(q * blockDim.x + threadIdx.x);
      const T v = md[C];
      if (v >= flT) {
        cm |= 1u << q;
        const unsigned Cl = (C - s2) & mask, Cr = (C + s2) & mask;
        const T nb = fmax(fmax(fmax(up[Cl], up[C]), fmax(up[Cr], md[Cl])),
                          fmax(fmax(md[Cr], dn[Cl]), fmax(dn[C], dn[Cr])));
        if (v > nb) fm |= 1u << q;
      }
    }
    if (!cand) cm = 0u;
    // one global atomic per row and list (a single hot counter took one
    // atomic per warp per 32 bins before: c5's dense B = N views were bound
    // by it); positions inside the row from a block scan
    const unsigned nf = (unsigned)__popc(fm), nc = (unsigned)__popc(cm);
    const unsigned xf = warp_incl_scan(nf), xc = warp_incl_scan(nc);
    if (lane == 31) { s_wf[warp] = xf; s_wc[warp] = xc; }
    __syncthreads();   // (also: every thread is done with the three rows)
    if (threadIdx.x == 0) {
      unsigned tf = 0, tc = 0;
      for (int w = 0; w < nwarps; ++w) {
        const unsigned a = s_wf[w], b = s_wc[w];
        s_wf[w] = tf;
        s_wc[w] = tc;
        tf += a;
        tc += b;
      }
      s_base[0] = tf ? atomicAdd(count, tf) : 0u;
      s_base[1] = tc ? atomicAdd(cand_count, tc) : 0u;
    }
    __syncthreads();
    unsigned pf = s_base[0] + s_wf[warp] + xf - nf;
    unsigned pc = s_base[1] + s_wc[warp] + xc - nc;
    const unsigned keyrow = ((s1inv * R) & mask) << lgB;
    while (fm) {
      const int q = __ffs(fm) - 1;
      fm &= fm - 1u;
      const unsigned C = (unsigned)(q * blockDim.x + threadIdx.x);
      list[pf++] = (int32_t)(keyrow | ((s2inv * C) & mask));
    }
    while (cm) {
      const int q = __ffs(cm) - 1;
      cm &= cm - 1u;
      cand[pc++] = (int32_t)(((size_t)R << lgB) | (unsigned)(q * blockDim.x + threadIdx.x));
    }
  }
  if (pub.slot) {
    __syncthreads();
    if (threadIdx.x == 0) publish_count(count, pub.done, pub.target, pub.slot, pub.seq, cand_count);
  }
}

template <typename T>
__global__ void k_permute_grid(const T* __restrict__ M, int lgN, unsigned s1i, unsigned s2i,
                               T* __restrict__ G) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* row = reinterpret_cast<T*>(smem_raw);
  const int N = 1 << lgN;
  const unsigned maskN = (unsigned)N - 1u;
  const unsigned r = blockIdx.x;
  const T* src = M + ((size_t)((s1i * r) & maskN) << lgN);
  for (int c = threadIdx.x; c < N; c += blockDim.x) row[c] = src[c];
  __syncthreads();
  T* dst = G + ((size_t)r << lgN);
  for (int c = threadIdx.x; c < N; c += blockDim.x) dst[c] = row[(s2i * (unsigned)c) & maskN];
}

// ---------------------------------------------------------------- scans
// Exclusive scan of each segment's per-block counts (one CTA per segment).
__global__ void k_scan_blocks(const unsigned* __restrict__ counts, int nblk,
                              unsigned* __restrict__ offsets, unsigned* __restrict__ totals) {
  pdl_wait();
  const int seg = blockIdx.x;
  const unsigned* c = counts + (size_t)seg * nblk;
  unsigned* o = offsets + (size_t)seg * nblk;
  const int per = (nblk + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per;
  const int b1 = min(b0 + per, nblk);
  unsigned local = 0;
  for (int b = b0; b < b1; ++b) local += c[b];
  // block exclusive scan of `local`
  __shared__ unsigned s_warp[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned inc = warp_incl_scan(local);
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    unsigned v = lane < nw ? s_warp[lane] : 0u;
    v = warp_incl_scan(v);
    s_warp[lane] = v;
  }
  __syncthreads();
  unsigned run = inc - local + (warp ? s_warp[warp - 1] : 0u);
  for (int b = b0; b < b1; ++b) {
    o[b] = run;
    run += c[b];
  }
  if (threadIdx.x == blockDim.x - 1 && totals) totals[seg] = run;
  if (nblk == 0 && threadIdx.x == 0 && totals) totals[seg] = 0;
}

// Block-exclusive scan over kCmpThreads values; returns exclusive prefix.
__device__ __forceinline__ unsigned block_excl_scan256(unsigned v, unsigned* s_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned inc = warp_incl_scan(v);
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    unsigned t = lane < (kCmpThreads / 32) ? s_warp[lane] : 0u;
    t = warp_incl_scan(t);
    if (lane < (kCmpThreads / 32)) s_warp[lane] = t;
  }
  __syncthreads();
  const unsigned r = inc - v + (warp ? s_warp[warp - 1] : 0u);
  __syncthreads();
  return r;
}

// Scatter the set bits of each segment to out[seg * out_stride + rank] (flat index).
__global__ void k_compact_bits(const uint32_t* __restrict__ bits, long seglen,
                               const unsigned* __restrict__ offsets, int32_t* __restrict__ out,
                               long out_stride) {
  pdl_wait();
  __shared__ unsigned s_warp[32];
  const int seg = blockIdx.y;
  const long wps = words_for(seglen);
  const long w = (long)blockIdx.x * kCmpWords + threadIdx.x;
  uint32_t word = (w < wps) ? bits[(size_t)seg * wps + w] : 0u;
  const unsigned pre = block_excl_scan256(__popc(word), s_warp);
  unsigned pos = offsets[(size_t)seg * gridDim.x + blockIdx.x] + pre;
  int32_t* o = out + (size_t)seg * out_stride;
  while (word) {
    const int b = __ffs(word) - 1;
    word &= word - 1u;
    o[pos++] = (int32_t)(w * 32 + b);
  }
}

// k_compact_bits of one segment without the scan launch: every CTA sums the
// block counts before its own (nblk <= a few thousand words, coalesced) —
// one launch less on the tuner's tail.
__global__ void k_compact_bits_self(const uint32_t* __restrict__ bits, long seglen,
                                    const unsigned* __restrict__ blk_counts,
                                    int32_t* __restrict__ out) {
  pdl_wait();
  __shared__ unsigned s_warp[32];
  __shared__ unsigned s_before;
  unsigned before = 0;
  for (int b = threadIdx.x; b < (int)blockIdx.x; b += blockDim.x) before += blk_counts[b];
  for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
  if (threadIdx.x == 0) s_before = 0u;
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && before) atomicAdd(&s_before, before);
  const long wps = words_for(seglen);
  const long w = (long)blockIdx.x * kCmpWords + threadIdx.x;
  uint32_t word = (w < wps) ? bits[w] : 0u;
  const unsigned pre = block_excl_scan256(__popc(word), s_warp);   // (barriers: s_before complete)
  unsigned pos = s_before + pre;
  while (word) {
    const int b = __ffs(word) - 1;
    word &= word - 1u;
    out[pos++] = (int32_t)(w * 32 + b);
  }
}

// ---------------------------------------------------------------- radix select
struct SelState {
  unsigned long long prefix;   // key bits fixed so far
  unsigned long long mask;     // which bits are fixed
  long long need;              // how many still to take among keys matching prefix
  long long take_all;          // 1: keep the whole segment (num >= seglen)
};

template <typename T>
__global__ void k_radix_hist(const T* __restrict__ vals, long seglen,
                             const SelState* __restrict__ st, int shift,
                             unsigned* __restrict__ hist) {
  pdl_wait();
  __shared__ unsigned sh[256];
  const int seg = blockIdx.y;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const SelState s = st[seg];
  if (!s.take_all) {
    const T* v = vals + (size_t)seg * seglen;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < seglen;
         e += (long)gridDim.x * blockDim.x) {
      const unsigned long long k = fkey(v[e]);
      if ((k & s.mask) == s.prefix) atomicAdd(&sh[(k >> shift) & 255u], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[(size_t)seg * 256 + i], sh[i]);
}

__global__ void k_radix_pick(SelState* __restrict__ st, unsigned* __restrict__ hist, int shift,
                             int nseg) {
  pdl_wait();
  const int seg = blockIdx.x * blockDim.x + threadIdx.x;
  if (seg >= nseg) return;
  SelState s = st[seg];
  unsigned* h = hist + (size_t)seg * 256;
  if (!s.take_all) {
    long long cum = 0;
    for (int d = 255; d >= 0; --d) {
      const long long c = h[d];
      if (cum + c >= s.need) {
        s.prefix |= (unsigned long long)d << shift;
        s.mask |= 255ull << shift;
        s.need -= cum;
        break;
      }
      cum += c;
    }
    st[seg] = s;
  }
  for (int d = 0; d < 256; ++d) h[d] = 0;
}

// All radix passes of the exact top-`need` selection of one short segment in
// ONE CTA (segments up to kSelSegMax keys, one CTA per segment): per 8-bit
// digit a shared histogram of the keys still matching the prefix, then warp 0
// finds the digit holding the need-th largest key (descending warp scan).
// Same SelState result as the k_radix_hist / k_radix_pick launch pairs, which
// stay for long segments (16 launches -> 1 for SFFT's B x B loops).
constexpr long kSelSegMax = 1L << 16;

template <typename T>
__global__ void __launch_bounds__(1024) k_radix_select_seg(const T* __restrict__ vals, long seglen,
                                                           SelState* __restrict__ st) {
  pdl_wait();
  __shared__ unsigned sh[256];
  __shared__ SelState s_st;
  const int seg = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) s_st = st[seg];
  __syncthreads();
  if (s_st.take_all) return;
  const T* v = vals + (size_t)seg * seglen;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const unsigned long long prefix = s_st.prefix, mask = s_st.mask;
    for (long e = tid; e < seglen; e += blockDim.x) {
      const unsigned long long k = fkey(v[e]);
      if ((k & mask) == prefix) atomicAdd(&sh[(k >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      // lane l owns digits 255 - 8l .. 248 - 8l (descending)
      unsigned c[8], lsum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) { c[i] = sh[255 - 8 * lane - i]; lsum += c[i]; }
      const unsigned incl = warp_incl_scan(lsum);
      const long long need = s_st.need;
      const unsigned hit = __ballot_sync(0xffffffffu, (long long)incl >= need);
      const int L0 = __ffs(hit) - 1;               // first lane reaching need (exists)
      if (lane == L0) {
        long long cum = (long long)(incl - lsum);
        for (int i = 0; i < 8; ++i) {
          if (cum + c[i] >= need) {
            const unsigned d = 255u - 8u * (unsigned)lane - (unsigned)i;
            s_st.prefix |= (unsigned long long)d << shift;
            s_st.mask |= 255ull << shift;
            s_st.need = need - cum;
            break;
          }
          cum += c[i];
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) st[seg] = s_st;
}

// per-block count of keys equal to the threshold (for tie ranks)
template <typename T>
__global__ void k_tie_counts(const T* __restrict__ vals, long seglen,
                             const SelState* __restrict__ st, unsigned* __restrict__ tie_blk) {
  pdl_wait();
  __shared__ unsigned s_warp[32];
  const int seg = blockIdx.y;
  const SelState s = st[seg];
  const T* v = vals + (size_t)seg * seglen;
  const long e0 = ((long)blockIdx.x * kCmpWords + threadIdx.x) * 32;
  unsigned c = 0;
  if (!s.take_all)
    for (int b = 0; b < 32; ++b) {
      const long e = e0 + b;
      if (e < seglen && fkey(v[e]) == s.prefix) ++c;
    }
  const unsigned pre = block_excl_scan256(c, s_warp);
  if (threadIdx.x == kCmpThreads - 1) tie_blk[(size_t)seg * gridDim.x + blockIdx.x] = pre + c;
}

// selection bitmask: key > T, or key == T with global tie rank < need
template <typename T>
__global__ void k_select_bits(const T* __restrict__ vals, long seglen,
                              const SelState* __restrict__ st, const unsigned* __restrict__ tie_off,
                              uint32_t* __restrict__ bits, unsigned* __restrict__ blk_counts) {
  pdl_wait();
  __shared__ unsigned s_warp[32];
  const int seg = blockIdx.y;
  const SelState s = st[seg];
  const T* v = vals + (size_t)seg * seglen;
  const long wps = words_for(seglen);
  const long w = (long)blockIdx.x * kCmpWords + threadIdx.x;
  uint32_t gt = 0, eq = 0;
  for (int b = 0; b < 32; ++b) {
    const long e = w * 32 + b;
    if (e < seglen) {
      if (s.take_all) {
        gt |= 1u << b;
      } else {
        const unsigned long long k = fkey(v[e]);
        if (k > s.prefix) gt |= 1u << b;
        else if (k == s.prefix) eq |= 1u << b;
      }
    }
  }
  const unsigned pre = block_excl_scan256(__popc(eq), s_warp);
  long long rank = (long long)tie_off[(size_t)seg * gridDim.x + blockIdx.x] + pre;
  uint32_t word = gt;
  uint32_t e2 = eq;
  while (e2) {
    const int b = __ffs(e2) - 1;
    e2 &= e2 - 1u;
    if (rank < s.need) word |= 1u << b;
    ++rank;
  }
  if (w < wps) bits[(size_t)seg * wps + w] = word;
  const unsigned tot = block_excl_scan256(__popc(word), s_warp);
  if (threadIdx.x == kCmpThreads - 1)
    blk_counts[(size_t)seg * gridDim.x + blockIdx.x] = tot + __popc(word);
}


// ---------------------------------------------------------------- one-CTA top-k
// Exact top-`num` selection (ties to the lowest index, engine.py:122-127) of a
// segment of n <= kTopkCtaMax values by ONE CTA of 1024 threads, each holding
// a contiguous run of `per` = ceil(n / 1024) <= 16 values in registers: the
// eight radix passes of k_radix_select_seg (same digit walk, same SelState
// result) histogram the register keys, then two block scans — tie ranks among
// the keys equal to the threshold, output positions — give every thread the
// selection mask of its run and the rank of its first selected value, so the
// caller emits the selected indices in ascending order without any of the
// k_tie_counts / k_select_bits / scan / compaction launches.
constexpr int kTopkCtaMax = 16384;
constexpr int kTopkPer = 16;

// selection key of the one-CTA top-k: any order-preserving injective key gives
// the same selection as fkey's 64-bit one, so float values use their own 32
// bits (4 radix passes instead of 8)
__device__ __forceinline__ unsigned long long tkey(double v) { return fkey(v); }
__device__ __forceinline__ unsigned long long tkey(float v) {
  const unsigned u = __float_as_uint(v);
  return (unsigned long long)((u & 0x80000000u) ? ~u : (u | 0x80000000u));
}


struct TopkScratch {
  unsigned hist[256];
  unsigned warp[32];
  unsigned long long prefix, mask;
  long long need;
};

__device__ __forceinline__ unsigned block_excl_scan1024(unsigned v, unsigned* s_warp,
                                                        unsigned* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned inc = warp_incl_scan(v);
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) s_warp[lane] = warp_incl_scan(s_warp[lane]);
  __syncthreads();
  const unsigned r = inc - v + (warp ? s_warp[warp - 1] : 0u);
  if (total) *total = s_warp[31];
  __syncthreads();   // s_warp is reused by the next scan
  return r;
}

// v[j] = value e0 + j of the thread's run (j < cnt); returns the selection mask
// of the run (bit j) and, in *pos, the number of selected values before it.
template <typename T>
__device__ __forceinline__ unsigned block_topk_mask(const T (&v)[kTopkPer], int cnt, int n,
                                                    long long num, TopkScratch& sc, unsigned* pos,
                                                    unsigned* total) {
  const int tid = threadIdx.x, lane = tid & 31;
  if (num >= (long long)n) {   // block-uniform: keep the whole segment
    const unsigned mask = cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u);
    *pos = block_excl_scan1024((unsigned)cnt, sc.warp, total);
    return mask;
  }
  if (tid == 0) { sc.prefix = 0ull; sc.mask = 0ull; sc.need = num; }
  for (int shift = (sizeof(T) == 4 ? 24 : 56); shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += blockDim.x) sc.hist[i] = 0;
    __syncthreads();
    const unsigned long long prefix = sc.prefix, mask = sc.mask;
#pragma unroll
    for (int j = 0; j < kTopkPer; ++j) {
      if (j < cnt) {
        const unsigned long long k = tkey(v[j]);
        if ((k & mask) == prefix) atomicAdd(&sc.hist[(k >> shift) & 255u], 1u);
      }
    }
    __syncthreads();
    if (tid < 32) {
      unsigned c[8], lsum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) { c[i] = sc.hist[255 - 8 * lane - i]; lsum += c[i]; }
      const unsigned incl = warp_incl_scan(lsum);
      const long long need = sc.need;
      const unsigned hit = __ballot_sync(0xffffffffu, (long long)incl >= need);
      const int L0 = __ffs(hit) - 1;
      if (lane == L0) {
        long long cum = (long long)(incl - lsum);
        for (int i = 0; i < 8; ++i) {
          if (cum + c[i] >= need) {
            const unsigned d = 255u - 8u * (unsigned)lane - (unsigned)i;
            sc.prefix |= (unsigned long long)d << shift;
            sc.mask |= 255ull << shift;
            sc.need = need - cum;
            break;
          }
          cum += c[i];
        }
      }
    }
    __syncthreads();
  }
  const unsigned long long thr = sc.prefix;
  const long long need = sc.need;
  unsigned gt = 0, eq = 0;
#pragma unroll
  for (int j = 0; j < kTopkPer; ++j) {
    if (j < cnt) {
      const unsigned long long k = tkey(v[j]);
      if (k > thr) gt |= 1u << j;
      else if (k == thr) eq |= 1u << j;
    }
  }
  long long rank = (long long)block_excl_scan1024((unsigned)__popc(eq), sc.warp, nullptr);
  unsigned sel = gt;
  while (eq) {
    const int b = __ffs(eq) - 1;
    eq &= eq - 1u;
    if (rank < need) sel |= 1u << b;
    ++rank;
  }
  *pos = block_excl_scan1024((unsigned)__popc(sel), sc.warp, total);
  return sel;
}

// Top-`num` bins of each segment as an ascending index list
// out[seg * out_stride + rank] (the location loops' top-d*k buckets,
// engine.py:122-127): one CTA per segment, seglen <= kTopkCtaMax.
template <typename T>
__global__ void __launch_bounds__(1024)
k_topk_list_seg(const T* __restrict__ vals, int seglen, long long num, int32_t* __restrict__ out,
                long out_stride) {
  pdl_wait();
  __shared__ TopkScratch sc;
  const int seg = blockIdx.x;
  const T* v0 = vals + (size_t)seg * seglen;
  const int per = (seglen + 1023) >> 10;
  const int e0 = min(seglen, (int)threadIdx.x * per);
  const int cnt = min(seglen, e0 + per) - e0;
  T v[kTopkPer];
#pragma unroll
  for (int j = 0; j < kTopkPer; ++j) v[j] = j < cnt ? v0[e0 + j] : (T)0;
  unsigned pos = 0;
  unsigned sel = block_topk_mask<T>(v, cnt, seglen, num, sc, &pos, nullptr);
  int32_t* o = out + (size_t)seg * out_stride;
  while (sel) {
    const int b = __ffs(sel) - 1;
    sel &= sel - 1u;
    o[pos++] = (int32_t)(e0 + b);
  }
}

}  // namespace sfft
