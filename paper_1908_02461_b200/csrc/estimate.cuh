// K6 / K7 — estimation and median-of-loops.
//   K6 replaces _estimate_arrays (engine.py:163-177): per coordinate (i, j) and
//      loop l:  q = sigma*i mod N,  u = floor((q + floor(w/2)) / w),
//      gain = F[(q_i - w u_i) mod N] * F[(q_j - w u_j) mod N],
//      val  = Z_l[u_i mod B, u_j mod B] * exp(-2 pi i ((tau1 i + tau2 j) mod N)/N) / gain
//      usable iff |gain| >= gain_floor (else 0 and excluded from the median).
//      The phase factor is tw[(tau1 i + tau2 j) mod N] from the same host table
//      (identical numpy expression, so identical values).
//   K7 replaces _median_select (engine.py:228-253): componentwise nan-median
//      over the usable loops (even count -> mean of the two middle values),
//      coordinates with no usable loop dropped, then top-k by |median| with
//      lexicographic (i, j) tie-break (select.cuh), then prune >= rel * max.
#pragma once
#include "common.cuh"
#include "select.cuh"

namespace sfft {

constexpr int kMaxLoops = 64;

template <typename T>
__global__ void k_estimate(const cplx<T>* __restrict__ spec, int nloops, const int32_t* __restrict__ keys,
                           const unsigned* __restrict__ m_dev, const Perm* __restrict__ perms,
                           int lgN, int lgB, const T* __restrict__ freq,
                           const cplx<T>* __restrict__ tw, double gain_floor,
                           cplx<T>* __restrict__ vals, uint8_t* __restrict__ usable, long stride,
                           bool natural_grid = false) {
  pdl_wait();
  using C = cplx<T>;
  const long m = *m_dev;
  const int N = 1 << lgN, B = 1 << lgB;
  const unsigned maskN = (unsigned)N - 1u, maskB = (unsigned)B - 1u;
  const int lgw = lgN - lgB;
  const unsigned hw = (unsigned)((1 << lgw) / 2);
  const long total = m * nloops;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x) {
    const int l = (int)(e / m);
    const long idx = e - (long)l * m;
    const Perm p = perms[l];
    const unsigned key = (unsigned)keys[idx];
    const unsigned i = key >> lgN, j = key & maskN;
    const unsigned qi = (p.s1 * i) & maskN, qj = (p.s2 * j) & maskN;
    const unsigned ui = (qi + hw) >> lgw, uj = (qj + hw) >> lgw;
    const unsigned oi = (qi - (ui << lgw)) & maskN, oj = (qj - (uj << lgw)) & maskN;
    const T gain = freq[oi] * freq[oj];
    const C ph = tw[(p.t1 * i + p.t2 * j) & maskN];
    C z;
    if (natural_grid) {
      // spec holds Y^ of the natural-order fold (coalesced fold writes): with
      // Z[a, b] = Y[s1 a + t1, s2 b + t2] (mod B),
      // Z^[a, b] = exp(+2 pi i (s1i t1 a + s2i t2 b) / B) Y^[s1i a, s2i b]
      const unsigned a = ui & maskB, b = uj & maskB;
      const unsigned ra = (p.s1i * a) & maskB, cb = (p.s2i * b) & maskB;
      const unsigned ex = (p.s1i * p.t1 * a + p.s2i * p.t2 * b) & maskB;
      const C w = tw[ex << lgw];
      z = cmul(spec[(size_t)l * B * B + (size_t)ra * B + cb], mk<T>(w.x, -w.y));
    } else {
      z = spec[(size_t)l * B * B + (size_t)(ui & maskB) * B + (uj & maskB)];
    }
    const bool ok = (double)fabs(gain) >= gain_floor;
    C v = cmul(z, ph);
    if (ok) { v.x = v.x / gain; v.y = v.y / gain; }
    else v = mk<T>(0, 0);
    vals[(size_t)l * stride + idx] = v;
    usable[(size_t)l * stride + idx] = ok ? 1 : 0;
  }
}

// B == N estimation shortcut: the all-pass window has gain 1 at every
// coordinate (freq = delta, offset 0) and Z_l[sigma*i, sigma*j] * phase_l
// equals x_hat[i, j] for every permutation (Lemma 1), so every loop's
// estimate is x_hat[i, j]: read it once.
template <typename T>
__global__ void k_estimate_dense(const cplx<T>* __restrict__ xhat, const int32_t* __restrict__ keys,
                                 const unsigned* __restrict__ m_dev, bool usable_all,
                                 cplx<T>* __restrict__ med, T* __restrict__ mags,
                                 uint8_t* __restrict__ alive, unsigned long long* __restrict__ peak) {
  pdl_wait();
  const long m = *m_dev;
  unsigned long long best = 0ull;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < m;
       i += (long)gridDim.x * blockDim.x) {
    const cplx<T> v = xhat[(uint32_t)keys[i]];
    med[i] = v;
    alive[i] = usable_all ? 1 : 0;
    const T a = usable_all ? cabs_(v) : (T)-1;
    mags[i] = a;
    if (usable_all) {
      const unsigned long long k = fkey(a);
      best = k > best ? k : best;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
    best = t > best ? t : best;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(peak, best);
}

// Same as k_estimate_dense, with x_hat[i, j] evaluated from the four-step
// factorisation instead of read from a stored spectrum: after the row pass and
// four-step pass A (twiddles applied), `A` row k1*L2 + n2 of column j holds
// the inputs of the length-L2 DFT that pass B would turn into rows
// k1 + L1*k2, so x_hat[k1 + L1 k2, j] = sum_n2 A[k1 L2 + n2, j] W_L2^(n2 k2)
// (W_L2^e = tw[e * N / L2]).  One warp per candidate, lanes split the n2 sum.
template <typename T>
__global__ void k_estimate_dense_fs(const cplx<T>* __restrict__ A, int lgN, int lgL1, int lgL2,
                                    const cplx<T>* __restrict__ tw,
                                    const int32_t* __restrict__ keys,
                                    const unsigned* __restrict__ m_dev, bool usable_all,
                                    cplx<T>* __restrict__ med, T* __restrict__ mags,
                                    uint8_t* __restrict__ alive,
                                    unsigned long long* __restrict__ peak) {
  pdl_wait();
  using C = cplx<T>;
  const long m = *m_dev;
  const int lane = threadIdx.x & 31;
  const long warps = (long)gridDim.x * (blockDim.x >> 5);
  const unsigned maskN = (1u << lgN) - 1u;
  const int L2 = 1 << lgL2;
  const int tsh = lgN - lgL2;
  unsigned long long best = 0ull;
  for (long q = blockIdx.x * (long)(blockDim.x >> 5) + (threadIdx.x >> 5); q < m; q += warps) {
    const unsigned key = (unsigned)keys[q];
    const unsigned i = key >> lgN, j = key & maskN;
    const unsigned k1 = i & ((1u << lgL1) - 1u), k2 = i >> lgL1;
    C s = mk<T>(0, 0);
    for (int n2 = lane; n2 < L2; n2 += 32) {
      const C a = A[((size_t)((k1 << lgL2) + n2) << lgN) + j];
      s = cadd(s, cmul(a, tw[((n2 * k2) & (L2 - 1)) << tsh]));
    }
    for (int o = 16; o > 0; o >>= 1) {
      s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
    }
    if (lane == 0) {
      med[q] = s;
      alive[q] = usable_all ? 1 : 0;
      const T a = usable_all ? cabs_(s) : (T)-1;
      mags[q] = a;
      if (usable_all) {
        const unsigned long long k = fkey(a);
        best = k > best ? k : best;
      }
    }
  }
  if (lane == 0 && best) atomicMax(peak, best);
}

// Estimation from the dense spectrum (B < N with an untruncated window,
// S(B) = N): the hashed spectrum is the spectrum of g . y (y = permuted x,
// g = space window), i.e. the circular convolution of y^ with g^ = N F
// (F = freq row, DC-normalised; g sums to N), sampled at k w:
//   Z^[k1, k2] = sum_{d1, d2} F[d1] F[d2] y^[k1 w - d1, k2 w - d2],
//   y^[f1, f2] = e^{+2 pi i (f1 s1i t1 + f2 s2i t2) / N} x^[s1i f1, s2i f2].
// With q = s i = w u + o (the bucket u and offset o of _estimate_arrays,
// engine.py:163-177) and e = o + d, the reference's value
// Z^[u_i, u_j] e^{-2 pi i (t1 i + t2 j)/N} / (F[o_i] F[o_j]) is exactly
//   sum_{d1, d2} F[d1] F[d2] tw[t1 s1i e1 + t2 s2i e2] x^[i - s1i e1, j - s2i e2] / gain.
// F[d] vanishes (below 1e-14, roundoff of the host table) for |d| > R, R = 2
// at w = 2: 25 gathers of x^ per (candidate, loop) instead of a fold of x and
// a B x B FFT per loop.  Same usable/gain rule as k_estimate.
template <typename T, int R>
__global__ void k_estimate_conv(const cplx<T>* __restrict__ xhat, int nloops,
                                const int32_t* __restrict__ keys, const unsigned* __restrict__ m_dev,
                                const Perm* __restrict__ perms, int lgN, int lgB,
                                const T* __restrict__ freq, const cplx<T>* __restrict__ tw,
                                double gain_floor, cplx<T>* __restrict__ vals,
                                uint8_t* __restrict__ usable, long stride) {
  pdl_wait();
  using C = cplx<T>;
  constexpr int K = 2 * R + 1;
  const long m = *m_dev;
  const unsigned maskN = (1u << lgN) - 1u;
  const int lgw = lgN - lgB;
  const unsigned hw = (unsigned)((1 << lgw) / 2);
  const long total = m * nloops;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x) {
    const int l = (int)(e / m);
    const long idx = e - (long)l * m;
    const Perm p = perms[l];
    const unsigned key = (unsigned)keys[idx];
    const unsigned i = key >> lgN, j = key & maskN;
    const unsigned qi = (p.s1 * i) & maskN, qj = (p.s2 * j) & maskN;
    const unsigned ui = (qi + hw) >> lgw, uj = (qj + hw) >> lgw;
    const unsigned oi = (qi - (ui << lgw)) & maskN, oj = (qj - (uj << lgw)) & maskN;
    const T gain = freq[oi] * freq[oj];
    const bool ok = (double)fabs(gain) >= gain_floor;
    C v = mk<T>(0, 0);
    if (ok) {
      unsigned rowo[K];
      C c2[K];
      unsigned colv[K];
#pragma unroll
      for (int d = 0; d < K; ++d) {
        const unsigned e1 = (oi + (unsigned)(d - R)) & maskN;
        rowo[d] = ((i - p.s1i * e1) & maskN) << lgN;
        const unsigned e2 = (oj + (unsigned)(d - R)) & maskN;
        colv[d] = (j - p.s2i * e2) & maskN;
        const T f2 = freq[(unsigned)(d - R) & maskN];
        const C t2 = tw[(p.t2 * p.s2i * e2) & maskN];
        c2[d] = mk<T>(f2 * t2.x, f2 * t2.y);
      }
      C acc = mk<T>(0, 0);
#pragma unroll
      for (int d1 = 0; d1 < K; ++d1) {
        C inner = mk<T>(0, 0);
#pragma unroll
        for (int d2 = 0; d2 < K; ++d2) inner = cadd(inner, cmul(c2[d2], xhat[(size_t)rowo[d1] + colv[d2]]));
        const unsigned e1 = (oi + (unsigned)(d1 - R)) & maskN;
        const T f1 = freq[(unsigned)(d1 - R) & maskN];
        const C t1 = tw[(p.t1 * p.s1i * e1) & maskN];
        acc = cadd(acc, cmul(mk<T>(f1 * t1.x, f1 * t1.y), inner));
      }
      v = mk<T>(acc.x / gain, acc.y / gain);
    }
    vals[(size_t)l * stride + idx] = v;
    usable[(size_t)l * stride + idx] = ok ? 1 : 0;
  }
}

template <typename T>
__device__ __forceinline__ void isort(T* a, int n) {
  for (int i = 1; i < n; ++i) {
    const T v = a[i];
    int j = i - 1;
    while (j >= 0 && a[j] > v) { a[j + 1] = a[j]; --j; }
    a[j + 1] = v;
  }
}

template <typename T>
__device__ __forceinline__ T median_sorted(const T* a, int n) {
  return (n & 1) ? a[n / 2] : (a[n / 2 - 1] + a[n / 2]) / (T)2;
}

// componentwise median; dead coordinates get mag = -1.  The reference masks
// unusable loops with np.where(usable, vals, np.nan) on a COMPLEX array
// (engine.py:241-242): the fill value is nan + 0j, so np.nanmedian skips those
// loops for the real part but sees 0.0 for the imaginary part.  Restated as it
// is: real median over the usable loops, imaginary median over all loops with
// 0 where a loop is unusable (identical when every loop is usable, which is
// the case whenever gain_floor is below the window's passband gain).
template <typename T>
__global__ void k_median(const cplx<T>* __restrict__ vals, const uint8_t* __restrict__ usable,
                         int nloops, long stride, const unsigned* __restrict__ m_dev,
                         cplx<T>* __restrict__ med, T* __restrict__ mags,
                         uint8_t* __restrict__ alive, unsigned* __restrict__ alive_count,
                         unsigned long long* __restrict__ peak) {
  pdl_wait();
  const long m = *m_dev;
  unsigned cnt_alive = 0;
  unsigned long long best = 0ull;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < m;
       i += (long)gridDim.x * blockDim.x) {
    T re[kMaxLoops], im[kMaxLoops];
    int c = 0;
    for (int l = 0; l < nloops; ++l) {
      if (usable[(size_t)l * stride + i]) {
        const cplx<T> v = vals[(size_t)l * stride + i];
        re[c] = v.x;
        im[l] = v.y;
        ++c;
      } else {
        im[l] = (T)0;
      }
    }
    if (c == 0) {
      alive[i] = 0;
      mags[i] = (T)-1;
      med[i] = mk<T>(0, 0);
      continue;
    }
    isort(re, c);
    isort(im, nloops);
    const cplx<T> v = mk<T>(median_sorted(re, c), median_sorted(im, nloops));
    med[i] = v;
    alive[i] = 1;
    const T a = cabs_(v);
    mags[i] = a;
    ++cnt_alive;
    const unsigned long long k = fkey(a);
    best = k > best ? k : best;
  }
  for (int o = 16; o > 0; o >>= 1) {
    cnt_alive += __shfl_xor_sync(0xffffffffu, cnt_alive, o);
    unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
    best = t > best ? t : best;
  }
  if ((threadIdx.x & 31) == 0) {
    if (cnt_alive) atomicAdd(alive_count, cnt_alive);
    atomicMax(peak, best);
  }
}

// Final keep-bitmask: alive, selected by top-k (sel bits, or all when no cut),
// and |med| >= prune_rel * peak (when prune_rel > 0).
template <typename T>
__global__ void k_final_bits(const T* __restrict__ mags, const uint8_t* __restrict__ alive,
                             const uint32_t* __restrict__ sel_bits, long m,
                             const unsigned long long* __restrict__ peak, double prune_rel,
                             uint32_t* __restrict__ bits, unsigned* __restrict__ blk_counts) {
  pdl_wait();
  __shared__ unsigned s_warp[32];
  const long w = (long)blockIdx.x * kCmpWords + threadIdx.x;
  const long wps = words_for(m);
  const double floor_v = prune_rel > 0 ? prune_rel * fkey_inv(*peak) : -1.0;
  uint32_t word = 0;
  if (w < wps) {
    const uint32_t sel = sel_bits ? sel_bits[w] : 0xffffffffu;
    for (int b = 0; b < 32; ++b) {
      const long i = w * 32 + b;
      if (i < m && alive[i] && ((sel >> b) & 1u)) {
        if (prune_rel <= 0 || (double)mags[i] >= floor_v) word |= 1u << b;
      }
    }
    bits[w] = word;
  }
  const unsigned pre = block_excl_scan256(__popc(word), s_warp);
  if (threadIdx.x == kCmpThreads - 1) blk_counts[blockIdx.x] = pre + __popc(word);
}

// gather the kept entries (positions from compaction) into (i, j) and values
template <typename T>
__global__ void k_gather_out(const int32_t* __restrict__ pos, const unsigned* __restrict__ count,
                             const int32_t* __restrict__ keys, const cplx<T>* __restrict__ med,
                             int lgN, int64_t* __restrict__ out_ij, cplx<T>* __restrict__ out_v) {
  pdl_wait();
  const long n = *count;
  const unsigned maskN = (1u << lgN) - 1u;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    const int32_t p = pos[i];
    const unsigned key = (unsigned)keys[p];
    out_ij[2 * i] = key >> lgN;
    out_ij[2 * i + 1] = key & maskN;
    out_v[i] = med[p];
  }
}

// Fused K6 + K7 tail for a dense (B == N) estimate of a small candidate set
// with no top-k cut (engine.py:163-253 with b_estimate = N): ONE CTA reads
// x_hat at the m candidates (every loop's estimate is x_hat[i, j], see
// k_estimate_dense), takes the peak |v|, prunes against prune_rel * peak,
// compacts the survivors in key order and writes (i, j), values and the count
// straight into mapped host memory.  m is read from device memory, so the
// launch does not wait for the host to learn the candidate count: when
// m > limit (the host sized the launch for at most `limit` candidates, and
// limit <= k guarantees that no cut is needed) the kernel only reports m and
// the host takes the general path.  Publication: slot[2] = m, slot[3] = the
// NaN/Inf flag of the input scan, then (count, seq) as one 8-byte word after
// a system fence — the host spins on seq (no stream synchronisation).  Same
// predicate and order as k_estimate_dense + k_final_bits + compaction +
// k_gather_out.
constexpr unsigned kFinishSmallBytes = 128 * 1024;   // shared copy of the candidates' values
constexpr unsigned kFinishFallback = 0xffffffffu;
template <typename T>
constexpr unsigned finish_small_max() { return kFinishSmallBytes / (unsigned)sizeof(cplx<T>); }

template <typename T>
__global__ void __launch_bounds__(1024)
k_finish_dense_small(const cplx<T>* __restrict__ xhat, const int32_t* __restrict__ keys,
                     const unsigned* __restrict__ blk_counts, int nblk, unsigned* __restrict__ m_out,
                     unsigned limit, bool usable_all,
                     double prune_rel, const unsigned* __restrict__ nonfinite, int lgN,
                     int64_t* __restrict__ out_ij, cplx<T>* __restrict__ out_v,
                     volatile unsigned* slot, unsigned seq) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx<T>* s_v = reinterpret_cast<cplx<T>*>(smem_raw);   // [limit] x_hat at the candidates
  __shared__ unsigned long long s_best[32];
  __shared__ unsigned s_warp[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // m = the sum of the compaction's block counts (no scan launch before this
  // kernel), also stored for the general path's kernels
  unsigned msum = 0;
  for (int b = tid; b < nblk; b += blockDim.x) msum += blk_counts[b];
  for (int o = 16; o > 0; o >>= 1) msum += __shfl_xor_sync(0xffffffffu, msum, o);
  if (lane == 0) s_warp[warp] = msum;
  __syncthreads();
  msum = s_warp[lane];
  for (int o = 16; o > 0; o >>= 1) msum += __shfl_xor_sync(0xffffffffu, msum, o);
  __syncthreads();                                    // s_warp is reused below
  const unsigned m = msum;
  if (tid == 0) *m_out = m;
  const unsigned bad = nonfinite ? *nonfinite : 0u;
  // m and the NaN flag go to the slot first; the system fence that orders
  // them (and the results) before the (count, seq) word is the one at the end
  if (tid == 0) {
    slot[2] = m;
    slot[3] = bad;
  }
  auto publish = [&](unsigned count) {   // thread 0, after a system fence behind every output write
    *reinterpret_cast<volatile unsigned long long*>(slot) =
        ((unsigned long long)count << 32) | (unsigned long long)seq;
  };
  if (m > limit || m == 0u || bad || !usable_all) {   // block-uniform
    if (tid == 0) {
      __threadfence_system();
      publish(m > limit ? kFinishFallback : 0u);
    }
    return;
  }
  // gather: candidates interleaved over the threads (coalesced key reads),
  // every x_hat read of a thread in flight at once (one latency round)
  constexpr int kPerMax = (int)(kFinishSmallBytes / sizeof(cplx<T>) / 1024u);
  unsigned long long best = 0ull;
  {
    cplx<T> v[kPerMax];
#pragma unroll
    for (int j = 0; j < kPerMax; ++j) {
      const unsigned i = (unsigned)j * 1024u + (unsigned)tid;
      if (i < m) v[j] = xhat[(uint32_t)keys[i]];
    }
#pragma unroll
    for (int j = 0; j < kPerMax; ++j) {
      const unsigned i = (unsigned)j * 1024u + (unsigned)tid;
      if (i < m) {
        s_v[i] = v[j];
        const unsigned long long k = fkey(cabs_(v[j]));
        best = k > best ? k : best;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
    best = t > best ? t : best;
  }
  if (lane == 0) s_best[warp] = best;
  __syncthreads();                                    // s_v and s_best complete
  best = s_best[lane];
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
    best = t > best ? t : best;
  }
  const double floor_v = prune_rel > 0 ? prune_rel * fkey_inv(best) : -1.0;
  // ordered compaction: a contiguous run of candidates per thread
  const unsigned per = (m + 1023u) >> 10;            // <= 16 (fp32) / 8 (fp64)
  const unsigned i0 = min(m, (unsigned)tid * per), i1 = min(m, i0 + per);
  unsigned keep = 0;                                  // bit j: candidate i0 + j survives
  for (unsigned i = i0; i < i1; ++i) {
    const T a = cabs_(s_v[i]);
    if (prune_rel <= 0 || (double)a >= floor_v) keep |= 1u << (i - i0);
  }
  const unsigned cnt = (unsigned)__popc(keep);
  const unsigned inc = warp_incl_scan(cnt);
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) s_warp[lane] = warp_incl_scan(s_warp[lane]);
  __syncthreads();
  unsigned pos = inc - cnt + (warp ? s_warp[warp - 1] : 0u);
  const unsigned total = s_warp[31];
  const unsigned maskN = (1u << lgN) - 1u;
  while (keep) {
    const unsigned j = (unsigned)__ffs(keep) - 1u;
    keep &= keep - 1u;
    const unsigned key = (unsigned)keys[i0 + j];
    out_ij[2 * (size_t)pos] = key >> lgN;
    out_ij[2 * (size_t)pos + 1] = key & maskN;
    out_v[pos] = s_v[i0 + j];
    ++pos;
  }
  if (cnt || tid == 0) __threadfence_system();   // results, m and the flag land before the count
  __syncthreads();
  if (tid == 0) publish(total);
}


// Fused K7 tail (engine.py:228-253) for up to kTopkCtaMax candidates, ONE CTA:
// the exact top-k cut when more than k coordinates are alive (dead ones carry
// magnitude -1; block_topk_mask), the prune against prune_rel * peak, the
// ordered compaction and the gather of (i, j) / values into mapped host
// memory, then (count, seq) published to the slot the host spins on with the
// alive count in slot[2] (it decides the output order flag).  Replaces
// k_sel_init, k_radix_select_seg, k_tie_counts, k_select_bits, k_final_bits,
// two scans, the compaction, k_gather_out and the final stream
// synchronisation.  n_alive_host < 0: the alive count is read from
// alive_cnt (written by k_median).
template <typename T>
__global__ void __launch_bounds__(1024)
k_finish_cut_small(const cplx<T>* __restrict__ med, const T* __restrict__ mags,
                   const uint8_t* __restrict__ alive, int m, long long k, double prune_rel,
                   const unsigned long long* __restrict__ peak, long long n_alive_host,
                   const unsigned* __restrict__ alive_cnt, const int32_t* __restrict__ keys, int lgN,
                   int64_t* __restrict__ out_ij, cplx<T>* __restrict__ out_v,
                   volatile unsigned* slot, unsigned seq) {
  pdl_wait();
  __shared__ TopkScratch sc;
  const int tid = threadIdx.x;
  const long long n_alive = n_alive_host >= 0 ? n_alive_host : (long long)*alive_cnt;
  const int per = (m + 1023) >> 10;
  const int e0 = min(m, tid * per);
  const int cnt = min(m, e0 + per) - e0;
  T v[kTopkPer];
#pragma unroll
  for (int j = 0; j < kTopkPer; ++j) v[j] = j < cnt ? mags[e0 + j] : (T)-1;
  unsigned sel = cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u);
  unsigned dummy = 0;
  if (n_alive > k) sel = block_topk_mask<T>(v, cnt, m, k, sc, &dummy, nullptr);   // block-uniform
  const double floor_v = prune_rel > 0 ? prune_rel * fkey_inv(*peak) : -1.0;
  unsigned keep = 0;
#pragma unroll
  for (int j = 0; j < kTopkPer; ++j) {
    if (j < cnt && ((sel >> j) & 1u) && alive[e0 + j] &&
        (prune_rel <= 0 || (double)v[j] >= floor_v))
      keep |= 1u << j;
  }
  unsigned total = 0;
  unsigned pos = block_excl_scan1024((unsigned)__popc(keep), sc.warp, &total);
  const unsigned maskN = (1u << lgN) - 1u;
  const bool any = keep != 0u;
  if (tid == 0) slot[2] = (unsigned)n_alive;   // ordered before the count by the fence below
  while (keep) {
    const int j = __ffs(keep) - 1;
    keep &= keep - 1u;
    const unsigned key = (unsigned)keys[e0 + j];
    out_ij[2 * (size_t)pos] = key >> lgN;
    out_ij[2 * (size_t)pos + 1] = key & maskN;
    out_v[pos] = med[e0 + j];
    ++pos;
  }
  if (any || tid == 0) __threadfence_system();   // results and alive count land before the count
  __syncthreads();
  if (tid == 0) {
    *reinterpret_cast<volatile unsigned long long*>(slot) =
        ((unsigned long long)total << 32) | (unsigned long long)seq;
  }
}

}  // namespace sfft
