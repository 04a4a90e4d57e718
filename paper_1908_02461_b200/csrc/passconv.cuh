// Tuner pass at B = N/2 from the dense spectrum (restatement of
// binned_spectrum + |.|, hashing.py:308-337, for the one bin count where it
// is cheaper than the fold + B x B FFT).
//
// At B = N/2 the window is untruncated (S(B) = N), so the hashed spectrum of
// permutation p is the circular convolution of the permuted spectrum with the
// window's response F (DC-normalised, host table; |F[d]| <= 1e-14 for
// |d| > 2 at w = 2; in fp32 the |d| = 2 taps, |F| = 2.5e-9, are below the
// arithmetic's resolution and R = 1):
//   Z^[k1, k2] = sum_{d1, d2 in [-2, 2]} F[d1] F[d2] y^[2 k1 - d1, 2 k2 - d2],
//   y^[f1, f2] = e^{+2 pi i (f1 a1 + f2 a2)/N} x^[s1i f1, s2i f2],  a = s_inv * tau.
// The tuner only needs |Z^|; dropping the unit factor e^{2 pi i 2 (k1 a1 + k2 a2)/N}
//   |Z^[k1, k2]| = | sum_{d1} c1[d1] sum_{d2} c2[d2] x^[s1i (2 k1 - d1), s2i (2 k2 - d2)] |,
//   c[d] = F[d] e^{-2 pi i d a / N}.
// CTA = RB consecutive output rows k1: it streams the 2 RB + 3 source rows
// e = 2 k1 - d1 (natural rows s1i e of x^, whole rows, TMA bulk copies into a
// ring of shared-memory slots), gathers the 5 column taps of its CPT output
// columns per source row once, and adds them with weight c1[d1] to each of the
// (up to 3) output rows that source row feeds.  x^ is read ~(2 RB + 3)/(2 RB)
// times instead of the image once plus three passes over the B x B grid.
// Output: |Z^| in bucket order (so the local-maximum test uses the identity
// view) and the grid's peak key.
#pragma once
#include "common.cuh"

namespace sfft {

template <typename T, int CPT, int RB, int NS, int R>
__global__ void __launch_bounds__(256)
k_pass_conv(const cplx<T>* __restrict__ xhat, int lgN, Perm p, const T* __restrict__ freq,
            const cplx<T>* __restrict__ tw, T* __restrict__ mags,
            unsigned long long* __restrict__ peak) {
  pdl_wait();
  using C = cplx<T>;
  __shared__ __align__(8) unsigned long long s_bar[NS];
  extern __shared__ __align__(128) unsigned char smem_raw[];
  C* ring = reinterpret_cast<C*>(smem_raw);
  const int N = 1 << lgN;
  const int B = N >> 1;
  const unsigned maskN = (unsigned)N - 1u;
  const int tid = threadIdx.x;
  const int k10 = blockIdx.x * RB;
  const unsigned s1i = p.s1i, s2i = p.s2i;
  const unsigned a1 = (s1i * p.t1) & maskN, a2 = (s2i * p.t2) & maskN;
  // row taps in shared memory (indexed by the runtime d1 below), column taps
  // in registers
  constexpr int K = 2 * R + 1;
  __shared__ C s_c1[K];
  C c2[K];
#pragma unroll
  for (int d = 0; d < K; ++d) {
    const unsigned dd = (unsigned)(d - R);
    const T f = freq[dd & maskN];
    const C t2 = tw[(dd * a2) & maskN];
    c2[d] = mk<T>(f * t2.x, f * t2.y);
    if (tid == d) {
      const C t1 = tw[(dd * a1) & maskN];
      s_c1[d] = mk<T>(f * t1.x, f * t1.y);
    }
  }
  // output column k2 = q * blockDim + tid: coalesced stores
  unsigned cbase[CPT];
#pragma unroll
  for (int q = 0; q < CPT; ++q) cbase[q] = (s2i * 2u * (unsigned)(q * blockDim.x + tid)) & maskN;
  C acc[RB][CPT];
#pragma unroll
  for (int j = 0; j < RB; ++j)
#pragma unroll
    for (int q = 0; q < CPT; ++q) acc[j][q] = mk<T>(0, 0);

  constexpr int NE = 2 * (RB - 1) + 2 * R + 1;   // source rows e = 2 k10 - R ... 2 (k10 + RB - 1) + R
  const unsigned rowbytes = (unsigned)(N * sizeof(C));
  if (tid < NS) mbar_init(&s_bar[tid], 1);
  mbar_fence_init();
  __syncthreads();
  auto issue = [=](int ei) {
    const unsigned e = (unsigned)(2 * k10 - R + ei);
    const unsigned r = (s1i * e) & maskN;
    const int slot = ei % NS;
    mbar_expect_tx(&s_bar[slot], rowbytes);
    bulk_g2s(ring + (size_t)slot * N, xhat + ((size_t)r << lgN), rowbytes, &s_bar[slot]);
  };
  if (tid == 0)
    for (int i = 0; i < NS && i < NE; ++i) issue(i);
  for (int ei = 0; ei < NE; ++ei) {
    const int slot = ei % NS;
    mbar_wait(&s_bar[slot], (unsigned)(ei / NS) & 1u);
    const C* row = ring + (size_t)slot * N;
    C g[CPT];
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      C s = mk<T>(0, 0);
#pragma unroll
      for (int d = 0; d < K; ++d) {
        const C v = row[(cbase[q] - s2i * (unsigned)(d - R)) & maskN];
        s.x = fma(c2[d].x, v.x, fma(-c2[d].y, v.y, s.x));
        s.y = fma(c2[d].x, v.y, fma(c2[d].y, v.x, s.y));
      }
      g[q] = s;
    }
    // source row e = 2 k1 - d1 feeds output rows k1 = k10 + j with d1 = 2 (k10 + j) - e
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      const int d1 = 2 * j + R - ei;   // 2 (k10 + j) - (2 k10 - R + ei)
      if (d1 < -R || d1 > R) continue;
      const C w = s_c1[d1 + R];
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        acc[j][q].x = fma(w.x, g[q].x, fma(-w.y, g[q].y, acc[j][q].x));
        acc[j][q].y = fma(w.x, g[q].y, fma(w.y, g[q].x, acc[j][q].y));
      }
    }
    __syncthreads();   // every thread is done with this slot
    if (tid == 0 && ei + NS < NE) issue(ei + NS);
  }
  unsigned long long best = 0ull;
#pragma unroll
  for (int j = 0; j < RB; ++j)
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const T m = mag_(acc[j][q]);
      mags[(size_t)(k10 + j) * B + q * blockDim.x + tid] = m;
      const unsigned long long k = fkey(m);
      best = k > best ? k : best;
    }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
    best = t > best ? t : best;
  }
  if ((tid & 31) == 0) atomicMax(peak, best);
}


// k_pass_conv over a BAND of `nb` consecutive output rows per CTA, sized by
// the host for one wave of resident CTAs (c3: 293 CTAs of 7 rows instead of
// 512 CTAs of 4 rows on 296 slots, a 1.73-wave grid with a 27% tail).  The
// source rows stream through the same TMA ring in ascending order; only the
// R + 1 output rows that the current source row can feed are open at a time
// (acc[0] = the oldest), so the accumulators do not grow with the band, a
// finished row is written as soon as its last source row (e = 2 k1 + R) has
// been added, and a source row is tested against R + 1 rows instead of RB.
// Each output row receives its taps in the same ascending-e order and with
// the same expressions as in k_pass_conv: bit-identical |Z^|.  The halo
// (2 R rows per band) shrinks from (2 RB + 2 R - 1) / (2 RB) to
// (2 nb + 2 R - 1) / (2 nb) of x^.
template <typename T, int CPT, int NS, int R>
__global__ void __launch_bounds__(256)
k_pass_conv_band(const cplx<T>* __restrict__ xhat, int lgN, Perm p, const T* __restrict__ freq,
                 const cplx<T>* __restrict__ tw, int nb, T* __restrict__ mags,
                 unsigned long long* __restrict__ peak) {
  pdl_wait();
  using C = cplx<T>;
  __shared__ __align__(8) unsigned long long s_bar[NS];
  extern __shared__ __align__(128) unsigned char smem_raw[];
  C* ring = reinterpret_cast<C*>(smem_raw);
  const int N = 1 << lgN;
  const int B = N >> 1;
  const unsigned maskN = (unsigned)N - 1u;
  const int tid = threadIdx.x;
  const int k10 = blockIdx.x * nb;
  const int nbc = min(nb, B - k10);
  const unsigned s1i = p.s1i, s2i = p.s2i;
  const unsigned a1 = (s1i * p.t1) & maskN, a2 = (s2i * p.t2) & maskN;
  constexpr int K = 2 * R + 1;
  constexpr int NA = R + 1;
  __shared__ C s_c1[K];
  C c2[K];
#pragma unroll
  for (int d = 0; d < K; ++d) {
    const unsigned dd = (unsigned)(d - R);
    const T f = freq[dd & maskN];
    const C t2 = tw[(dd * a2) & maskN];
    c2[d] = mk<T>(f * t2.x, f * t2.y);
    if (tid == d) {
      const C t1 = tw[(dd * a1) & maskN];
      s_c1[d] = mk<T>(f * t1.x, f * t1.y);
    }
  }
  unsigned cbase[CPT];
#pragma unroll
  for (int q = 0; q < CPT; ++q) cbase[q] = (s2i * 2u * (unsigned)(q * blockDim.x + tid)) & maskN;
  C acc[NA][CPT];
#pragma unroll
  for (int a = 0; a < NA; ++a)
#pragma unroll
    for (int q = 0; q < CPT; ++q) acc[a][q] = mk<T>(0, 0);

  const int NE = 2 * (nbc - 1) + 2 * R + 1;   // source rows e = 2 k10 - R ... 2 (k10 + nbc - 1) + R
  const unsigned rowbytes = (unsigned)(N * sizeof(C));
  if (tid < NS) mbar_init(&s_bar[tid], 1);
  mbar_fence_init();
  __syncthreads();
  auto issue = [=](int ei) {
    const unsigned e = (unsigned)(2 * k10 - R + ei);
    const unsigned r = (s1i * e) & maskN;
    const int slot = ei % NS;
    mbar_expect_tx(&s_bar[slot], rowbytes);
    bulk_g2s(ring + (size_t)slot * N, xhat + ((size_t)r << lgN), rowbytes, &s_bar[slot]);
  };
  if (tid == 0)
    for (int i = 0; i < NS && i < NE; ++i) issue(i);
  unsigned long long best = 0ull;
  int kcur = 0;                                // acc[a] = output row k10 + kcur + a
  int slot = 0;
  unsigned phase = 0;
  for (int ei = 0; ei < NE; ++ei) {
    mbar_wait(&s_bar[slot], (phase >> slot) & 1u);
    phase ^= 1u << slot;
    const C* row = ring + (size_t)slot * N;
    C g[CPT];
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      C s = mk<T>(0, 0);
#pragma unroll
      for (int d = 0; d < K; ++d) {
        const C v = row[(cbase[q] - s2i * (unsigned)(d - R)) & maskN];
        s.x = fma(c2[d].x, v.x, fma(-c2[d].y, v.y, s.x));
        s.y = fma(c2[d].x, v.y, fma(c2[d].y, v.x, s.y));
      }
      g[q] = s;
    }
    const int erel = ei - R;                   // source row e = 2 k10 + erel
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      const int j = kcur + a;
      const int d1 = 2 * j - erel;
      if (j >= nbc || d1 < -R || d1 > R) continue;   // block-uniform
      const C w = s_c1[d1 + R];
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        acc[a][q].x = fma(w.x, g[q].x, fma(-w.y, g[q].y, acc[a][q].x));
        acc[a][q].y = fma(w.x, g[q].y, fma(w.y, g[q].x, acc[a][q].y));
      }
    }
    __syncthreads();   // every thread is done with this slot
    if (tid == 0 && ei + NS < NE) issue(ei + NS);
    slot = slot + 1 == NS ? 0 : slot + 1;
    if (erel == 2 * kcur + R) {                // output row k10 + kcur is complete
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const T m = mag_(acc[0][q]);
        mags[(size_t)(k10 + kcur) * B + q * blockDim.x + tid] = m;
        const unsigned long long k = fkey(m);
        best = k > best ? k : best;
      }
#pragma unroll
      for (int a = 0; a + 1 < NA; ++a)
#pragma unroll
        for (int q = 0; q < CPT; ++q) acc[a][q] = acc[a + 1][q];
#pragma unroll
      for (int q = 0; q < CPT; ++q) acc[NA - 1][q] = mk<T>(0, 0);
      ++kcur;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
    best = t > best ? t : best;
  }
  if ((tid & 31) == 0) atomicMax(peak, best);
}

}  // namespace sfft
