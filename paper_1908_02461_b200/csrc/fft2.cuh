// K2 (large grids) — Stockham radix-16 FFT passes for B x B grids and the
// dense N x N image (replaces corefft.fft2d, corefft.py:101-109, for B >= 128).
//
// One 1D transform of length L runs in shared memory as Stockham autosort
// passes: every thread owns exactly 16 complex registers per pass — one
// radix-16 butterfly group, or 16/R groups of a smaller radix R for the last
// pass — so a pass is: load (smem), twiddle W_{Ns*R}^{(j mod Ns) r}, R-point
// DFT in registers with compile-time constant twiddles, store (smem).  Rows
// in shared memory use a padded index i + i/16 (+1 per row) so both the
// strided loads and the scattered Stockham stores are bank-conflict free.
//
// 2D grid = row pass + column pass.  Column pass: for L <= 512 a CTA stages
// `cc` adjacent columns (>= 128 B per row segment) and transforms them in
// smem; for L > 512 the columns use the four-step split L = L1 * L2:
//   pass A (in place): length-L1 DFTs over rows n2 + L2*n1, twiddle W_L^{n2 k1}
//   pass B (out of place): length-L2 DFTs over the contiguous rows L2*k1 + n2,
//                          written to row k1 + L1*k2.
// The final pass can write |Z| (np.abs == hypot) and a per-grid peak
// (order-independent atomicMax on an order-preserving key) instead of, or in
// addition to, the complex spectrum: the tuner only needs magnitudes.
#pragma once
#include <type_traits>
#include <utility>
#include <cooperative_groups.h>
#include "common.cuh"

namespace sfft {

__device__ __forceinline__ int padi(int i) { return i + (i >> 4); }
__host__ __device__ inline int pad_row(int L) { return L + (L >> 4) + 1; }

// cos/sin(2*pi*k/16), k = 0..15
__device__ __forceinline__ double c16(int k) {
  constexpr double t[16] = {1.0, 0.92387953251128674, 0.70710678118654757, 0.38268343236508978,
                            0.0, -0.38268343236508978, -0.70710678118654757, -0.92387953251128674,
                            -1.0, -0.92387953251128674, -0.70710678118654757, -0.38268343236508978,
                            0.0, 0.38268343236508978, 0.70710678118654757, 0.92387953251128674};
  return t[k & 15];
}
__device__ __forceinline__ double s16(int k) { return c16(k + 12); }  // sin(x) = cos(x - pi/2)

template <typename C>
__device__ __forceinline__ C mul_negi(C a) {  // a * (-i)
  C z; z.x = a.y; z.y = -a.x; return z;
}

// v[r] *= w^r for r = 1..R-1 from one table twiddle w: powers by repeated
// squaring / products (<= 3 roundings deep), instead of R-1 table loads.
template <typename T, int R>
__device__ __forceinline__ void twiddle_powers(cplx<T>* v, cplx<T> w) {
  using C = cplx<T>;
  C p[16];
  p[1] = w;
#pragma unroll
  for (int r = 2; r < R; ++r) p[r] = (r & 1) ? cmul(p[r - 1], w) : cmul(p[r >> 1], p[r >> 1]);
#pragma unroll
  for (int r = 1; r < R; ++r) v[r] = cmul(v[r], p[r]);
}

// forward R-point DFT in registers (natural order in and out), R in {2,4,8,16}
template <typename T, int R>
__device__ __forceinline__ void dft_reg(cplx<T>* v) {
  using C = cplx<T>;
  // bit reversal
#pragma unroll
  for (int i = 0; i < R; ++i) {
    int j = 0;
#pragma unroll
    for (int b = 1, ib = i; b < R; b <<= 1, ib >>= 1) j = (j << 1) | (ib & 1);
    if (j > i) { C t = v[i]; v[i] = v[j]; v[j] = t; }
  }
#pragma unroll
  for (int h = 1; h < R; h <<= 1) {
#pragma unroll
    for (int k = 0; k < R; k += 2 * h) {
#pragma unroll
      for (int j = 0; j < h; ++j) {
        const int e = j * (16 / (2 * h));  // W_{2h}^j = W_16^e
        C t = v[k + j + h];
        if (e == 4) {
          t = mul_negi(t);
        } else if (e != 0) {
          C w;
          w.x = (T)c16(e);
          w.y = (T)-s16(e);
          t = cmul(t, w);
        }
        v[k + j + h] = csub(v[k + j], t);
        v[k + j] = cadd(v[k + j], t);
      }
    }
  }
}

// One Stockham pass of radix 2^LGR over `rows` rows (stride rs) of length 2^lgL.
// blockDim.x * 16 == rows * L must hold.
template <typename T, int LGR, int IPT = 1>
__device__ __forceinline__ void stockham_pass(cplx<T>* s, int lgL, int rs, int lgNs,
                                              const cplx<T>* __restrict__ tw, int lgN) {
  using C = cplx<T>;
  constexpr int R = 1 << LGR;
  constexpr int K = IPT * 16 / R;
  const int per_lg = lgL - LGR;
  const int per = 1 << per_lg;
  C v[16 * IPT];
#pragma unroll
  for (int q = 0; q < K; ++q) {
    const int it = threadIdx.x + q * blockDim.x;
    const int row = it >> per_lg, j = it & (per - 1);
    const C* sr = s + row * rs;
#pragma unroll
    for (int r = 0; r < R; ++r) v[q * R + r] = sr[padi(j + r * per)];
  }
  __syncthreads();
  const int Ns = 1 << lgNs;
  const int tsh = lgN - lgNs - LGR;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    const int it = threadIdx.x + q * blockDim.x;
    const int row = it >> per_lg, j = it & (per - 1);
    const int jm = j & (Ns - 1);
    if (lgNs > 0) twiddle_powers<T, R>(&v[q * R], __ldg(tw + (jm << tsh)));
    dft_reg<T, R>(&v[q * R]);
    C* sr = s + row * rs;
    const int base = ((j >> lgNs) << (lgNs + LGR)) + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) sr[padi(base + r * Ns)] = v[q * R + r];
  }
  __syncthreads();
}

// Full length-2^lgL transform of `rows` smem rows (natural order in/out).
template <typename T>
__device__ __forceinline__ void stockham(cplx<T>* s, int lgL, int rs, const cplx<T>* tw,
                                         int lgN) {
  int lgNs = 0;
  while (lgNs < lgL) {
    const int rem = lgL - lgNs;
    if (rem >= 4) { stockham_pass<T, 4>(s, lgL, rs, lgNs, tw, lgN); lgNs += 4; }
    else if (rem == 3) { stockham_pass<T, 3>(s, lgL, rs, lgNs, tw, lgN); lgNs += 3; }
    else if (rem == 2) { stockham_pass<T, 2>(s, lgL, rs, lgNs, tw, lgN); lgNs += 2; }
    else { stockham_pass<T, 1>(s, lgL, rs, lgNs, tw, lgN); lgNs += 1; }
  }
}

// per-thread running peak in the arithmetic type (|z| >= 0 and finite
// inputs: max in T then one order-preserving key per warp equals the max key)
template <typename T>
__device__ __forceinline__ void emit_mag(T m, T& best) {
  best = fmax(best, m);
}

template <typename T>
__device__ __forceinline__ void flush_peak(T best, unsigned long long* peak) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) atomicMax(peak, fkey(best));
}

// Last Stockham pass (radix 2^LGR, Ns = L/R) read from smem, written straight
// to global memory through `st(seq, k, value)`; COLMAP: consecutive threads
// take consecutive sequences (columns) so global stores coalesce across
// columns, else consecutive j (contiguous rows).
template <typename T, int LGR, bool COLMAP, int IPT, typename St>
__device__ __forceinline__ void stockham_last(const cplx<T>* s, int lgL, int rs, int nseq_lg,
                                              const cplx<T>* __restrict__ tw, int lgN, St st) {
  using C = cplx<T>;
  constexpr int R = 1 << LGR;
  constexpr int K = IPT * 16 / R;
  const int per_lg = lgL - LGR;
  const int per = 1 << per_lg;  // == Ns
  const int tsh = lgN - lgL;
  C v[16 * IPT];
#pragma unroll
  for (int q = 0; q < K; ++q) {
    const int it = threadIdx.x + q * blockDim.x;
    int seq, j;
    if (COLMAP) { seq = it & ((1 << nseq_lg) - 1); j = it >> nseq_lg; }
    else { seq = it >> per_lg; j = it & (per - 1); }
    const C* sr = s + seq * rs;
#pragma unroll
    for (int r = 0; r < R; ++r) v[q * R + r] = sr[padi(j + r * per)];
    twiddle_powers<T, R>(&v[q * R], __ldg(tw + (j << tsh)));
    dft_reg<T, R>(&v[q * R]);
#pragma unroll
    for (int r = 0; r < R; ++r) st(seq, j + r * per, v[q * R + r]);
  }
}

// Whole transform of 2^nseq_lg sequences of length L >= 16 (blockDim.x * 16 ==
// nseq * L): pass 1 (radix 16) gathers its inputs straight from global memory
// through `ld(seq, u)`, middle passes run in smem, the last pass stores
// through `st`.  One smem round trip for L <= 256, two for L <= 4096.
template <typename T, bool COLMAP, int IPT = 1, int LG = 0, typename Ld, typename St>
__device__ __forceinline__ void fft_tile(cplx<T>* s, int lgL, int nseq_lg, int rs,
                                         const cplx<T>* __restrict__ tw, int lgN, Ld ld, St st) {
  using C = cplx<T>;
  if (LG > 0) lgL = LG;   // compile-time length: only the passes it needs are emitted
  const int L = 1 << lgL;
  const int per_lg = lgL - 4;
  const int per = L >> 4;
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const int it = threadIdx.x + q * blockDim.x;
    int seq, j;
    if (COLMAP) { seq = it & ((1 << nseq_lg) - 1); j = it >> nseq_lg; }
    else { seq = it >> per_lg; j = it & (per - 1); }
    C v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = ld(seq, j + r * per);
    dft_reg<T, 16>(v);
    if (lgL == 4) {
#pragma unroll
      for (int r = 0; r < 16; ++r) st(seq, r, v[r]);
    } else {
      C* sr = s + seq * rs;
#pragma unroll
      for (int r = 0; r < 16; ++r) sr[padi(j * 16 + r)] = v[r];
    }
  }
  if (lgL == 4) return;
  __syncthreads();
  int lgNs = 4;
  // middle passes: leave exactly the last pass's bits (4, or the remainder)
  while (lgL - lgNs > 4) {
    const int rem = lgL - lgNs - 4;           // bits to spend before the final radix-16
    if (rem >= 4) { stockham_pass<T, 4, IPT>(s, lgL, rs, lgNs, tw, lgN); lgNs += 4; }
    else if (rem == 3) { stockham_pass<T, 3, IPT>(s, lgL, rs, lgNs, tw, lgN); lgNs += 3; }
    else if (rem == 2) { stockham_pass<T, 2, IPT>(s, lgL, rs, lgNs, tw, lgN); lgNs += 2; }
    else { stockham_pass<T, 1, IPT>(s, lgL, rs, lgNs, tw, lgN); lgNs += 1; }
  }
  const int last = lgL - lgNs;
  if (last == 4) stockham_last<T, 4, COLMAP, IPT>(s, lgL, rs, nseq_lg, tw, lgN, st);
  else if (last == 3) stockham_last<T, 3, COLMAP, IPT>(s, lgL, rs, nseq_lg, tw, lgN, st);
  else if (last == 2) stockham_last<T, 2, COLMAP, IPT>(s, lgL, rs, nseq_lg, tw, lgN, st);
  else stockham_last<T, 1, COLMAP, IPT>(s, lgL, rs, nseq_lg, tw, lgN, st);
}

// Row pass: CTA = `rows` rows of length L (blockDim = rows * L / 16).
template <typename T, typename Tin, bool WC, bool WM, int IPT = 1, int LG = 0>
__global__ void __launch_bounds__(512, (sizeof(T) == 4) ? 2 : 1)
k_fftr(const Tin* src, cplx<T>* dst, T* __restrict__ mags, unsigned long long* __restrict__ peak,
       int lgL, int grid_lg, const cplx<T>* __restrict__ tw, int lgN,
       unsigned* __restrict__ nonfinite = nullptr) {
  pdl_wait();
  using C = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s = reinterpret_cast<C*>(smem_raw);
  const int rows_lg = __ffs((blockDim.x * 16 * IPT) >> lgL) - 1;
  const size_t e0 = ((size_t)blockIdx.x << rows_lg) << lgL;
  T best = 0;
  bool bad = false;
  auto ld = [&](int seq, int u) {
    const Tin w = src[e0 + ((size_t)seq << lgL) + u];
    if (nonfinite) bad |= !isfinite(w.x) || !isfinite(w.y);   // as_complex_matrix check
    return mk<T>((T)w.x, (T)w.y);
  };
  auto st = [&](int seq, int k, C v) {
    const size_t o = e0 + ((size_t)seq << lgL) + k;
    if (WC) dst[o] = v;
    if (WM) {
      const T m = mag_(v);
      mags[o] = m;
      emit_mag(m, best);
    }
  };
  fft_tile<T, false, IPT, LG>(s, lgL, rows_lg, pad_row(1 << lgL), tw, lgN, ld, st);
  if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1u);
  if (WM && peak) flush_peak(best, peak + (e0 >> grid_lg));
}

// Column pass for L <= 512: CTA = `cc` adjacent columns of one grid (W = L).
template <typename T, bool WC, bool WM, int LG = 0>
__global__ void __launch_bounds__(512, (sizeof(T) == 4) ? 2 : 1)
k_fftc(const cplx<T>* src, cplx<T>* dst, T* __restrict__ mags,
       unsigned long long* __restrict__ peak, int lgL, int lgcc, const cplx<T>* __restrict__ tw,
       int lgN) {
  pdl_wait();
  using C = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s = reinterpret_cast<C*>(smem_raw);
  const size_t g = blockIdx.y;
  const size_t gbase = (g << (2 * lgL)) + ((size_t)blockIdx.x << lgcc);
  T best = 0;
  auto ld = [&](int c, int u) { return src[gbase + ((size_t)u << lgL) + c]; };
  auto st = [&](int c, int k, C v) {
    const size_t o = gbase + ((size_t)k << lgL) + c;
    if (WC) dst[o] = v;
    if (WM) {
      const T m = mag_(v);
      mags[o] = m;
      emit_mag(m, best);
    }
  };
  fft_tile<T, true, 1, LG>(s, lgL, lgcc, pad_row(1 << lgL), tw, lgN, ld, st);
  if (WM && peak) flush_peak(best, peak + g);
}

// Single-pass column FFT for 1024 <= L <= 4096: CTA = cc adjacent columns
// (cc * sizeof(C) >= 32 B, one full sector per row segment) held whole in
// shared memory, IPT radix-16 groups per thread.  Replaces the four-step
// A + B pair: one read and one write of the grid instead of two each.
template <typename T, bool WC, bool WM, int IPT, int LG = 0>
__global__ void __launch_bounds__(512, 1)
k_fftc1(const cplx<T>* src, cplx<T>* dst, T* __restrict__ mags,
        unsigned long long* __restrict__ peak, int lgL, int lgcc, const cplx<T>* __restrict__ tw,
        int lgN) {
  pdl_wait();
  using C = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s = reinterpret_cast<C*>(smem_raw);
  const size_t g = blockIdx.y;
  const size_t gbase = (g << (2 * lgL)) + ((size_t)blockIdx.x << lgcc);
  T best = 0;
  auto ld = [&](int c, int u) { return src[gbase + ((size_t)u << lgL) + c]; };
  auto st = [&](int c, int k, C v) {
    const size_t o = gbase + ((size_t)k << lgL) + c;
    if (WC) dst[o] = v;
    if (WM) {
      const T m = mag_(v);
      mags[o] = m;
      emit_mag(m, best);
    }
  };
  fft_tile<T, true, IPT, LG>(s, lgL, lgcc, pad_row(1 << lgL), tw, lgN, ld, st);
  if (WM && peak) flush_peak(best, peak + g);
}

// Four-step column pass A (in place): length-L1 DFTs over rows n2 + L2*n1, then
// twiddle by W_L^{n2 k1}; grid = (column tiles, n2, grid index).
template <typename T, int LG1 = 0>
__global__ void __launch_bounds__(512, (sizeof(T) == 4) ? 2 : 1)
k_fftcA(cplx<T>* data, int lgL1, int lgL2, int lgcc, const cplx<T>* __restrict__ tw, int lgN) {
  pdl_wait();
  using C = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s = reinterpret_cast<C*>(smem_raw);
  const int lgL = lgL1 + lgL2;
  const int n2 = blockIdx.y;
  const size_t gbase = ((size_t)blockIdx.z << (2 * lgL)) + ((size_t)blockIdx.x << lgcc);
  const int tsh = lgN - lgL;
  auto ld = [&](int c, int n1) { return data[gbase + ((size_t)(n2 + (n1 << lgL2)) << lgL) + c]; };
  auto st = [&](int c, int k1, C v) {
    if (n2 && k1) v = cmul(v, __ldg(tw + ((n2 * k1) << tsh)));
    data[gbase + ((size_t)(n2 + (k1 << lgL2)) << lgL) + c] = v;
  };
  fft_tile<T, true, 1, LG1>(s, lgL1, lgcc, pad_row(1 << lgL1), tw, lgN, ld, st);
}

// Four-step column pass B: length-L2 DFTs over rows L2*k1 + n2 -> row k1 + L1*k2.
template <typename T, bool WC, bool WM, int LG2 = 0>
__global__ void __launch_bounds__(512, (sizeof(T) == 4) ? 2 : 1)
k_fftcB(const cplx<T>* __restrict__ src, cplx<T>* __restrict__ dst, T* __restrict__ mags,
        unsigned long long* __restrict__ peak, int lgL1, int lgL2, int lgcc,
        const cplx<T>* __restrict__ tw, int lgN) {
  pdl_wait();
  using C = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s = reinterpret_cast<C*>(smem_raw);
  const int lgL = lgL1 + lgL2;
  const int k1 = blockIdx.y;
  const size_t g = blockIdx.z;
  const size_t gbase = (g << (2 * lgL)) + ((size_t)blockIdx.x << lgcc);
  T best = 0;
  auto ld = [&](int c, int n2) { return src[gbase + ((size_t)((k1 << lgL2) + n2) << lgL) + c]; };
  auto st = [&](int c, int k2, C v) {
    const size_t o = gbase + ((size_t)(k1 + (k2 << lgL1)) << lgL) + c;
    if (WC) dst[o] = v;
    if (WM) {
      const T m = mag_(v);
      mags[o] = m;
      emit_mag(m, best);
    }
  };
  fft_tile<T, true, 1, LG2>(s, lgL2, lgcc, pad_row(1 << lgL2), tw, lgN, ld, st);
  if (WM && peak) flush_peak(best, peak + g);
}

// Length-2^LG transform of 2^nseq_lg sequences whose first radix-16 pass
// gathers from global memory through ld(seq, u) (consecutive threads take
// consecutive sequences, then consecutive j); every later pass runs in shared
// memory and the result stays there in natural order (padded rows, stride rs).
template <typename T, int LG, typename Ld>
__device__ __forceinline__ void fft_tile_smem(cplx<T>* s, int nseq_lg, int rs,
                                              const cplx<T>* __restrict__ tw, int lgN, Ld ld) {
  using C = cplx<T>;
  constexpr int per = (1 << LG) >> 4;
  {
    const int it = threadIdx.x;
    const int seq = it & ((1 << nseq_lg) - 1), j = it >> nseq_lg;
    C v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = ld(seq, j + r * per);
    dft_reg<T, 16>(v);
    C* sr = s + seq * rs;
#pragma unroll
    for (int r = 0; r < 16; ++r) sr[padi(j * 16 + r)] = v[r];
  }
  __syncthreads();
  int lgNs = 4;
#pragma unroll
  for (int pass = 0; pass < 4; ++pass) {
    if (lgNs >= LG) break;
    const int rem = LG - lgNs;
    if (rem >= 4) { stockham_pass<T, 4>(s, LG, rs, lgNs, tw, lgN); lgNs += 4; }
    else if (rem == 3) { stockham_pass<T, 3>(s, LG, rs, lgNs, tw, lgN); lgNs += 3; }
    else if (rem == 2) { stockham_pass<T, 2>(s, LG, rs, lgNs, tw, lgN); lgNs += 2; }
    else { stockham_pass<T, 1>(s, LG, rs, lgNs, tw, lgN); lgNs += 1; }
  }
}

// Row pass for rows too long for one CTA's shared memory (fp64, L = 16384:
// 278 KB padded): a 2-CTA cluster per row.  CTA q transforms the elements
// 2u + q to E_q[k'] in its shared memory; after a cluster barrier it reads
// E_0 and E_1 for its half of k' (the peer's through DSMEM) and writes the
// radix-2 outputs X[k'] = E_0 + W_L^k' E_1, X[k' + L/2] = E_0 - W_L^k' E_1.
// Complex output only (the dense row pass), with the NaN/Inf check.
template <typename T, typename Tin, int LGM>
__global__ void __launch_bounds__(512, 1)
k_fftr_cl2(const Tin* __restrict__ src, cplx<T>* __restrict__ dst,
           const cplx<T>* __restrict__ tw, int lgN, unsigned* __restrict__ nonfinite) {
  pdl_wait();
  namespace cg = cooperative_groups;
  using C = cplx<T>;
  constexpr int M = 1 << LGM;
  constexpr int lgL = LGM + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s = reinterpret_cast<C*>(smem_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const size_t base = (size_t)(blockIdx.x >> 1) << lgL;
  bool bad = false;
  auto ld = [&](int, int u) {
    const Tin w = src[base + 2 * (size_t)u + q];
    if (nonfinite) bad |= !isfinite(w.x) || !isfinite(w.y);
    return mk<T>((T)w.x, (T)w.y);
  };
  fft_tile_smem<T, LGM>(s, 0, pad_row(M), tw, lgN, ld);
  cl.sync();
  const C* e0s = cl.map_shared_rank(s, 0);
  const C* e1s = cl.map_shared_rank(s, 1);
  const int tsh = lgN - lgL;
  for (int kk = q * (M / 2) + threadIdx.x; kk < (q + 1) * (M / 2); kk += blockDim.x) {
    const C e0 = e0s[padi(kk)];
    C e1 = e1s[padi(kk)];
    if (kk) e1 = cmul(e1, __ldg(tw + ((size_t)kk << tsh)));
    dst[base + kk] = cadd(e0, e1);
    dst[base + kk + M] = csub(e0, e1);
  }
  cl.sync();   // the peer has finished reading this CTA's shared memory
  if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1u);
}

// ---------------------------------------------------------------- dispatch
// Calls f(std::integral_constant<int, lg>) for LO <= lg <= HI, else
// f(std::integral_constant<int, 0>) (runtime length): a compile-time length
// emits only the Stockham passes that length needs, which keeps the kernel
// small enough for the instruction cache (measured: k_fftcB at B = 2048
// 25.3 -> 17.8 us).
template <int LO, int HI, typename F>
inline void with_lg(int lg, F&& f) {
  if constexpr (LO <= HI) {
    if (lg == LO) {
      f(std::integral_constant<int, LO>{});
      return;
    }
    with_lg<LO + 1, HI>(lg, std::forward<F>(f));
  } else {
    f(std::integral_constant<int, 0>{});
  }
}

// ---------------------------------------------------------------- geometry
struct FftPlan2D {
  int lgL;
  int rows_per_cta, row_threads, row_ipt;   // row pass
  bool four_step;
  int lgL1, lgL2;                      // four-step split
  int lgccA, thrA, lgccB, thrB;        // column tiles (A, B) or single pass (B)
  size_t smem_row, smem_A, smem_B;
  bool col1;                           // single-pass wide column tile (k_fftc1)
  int lgcc1, thr1, ipt1;
  size_t smem_1;
};

template <typename T>
inline FftPlan2D plan_fft2d(int lgL) {
  FftPlan2D p{};
  const size_t cs = sizeof(cplx<T>);
  const int L = 1 << lgL;
  p.lgL = lgL;
  // row pass: rows*L/16 threads, about 256
  int rows = L >= 4096 ? 1 : 4096 / L;
  if (rows > L) rows = L;
  p.rows_per_cta = rows;
  p.row_ipt = (rows * L / 16 > 512) ? 2 : 1;     // L = 16384: two radix-16 groups per thread
  p.row_threads = rows * L / 16 / p.row_ipt;
  p.smem_row = (size_t)rows * pad_row(L) * cs;
  auto tile = [&](int lgLc, int& lgcc, int& thr, size_t& sm) {
    const int Lc = 1 << lgLc;
    int lc = 0;
    while ((1 << lc) * Lc < 4096) ++lc;                     // ~256 threads
    while ((1 << lc) * (int)cs < 128) ++lc;                 // >= 128 B per row segment
    while ((1 << lc) > L) --lc;
    while (lc > 0 && (size_t)(1 << lc) * pad_row(Lc) * cs > 96 * 1024) --lc;
    lgcc = lc;
    thr = (1 << lc) * Lc / 16;
    sm = (size_t)(1 << lc) * pad_row(Lc) * cs;
  };
  p.four_step = lgL > 9;
  // single-pass column tile of the narrowest full-sector width: faster than
  // four-step at L = 1024 (measured 12.5 vs 20.5 us, 1024^2 fp32); at 2048 it
  // ties and at 4096 (one 139 KB CTA per SM) it loses to four-step A + B
  p.col1 = false;
  if (lgL == 10) {
    int lc = 0;
    while ((1 << lc) * (int)cs < 32) ++lc;
    const int ipt = (1 << lc) * L / 16 > 512 ? 2 : 1;
    p.col1 = true;
    p.lgcc1 = lc;
    p.ipt1 = ipt;
    p.thr1 = (1 << lc) * L / 16 / ipt;
    p.smem_1 = (size_t)(1 << lc) * pad_row(L) * cs;
  }
  if (p.four_step) {
    p.lgL1 = (lgL + 1) / 2;
    p.lgL2 = lgL - p.lgL1;
    tile(p.lgL1, p.lgccA, p.thrA, p.smem_A);
    tile(p.lgL2, p.lgccB, p.thrB, p.smem_B);
  } else {
    tile(lgL, p.lgccB, p.thrB, p.smem_B);
  }
  return p;
}

}  // namespace sfft
