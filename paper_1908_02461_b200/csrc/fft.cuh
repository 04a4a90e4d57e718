// K2 — bucket FFTs (replaces corefft.fft2d / _fft1d_batch, corefft.py:77-109).
//
// Unscaled forward DFT  X[k] = sum_u x[u] * exp(-2*pi*i*k*u/L)  along rows
// then columns, exactly the reference convention.  Each 1D transform runs in
// shared memory: the sequence is staged in bit-reversed order, then radix-4
// stages (two radix-2 DIT stages merged in registers) and at most one radix-2
// stage, in place.  Twiddles come from ONE table per image side N,
// tw[k] = exp(-2*pi*i*k/N), built on the host with the same numpy expression
// the reference uses (hashing/engine phase factors); W_m^p = tw[p*N/m].
//
// Grid shapes:
//   * B*B*sizeof(C) <= kSmall2DBytes : one CTA transforms a whole B x B grid
//     (optionally fused with the fold's partial-sum reduction and the
//     bucket permutation, see fold.cuh).
//   * otherwise: a row pass (CTA = several rows, coalesced) and a column pass
//     (CTA = a group of >= 32 B of adjacent columns, sector-efficient).
#pragma once
#include "common.cuh"

namespace sfft {

constexpr int kSmall2DBytes = 64 * 1024;

// In-place DIT stages over `count` sequences of length 2^lgL living in smem.
// Element e of sequence s is at base[s*ss + e*es].  Input must be bit-reversed.
// Must be called by all threads of the block (contains __syncthreads).
template <typename T>
__device__ void fft_stages(cplx<T>* base, int count, int lgL, int es, int ss,
                           const cplx<T>* __restrict__ tw, int lgN) {
  using C = cplx<T>;
  const int L = 1 << lgL;
  const int tid = threadIdx.x, nth = blockDim.x;
  int lgh = 0;
  while (lgh < lgL) {
    const int h = 1 << lgh;
    if (lgh + 2 <= lgL) {
      const int per = L >> 2;
      const int total = count * per;
      for (int g = tid; g < total; g += nth) {
        const int s = g >> (lgL - 2);
        const int q = g & (per - 1);
        const int j = q & (h - 1);
        const int k = (q >> lgh) << (lgh + 2);
        C* d = base + (size_t)s * ss;
        const int i0 = (k + j) * es, i1 = (k + j + h) * es, i2 = (k + j + 2 * h) * es,
                  i3 = (k + j + 3 * h) * es;
        C a = d[i0], b = d[i1], c = d[i2], e = d[i3];
        const C w1 = tw[j << (lgN - lgh - 1)];
        const C w2 = tw[j << (lgN - lgh - 2)];
        const C w3 = tw[(j + h) << (lgN - lgh - 2)];
        C t = cmul(b, w1); b = csub(a, t); a = cadd(a, t);
        t = cmul(e, w1); e = csub(c, t); c = cadd(c, t);
        t = cmul(c, w2); c = csub(a, t); a = cadd(a, t);
        t = cmul(e, w3); e = csub(b, t); b = cadd(b, t);
        d[i0] = a; d[i1] = b; d[i2] = c; d[i3] = e;
      }
      lgh += 2;
    } else {
      const int per = L >> 1;
      const int total = count * per;
      for (int g = tid; g < total; g += nth) {
        const int s = g >> (lgL - 1);
        const int q = g & (per - 1);
        const int j = q & (h - 1);
        const int k = (q >> lgh) << (lgh + 1);
        C* d = base + (size_t)s * ss;
        const int i0 = (k + j) * es, i1 = (k + j + h) * es;
        C a = d[i0], b = d[i1];
        const C w = tw[j << (lgN - lgh - 1)];
        C t = cmul(b, w); b = csub(a, t); a = cadd(a, t);
        d[i0] = a; d[i1] = b;
      }
      lgh += 1;
    }
    __syncthreads();
  }
}

// Whole-grid 2D FFT of `ngrids` B x B grids, one CTA per grid, in place.
// Rows padded to B + 1 elements (bank-conflict-free column stages), length-B
// twiddles staged in shared memory: dynamic smem = (B (B + 1) + B) elements.
template <typename T>
__global__ void k_fft2d_small(cplx<T>* __restrict__ grids, int lgB,
                              const cplx<T>* __restrict__ tw, int lgN) {
  pdl_wait();
  using C = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s = reinterpret_cast<C*>(smem_raw);
  const int B = 1 << lgB, BB = B * B, RS = B + 1;
  C* tws = s + (size_t)B * RS;
  C* g = grids + (size_t)blockIdx.x * BB;
  for (int k = threadIdx.x; k < B; k += blockDim.x) tws[k] = tw[k << (lgN - lgB)];
  for (int e = threadIdx.x; e < BB; e += blockDim.x) {
    const int u = e >> lgB, v = e & (B - 1);
    s[bitrev(u, lgB) * RS + bitrev(v, lgB)] = g[e];
  }
  __syncthreads();
  fft_stages<T>(s, B, lgB, 1, RS, tws, lgB);    // rows
  fft_stages<T>(s, B, lgB, RS, 1, tws, lgB);    // columns
  for (int e = threadIdx.x; e < BB; e += blockDim.x) g[e] = s[(e >> lgB) * RS + (e & (B - 1))];
}

// Row pass over `nrows` rows of length B (rows of all grids concatenated).
// If `src` is non-null the rows are read from an input image (Tin) instead of
// `dst` (used for the dense transform of the image itself).
template <typename T, typename Tin>
__global__ void k_fft_rows(const Tin* __restrict__ src, cplx<T>* __restrict__ dst, int lgB,
                           long nrows, int rows_per_cta, const cplx<T>* __restrict__ tw,
                           int lgN) {
  pdl_wait();
  using C = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s = reinterpret_cast<C*>(smem_raw);
  const int B = 1 << lgB;
  const long row0 = (long)blockIdx.x * rows_per_cta;
  const int nr = (int)min((long)rows_per_cta, nrows - row0);
  const int tot = nr << lgB;
  if (src) {
    const Tin* in = src + (row0 << lgB);
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
      const int r = e >> lgB, i = e & (B - 1);
      s[(r << lgB) + bitrev(i, lgB)] = load_c<T>(in + e);
    }
  } else {
    const C* in = dst + (row0 << lgB);
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
      const int r = e >> lgB, i = e & (B - 1);
      s[(r << lgB) + bitrev(i, lgB)] = in[e];
    }
  }
  __syncthreads();
  fft_stages<T>(s, nr, lgB, 1, B, tw, lgN);
  C* out = dst + (row0 << lgB);
  for (int e = threadIdx.x; e < tot; e += blockDim.x) out[e] = s[e];
}

// Column pass: CTA = `cpc` adjacent columns of one grid.
template <typename T>
__global__ void k_fft_cols(cplx<T>* __restrict__ grids, int lgB, int cpc,
                           const cplx<T>* __restrict__ tw, int lgN) {
  pdl_wait();
  using C = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s = reinterpret_cast<C*>(smem_raw);
  const int B = 1 << lgB;
  const int groups = B / cpc;
  const long g = blockIdx.x / groups;
  const int c0 = (blockIdx.x % groups) * cpc;
  C* base = grids + (g << (2 * lgB)) + c0;
  const int tot = B * cpc;
  for (int e = threadIdx.x; e < tot; e += blockDim.x) {
    const int u = e / cpc, cc = e - u * cpc;
    s[cc * B + bitrev(u, lgB)] = base[(size_t)u * B + cc];
  }
  __syncthreads();
  fft_stages<T>(s, cpc, lgB, 1, B, tw, lgN);
  for (int e = threadIdx.x; e < tot; e += blockDim.x) {
    const int u = e / cpc, cc = e - u * cpc;
    base[(size_t)u * B + cc] = s[cc * B + u];
  }
}

// ---------------------------------------------------------------- launchers
constexpr size_t kMaxDynSmem = 200 * 1024;

template <typename T>
inline int fft_cols_per_cta(int B) {
  // >= 32 B of adjacent columns per row segment when it fits, grown while the
  // staging buffer stays small; 0 = the column does not fit in shared memory
  const size_t col = (size_t)B * sizeof(cplx<T>);
  int cpc = (int)(32 / sizeof(cplx<T>));
  while (cpc > 1 && (size_t)cpc * col > kMaxDynSmem) cpc /= 2;
  if ((size_t)cpc * col > kMaxDynSmem) return 0;
  while (cpc * 2 <= B && (size_t)cpc * 2 * col <= 48 * 1024 && cpc < 16) cpc *= 2;
  return cpc > B ? B : cpc;
}

template <typename T>
inline int fft_rows_per_cta(int B) {
  const size_t row = (size_t)B * sizeof(cplx<T>);
  if (row > kMaxDynSmem) return 0;
  int r = 1;
  while ((size_t)r * 2 * row <= 32 * 1024 && r * 2 * B <= 8192) r *= 2;
  return r;
}

}  // namespace sfft
