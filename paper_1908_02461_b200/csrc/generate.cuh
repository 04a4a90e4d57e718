// Device-side workload generator: the planted
// k-sparse-spectrum image plus complex Gaussian noise of the BASELINE configs,
// built in HBM so that large batches (c4: 2048 x 8 MB) and 2 GiB images (c5)
// are never generated on the host.
//
//   x = ifft2(S) + sd * (n1 + i n2),  S = the k planted coefficients
//
// ifft2(S) = conj(fft2(conj(S))) / N^2 (the reference's unscaled-inverse
// convention, corefft.py:112-118): the conjugated coefficients are scattered
// into the zeroed output grid, the library's own forward FFT runs in place,
// and one elementwise pass conjugates, scales and adds the noise.
//
// Noise: counter-based Philox4x32-10 keyed by the 64-bit noise seed, counter
// = element index, one 128-bit draw per element -> two 53-bit uniforms ->
// Box-Muller (n1 = r cos t, n2 = r sin t, r = sqrt(-2 ln u1), t = 2 pi u2),
// computed in double.  The stream is independent of the launch geometry, so
// tests/test_generator.py restates it in numpy bit for bit (up to libm ulps).
#pragma once
#include "common.cuh"

namespace sfft {

struct Philox4 {
  uint32_t v[4];
};

__host__ __device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                                           uint32_t c3, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)M0 * c0, p1 = (uint64_t)M1 * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += W0;
    k1 += W1;
  }
  Philox4 o;
  o.v[0] = c0;
  o.v[1] = c1;
  o.v[2] = c2;
  o.v[3] = c3;
  return o;
}

// conj(coeff) scattered at flat index (row, col); the grid is zeroed first
template <typename T>
__global__ void k_gen_scatter(cplx<T>* __restrict__ grid, int lgN, const int64_t* __restrict__ rows,
                              const int64_t* __restrict__ cols, const double2* __restrict__ coeffs,
                              int k) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  const double2 c = coeffs[i];
  grid[((size_t)rows[i] << lgN) + (size_t)cols[i]] = mk<T>((T)c.x, (T)-c.y);
}

// x = conj(y) / N^2 + sd * (n1 + i n2), in place
template <typename T>
__global__ void k_gen_finish(cplx<T>* __restrict__ grid, long total, double inv, double sd,
                             uint32_t k0, uint32_t k1) {
  pdl_wait();
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x) {
    const cplx<T> y = grid[e];
    double re = (double)y.x * inv, im = -(double)y.y * inv;
    if (sd > 0.0) {
      const Philox4 r = philox4x32_10((uint32_t)e, (uint32_t)((unsigned long long)e >> 32), 0u, 0u,
                                      k0, k1);
      // 53-bit uniforms; u1 in (0, 1] so the log is finite
      const double u1 = 1.0 - (double)(((uint64_t)(r.v[0] >> 5) << 26) | (r.v[1] >> 6)) *
                                  (1.0 / 9007199254740992.0);
      const double u2 = (double)(((uint64_t)(r.v[2] >> 5) << 26) | (r.v[3] >> 6)) *
                        (1.0 / 9007199254740992.0);
      const double rad = sqrt(-2.0 * log(u1));
      double sn, cs;
      sincospi(2.0 * u2, &sn, &cs);
      re += sd * rad * cs;
      im += sd * rad * sn;
    }
    grid[e] = mk<T>((T)re, (T)im);
  }
}

}  // namespace sfft
