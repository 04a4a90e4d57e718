// K1 — fused permute + window + fold into B x B buckets.
// Replaces the gather/window/reshape-sum of binned_spectrum
// (/root/reference/pkg/src/sfft2d/hashing.py:308-337).
//
// Restatement used here.  The reference gathers
//   block[u, v] = g[u] g[v] x[s1*u + t1, s2*v + t2]    (u, v over the support)
// and folds u, v modulo B.  Substituting r = s1*u + t1 (a bijection mod N)
// and using B | N, the bucket of row r is  pi1(r mod B)  with
//   pi1(rho) = s1^-1 * (rho - t1) mod B,
// so with natural-order weights  wr[r] = g[s1^-1 (r - t1) mod N]  (zero outside
// the window support) the folded grid is
//   y[pi1(rho), pi2(kappa)] = sum_{r = rho mod B} sum_{c = kappa mod B} wr[r] wc[c] x[r, c].
// The image is therefore streamed in natural (coalesced) row-major order, rows
// with zero weight are skipped, and NL permutations (hash loops) share one read.
//
// Work split: CTA (kappa-tile, rho, z).  Threads own CPT adjacent columns of a
// tile of TW columns; a CTA visits rows rho + j*B for j in its alias chunk z
// and every column congruent to its tile.  Row weights for the chunk are
// staged in shared memory; per column the row sum is accumulated first, then
// scaled by the column weight (2*NL FMA per complex element).  With Z > 1 the
// CTAs write natural-order partials [Z][NL][B][B] that a second kernel sums in
// a fixed order (deterministic, no float atomics) while applying pi1/pi2 —
// fused with the whole 2D FFT when the grid fits one CTA's shared memory.
#pragma once
#include "common.cuh"
#include "fft.cuh"
#include <cooperative_groups.h>

namespace sfft {

constexpr int kFoldThreads = 256;
constexpr int kFoldMaxRows = 256;  // row aliases per chunk (smem weight tile)

template <typename Tin, typename T, int CPT> struct ColLoad;
template <> struct ColLoad<float2, float, 1> {
  __device__ static void ld(const float2* p, float2* v) { v[0] = __ldg(p); }
};
template <> struct ColLoad<float2, double, 1> {
  __device__ static void ld(const float2* p, double2* v) {
    float2 a = __ldg(p); v[0] = make_double2(a.x, a.y);
  }
};
template <> struct ColLoad<double2, double, 1> {
  __device__ static void ld(const double2* p, double2* v) { v[0] = __ldg(p); }
};
template <> struct ColLoad<double2, float, 1> {
  __device__ static void ld(const double2* p, float2* v) {
    double2 a = __ldg(p); v[0] = make_float2((float)a.x, (float)a.y);
  }
};
template <> struct ColLoad<float2, float, 2> {
  __device__ static void ld(const float2* p, float2* v) {
    float4 a = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = make_float2(a.x, a.y); v[1] = make_float2(a.z, a.w);
  }
};
template <> struct ColLoad<float2, double, 2> {
  __device__ static void ld(const float2* p, double2* v) {
    float4 a = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = make_double2(a.x, a.y); v[1] = make_double2(a.z, a.w);
  }
};
template <> struct ColLoad<double2, double, 2> {
  __device__ static void ld(const double2* p, double2* v) { v[0] = __ldg(p); v[1] = __ldg(p + 1); }
};
template <> struct ColLoad<double2, float, 2> {
  __device__ static void ld(const double2* p, float2* v) {
    double2 a = __ldg(p), b = __ldg(p + 1);
    v[0] = make_float2((float)a.x, (float)a.y); v[1] = make_float2((float)b.x, (float)b.y);
  }
};

struct FoldGeom {
  int lgN, lgB;
  int TW;        // tile width in columns (threads * CPT)
  int ktiles;    // kappa tiles per rho (B >= TW ? B / TW : 1)
  int Z;         // row-alias chunks
  int rpc;       // row aliases per chunk
  int tab;       // byte offset of the smem copy of the window table (-1: none)
};

template <typename Tin, typename T, int NL, int CPT, int MU = 1>
__global__ void __launch_bounds__(kFoldThreads)
k_fold(const Tin* __restrict__ x, const T* __restrict__ space, PermPack pp, int nloops,
       FoldGeom gm, bool natural, cplx<T>* __restrict__ dst,
       unsigned long long* __restrict__ zero_peak = nullptr) {
  pdl_wait();
  using C = cplx<T>;
  if (zero_peak && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0)
    *zero_peak = 0ull;
  __shared__ T s_w[NL * kFoldMaxRows];
  __shared__ int s_rows[kFoldMaxRows];
  __shared__ int s_nnz;
  extern __shared__ __align__(16) unsigned char smem_raw[];   // [NL][TW] reduction (B < TW)

  const int N = 1 << gm.lgN, B = 1 << gm.lgB;
  const unsigned maskN = (unsigned)N - 1u, maskB = (unsigned)B - 1u;
  const int rho = blockIdx.y;
  const int z = blockIdx.z;
  const int aliases = N >> gm.lgB;
  const int j0 = z * gm.rpc;
  const int cnt = min(gm.rpc, aliases - j0);
  const int tid = threadIdx.x;

  // ---- window table in shared memory (column weights are gathered at an
  // odd stride, which is bank-conflict free in smem but 32 sectors per warp
  // load from L1)
  const T* wt = space;
  if (gm.tab >= 0) {
    T* tsm = reinterpret_cast<T*>(smem_raw + gm.tab);
    constexpr int V = 16 / sizeof(T);
    for (int i = tid * V; i < N; i += blockDim.x * V)
      *reinterpret_cast<uint4*>(tsm + i) = __ldg(reinterpret_cast<const uint4*>(space + i));
    wt = tsm;
  }
  // ---- row weights of this chunk, and the compacted list of useful rows
  for (int jj = tid; jj < cnt; jj += blockDim.x) {
    const unsigned r = (unsigned)(rho + (j0 + jj) * B);
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      T w = (T)0;
      if (l < nloops) w = __ldg(space + ((pp.p[l].s1i * (r - pp.p[l].t1)) & maskN));
      s_w[l * kFoldMaxRows + jj] = w;
    }
  }
  __syncthreads();
  if (tid < 32) {
    int base = 0;
    for (int c0 = 0; c0 < cnt; c0 += 32) {
      const int jj = c0 + tid;
      bool nz = false;
      if (jj < cnt) {
#pragma unroll
        for (int l = 0; l < NL; ++l) nz |= (s_w[l * kFoldMaxRows + jj] != (T)0);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, nz);
      if (nz) s_rows[base + __popc(bal & ((1u << tid) - 1u))] = jj;
      base += __popc(bal);
    }
    if (tid == 0) s_nnz = base;
  }
  __syncthreads();
  const int nnz = s_nnz;

  // ---- stream the image
  const int cp = tid * CPT;
  const int step = max(B, gm.TW);
  const int cbase = (B >= gm.TW) ? blockIdx.x * gm.TW : 0;
  const int ncb = N / step;
  C acc[NL][CPT];
#pragma unroll
  for (int l = 0; l < NL; ++l)
#pragma unroll
    for (int q = 0; q < CPT; ++q) acc[l][q] = mk<T>(0, 0);

  if (nnz > 0) {
    // MU column blocks per step: MU independent loads per row, rows unrolled
    // by 2, so a thread keeps 2*MU 16-byte loads in flight
    for (int m0 = 0; m0 < ncb; m0 += MU) {
      T wc[MU][NL][CPT];
      bool any = false;
#pragma unroll
      for (int mu = 0; mu < MU; ++mu) {
        const int c = cbase + (m0 + mu) * step + cp;
#pragma unroll
        for (int l = 0; l < NL; ++l)
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            T w = (T)0;
            if (l < nloops && m0 + mu < ncb)
              w = wt[(pp.p[l].s2i * ((unsigned)(c + q) - pp.p[l].t2)) & maskN];
            wc[mu][l][q] = w;
            any |= (w != (T)0);
          }
      }
      if (!any) continue;
      C u[MU][NL][CPT];
#pragma unroll
      for (int mu = 0; mu < MU; ++mu)
#pragma unroll
        for (int l = 0; l < NL; ++l)
#pragma unroll
          for (int q = 0; q < CPT; ++q) u[mu][l][q] = mk<T>(0, 0);
      const Tin* col = x + cbase + m0 * step + cp;
#pragma unroll 2
      for (int i = 0; i < nnz; ++i) {
        const int jj = s_rows[i];
        const size_t r = (size_t)(rho + (j0 + jj) * B);
        C v[MU][CPT];
#pragma unroll
        for (int mu = 0; mu < MU; ++mu)
          if (m0 + mu < ncb) ColLoad<Tin, T, CPT>::ld(col + mu * step + (r << gm.lgN), v[mu]);
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const T wr = s_w[l * kFoldMaxRows + jj];
#pragma unroll
          for (int mu = 0; mu < MU; ++mu)
#pragma unroll
            for (int q = 0; q < CPT; ++q) {
              u[mu][l][q].x = fma(wr, v[mu][q].x, u[mu][l][q].x);
              u[mu][l][q].y = fma(wr, v[mu][q].y, u[mu][l][q].y);
            }
        }
      }
#pragma unroll
      for (int mu = 0; mu < MU; ++mu)
#pragma unroll
        for (int l = 0; l < NL; ++l)
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            acc[l][q].x = fma(wc[mu][l][q], u[mu][l][q].x, acc[l][q].x);
            acc[l][q].y = fma(wc[mu][l][q], u[mu][l][q].y, acc[l][q].y);
          }
    }
  }

  // ---- emit (rho, kappa) values
  const size_t BB = (size_t)B * B;
  if (B >= gm.TW) {
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      if (l >= nloops) break;
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const unsigned kap = (unsigned)(cbase + cp + q);
        if (gm.Z == 1) {
          const unsigned a = natural ? (unsigned)rho : (pp.p[l].s1i * ((unsigned)rho - pp.p[l].t1)) & maskB;
          const unsigned b = natural ? kap : (pp.p[l].s2i * (kap - pp.p[l].t2)) & maskB;
          dst[l * BB + (size_t)a * B + b] = acc[l][q];
        } else {
          dst[((size_t)z * nloops + l) * BB + (size_t)rho * B + kap] = acc[l][q];
        }
      }
    }
  } else {
    C* red = reinterpret_cast<C*>(smem_raw);
#pragma unroll
    for (int l = 0; l < NL; ++l)
#pragma unroll
      for (int q = 0; q < CPT; ++q) red[l * gm.TW + cp + q] = acc[l][q];
    __syncthreads();
    const int reps = gm.TW / B;
    for (int e = tid; e < nloops * B; e += blockDim.x) {
      const int l = e / B;
      const int kap = e - l * B;
      C s = mk<T>(0, 0);
      for (int a = 0; a < reps; ++a) s = cadd(s, red[l * gm.TW + kap + a * B]);
      if (gm.Z == 1) {
        const unsigned ra = natural ? (unsigned)rho : (pp.p[l].s1i * ((unsigned)rho - pp.p[l].t1)) & maskB;
        const unsigned cb = natural ? (unsigned)kap : (pp.p[l].s2i * ((unsigned)kap - pp.p[l].t2)) & maskB;
        dst[l * BB + (size_t)ra * B + cb] = s;
      } else {
        dst[((size_t)z * nloops + l) * BB + (size_t)rho * B + kap] = s;
      }
    }
  }
}

// Multi-loop fold for B < 512 (the SFFT's L location / estimation loops, all
// from one read of x): CTA = (column tile of TWC <= 512 columns, bucket row
// rho, row chunk z).  Each thread owns 2 adjacent columns for the whole CTA,
// so the row sums u_l(c) = sum_r wr_l[r] x[r, c] stay in registers and are
// scaled by wc_l(c) once at the end; rows are unrolled by UNR with all UNR
// 16-byte loads issued before the first FMA (UNR loads in flight per thread —
// k_fold's per-column-block loop kept 2, which held the 8-loop c3 fold at
// 0.23 of HBM).  The TWC / B aliases of each kappa inside the tile are summed
// in shared memory in a fixed order; the tile's row of the bucket grid goes
// to partial (tile, z) [Zp][NL][B][B] (natural order), or straight to the
// grid when Zp == 1.
template <typename Tin, typename T, int NL, int UNR>
__global__ void __launch_bounds__(256)
k_fold_ml(const Tin* __restrict__ x, const T* __restrict__ space, PermPack pp, int nloops,
          int lgN, int lgB, int TWC, int rpc, bool natural, int zp, cplx<T>* __restrict__ dst,
          unsigned* __restrict__ nonfinite = nullptr) {
  pdl_wait();
  using C = cplx<T>;
  __shared__ T s_w[NL * kFoldMaxRows];
  __shared__ int s_rows[kFoldMaxRows];
  __shared__ int s_nnz;
  extern __shared__ __align__(16) unsigned char smem_raw[];   // [NL][TWC] alias reduction
  const int N = 1 << lgN, B = 1 << lgB;
  const unsigned maskN = (unsigned)N - 1u, maskB = (unsigned)B - 1u;
  const int tile = blockIdx.x, rho = blockIdx.y, z = blockIdx.z;
  const int aliases = N >> lgB;
  const int j0 = z * rpc;
  const int cnt = min(rpc, aliases - j0);
  const int tid = threadIdx.x;
  for (int jj = tid; jj < cnt; jj += blockDim.x) {
    const unsigned r = (unsigned)(rho + (j0 + jj) * B);
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      T w = (T)0;
      if (l < nloops) w = __ldg(space + ((pp.p[l].s1i * (r - pp.p[l].t1)) & maskN));
      s_w[l * kFoldMaxRows + jj] = w;
    }
  }
  __syncthreads();
  if (tid < 32) {
    int base = 0;
    for (int c0 = 0; c0 < cnt; c0 += 32) {
      const int jj = c0 + tid;
      bool nz = false;
      if (jj < cnt) {
#pragma unroll
        for (int l = 0; l < NL; ++l) nz |= (s_w[l * kFoldMaxRows + jj] != (T)0);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, nz);
      if (nz) s_rows[base + __popc(bal & ((1u << tid) - 1u))] = jj;
      base += __popc(bal);
    }
    if (tid == 0) s_nnz = base;
  }
  __syncthreads();
  const int nnz = s_nnz;
  const int cc = tid * 2;                       // column inside the tile
  const bool act = cc < TWC;
  const int c0 = tile * TWC + cc;
  C u[NL][2];
#pragma unroll
  for (int l = 0; l < NL; ++l) { u[l][0] = mk<T>(0, 0); u[l][1] = mk<T>(0, 0); }
  bool bad = false;   // NaN/Inf among the samples read (as_complex_matrix, corefft.py:49-50)
  if (act) {
    const Tin* col = x + c0;
    for (int i = 0; i < nnz; i += UNR) {
      C v[UNR][2];
      int jr[UNR];
#pragma unroll
      for (int k = 0; k < UNR; ++k) {
        jr[k] = (i + k < nnz) ? s_rows[i + k] : -1;
        if (jr[k] >= 0) {
          const size_t r = (size_t)(rho + (j0 + jr[k]) * B);
          ColLoad<Tin, T, 2>::ld(col + (r << lgN), v[k]);
        } else {
          v[k][0] = mk<T>(0, 0);
          v[k][1] = mk<T>(0, 0);
        }
      }
      if (nonfinite) {
#pragma unroll
        for (int k = 0; k < UNR; ++k)
          bad |= !isfinite(v[k][0].x) || !isfinite(v[k][0].y) || !isfinite(v[k][1].x) ||
                 !isfinite(v[k][1].y);
      }
#pragma unroll
      for (int k = 0; k < UNR; ++k) {
        if (jr[k] < 0) break;
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const T wr = s_w[l * kFoldMaxRows + jr[k]];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            u[l][q].x = fma(wr, v[k][q].x, u[l][q].x);
            u[l][q].y = fma(wr, v[k][q].y, u[l][q].y);
          }
        }
      }
    }
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && (tid & 31) == 0) atomicOr(nonfinite, 1u);
  C* red = reinterpret_cast<C*>(smem_raw);
  if (act) {
#pragma unroll
    for (int l = 0; l < NL; ++l)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        T w = (T)0;
        if (l < nloops) w = __ldg(space + ((pp.p[l].s2i * ((unsigned)(c0 + q) - pp.p[l].t2)) & maskN));
        red[l * TWC + cc + q] = mk<T>(w * u[l][q].x, w * u[l][q].y);
      }
  }
  __syncthreads();
  const size_t BB = (size_t)B * B;
  const int reps = TWC >> lgB;
  C* resv = red + (size_t)NL * TWC;             // [nloops][B] row of this tile
  for (int e = tid; e < nloops * B; e += blockDim.x) {
    const int l = e >> lgB;
    const int kap = e & (B - 1);
    C s = mk<T>(0, 0);
    for (int a = 0; a < reps; ++a) s = cadd(s, red[l * TWC + kap + (a << lgB)]);
    resv[e] = s;
  }
  // the cluster's tiles (consecutive along x) are summed through distributed
  // shared memory in rank order; each CTA of the cluster emits a slice
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int csz = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  cl.sync();
  const int tot = nloops * B;
  const int per = (tot + csz - 1) / csz;
  for (int e = rank * per + tid; e < min(tot, (rank + 1) * per); e += blockDim.x) {
    C s = mk<T>(0, 0);
    for (int q = 0; q < csz; ++q) s = cadd(s, cl.map_shared_rank(resv, q)[e]);
    const int l = e >> lgB;
    const int kap = e & (B - 1);
    if (zp == 1) {
      const unsigned ra = natural ? (unsigned)rho : (pp.p[l].s1i * ((unsigned)rho - pp.p[l].t1)) & maskB;
      const unsigned cb = natural ? (unsigned)kap : (pp.p[l].s2i * ((unsigned)kap - pp.p[l].t2)) & maskB;
      dst[l * BB + (size_t)ra * B + cb] = s;
    } else {
      const size_t part = (size_t)(tile / csz) * gridDim.z + z;
      dst[(part * nloops + l) * BB + (size_t)rho * B + kap] = s;
    }
  }
  cl.sync();   // peers have finished reading this CTA's shared memory
}

// Ring-buffered single-loop fold for B < TW (= 512 columns per tile, 256
// threads x 2 columns): the same sums, geometry and outputs as
// k_fold<Tin, T, 1, 2, *> (CTA (rho, chunk z), rows rho + j B of the chunk
// with nonzero window weight), but the rows are moved by the TMA engine:
// thread 0 streams each row's 32 KB segment into one of `nslot`
// shared-memory slots with cp.async.bulk (completion on the slot's
// mbarrier), so up to nslot rows per CTA are in flight without holding
// registers; every thread then folds its 2 columns per 512-column block from
// shared memory.  Column weights stay in registers for the whole CTA.
constexpr int kRingSegBytes = 32 * 1024;

// two adjacent complex inputs from shared memory, converted to cplx<T>
template <typename T>
__device__ __forceinline__ void lds_pair(const float2* p, cplx<T>* v) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  v[0] = mk<T>((T)a.x, (T)a.y);
  v[1] = mk<T>((T)a.z, (T)a.w);
}
template <typename T>
__device__ __forceinline__ void lds_pair(const double2* p, cplx<T>* v) {
  const double2 a = p[0], b = p[1];
  v[0] = mk<T>((T)a.x, (T)a.y);
  v[1] = mk<T>((T)b.x, (T)b.y);
}

template <typename Tin, typename T>
__global__ void __launch_bounds__(256, 1)
k_fold_ring(const Tin* __restrict__ x, const T* __restrict__ space, Perm p, FoldGeom gm,
            bool natural, int nslot, cplx<T>* __restrict__ dst,
            unsigned long long* __restrict__ zero_peak = nullptr) {
  pdl_wait();
  using C = cplx<T>;
  constexpr int SEGC = kRingSegBytes / (int)sizeof(Tin);   // columns per row segment
  constexpr int NB = SEGC / 512;                            // 512-column blocks per segment
  if (zero_peak && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) *zero_peak = 0ull;
  __shared__ T s_w[kFoldMaxRows];
  __shared__ int s_rows[kFoldMaxRows];
  __shared__ int s_nnz;
  __shared__ __align__(8) unsigned long long s_bar[8];
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Tin* ring = reinterpret_cast<Tin*>(smem_raw);
  C* red = reinterpret_cast<C*>(smem_raw + (size_t)nslot * kRingSegBytes);

  const int N = 1 << gm.lgN, B = 1 << gm.lgB;
  const unsigned maskN = (unsigned)N - 1u, maskB = (unsigned)B - 1u;
  const int rho = blockIdx.y, z = blockIdx.z;
  const int aliases = N >> gm.lgB;
  const int j0 = z * gm.rpc;
  const int cnt = min(gm.rpc, aliases - j0);
  const int tid = threadIdx.x;

  for (int jj = tid; jj < cnt; jj += blockDim.x) {
    const unsigned r = (unsigned)(rho + (j0 + jj) * B);
    s_w[jj] = __ldg(space + ((p.s1i * (r - p.t1)) & maskN));
  }
  if (tid < nslot) mbar_init(&s_bar[tid], 1);
  mbar_fence_init();
  __syncthreads();
  if (tid < 32) {
    int base = 0;
    for (int c0 = 0; c0 < cnt; c0 += 32) {
      const int jj = c0 + tid;
      const bool nz = jj < cnt && s_w[jj] != (T)0;
      const unsigned bal = __ballot_sync(0xffffffffu, nz);
      if (nz) s_rows[base + __popc(bal & ((1u << tid) - 1u))] = jj;
      base += __popc(bal);
    }
    if (tid == 0) s_nnz = base;
  }
  __syncthreads();
  const int nnz = s_nnz;
  const int cp = tid * 2;
  C acc[2] = {mk<T>(0, 0), mk<T>(0, 0)};
  unsigned use = 0;                        // completed uses of the ring (phase tracking)
  for (int cg = 0; cg < N / SEGC; ++cg) {
    T wc[NB][2];
    bool any = false;
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const unsigned c = (unsigned)(cg * SEGC + b * 512 + cp + q);
        wc[b][q] = __ldg(space + ((p.s2i * (c - p.t2)) & maskN));
        any |= wc[b][q] != (T)0;
      }
    if (!__syncthreads_or(any)) continue;   // no column of this segment carries weight
    C u[NB][2];
#pragma unroll
    for (int b = 0; b < NB; ++b) u[b][0] = u[b][1] = mk<T>(0, 0);
    auto issue = [&](int i) {
      const int slot = (int)((use + i) % nslot);
      const size_t r = (size_t)(rho + (j0 + s_rows[i]) * B);
      mbar_expect_tx(&s_bar[slot], kRingSegBytes);
      bulk_g2s(ring + (size_t)slot * SEGC, x + (r << gm.lgN) + (size_t)cg * SEGC, kRingSegBytes,
               &s_bar[slot]);
    };
    if (tid == 0)
      for (int i = 0; i < min(nslot, nnz); ++i) issue(i);
    for (int i = 0; i < nnz; ++i) {
      const unsigned k = use + i;
      const int slot = (int)(k % nslot);
      mbar_wait(&s_bar[slot], (k / nslot) & 1u);
      const T wr = s_w[s_rows[i]];
      const Tin* row = ring + (size_t)slot * SEGC;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        C v[2];
        lds_pair<T>(row + b * 512 + cp, v);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          u[b][q].x = fma(wr, v[q].x, u[b][q].x);
          u[b][q].y = fma(wr, v[q].y, u[b][q].y);
        }
      }
      __syncthreads();                       // every thread is done with this slot
      if (tid == 0 && i + nslot < nnz) issue(i + nslot);
    }
    use += (unsigned)nnz;
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        acc[q].x = fma(wc[b][q], u[b][q].x, acc[q].x);
        acc[q].y = fma(wc[b][q], u[b][q].y, acc[q].y);
      }
  }
  // ---- column aliases within the 512-column tile -> B bucket columns
  red[cp] = acc[0];
  red[cp + 1] = acc[1];
  __syncthreads();
  const size_t BB = (size_t)B * B;
  const int reps = 512 / B;
  for (int kap = tid; kap < B; kap += blockDim.x) {
    C s = mk<T>(0, 0);
    for (int a = 0; a < reps; ++a) s = cadd(s, red[kap + a * B]);
    if (gm.Z == 1) {
      const unsigned ra = natural ? (unsigned)rho : (p.s1i * ((unsigned)rho - p.t1)) & maskB;
      const unsigned cb = natural ? (unsigned)kap : (p.s2i * ((unsigned)kap - p.t2)) & maskB;
      dst[(size_t)ra * B + cb] = s;
    } else {
      dst[(size_t)z * BB + (size_t)rho * B + kap] = s;
    }
  }
}

// k_fold_ring for TWO hash passes from one read (see k_fold_wide2): pass t's
// natural fold at B < 512 (permutation p, window `space`) and the next pass's
// at 2B <= 512 (permutation q, window `space2`).  CTA (rho, z) streams the rows
// rho + jB of its alias chunk; for the 2B grid those rows are bucket row
// rho + (j & 1) B.  Every bucket column of both grids is (cp + q) mod B or 2B
// for the thread's columns cp + q (512 = 0 mod 2B), so each thread keeps
// acc (B) and acc2[j & 1] (2B) for its two columns; the weight products
// wr * wc are formed per row and block (no per-block row sums u[] — those
// would not fit twice in registers).  Rows with a zero weight in both passes
// are skipped.  Partials [Z][B][B] and [Z][2B][2B] (Z = 1: the grids).
// SAME: the second pass has the same B (the tuner's first two passes, whose
// B does not change after a pass without a ratio, tuner.py:182-207): its rows
// all go to bucket row rho, window `space2` = `space`.
template <typename Tin, typename T, bool SAME = false>
__global__ void __launch_bounds__(256)
k_fold_ring2(const Tin* __restrict__ x, const T* __restrict__ space,
             const T* __restrict__ space2, Perm p, Perm q, FoldGeom gm, int nslot,
             cplx<T>* __restrict__ dst, cplx<T>* __restrict__ dst2,
             unsigned long long* __restrict__ zero_peak = nullptr) {
  pdl_wait();
  using C = cplx<T>;
  constexpr int SEGC = kRingSegBytes / (int)sizeof(Tin);
  constexpr int NB = SEGC / 512;
  if (zero_peak && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) *zero_peak = 0ull;
  __shared__ T s_w[kFoldMaxRows], s_w2[kFoldMaxRows];
  __shared__ int s_rows[kFoldMaxRows];
  __shared__ int s_nnz;
  __shared__ __align__(8) unsigned long long s_bar[8];
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Tin* ring = reinterpret_cast<Tin*>(smem_raw);
  C* red = reinterpret_cast<C*>(smem_raw + (size_t)nslot * kRingSegBytes);   // 3 x 512

  const int N = 1 << gm.lgN, B = 1 << gm.lgB;
  const unsigned maskN = (unsigned)N - 1u;
  const int rho = blockIdx.y, z = blockIdx.z;
  const int aliases = N >> gm.lgB;
  const int j0 = z * gm.rpc;
  const int cnt = min(gm.rpc, aliases - j0);
  const int tid = threadIdx.x;
  for (int jj = tid; jj < cnt; jj += blockDim.x) {
    const unsigned r = (unsigned)(rho + (j0 + jj) * B);
    s_w[jj] = __ldg(space + ((p.s1i * (r - p.t1)) & maskN));
    s_w2[jj] = __ldg(space2 + ((q.s1i * (r - q.t1)) & maskN));
  }
  if (tid < nslot) mbar_init(&s_bar[tid], 1);
  mbar_fence_init();
  __syncthreads();
  if (tid < 32) {
    int base = 0;
    for (int c0 = 0; c0 < cnt; c0 += 32) {
      const int jj = c0 + tid;
      const bool nz = jj < cnt && (s_w[jj] != (T)0 || s_w2[jj] != (T)0);
      const unsigned bal = __ballot_sync(0xffffffffu, nz);
      if (nz) s_rows[base + __popc(bal & ((1u << tid) - 1u))] = jj;
      base += __popc(bal);
    }
    if (tid == 0) s_nnz = base;
  }
  __syncthreads();
  const int nnz = s_nnz;
  const int cp = tid * 2;
  C acc[2], acc2[2][2];                       // acc2[row parity][column]
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    acc[k] = mk<T>(0, 0);
    acc2[0][k] = acc2[1][k] = mk<T>(0, 0);
  }
  unsigned use = 0;
  for (int cg = 0; cg < N / SEGC; ++cg) {
    T wc[NB][2], wc2[NB][2];
    bool any = false;
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const unsigned c = (unsigned)(cg * SEGC + b * 512 + cp + k);
        wc[b][k] = __ldg(space + ((p.s2i * (c - p.t2)) & maskN));
        wc2[b][k] = __ldg(space2 + ((q.s2i * (c - q.t2)) & maskN));
        any |= (wc[b][k] != (T)0) | (wc2[b][k] != (T)0);
      }
    if (!__syncthreads_or(any)) continue;
    auto issue = [&](int i) {
      const int slot = (int)((use + i) % nslot);
      const size_t r = (size_t)(rho + (j0 + s_rows[i]) * B);
      mbar_expect_tx(&s_bar[slot], kRingSegBytes);
      bulk_g2s(ring + (size_t)slot * SEGC, x + (r << gm.lgN) + (size_t)cg * SEGC, kRingSegBytes,
               &s_bar[slot]);
    };
    if (tid == 0)
      for (int i = 0; i < min(nslot, nnz); ++i) issue(i);
    for (int i = 0; i < nnz; ++i) {
      const unsigned k = use + i;
      const int slot = (int)(k % nslot);
      mbar_wait(&s_bar[slot], (k / nslot) & 1u);
      const int jr = s_rows[i];
      const T wr = s_w[jr], wr2 = s_w2[jr];
      const int par = SAME ? 0 : ((j0 + jr) & 1);
      const Tin* row = ring + (size_t)slot * SEGC;
      C t1[2] = {mk<T>(0, 0), mk<T>(0, 0)}, t2[2] = {mk<T>(0, 0), mk<T>(0, 0)};
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        C v[2];
        lds_pair<T>(row + b * 512 + cp, v);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          t1[kk].x = fma(wc[b][kk], v[kk].x, t1[kk].x);
          t1[kk].y = fma(wc[b][kk], v[kk].y, t1[kk].y);
          t2[kk].x = fma(wc2[b][kk], v[kk].x, t2[kk].x);
          t2[kk].y = fma(wc2[b][kk], v[kk].y, t2[kk].y);
        }
      }
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        acc[kk].x = fma(wr, t1[kk].x, acc[kk].x);
        acc[kk].y = fma(wr, t1[kk].y, acc[kk].y);
        if (par) {
          acc2[1][kk].x = fma(wr2, t2[kk].x, acc2[1][kk].x);
          acc2[1][kk].y = fma(wr2, t2[kk].y, acc2[1][kk].y);
        } else {
          acc2[0][kk].x = fma(wr2, t2[kk].x, acc2[0][kk].x);
          acc2[0][kk].y = fma(wr2, t2[kk].y, acc2[0][kk].y);
        }
      }
      __syncthreads();                       // every thread is done with this slot
      if (tid == 0 && i + nslot < nnz) issue(i + nslot);
    }
    use += (unsigned)nnz;
  }
  // column aliases within the 512-column tile -> bucket columns (B and 2B)
  red[cp] = acc[0];
  red[cp + 1] = acc[1];
  red[512 + cp] = acc2[0][0];
  red[512 + cp + 1] = acc2[0][1];
  red[1024 + cp] = acc2[1][0];
  red[1024 + cp + 1] = acc2[1][1];
  __syncthreads();
  const size_t BB = (size_t)B * B, B2 = (size_t)B << 1;
  for (int kap = tid; kap < B; kap += blockDim.x) {
    C sum = mk<T>(0, 0);
    for (int a = 0; a < 512 / B; ++a) sum = cadd(sum, red[kap + a * B]);
    dst[(size_t)z * BB + (size_t)rho * B + kap] = sum;
  }
  if (SAME) {
    for (int kap = tid; kap < B; kap += blockDim.x) {
      C sum = mk<T>(0, 0);
      for (int a = 0; a < 512 / B; ++a) sum = cadd(sum, red[512 + kap + a * B]);
      dst2[(size_t)z * BB + (size_t)rho * B + kap] = sum;
    }
    return;
  }
  for (int e = tid; e < 2 * (int)B2; e += blockDim.x) {
    const int par = e / (int)B2, kap = e - par * (int)B2;
    C sum = mk<T>(0, 0);
    for (int a = 0; a < 512 / (int)B2; ++a) sum = cadd(sum, red[512 * (1 + par) + kap + a * (int)B2]);
    dst2[(size_t)z * 4 * BB + (size_t)(rho + par * B) * B2 + kap] = sum;
  }
}

// Deterministic sum of Z partials with 8 independent accumulators (keeps 8
// loads in flight; the combination order is fixed, so results are
// reproducible bit for bit).
template <typename C>
__device__ __forceinline__ C sum_partials(const C* __restrict__ p, size_t stride, int Z) {
  C a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i].x = 0; a[i].y = 0; }
  int z = 0;
  for (; z + 8 <= Z; z += 8) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = cadd(a[i], p[(size_t)(z + i) * stride]);
  }
  for (int i = 0; z < Z; ++z, ++i) a[i] = cadd(a[i], p[(size_t)z * stride]);
  return cadd(cadd(cadd(a[0], a[1]), cadd(a[2], a[3])), cadd(cadd(a[4], a[5]), cadd(a[6], a[7])));
}

// Single-loop fold for B >= 512 (every output sums only (N/B)^2 <= 1024
// samples): CTA = 512 columns (2 per thread, 16-byte loads) x RH consecutive
// output rows rho; for each column alias and row alias the RH row loads are
// independent, and row aliases are unrolled by 4, so a thread keeps 4*RH
// 16-byte loads in flight.  Writes the permuted grid directly (Z = 1).
template <typename Tin, typename T, int RH>
__global__ void __launch_bounds__(256)
k_fold_wide(const Tin* __restrict__ x, const T* __restrict__ space, Perm p, int lgN, int lgB,
            bool natural, cplx<T>* __restrict__ y,
            unsigned long long* __restrict__ zero_peak = nullptr) {
  pdl_wait();
  using C = cplx<T>;
  __shared__ T s_w[RH * 32];
  if (zero_peak && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *zero_peak = 0ull;
  const int B = 1 << lgB;
  const unsigned maskN = (1u << lgN) - 1u, maskB = (unsigned)B - 1u;
  const int A = 1 << (lgN - lgB);            // aliases per axis (<= 32)
  const int rho0 = blockIdx.y * RH;
  const int kap = blockIdx.x * 512 + threadIdx.x * 2;
  for (int e = threadIdx.x; e < RH * A; e += blockDim.x) {
    const int r = e / A, j = e - r * A;
    s_w[r * 32 + j] = __ldg(space + ((p.s1i * ((unsigned)(rho0 + r + (j << lgB)) - p.t1)) & maskN));
  }
  __syncthreads();
  C acc[RH][2];
#pragma unroll
  for (int r = 0; r < RH; ++r) acc[r][0] = acc[r][1] = mk<T>(0, 0);
  // two column aliases per step: 2*RH independent row loads per row alias,
  // row aliases unrolled by 4
  for (int i0 = 0; i0 < A; i0 += 2) {
    const int ni = (i0 + 1 < A) ? 2 : 1;
    T wc[2][2];
    C u[2][RH][2];
#pragma unroll
    for (int ii = 0; ii < 2; ++ii) {
      const int c = kap + ((i0 + ii) << lgB);
      wc[ii][0] = ii < ni ? __ldg(space + ((p.s2i * ((unsigned)c - p.t2)) & maskN)) : (T)0;
      wc[ii][1] = ii < ni ? __ldg(space + ((p.s2i * ((unsigned)c + 1u - p.t2)) & maskN)) : (T)0;
#pragma unroll
      for (int r = 0; r < RH; ++r) u[ii][r][0] = u[ii][r][1] = mk<T>(0, 0);
    }
#pragma unroll 4
    for (int j = 0; j < A; ++j) {
      C v[2][RH][2];
#pragma unroll
      for (int ii = 0; ii < 2; ++ii)
#pragma unroll
        for (int r = 0; r < RH; ++r)
          if (ii < ni)
            ColLoad<Tin, T, 2>::ld(x + kap + ((i0 + ii) << lgB) + ((size_t)(rho0 + r + (j << lgB)) << lgN),
                                   v[ii][r]);
#pragma unroll
      for (int ii = 0; ii < 2; ++ii)
#pragma unroll
        for (int r = 0; r < RH; ++r) {
          if (ii >= ni) continue;
          const T w = s_w[r * 32 + j];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            u[ii][r][q].x = fma(w, v[ii][r][q].x, u[ii][r][q].x);
            u[ii][r][q].y = fma(w, v[ii][r][q].y, u[ii][r][q].y);
          }
        }
    }
#pragma unroll
    for (int ii = 0; ii < 2; ++ii)
#pragma unroll
      for (int r = 0; r < RH; ++r) {
        acc[r][0].x = fma(wc[ii][0], u[ii][r][0].x, acc[r][0].x);
        acc[r][0].y = fma(wc[ii][0], u[ii][r][0].y, acc[r][0].y);
        acc[r][1].x = fma(wc[ii][1], u[ii][r][1].x, acc[r][1].x);
        acc[r][1].y = fma(wc[ii][1], u[ii][r][1].y, acc[r][1].y);
      }
  }
  const unsigned b0 = natural ? (unsigned)kap : (p.s2i * ((unsigned)kap - p.t2)) & maskB;
  const unsigned b1 = natural ? (unsigned)kap + 1u : (p.s2i * ((unsigned)kap + 1u - p.t2)) & maskB;
#pragma unroll
  for (int r = 0; r < RH; ++r) {
    const unsigned a = natural ? (unsigned)(rho0 + r) : (p.s1i * ((unsigned)(rho0 + r) - p.t1)) & maskB;
    y[(size_t)a * B + b0] = acc[r][0];
    y[(size_t)a * B + b1] = acc[r][1];
  }
}

// k_fold_wide for TWO hash passes from one read of x: pass t's natural fold
// Y1 at B (permutation p, window `space`) and, speculatively, the next pass's
// natural fold Y2 at 2B (permutation q, window `space2`).  The tuner almost
// always doubles B (tuner.py:121-130, ratio > delta2), and the next pass's
// permutation is already known (draws do not depend on B), so one HBM read of
// the image serves both passes; if the count of pass t sends the tuner
// elsewhere, Y2 is discarded.  Bucket row rho of Y1 collects rows
// rho + jB; Y2's rows rho and rho + B are the even / odd j of the same rows
// (columns likewise), so the CTA that owns Y1's (rho, kappa) owns Y2's four
// buckets (rho + {0, B}, kappa + {0, B}).  CTA = one bucket row x 256 columns;
// 16 row-segment loads in flight per thread (~136 registers, 3 CTAs per SM).
template <typename Tin, typename T>
__global__ void __launch_bounds__(128)
k_fold_wide2(const Tin* __restrict__ x, const T* __restrict__ space, const T* __restrict__ space2,
             Perm p, Perm q, int lgN, int lgB, cplx<T>* __restrict__ y, cplx<T>* __restrict__ y2,
             unsigned long long* __restrict__ zero_peak) {
  pdl_wait();
  using C = cplx<T>;
  __shared__ T s_w[32], s_w2[32];
  if (zero_peak && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *zero_peak = 0ull;
  const int B = 1 << lgB;
  const unsigned maskN = (1u << lgN) - 1u;
  const int A = 1 << (lgN - lgB);            // aliases per axis (4 .. 32, even)
  const int rho = blockIdx.y;
  const int kap = blockIdx.x * 256 + threadIdx.x * 2;   // 128 threads x 2 columns
  for (int j = threadIdx.x; j < A; j += blockDim.x) {
    const unsigned r = (unsigned)(rho + (j << lgB));
    s_w[j] = __ldg(space + ((p.s1i * (r - p.t1)) & maskN));
    s_w2[j] = __ldg(space2 + ((q.s1i * (r - q.t1)) & maskN));
  }
  __syncthreads();
  C acc[2], acc2[2][2][2];                   // acc2[column parity][row parity][column]
#pragma unroll
  for (int cq = 0; cq < 2; ++cq) {
    acc[cq] = mk<T>(0, 0);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) acc2[a][b][cq] = mk<T>(0, 0);
  }
  for (int i0 = 0; i0 < A; i0 += 2) {         // column aliases i0 (even), i0 + 1 (odd)
    T wc[2][2], wc2[2][2];
    C u[2][2], u2[2][2][2];                  // [ii][cq], [ii][row parity][cq]
#pragma unroll
    for (int ii = 0; ii < 2; ++ii)
#pragma unroll
      for (int cq = 0; cq < 2; ++cq) {
        const unsigned c = (unsigned)(kap + ((i0 + ii) << lgB) + cq);
        wc[ii][cq] = __ldg(space + ((p.s2i * (c - p.t2)) & maskN));
        wc2[ii][cq] = __ldg(space2 + ((q.s2i * (c - q.t2)) & maskN));
        u[ii][cq] = mk<T>(0, 0);
        u2[ii][0][cq] = u2[ii][1][cq] = mk<T>(0, 0);
      }
    // row aliases in batches of JB = 8: all 16 row-segment loads of a batch are
    // issued before the first FMA (fp64 too: JB = 4 halved the registers but
    // measured 61 -> 71 us — loads in flight matter more than occupancy here)
    constexpr int JB = 8;
    for (int jb = 0; jb < A; jb += JB) {
      C v[JB][2][2];                         // [row alias in batch][ii][cq]
#pragma unroll
      for (int jj = 0; jj < JB; ++jj)
#pragma unroll
        for (int ii = 0; ii < 2; ++ii)
          if (jj < 4 || A > 4)
            ColLoad<Tin, T, 2>::ld(x + kap + ((i0 + ii) << lgB) + ((size_t)(rho + ((jb + jj) << lgB)) << lgN),
                                   v[jj][ii]);
#pragma unroll
      for (int jj = 0; jj < JB; ++jj) {
        if (jj >= 4 && A <= 4) break;
        const int jp = jj & 1;
        const T w = s_w[jb + jj], w2 = s_w2[jb + jj];
#pragma unroll
        for (int ii = 0; ii < 2; ++ii)
#pragma unroll
          for (int cq = 0; cq < 2; ++cq) {
            const C vv = v[jj][ii][cq];
            u[ii][cq].x = fma(w, vv.x, u[ii][cq].x);
            u[ii][cq].y = fma(w, vv.y, u[ii][cq].y);
            u2[ii][jp][cq].x = fma(w2, vv.x, u2[ii][jp][cq].x);
            u2[ii][jp][cq].y = fma(w2, vv.y, u2[ii][jp][cq].y);
          }
      }
    }
#pragma unroll
    for (int ii = 0; ii < 2; ++ii)
#pragma unroll
      for (int cq = 0; cq < 2; ++cq) {
        acc[cq].x = fma(wc[ii][cq], u[ii][cq].x, acc[cq].x);
        acc[cq].y = fma(wc[ii][cq], u[ii][cq].y, acc[cq].y);
#pragma unroll
        for (int jp = 0; jp < 2; ++jp) {
          acc2[ii][jp][cq].x = fma(wc2[ii][cq], u2[ii][jp][cq].x, acc2[ii][jp][cq].x);
          acc2[ii][jp][cq].y = fma(wc2[ii][cq], u2[ii][jp][cq].y, acc2[ii][jp][cq].y);
        }
      }
  }
  y[(size_t)rho * B + kap] = acc[0];
  y[(size_t)rho * B + kap + 1] = acc[1];
  const size_t B2 = (size_t)B << 1;
#pragma unroll
  for (int ii = 0; ii < 2; ++ii)
#pragma unroll
    for (int jp = 0; jp < 2; ++jp) {
      C* o = y2 + (size_t)(rho + jp * B) * B2 + kap + ii * B;
      o[0] = acc2[ii][jp][0];
      o[1] = acc2[ii][jp][1];
    }
}

// Sum the Z partials in fixed order and scatter to the permuted bucket grid.
template <typename T>
__global__ void k_fold_reduce(const cplx<T>* __restrict__ part, int Z, int nloops, int lgB,
                              PermPack pp, cplx<T>* __restrict__ y) {
  pdl_wait();
  using C = cplx<T>;
  const int B = 1 << lgB;
  const size_t BB = (size_t)B * B;
  const size_t total = BB * nloops;
  const unsigned maskB = (unsigned)B - 1u;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
       e += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(e / BB);
    const size_t rem = e - l * BB;
    const unsigned rho = (unsigned)(rem >> lgB), kap = (unsigned)(rem & maskB);
    const C s = sum_partials(part + (size_t)l * BB + rem, (size_t)nloops * BB, Z);
    const unsigned a = (pp.p[l].s1i * (rho - pp.p[l].t1)) & maskB;
    const unsigned b = (pp.p[l].s2i * (kap - pp.p[l].t2)) & maskB;
    y[l * BB + (size_t)a * B + b] = s;
  }
}

// Small grids: reduce partials + permute + whole 2D FFT in one CTA per loop.
// Rows padded to B + 1 elements (the column stages are then bank-conflict
// free) and the length-B twiddles staged in shared memory; dynamic smem =
// small_fft_smem<T>(lgB).
template <typename T>
__host__ __device__ inline size_t small_fft_smem(int lgB) {
  const size_t B = (size_t)1 << lgB;
  return (B * (B + 1) + B) * sizeof(cplx<T>);
}

template <typename T>
__global__ void __launch_bounds__(1024) k_fold_reduce_fft_small(const cplx<T>* __restrict__ part, int Z, int nloops,
                                        int lgB, PermPack pp, const cplx<T>* __restrict__ tw,
                                        int lgN, cplx<T>* __restrict__ spec) {
  pdl_wait();
  using C = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s = reinterpret_cast<C*>(smem_raw);
  const int B = 1 << lgB;
  const int BB = B * B;
  const int RS = B + 1;
  C* tws = s + (size_t)B * RS;
  const int l = blockIdx.x;
  const unsigned maskB = (unsigned)B - 1u;
  for (int k = threadIdx.x; k < B; k += blockDim.x) tws[k] = tw[k << (lgN - lgB)];
  for (int e = threadIdx.x; e < BB; e += blockDim.x) {
    const unsigned rho = (unsigned)(e >> lgB), kap = (unsigned)(e & (B - 1));
    const C v = sum_partials(part + (size_t)l * BB + e, (size_t)nloops * BB, Z);
    const unsigned a = (pp.p[l].s1i * (rho - pp.p[l].t1)) & maskB;
    const unsigned b = (pp.p[l].s2i * (kap - pp.p[l].t2)) & maskB;
    s[bitrev(a, lgB) * RS + bitrev(b, lgB)] = v;
  }
  __syncthreads();
  fft_stages<T>(s, B, lgB, 1, RS, tws, lgB);
  fft_stages<T>(s, B, lgB, RS, 1, tws, lgB);
  C* out = spec + (size_t)l * BB;
  for (int e = threadIdx.x; e < BB; e += blockDim.x) out[e] = s[(e >> lgB) * RS + (e & (B - 1))];
}

// Tuner pass for small grids (B*B*sizeof(C) <= kSmall2DBytes), one CTA:
// reduce the fold partials (or take the already permuted grid), 2D FFT in
// shared memory, |Z| and its peak, strict 8-neighbour toroidal maxima above
// floor_rel * peak, appended (unordered) to `list` with the count in `count`.
template <typename T, int kSlots = 4>
__global__ void __launch_bounds__(1024)
k_small_pass(const cplx<T>* __restrict__ part, int Z, bool permuted, int lgB, Perm p,
             const cplx<T>* __restrict__ tw, int lgN, double floor_rel,
             int32_t* __restrict__ list, unsigned* __restrict__ count,
             Publish pub = Publish{nullptr, 0, nullptr, 0}, uint32_t* __restrict__ bm = nullptr) {
  pdl_wait();
  using C = cplx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s = reinterpret_cast<C*>(smem_raw);
  const int B = 1 << lgB, BB = B * B;
  // rows padded to B + 1 elements: the column pass (stride RS) is then free
  // of shared-memory bank conflicts (stride B put a warp on one bank)
  const int RS = B + 1;
  T* m = reinterpret_cast<T*>(s + (size_t)B * RS);
  __shared__ unsigned long long s_peak;
  __shared__ unsigned s_n;
  __shared__ unsigned s_rowflag[2];   // B <= 64: bin rows holding a maximum
  if (threadIdx.x == 0) { s_peak = 0; s_n = 0; s_rowflag[0] = 0u; s_rowflag[1] = 0u; }
  const unsigned maskB = (unsigned)B - 1u;
  // tpe threads per bin split the Z partials (fixed combination order:
  // deterministic); a shuffle tree joins the slices
  const int tpe_lg = BB >= (int)blockDim.x ? 0 : min(5, __ffs(blockDim.x / BB) - 1);
  const int tpe = 1 << tpe_lg;
  const int zs = (Z + tpe - 1) >> tpe_lg;
  // up to kSlots slots per thread (1 when the grid's bins x slices fit the
  // block: B <= 32), their partial sums loaded together (all loads in
  // flight before the first use)
  C vv[kSlots];
  const int total = BB << tpe_lg;
  const C* src[kSlots];
  int zn[kSlots];
  int zmax = 0;
#pragma unroll
  for (int u = 0; u < kSlots; ++u) {
    const int t = threadIdx.x + u * blockDim.x;
    vv[u] = mk<T>(0, 0);
    zn[u] = 0;
    src[u] = part;
    if (t < total) {
      const int e = t >> tpe_lg, sl = t & (tpe - 1);
      const int z0 = permuted ? 0 : sl * zs;
      zn[u] = permuted ? 1 : max(0, min(zs, Z - z0));
      src[u] = part + (size_t)z0 * BB + e;
      zmax = max(zmax, zn[u]);
    }
  }
  // partials in a fixed order per bin; the slots' loads are independent and
  // the z loop is unrolled, so up to 4 x 4 loads per thread are in flight
#pragma unroll 4
  for (int z = 0; z < zmax; ++z)
#pragma unroll
    for (int u = 0; u < kSlots; ++u)
      if (z < zn[u]) vv[u] = cadd(vv[u], src[u][(size_t)z * BB]);
#pragma unroll
  for (int u = 0; u < kSlots; ++u) {
    const int t = threadIdx.x + u * blockDim.x;
    if (t >= total) break;
    const int e = t >> tpe_lg, sl = t & (tpe - 1);
    C v = vv[u];
    for (int o = 1; o < tpe; o <<= 1) {
      const C w = mk<T>(__shfl_down_sync(0xffffffffu, v.x, o), __shfl_down_sync(0xffffffffu, v.y, o));
      v = cadd(v, w);
    }
    if (sl == 0) {
      unsigned a = (unsigned)(e >> lgB), b = (unsigned)(e & (B - 1));
      if (!permuted) {
        a = (p.s1i * (a - p.t1)) & maskB;
        b = (p.s2i * (b - p.t2)) & maskB;
      }
      s[bitrev(a, lgB) * RS + bitrev(b, lgB)] = v;
    }
  }
  // twiddles of a length-B transform, W_B^k = tw[k * N / B], staged in smem
  C* tws = reinterpret_cast<C*>(m + BB);
  for (int k = threadIdx.x; k < B; k += blockDim.x) tws[k] = tw[k << (lgN - lgB)];
  __syncthreads();
  fft_stages<T>(s, B, lgB, 1, RS, tws, lgB);    // rows
  fft_stages<T>(s, B, lgB, RS, 1, tws, lgB);    // columns
  unsigned long long best = 0;
  for (int e = threadIdx.x; e < BB; e += blockDim.x) {
    const T v = cabs_(s[(e >> lgB) * RS + (e & (B - 1))]);
    m[e] = v;
    const unsigned long long k = fkey(v);
    best = k > best ? k : best;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
    best = t > best ? t : best;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(&s_peak, best);
  __syncthreads();
  const double pk = fkey_inv(s_peak);
  const double fl = floor_rel * pk;
  for (int e0 = 0; e0 < BB; e0 += blockDim.x) {
    const int e = e0 + threadIdx.x;
    bool f = false;
    if (pk > 0.0 && e < BB) {
      const unsigned r = (unsigned)(e >> lgB), c = (unsigned)(e & (B - 1));
      const T v = m[e];
      if ((double)v >= fl) {
        const unsigned rm = (r - 1u) & maskB, rp = (r + 1u) & maskB;
        const unsigned cm = (c - 1u) & maskB, cp = (c + 1u) & maskB;
        f = (v > m[(rm << lgB) | cm]) & (v > m[(rm << lgB) | c]) & (v > m[(rm << lgB) | cp]) &
            (v > m[(r << lgB) | cm]) & (v > m[(r << lgB) | cp]) & (v > m[(rp << lgB) | cm]) &
            (v > m[(rp << lgB) | c]) & (v > m[(rp << lgB) | cp]);
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    // the vote bitmap of the pass (k_vote_bitmap's layout: bin bits, then
    // row flags), written whole: every word of the grid once
    if (bm && (threadIdx.x & 31) == 0 && (e - (int)(threadIdx.x & 31)) < BB)
      bm[(e - (int)(threadIdx.x & 31)) >> 5] = bal;
    if (bal) {
      unsigned base = 0;
      if ((threadIdx.x & 31) == 0) base = atomicAdd(&s_n, (unsigned)__popc(bal));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (f) {
        list[base + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u))] = e;
        if (bm) atomicOr(&s_rowflag[(e >> lgB) >> 5], 1u << ((e >> lgB) & 31));
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (bm) {
      uint32_t* flags = bm + (((BB + 31) / 32 + 3) & ~3);
      flags[0] = s_rowflag[0];
      if (B > 32) flags[1] = s_rowflag[1];
    }
    *count = s_n;
    // a single CTA: the count goes to the host's slot directly (no ticket,
    // fences or count read-back: three L2 round trips off every small pass)
    if (pub.slot)
      *reinterpret_cast<volatile unsigned long long*>(pub.slot) =
          ((unsigned long long)s_n << 32) | (unsigned long long)pub.seq;
  }
}

inline FoldGeom fold_geometry(int lgN, int lgB, int cpt) {
  FoldGeom g;
  g.lgN = lgN;
  g.lgB = lgB;
  const int N = 1 << lgN, B = 1 << lgB;
  g.TW = min(N, kFoldThreads * cpt);
  g.ktiles = B >= g.TW ? B / g.TW : 1;
  const int aliases = N / B;
  const long per_z = (long)B * g.ktiles;
  const long target = 8L * kNumSMs;
  int Z = (int)((target + per_z - 1) / per_z);
  if (Z < 1) Z = 1;
  if (Z > aliases) Z = aliases;
  int rpc = (aliases + Z - 1) / Z;
  if (rpc > kFoldMaxRows) rpc = kFoldMaxRows;
  g.rpc = rpc;
  g.Z = (aliases + rpc - 1) / rpc;
  g.tab = -1;
  return g;
}

}  // namespace sfft
