// K5 — reverse hashing and voting.
// Replaces _unhash_axis/_unhash_grid (hashing.py:368-386) plus
//   * SFFT per-loop dedup + vote (engine.py:141-160): a coordinate counts once
//     per loop -> a per-coordinate bitmask byte, bit l = "loop l hit it";
//   * tuner votes with multiplicity (tuner.py:175-179, 228-240) -> a per-
//     coordinate byte counter (a strict local maximum's expanded 3x3 preimage
//     can overlap at most 4 others at w = 1 and none at w >= 2, so tallies are
//     bounded by 4 * passes; when that bound exceeds 255 the counters are 32 bit).
// Bytes are packed four to a 32-bit word and updated with atomicOr / atomicAdd
// on the containing word (no carry can cross a byte: bounded above).
//
// Preimage of bin c along one axis with w = N/B and expand e:
//   t in [c*w - floor(w/2) - e, c*w + ceil(w/2) + e)  (length min(w + 2e, N)),
//   coordinate = sigma^-1 * t mod N.
#pragma once
#include "common.cuh"
#include "select.cuh"

namespace sfft {

enum VoteMode { kVoteOrBit = 0, kVoteAdd8 = 1, kVoteAdd32 = 2 };

// bins: flat bin indices (bi*B + bj) per segment, `counts[seg]` valid entries
// (or uniform `count` when counts == nullptr); one permutation per segment.
// budget > 0: skip the whole segment when nb * len^2 > budget (the tuner's
// vote budget, tuner.py:165,175, evaluated on the device so the vote can be
// queued before the host learns the count).
__global__ void k_vote(const int32_t* __restrict__ bins, long seg_stride, const unsigned* counts,
                       long count, const Perm* __restrict__ perms, int lgN, int lgB, int expand,
                       int mode, int bit0, uint32_t* __restrict__ hist, long long budget = 0,
                       Perm pval = Perm{0, 0, 0, 0, 0, 0}) {
  pdl_wait();
  const int seg = blockIdx.y;
  const long nb = counts ? (long)counts[seg] : count;
  const int N = 1 << lgN;
  const unsigned maskN = (unsigned)N - 1u;
  const int w = N >> lgB;
  int len, shiftlo;
  if (w == 1 && expand == 0) {
    len = 1;
    shiftlo = 0;
  } else {
    len = min(w + 2 * expand, N);
    shiftlo = w / 2 + expand;
  }
  const long per = (long)len * len;
  const long total = nb * per;
  if (budget > 0 && total > budget) return;
  const Perm p = perms ? perms[seg] : pval;   // by value for single-segment tuner votes
  const int32_t* sb = bins + seg * seg_stride;
  const unsigned bitv = 1u << ((bit0 + seg) & 7);
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x) {
    const long q = e / per;
    const int rem = (int)(e - q * per);
    const int a = rem / len, b = rem - a * len;
    const unsigned bin = (unsigned)sb[q];
    const unsigned bi = bin >> lgB, bj = bin & ((1u << lgB) - 1u);
    const unsigned ti = (unsigned)((int)(bi * w) - shiftlo + a) & maskN;
    const unsigned tj = (unsigned)((int)(bj * w) - shiftlo + b) & maskN;
    const unsigned ii = (p.s1i * ti) & maskN, jj = (p.s2i * tj) & maskN;
    const size_t key = ((size_t)ii << lgN) | jj;
    if (mode == kVoteAdd32) {
      atomicAdd(hist + key, 1u);
    } else {
      const unsigned sh = (unsigned)(key & 3u) * 8u;
      if (mode == kVoteAdd8) atomicAdd(hist + (key >> 2), 1u << sh);
      else atomicOr(hist + (key >> 2), bitv << sh);
    }
  }
}

// Deferred tuner vote (kVoteAdd8 tallies, tuner.py:175-179, 228-240).
// Instead of adding every voting pass into an N^2 histogram in HBM, the tuner
// archives each pass's maxima list (a few KB) and ONE kernel at the end
// computes the tallies of a tile of G consecutive keys (R = G / N natural rows)
// in shared memory from all archived passes, then thresholds them straight
// into the compaction bitmask (k_hist_bits' output) — the histogram never
// touches HBM.  Per pass, for row i of the tile:
//   coordinate (i, j) is in the preimage of maximum (a, b) iff t = s1 i mod N
//   lies in T_a and v = s2 j mod N lies in T_b, where
//   T_c = [c w - floor(w/2) - 1, c w + ceil(w/2) + 1) mod N  (expand = 1),
// so row i gains, at every j = s2^-1 v with v in T_b, the number of maxima
// (a, b) whose bin row a has t in T_a (at most 3 bin rows).
//   * bitmap passes (B <= 512): the pass's B x B maxima bitmap is built in
//     shared memory; [A] lists each row's active bin columns b with their
//     multiplicity, [B] scatters the increments with shared atomics;
//   * list passes (B >= 1024, at most kLazyScan maxima): every maximum's
//     len x len preimage is tested against the tile's rows.
// Passes with more maxima at B >= 1024 were voted into `hist_init` with
// k_vote (one atomic per coordinate) and seed the tile.  Bytes cannot carry:
// tallies are bounded by 4 * passes <= 255 in this mode.
constexpr int kLazyMax = 40;        // archived passes (tuner passes + confirmations + fallback)
constexpr int kLazyScan = 8192;     // list passes: maxima scanned by every CTA
constexpr int kLazyMaxRows = 128;   // R = G / N, G >= 8192 keys, N >= 256... capped
struct LazyPass {
  Perm p;
  int lgB;
  int count;
  long long off;                    // list passes: first entry in the list archive;
                                    // bitmap passes: first word of the bitmap archive
  int soff;                         // bitmap passes: first word in k_vote_lazy2's shared copy
};

// words of one archived bitmap pass: B^2 bits, then B row-flag bits, each
// padded to whole 16-byte chunks (cp.async granules)
__host__ __device__ inline int lazy_bm_words(int lgB) {
  const int B = 1 << lgB;
  return (((B * B + 31) / 32 + 3) & ~3) + (((B + 31) / 32 + 3) & ~3);
}

// Archive one bitmap pass: maxima bitmap + row flags of the pass's list into a
// zeroed region (tuner pass order; runs on the main stream after the maxima
// kernel, one thread per maximum).
__global__ void k_vote_bitmap(const int32_t* __restrict__ list, const unsigned* __restrict__ count_p,
                              int lgB, uint32_t* __restrict__ bm) {
  pdl_wait();
  const int B = 1 << lgB;
  uint32_t* flags = bm + (((B * B + 31) / 32 + 3) & ~3);
  const unsigned cnt = *count_p;
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += gridDim.x * blockDim.x) {
    const unsigned bin = (unsigned)list[e];
    atomicOr(&bm[bin >> 5], 1u << (bin & 31u));
    const unsigned a = bin >> lgB;
    atomicOr(&flags[a >> 5], 1u << (a & 31u));
  }
}
struct LazyPasses {
  LazyPass v[kLazyMax];
  int n;
  int lgBmax;                       // largest B of a bitmap pass (sizes the bitmap / lists)
};

__device__ __forceinline__ void lazy_add(uint32_t* tal, unsigned key, unsigned inc) {
  atomicAdd(&tal[key >> 2], inc << ((key & 3u) * 8u));
}

__global__ void __launch_bounds__(256) k_vote_lazy(const int32_t* __restrict__ arch,
                                                    const uint32_t* __restrict__ bmarch, LazyPasses lp,
                                                    int lgN, int lgG,
                                                    const uint32_t* __restrict__ hist_init,
                                                    uint32_t* __restrict__ hist_out, unsigned thr,
                                                    uint32_t* __restrict__ bits,
                                                    unsigned* __restrict__ blk_counts) {
  pdl_wait();
  extern __shared__ __align__(16) uint32_t sm_vote[];
  __shared__ int s_nlist[kLazyMaxRows];
  __shared__ unsigned s_warp[32];
  const int N = 1 << lgN, G = 1 << lgG, R = G >> lgN;
  const unsigned maskN = (unsigned)N - 1u;
  const int tid = threadIdx.x, nt = blockDim.x;
  const size_t k0 = (size_t)blockIdx.x << lgG;
  const unsigned i0 = (unsigned)(k0 >> lgN);
  const int Bmax = 1 << lp.lgBmax;
  const int bmw = lazy_bm_words(lp.lgBmax);
  uint32_t* s_tal = sm_vote;                                   // G bytes
  uint32_t* s_bm0 = s_tal + G / 4;                             // two bitmap buffers
  int* s_list = (int*)(s_bm0 + 2 * bmw);                       // R x Bmax entries
  uint4* t4 = reinterpret_cast<uint4*>(s_tal);
  // bitmap passes arrive by cp.async, the next one while the current is used
  auto fetch = [&](int ps, int buf) {
    const int words = lazy_bm_words(lp.v[ps].lgB);
    const uint32_t* src = bmarch + lp.v[ps].off;
    uint32_t* dst = s_bm0 + buf * bmw;
    for (int e = tid * 4; e < words; e += nt * 4) cp_async16(dst + e, src + e);
    cp_async_commit();
  };
  auto next_bitmap = [&](int from) {
    for (int q = from; q < lp.n; ++q)
      if (lp.v[q].lgB <= lp.lgBmax) return q;
    return -1;
  };
  int cur = next_bitmap(0), buf = 0;
  if (cur >= 0) fetch(cur, 0);
  if (hist_init) {
    const uint4* h4 = reinterpret_cast<const uint4*>(hist_init + k0 / 4);
    for (int e = tid; e < G / 16; e += nt) t4[e] = h4[e];
  } else {
    for (int e = tid; e < G / 16; e += nt) t4[e] = make_uint4(0u, 0u, 0u, 0u);
  }
  for (int r = tid; r < R; r += nt) s_nlist[r] = 0;
  for (int ps = 0; ps < lp.n; ++ps) {
    const LazyPass& P = lp.v[ps];
    const int lgB = P.lgB, B = 1 << lgB;
    const unsigned maskB = (unsigned)B - 1u;
    const int lgw = lgN - lgB, w = 1 << lgw;
    const int len = (w == 1) ? 3 : w + 2;
    const int shiftlo = w / 2 + 1;   // floor(w/2) + expand
    const int32_t* L = arch + P.off;
    if (lgB <= lp.lgBmax) {
      // ---- bitmap pass: its bitmap (k_vote_bitmap) is in buffer `buf`
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      __syncthreads();
      const uint32_t* s_bits = s_bm0 + buf * bmw;
      const uint32_t* s_flag = s_bits + (((B * B + 31) / 32 + 3) & ~3);
      const int nxt = next_bitmap(ps + 1);
      if (nxt >= 0) fetch(nxt, buf ^ 1);   // overlaps [A] and [B] of this pass
      buf ^= 1;
      // [A] item (row r, 32-column chunk q): bin rows a with
      //     t + shiftlo - len < a w <= t + shiftlo, and their maxima in the chunk
      const int chunks = (B + 31) / 32;
      const unsigned cmask = B >= 32 ? 0xffffffffu : ((1u << B) - 1u);
      for (int item = tid; item < R * chunks; item += nt) {
        const int r = item / chunks, q = item - r * chunks;
        const unsigned t = (P.p.s1 * (i0 + (unsigned)r)) & maskN;
        const int hi = (int)((t + (unsigned)N + (unsigned)shiftlo) >> lgw);
        const int lo = (int)((t + (unsigned)N + (unsigned)shiftlo - (unsigned)len + (unsigned)w) >> lgw);
        unsigned rb[3];
        int na = 0;
        unsigned any = 0;
        for (int a = lo; a <= hi; ++a) {
          const unsigned am = (unsigned)a & maskB;
          if (!((s_flag[am >> 5] >> (am & 31u)) & 1u)) continue;
          const unsigned bit0 = am * (unsigned)B + (unsigned)q * 32u;
          rb[na] = B >= 32 ? s_bits[bit0 >> 5] : (s_bits[bit0 >> 5] >> (bit0 & 31u)) & cmask;
          any |= rb[na++];
        }
        while (any) {
          const int k = __ffs(any) - 1;
          any &= any - 1u;
          int m = 0;
          for (int u = 0; u < na; ++u) m += (rb[u] >> k) & 1u;
          const int slot = atomicAdd(&s_nlist[r], 1);
          s_list[r * Bmax + slot] = ((q * 32 + k) << 8) | m;
        }
      }
      __syncthreads();
      // [B] scatter every row's increments into the tile: the row's nt / R
      //     threads walk its entries; preimage offsets rr < w as
      //     (entry, rr) = (e >> lgw, e & (w - 1)), the two expand offsets
      //     rr = w, w + 1 separately (no integer division by len)
      {
        const int tpr = nt / R;                 // threads per row (R <= nt, both powers of 2)
        const int r = tid / tpr, l = tid - r * tpr;
        const int nl = s_nlist[r];
        const int* lst = s_list + r * Bmax;
        const unsigned rowkey = (unsigned)r << lgN;
        const int nmain = w == 1 ? nl * 3 : nl << lgw;
        for (int e = l; e < nmain; e += tpr) {
          int q, rr;
          if (w == 1) { q = e / 3; rr = e - q * 3; } else { q = e >> lgw; rr = e & (w - 1); }
          const int ent = lst[q];
          const unsigned v = ((unsigned)(ent >> 8) * (unsigned)w - (unsigned)shiftlo + (unsigned)rr) & maskN;
          lazy_add(s_tal, rowkey | ((P.p.s2i * v) & maskN), (unsigned)(ent & 255));
        }
        if (w > 1) {
          for (int e = l; e < 2 * nl; e += tpr) {
            const int ent = lst[e >> 1];
            const unsigned rr = (unsigned)w + (unsigned)(e & 1);
            const unsigned v = ((unsigned)(ent >> 8) * (unsigned)w - (unsigned)shiftlo + rr) & maskN;
            lazy_add(s_tal, rowkey | ((P.p.s2i * v) & maskN), (unsigned)(ent & 255));
          }
        }
      }
      __syncthreads();
      for (int r = tid; r < R; r += nt) s_nlist[r] = 0;
    } else {
      // ---- list pass: the preimage rows of maximum (a, b) are s1^-1 t, t in T_a
      for (int e = tid; e < P.count; e += nt) {
        const unsigned bin = (unsigned)L[e];
        const unsigned a = bin >> lgB, b = bin & maskB;
        for (int u = 0; u < len; ++u) {
          const unsigned t = (a * (unsigned)w - (unsigned)shiftlo + (unsigned)u) & maskN;
          const unsigned r = ((P.p.s1i * t) & maskN) - i0;
          if (r >= (unsigned)R) continue;
          for (int v = 0; v < len; ++v) {
            const unsigned tv = (b * (unsigned)w - (unsigned)shiftlo + (unsigned)v) & maskN;
            lazy_add(s_tal, (r << lgN) | ((P.p.s2i * tv) & maskN), 1u);
          }
        }
      }
      __syncthreads();
    }
  }
  if (hist_out) {
    uint4* h4 = reinterpret_cast<uint4*>(hist_out + k0 / 4);
    for (int e = tid; e < G / 16; e += nt) h4[e] = t4[e];
  }
  if (bits) {
    // kCmpElems keys per compaction block: word tid of every block in the tile
    for (int blk = 0; blk < G / kCmpElems; ++blk) {
      const int wl = blk * kCmpWords + tid;   // 32 keys = 8 tally words
      // bytewise h >= thr (SIMD compare), byte flags packed to 4 bits per word
      uint32_t word = 0;
      const unsigned thr4 = thr * 0x01010101u;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t m = __vcmpgeu4(s_tal[wl * 8 + u], thr4) & 0x01010101u;
        word |= ((m | (m >> 7) | (m >> 14) | (m >> 21)) & 15u) << (u * 4);
      }
      bits[(k0 >> 5) + wl] = word;
      const unsigned pre = block_excl_scan256(__popc(word), s_warp);
      if (tid == kCmpThreads - 1) blk_counts[(k0 >> lgG) * (G / kCmpElems) + blk] = pre + __popc(word);
      __syncthreads();
    }
  }
}

// dynamic shared memory of k_vote_lazy
// Barrier-free variant of k_vote_lazy (the same tallies): EVERY bitmap pass
// (bm_words words at the head of the bitmap archive) is staged in shared
// memory once, then each warp takes (tile row, bitmap pass) items on its
// own — the lanes scan the row's candidate bin rows chunk by chunk, and every
// maximum's w + 2 column preimages are spread over the lanes — so the block
// synchronises only before and after the tallies.  (k_vote_lazy, one pass at
// a time with three block barriers per pass, spent its time at those
// barriers: ncu stall "barrier" 6.2 per issued instruction, shared atomics at
// 7% of the pipe's peak, c3.)  List passes as in k_vote_lazy, strided over
// all warps.
__global__ void __launch_bounds__(256) k_vote_lazy2(const int32_t* __restrict__ arch,
                                                     const uint32_t* __restrict__ bmarch,
                                                     int /*smem bitmap words*/, LazyPasses lp, int lgN, int lgG,
                                                     const uint32_t* __restrict__ hist_init,
                                                     uint32_t* __restrict__ hist_out, unsigned thr,
                                                     uint32_t* __restrict__ bits,
                                                     unsigned* __restrict__ blk_counts) {
  pdl_wait();
  extern __shared__ __align__(16) uint32_t sm_vote[];
  __shared__ unsigned s_warp[32];
  const int N = 1 << lgN, G = 1 << lgG, R = G >> lgN;
  const unsigned maskN = (unsigned)N - 1u;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
  const size_t k0 = (size_t)blockIdx.x << lgG;
  const unsigned i0 = (unsigned)(k0 >> lgN);
  uint32_t* s_tal = sm_vote;            // G bytes
  uint32_t* s_bm = s_tal + G / 4;       // every bitmap pass, at its soff
  uint4* t4 = reinterpret_cast<uint4*>(s_tal);
  for (int ps = 0; ps < lp.n; ++ps) {
    if (lp.v[ps].lgB > lp.lgBmax) continue;
    const int words = lazy_bm_words(lp.v[ps].lgB);
    const uint32_t* src = bmarch + lp.v[ps].off;
    uint32_t* dst = s_bm + lp.v[ps].soff;
    for (int e = tid * 4; e < words; e += nt * 4) cp_async16(dst + e, src + e);
  }
  cp_async_commit();
  if (hist_init) {
    const uint4* h4 = reinterpret_cast<const uint4*>(hist_init + k0 / 4);
    for (int e = tid; e < G / 16; e += nt) t4[e] = h4[e];
  } else {
    for (int e = tid; e < G / 16; e += nt) t4[e] = make_uint4(0u, 0u, 0u, 0u);
  }
  // bitmap passes, in archive order
  int nbm = 0;
  for (int ps = 0; ps < lp.n; ++ps) nbm += lp.v[ps].lgB <= lp.lgBmax;
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  const int items = R * nbm;
  for (int item = warp; item < items; item += nwarps) {
    const int r = item % R;
    int k = item / R, ps = 0;
    for (;; ++ps)   // the k-th bitmap pass
      if (lp.v[ps].lgB <= lp.lgBmax && k-- == 0) break;
    const LazyPass& P = lp.v[ps];
    const int lgB = P.lgB, B = 1 << lgB;
    const unsigned maskB = (unsigned)B - 1u;
    const int lgw = lgN - lgB, w = 1 << lgw;
    const int len = (w == 1) ? 3 : w + 2;
    const int shiftlo = w / 2 + 1;   // floor(w/2) + expand
    const uint32_t* s_bits = s_bm + P.soff;
    const uint32_t* s_flag = s_bits + (((B * B + 31) / 32 + 3) & ~3);
    const unsigned t = (P.p.s1 * (i0 + (unsigned)r)) & maskN;
    const int hi = (int)((t + (unsigned)N + (unsigned)shiftlo) >> lgw);
    const int lo = (int)((t + (unsigned)N + (unsigned)shiftlo - (unsigned)len + (unsigned)w) >> lgw);
    const int chunks = (B + 31) / 32;
    const unsigned cmask = B >= 32 ? 0xffffffffu : ((1u << B) - 1u);
    const unsigned rowkey = (unsigned)r << lgN;
    for (int q0 = 0; q0 < chunks; q0 += 32) {
      const int q = q0 + lane;
      unsigned rb[3] = {0u, 0u, 0u};
      int na = 0;
      unsigned any = 0u;
      if (q < chunks) {
        for (int a = lo; a <= hi; ++a) {
          const unsigned am = (unsigned)a & maskB;
          if (!((s_flag[am >> 5] >> (am & 31u)) & 1u)) continue;
          const unsigned bit0 = am * (unsigned)B + (unsigned)q * 32u;
          rb[na] = B >= 32 ? s_bits[bit0 >> 5] : (s_bits[bit0 >> 5] >> (bit0 & 31u)) & cmask;
          any |= rb[na++];
        }
      }
      // every lane's maxima in turn; the warp spreads each one's len column
      // preimages over its lanes
      unsigned ballot = __ballot_sync(0xffffffffu, any != 0u);
      while (ballot) {
        const int src = __ffs(ballot) - 1;
        unsigned bitsrc = __shfl_sync(0xffffffffu, any, src);
        const unsigned r0 = __shfl_sync(0xffffffffu, rb[0], src);
        const unsigned r1 = __shfl_sync(0xffffffffu, rb[1], src);
        const unsigned r2 = __shfl_sync(0xffffffffu, rb[2], src);
        const int qs = __shfl_sync(0xffffffffu, q, src);
        while (bitsrc) {
          const int kk = __ffs(bitsrc) - 1;
          bitsrc &= bitsrc - 1u;
          const unsigned m = ((r0 >> kk) & 1u) + ((r1 >> kk) & 1u) + ((r2 >> kk) & 1u);
          const unsigned b = (unsigned)(qs * 32 + kk);
          for (int rr = lane; rr < len; rr += 32) {
            const unsigned v = (b * (unsigned)w - (unsigned)shiftlo + (unsigned)rr) & maskN;
            lazy_add(s_tal, rowkey | ((P.p.s2i * v) & maskN), m);
          }
        }
        ballot &= ballot - 1u;
      }
    }
  }
  // list passes: every maximum's len x len preimage tested against the tile
  for (int ps = 0; ps < lp.n; ++ps) {
    const LazyPass& P = lp.v[ps];
    if (P.lgB <= lp.lgBmax) continue;
    const int lgB = P.lgB;
    const unsigned maskB = (1u << lgB) - 1u;
    const int lgw = lgN - lgB, w = 1 << lgw;
    const int len = (w == 1) ? 3 : w + 2;
    const int shiftlo = w / 2 + 1;
    const int32_t* L = arch + P.off;
    for (int e = tid; e < P.count; e += nt) {
      const unsigned bin = (unsigned)L[e];
      const unsigned a = bin >> lgB, b = bin & maskB;
      for (int u = 0; u < len; ++u) {
        const unsigned tt = (a * (unsigned)w - (unsigned)shiftlo + (unsigned)u) & maskN;
        const unsigned r = ((P.p.s1i * tt) & maskN) - i0;
        if (r >= (unsigned)R) continue;
        for (int v = 0; v < len; ++v) {
          const unsigned tv = (b * (unsigned)w - (unsigned)shiftlo + (unsigned)v) & maskN;
          lazy_add(s_tal, (r << lgN) | ((P.p.s2i * tv) & maskN), 1u);
        }
      }
    }
  }
  __syncthreads();
  if (hist_out) {
    uint4* h4 = reinterpret_cast<uint4*>(hist_out + k0 / 4);
    for (int e = tid; e < G / 16; e += nt) h4[e] = t4[e];
  }
  if (bits) {
    for (int blk = 0; blk < G / kCmpElems; ++blk) {
      const int wl = blk * kCmpWords + tid;
      uint32_t word = 0;
      const unsigned thr4 = thr * 0x01010101u;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t m = __vcmpgeu4(s_tal[wl * 8 + u], thr4) & 0x01010101u;
        word |= ((m | (m >> 7) | (m >> 14) | (m >> 21)) & 15u) << (u * 4);
      }
      bits[(k0 >> 5) + wl] = word;
      const unsigned pre = block_excl_scan256(__popc(word), s_warp);
      if (tid == kCmpThreads - 1) blk_counts[(k0 >> lgG) * (G / kCmpElems) + blk] = pre + __popc(word);
      __syncthreads();
    }
  }
}

inline size_t vote_lazy_smem(int lgN, int lgG, int lgBmax) {
  const long G = 1L << lgG, Bm = 1L << lgBmax, R = G >> lgN;
  return (size_t)(G / 4 + 2L * lazy_bm_words(lgBmax) + R * Bm) * 4;
}

// Fold one group's loop-bit masks into per-coordinate loop counts (L > 8).
__global__ void k_mask_to_counts(uint32_t* __restrict__ masks, uint32_t* __restrict__ counts,
                                 long nwords) {
  pdl_wait();
  for (long w = blockIdx.x * (long)blockDim.x + threadIdx.x; w < nwords;
       w += (long)gridDim.x * blockDim.x) {
    const uint32_t m = masks[w];
    if (!m) continue;
    uint32_t add = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) add |= (uint32_t)__popc((m >> (8 * b)) & 255u) << (8 * b);
    counts[w] += add;
    masks[w] = 0;
  }
}

// value of coordinate `key` in a histogram of the given mode
__device__ __forceinline__ unsigned hist_value(const uint32_t* hist, size_t key, int mode) {
  if (mode == kVoteAdd32) return hist[key];
  const unsigned byte = (hist[key >> 2] >> ((key & 3u) * 8u)) & 255u;
  return mode == kVoteOrBit ? (unsigned)__popc(byte) : byte;
}

// bitmask of coordinates with value >= thr (block = 8192 coordinates)
__global__ void k_hist_bits(const uint32_t* __restrict__ hist, long nkeys, int mode, unsigned thr,
                            uint32_t* __restrict__ bits, unsigned* __restrict__ blk_counts) {
  pdl_wait();
  __shared__ unsigned s_warp[32];
  const long w = (long)blockIdx.x * kCmpWords + threadIdx.x;
  const long wps = words_for(nkeys);
  uint32_t word = 0;
  if (w < wps) {
    const long k0 = w * 32;
    if (mode == kVoteAdd32) {
      for (int b = 0; b < 32; ++b)
        if (k0 + b < nkeys && hist[k0 + b] >= thr) word |= 1u << b;
    } else {
      // 32 keys = 8 packed words = two 16-byte loads
      const uint4* h4 = reinterpret_cast<const uint4*>(hist + k0 / 4);
      const uint4 u0 = h4[0], u1 = h4[1];
      const uint32_t hw[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (!hw[i]) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          unsigned v = (hw[i] >> (8 * b)) & 255u;
          if (mode == kVoteOrBit) v = __popc(v);
          if (v >= thr) word |= 1u << (i * 4 + b);
        }
      }
    }
    bits[w] = word;
  }
  const unsigned pre = block_excl_scan256(__popc(word), s_warp);
  if (threadIdx.x == kCmpThreads - 1) blk_counts[blockIdx.x] = pre + __popc(word);
}

// tallies of compacted keys
__global__ void k_gather_tallies(const uint32_t* __restrict__ hist, int mode,
                                 const int32_t* __restrict__ keys, const unsigned* __restrict__ m,
                                 int32_t* __restrict__ tallies) {
  pdl_wait();
  const long n = *m;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x)
    tallies[i] = (int32_t)hist_value(hist, (size_t)(uint32_t)keys[i], mode);
}

}  // namespace sfft
