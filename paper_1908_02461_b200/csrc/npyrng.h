// Host-side restatement of numpy's default_rng(seed) for an integer seed:
// SeedSequence entropy mixing (numpy/random/bit_generator.pyx, after
// O'Neill's seed_seq) and the PCG64 (XSL-RR 128/64) bit generator
// (numpy/random/src/pcg64), exposed through numpy's bitgen_t layout so that
// numpy's own bounded-integer routine (random_bounded_uint64_fill, linked from
// libnpyrandom.a) draws from it exactly as Generator.integers does.
//
// Used for the SFFT per-loop streams of the reference,
//   loop_rngs[i] = np.random.default_rng(rng.integers(2**63))  (engine.py:268)
// so the 2L child generators are built natively instead of in Python
// (~20 us each there).  Pinned against numpy itself by tests/test_host.py
// (PCG64 states, raw draws and the SFFT permutation lists).
#pragma once
#include <stdint.h>

#include <vector>

namespace npyrng {

// numpy/random/bitgen.h
struct bitgen_t {
  void* state;
  uint64_t (*next_uint64)(void* st);
  uint32_t (*next_uint32)(void* st);
  double (*next_double)(void* st);
  uint64_t (*next_raw)(void* st);
};

struct Pcg64 {
  unsigned __int128 state = 0, inc = 0;
  int has_uint32 = 0;
  uint32_t uinteger = 0;
};

constexpr unsigned __int128 kPcgMult =
    ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | (unsigned __int128)0x4385DF649FCCF645ull;

inline void pcg_step(Pcg64* s) { s->state = s->state * kPcgMult + s->inc; }

inline uint64_t pcg_next64(Pcg64* s) {
  pcg_step(s);   // step, then output the new state (pcg_setseq_128_xsl_rr_64_random_r)
  const uint64_t x = (uint64_t)(s->state >> 64) ^ (uint64_t)s->state;
  const unsigned rot = (unsigned)(s->state >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

inline uint64_t bg_next64(void* st) { return pcg_next64((Pcg64*)st); }
inline uint32_t bg_next32(void* st) {   // pcg64_next32: halves of one 64-bit draw
  Pcg64* s = (Pcg64*)st;
  if (s->has_uint32) {
    s->has_uint32 = 0;
    return s->uinteger;
  }
  const uint64_t v = pcg_next64(s);
  s->has_uint32 = 1;
  s->uinteger = (uint32_t)(v >> 32);
  return (uint32_t)(v & 0xffffffffu);
}
inline double bg_double(void* st) { return (double)(pcg_next64((Pcg64*)st) >> 11) * (1.0 / 9007199254740992.0); }

inline void bind(bitgen_t* bg, Pcg64* s) {
  bg->state = s;
  bg->next_uint64 = bg_next64;
  bg->next_uint32 = bg_next32;
  bg->next_double = bg_double;
  bg->next_raw = bg_next64;
}

// SeedSequence(entropy).generate_state(4, uint64) for a non-negative int
// entropy (pool_size 4, no spawn key)
inline void seed_sequence_state(uint64_t entropy, uint64_t out[4]) {
  const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu,
                 MULT_B = 0x58f38dedu, MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  const int XSHIFT = 16;
  // _coerce_to_uint32_array(int): little-endian 32-bit words, at least one
  std::vector<uint32_t> ent;
  uint64_t v = entropy;
  do {
    ent.push_back((uint32_t)(v & 0xffffffffu));
    v >>= 32;
  } while (v);
  uint32_t hc = INIT_A;
  auto hashmix = [&](uint32_t value) {
    value ^= hc;
    hc *= MULT_A;
    value *= hc;
    value ^= value >> XSHIFT;
    return value;
  };
  auto mix = [&](uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    r ^= r >> XSHIFT;
    return r;
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < (int)ent.size() ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (size_t s = 4; s < ent.size(); ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s]));
  uint32_t w[8];
  uint32_t hb = INIT_B;
  for (int i = 0; i < 8; ++i) {
    uint32_t dv = pool[i & 3];
    dv ^= hb;
    hb *= MULT_B;
    dv *= hb;
    dv ^= dv >> XSHIFT;
    w[i] = dv;
  }
  for (int i = 0; i < 4; ++i) out[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
}

// np.random.default_rng(seed) -> PCG64 state (pcg64_set_seed + srandom_r)
inline void default_rng(uint64_t seed, Pcg64* s) {
  uint64_t st[4];
  seed_sequence_state(seed, st);
  const unsigned __int128 initstate = ((unsigned __int128)st[0] << 64) | st[1];
  const unsigned __int128 initseq = ((unsigned __int128)st[2] << 64) | st[3];
  s->state = 0;
  s->inc = (initseq << 1) | 1u;
  pcg_step(s);
  s->state += initstate;
  pcg_step(s);
  s->has_uint32 = 0;
  s->uinteger = 0;
}

}  // namespace npyrng
