// pcg64.cuh — NumPy-exact SeedSequence + PCG64 (XSL-RR 128/64) streams,
// usable on host and device.
//
// Restates the published NumPy algorithms the reference depends on
// (numpy>=1.24, pkg/pyproject.toml:10): SeedSequence pool mixing and
// generate_state (bit_generator.pyx), PCG64 seeding (pcg64_set_seed:
// state=0, inc=(initseq<<1)|1, step, state+=initstate, step), the buffered
// next_uint32 (low half first), next_double = (u64>>11)*2^-53,
// Generator.uniform = low + (high-low)*next_double, and random_interval's
// masked rejection over next_uint32 (distributions.c) as consumed by the
// Fisher-Yates shuffle behind Generator.permutation (pnn.py:238).
#pragma once
#include <stdint.h>

#include "../../include/bbml.h"

#if defined(__CUDACC__)
#define BBML_HD __host__ __device__ __forceinline__
#else
#define BBML_HD inline
#endif

namespace bbml {

typedef unsigned __int128 u128;

struct SeedSeq {
  uint32_t pool[4];

  BBML_HD static uint32_t hashmix(uint32_t v, uint32_t& hc) {
    v ^= hc;
    hc *= 0x931E8875u;
    v *= hc;
    return v ^ (v >> 16);
  }
  BBML_HD static uint32_t mix(uint32_t x, uint32_t y) {
    uint32_t r = 0xCA01F9DDu * x - 0x4973F715u * y;
    return r ^ (r >> 16);
  }
  BBML_HD void init(const uint32_t* w, int n) {
    uint32_t hc = 0x43B0D7E5u;
    for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n ? w[i] : 0u, hc);
    for (int s = 0; s < 4; ++s)
      for (int d = 0; d < 4; ++d)
        if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
    for (int s = 4; s < n; ++s)
      for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(w[s], hc));
  }
  // generate_state(n_out, uint32)
  BBML_HD void generate(uint32_t* out, int n_out) const {
    uint32_t hc = 0x8B51F9DDu;
    for (int i = 0; i < n_out; ++i) {
      uint32_t v = pool[i & 3];
      v ^= hc;
      hc *= 0x58F38DEDu;
      v *= hc;
      out[i] = v ^ (v >> 16);
    }
  }
};

struct Pcg64 {
  u128 state, inc;
  uint32_t buf32;
  int has32;

  BBML_HD static u128 mult() {
    return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
  }
  BBML_HD void step() { state = state * mult() + inc; }

  // default_rng(SeedSequence(words))
  BBML_HD void seed_words(const uint32_t* w, int n) {
    SeedSeq ss;
    ss.init(w, n);
    uint32_t o[8];
    ss.generate(o, 8);
    uint64_t s0 = (uint64_t)o[0] | ((uint64_t)o[1] << 32);
    uint64_t s1 = (uint64_t)o[2] | ((uint64_t)o[3] << 32);
    uint64_t s2 = (uint64_t)o[4] | ((uint64_t)o[5] << 32);
    uint64_t s3 = (uint64_t)o[6] | ((uint64_t)o[7] << 32);
    u128 initstate = ((u128)s0 << 64) | s1;
    u128 initseq = ((u128)s2 << 64) | s3;
    state = 0;
    inc = (initseq << 1) | 1;
    step();
    state += initstate;
    step();
    has32 = 0;
    buf32 = 0;
  }

  BBML_HD void seed(const bbml_seed& sd) {
    if (sd.mode == 1) {
      // experiment.series_seed: SeedSequence(entropy).generate_state(1, u64)
      SeedSeq ss;
      ss.init(sd.words, sd.n_words);
      uint32_t o[2];
      ss.generate(o, 2);
      uint32_t w[2] = {o[0], o[1]};
      // int -> uint32 words: 0 -> [0]; < 2^32 -> one word
      seed_words(w, o[1] ? 2 : 1);
    } else {
      seed_words(sd.words, sd.n_words);
    }
  }

  BBML_HD uint64_t next64() {
    step();
    uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    uint64_t x = hi ^ lo;
    unsigned rot = (unsigned)(hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  BBML_HD uint32_t next32() {
    if (has32) {
      has32 = 0;
      return buf32;
    }
    uint64_t v = next64();
    has32 = 1;
    buf32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  BBML_HD double next_double() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }

  // Generator.uniform(low, high): low + (high - low) * u, no FMA contraction.
  BBML_HD double uniform(double low, double high) {
    double u = next_double();
#if defined(__CUDA_ARCH__)
    return __dadd_rn(low, __dmul_rn(__dsub_rn(high, low), u));
#else
    volatile double range = high - low;
    volatile double prod = range * u;
    return low + prod;
#endif
  }

  // random_interval(mx) for mx < 2^32 (masked rejection on the 32-bit stream)
  BBML_HD uint32_t interval32(uint32_t mx) {
    if (mx == 0) return 0;
    uint32_t mask = mx;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    uint32_t v;
    do {
      v = next32() & mask;
    } while (v > mx);
    return v;
  }
};

}  // namespace bbml
