// Host-side per-user minibatch orders, bit-exact with the reference.
//
// The reference draws every user's epoch shuffles on the host:
//   seed  = derive_seed(ctx, "user", uid)        fedsim/core/seeds.py:18-33
//         = first 8 bytes (little endian) of sha256(repr parts joined by \x1f) & (2^63 - 1)
//   rng   = numpy.random.default_rng(seed)       PCG64 seeded by SeedSequence
//   perms = [rng.permutation(n) for _ in range(E)]   fedsim/models/models.py:252-255
// In numpy that chain costs ~19 us per user (hard part 2),
// i.e. ~19 ms of host time per 1000-user context.  This file restates the
// three algorithms natively (numpy >= 1.17 SeedSequence / PCG64 /
// Generator.permutation; restated in SURVEY.md appendix C) so the engine
// produces the identical int32 permutations in ~1 us per user.
#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/fedsim_b200.h"

namespace {

// ------------------------------------------------------------------ SHA-256
struct Sha256 {
  uint32_t h[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                   0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
  uint8_t buf[64];
  uint64_t len = 0;
  size_t fill = 0;

  static uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

  void block(const uint8_t* p) {
    static const uint32_t k[64] = {
        0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
        0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
        0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
        0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
        0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
        0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
        0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
        0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
      w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
    for (int i = 16; i < 64; ++i) {
      const uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      const uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int i = 0; i < 64; ++i) {
      const uint32_t t1 = hh + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + k[i] + w[i];
      const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
      hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
  }
  void update(const uint8_t* p, size_t n) {
    len += n;
    while (n) {
      const size_t take = (64 - fill) < n ? (64 - fill) : n;
      memcpy(buf + fill, p, take);
      fill += take;
      p += take;
      n -= take;
      if (fill == 64) {
        block(buf);
        fill = 0;
      }
    }
  }
  void digest(uint8_t out[32]) {
    const uint64_t bits = len * 8;
    const uint8_t one = 0x80, zero = 0;
    update(&one, 1);
    while (fill != 56) update(&zero, 1);
    uint8_t lenb[8];
    for (int i = 0; i < 8; ++i) lenb[i] = (uint8_t)(bits >> (56 - 8 * i));
    update(lenb, 8);
    for (int i = 0; i < 8; ++i) {
      out[4 * i] = (uint8_t)(h[i] >> 24);
      out[4 * i + 1] = (uint8_t)(h[i] >> 16);
      out[4 * i + 2] = (uint8_t)(h[i] >> 8);
      out[4 * i + 3] = (uint8_t)h[i];
    }
  }
};

uint64_t seed_from_digest(const uint8_t d[32]) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | d[i];
  return v & ((1ULL << 63) - 1);
}

// ----------------------------------------------------- SeedSequence (numpy)
constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
constexpr uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;

struct HashMix {
  uint32_t c = INIT_A;
  uint32_t operator()(uint32_t v) {
    v ^= c;
    c *= MULT_A;
    v *= c;
    return v ^ (v >> 16);
  }
};
uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = MIX_L * x - MIX_R * y;
  return r ^ (r >> 16);
}

// generate_state(4, uint64) of SeedSequence(seed) for a non-negative int seed
void seed_sequence_state(uint64_t seed, uint64_t out[4]) {
  uint32_t ent[2];
  int nent = 0;
  ent[nent++] = (uint32_t)seed;
  if (seed >> 32) ent[nent++] = (uint32_t)(seed >> 32);
  uint32_t pool[4];
  HashMix hm;
  for (int i = 0; i < 4; ++i) pool[i] = hm(i < nent ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hm(pool[s]));
  // (no entropy words beyond the pool size for seeds < 2^128)
  uint32_t hc = INIT_B;
  uint32_t w[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hc;
    hc *= MULT_B;
    v *= hc;
    w[i] = v ^ (v >> 16);
  }
  for (int i = 0; i < 4; ++i) out[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
}

// ------------------------------------------------------------ PCG64 (numpy)
using u128 = unsigned __int128;
struct Pcg64 {
  u128 state, inc;
  bool has32 = false;
  uint32_t buf32 = 0;
  static constexpr u128 MULT = ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
  void step() { state = state * MULT + inc; }
  explicit Pcg64(const uint64_t v[4]) {
    const u128 initstate = ((u128)v[0] << 64) | v[1];
    const u128 initseq = ((u128)v[2] << 64) | v[3];
    state = 0;
    inc = (initseq << 1) | 1;
    step();
    state += initstate;
    step();
  }
  uint64_t next64() {
    step();
    const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
    const unsigned rot = (unsigned)(state >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  uint32_t next32() {
    if (has32) {
      has32 = false;
      return buf32;
    }
    const uint64_t n = next64();
    has32 = true;
    buf32 = (uint32_t)(n >> 32);
    return (uint32_t)n;
  }
  // numpy random_interval: masked rejection sampling in [0, max]
  uint64_t interval(uint64_t max) {
    if (max == 0) return 0;
    uint64_t mask = max;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
    mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
    uint64_t v;
    if (max <= 0xffffffffULL) {
      while ((v = (next32() & mask)) > max) {
      }
    } else {
      while ((v = (next64() & mask)) > max) {
      }
    }
    return v;
  }
};

}  // namespace

extern "C" {

int fb_derive_seed(const uint8_t* data, int64_t len, uint64_t* out) {
  if (!data || len < 0 || !out) return FB_ERR_ARG;
  Sha256 h;
  h.update(data, (size_t)len);
  uint8_t d[32];
  h.digest(d);
  *out = seed_from_digest(d);
  return FB_OK;
}

int fb_user_permutations(uint64_t context_seed, const uint8_t* id_reprs, const int64_t* id_off, int num_users,
                         const int32_t* num_rows, int epochs, int32_t* perms_out, const int64_t* perm_off) {
  if (num_users < 0 || epochs < 0 || (num_users > 0 && (!id_reprs || !id_off || !num_rows || !perm_off)))
    return FB_ERR_ARG;
  // prefix "<ctx>\x1f'user'\x1f" shared by every user (repr(int) + sep + repr("user") + sep)
  const std::string prefix = std::to_string(context_seed) + "\x1f'user'\x1f";
  const uint8_t sep = 0x1f;
  for (int u = 0; u < num_users; ++u) {
    Sha256 h;
    h.update(reinterpret_cast<const uint8_t*>(prefix.data()), prefix.size());
    h.update(id_reprs + id_off[u], (size_t)(id_off[u + 1] - id_off[u]));
    h.update(&sep, 1);
    uint8_t d[32];
    h.digest(d);
    uint64_t st[4];
    seed_sequence_state(seed_from_digest(d), st);
    Pcg64 rng(st);
    const int n = num_rows[u];
    int32_t* out = perms_out + perm_off[u];
    for (int e = 0; e < epochs; ++e) {
      int32_t* a = out + (int64_t)e * n;
      for (int i = 0; i < n; ++i) a[i] = i;
      for (int i = n - 1; i > 0; --i) {
        const int j = (int)rng.interval((uint64_t)i);
        const int32_t t = a[i];
        a[i] = a[j];
        a[j] = t;
      }
    }
  }
  return FB_OK;
}

}  // extern "C"
