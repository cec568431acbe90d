// Host-side per-iteration draws of the lookahead producer, bit-exact with the
// reference's numpy streams (reference rng.py:14-24, solvers.py:250-262,384,395):
//
//   substream(seed, name, t) = Generator(PCG64(SeedSequence((seed, crc32(name), t))))
//   block_t  = sort(substream(seed, "block", t).choice(n, b, replace=False))
//   crc_t    = zlib.crc32(block_t as little-endian int64 bytes)
//   omega_t  = PCG64 state words of substream(seed, "omega", t) (the device
//              generator, rng.cu, expands them into the b x r sketch matrix)
//   v0_t     = substream(seed, "power", t).standard_normal(b), normalised
//
// Restated from numpy's published algorithms (numpy 2.3): SeedSequence's
// hash mixing (bit_generator.pyx), PCG64 XSL-RR 128/64 seeding and 32-bit
// buffering (pcg64.h), Generator.choice without replacement -- Floyd's
// algorithm with a hash set, or a tail shuffle when n > 10000 and b > n/50
// (_generator.pyx) -- Lemire's bounded integers (distributions.c) and the
// 256-step ziggurat (distributions.c, tables in ziggurat_tables.cuh). Pinned
// against numpy in tests/test_host_draws.py.
//
// In C so that the producer's per-iteration draws run without the GIL and on
// several host threads: done in Python they held the interpreter ~0.4 ms per
// iteration and kept the solver thread from enqueueing its launches.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>
#include <algorithm>

#include "common.cuh"
#define SAP_ZIG_QUAL static const
#include "ziggurat_tables.cuh"

namespace sap {
int fail(int code, const char *fmt, ...);
}

namespace {

using u128 = unsigned __int128;

// ---- crc32 (zlib: reflected polynomial 0xEDB88320) -----------------------------
struct Crc32Table {
  uint32_t t[256];
  Crc32Table() {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      t[i] = c;
    }
  }
};
const Crc32Table kCrc;

uint32_t crc32(const void* data, size_t len) {
  const uint8_t* p = static_cast<const uint8_t*>(data);
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < len; ++i) c = kCrc.t[(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

// ---- SeedSequence (pool size 4, no spawn key) --------------------------------------
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

// entropy words of an int: little-endian 32-bit words, [0] for zero
int int_words(uint64_t x, uint32_t* out) {
  if (x == 0) { out[0] = 0; return 1; }
  int k = 0;
  while (x) { out[k++] = static_cast<uint32_t>(x); x >>= 32; }
  return k;
}

// 4 uint64 words = SeedSequence(key).generate_state(4, uint64)
void seed_sequence_state(const uint64_t* key, int nkey, uint64_t out[4]) {
  uint32_t ent[16];
  int ne = 0;
  for (int i = 0; i < nkey; ++i) ne += int_words(key[i], ent + ne);
  uint32_t hc = kInitA;
  auto hashmix = [&hc](uint32_t v) {
    v ^= hc;
    hc *= kMultA;
    v *= hc;
    v ^= v >> 16;
    return v;
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = kMixL * x - kMixR * y;
    return r ^ (r >> 16);
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < ne ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (int s = 4; s < ne; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s]));
  uint32_t hb = kInitB, w[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  for (int i = 0; i < 4; ++i) out[i] = static_cast<uint64_t>(w[2 * i]) | (static_cast<uint64_t>(w[2 * i + 1]) << 32);
}

// ---- PCG64 ----------------------------------------------------------------------
const u128 kPcgMult = (static_cast<u128>(2549297995355413924ull) << 64) + 4865540595714422341ull;

struct Pcg64 {
  u128 state, inc;
  bool has32 = false;
  uint32_t buf32 = 0;

  explicit Pcg64(const uint64_t w[4]) {  // pcg64_set_seed(seed = w[0:2], inc = w[2:4])
    u128 s = (static_cast<u128>(w[0]) << 64) | w[1];
    u128 q = (static_cast<u128>(w[2]) << 64) | w[3];
    state = 0;
    inc = (q << 1) | 1u;
    state = state * kPcgMult + inc;
    state += s;
    state = state * kPcgMult + inc;
  }
  uint64_t next64() {
    state = state * kPcgMult + inc;
    uint64_t hi = static_cast<uint64_t>(state >> 64), lo = static_cast<uint64_t>(state);
    uint64_t x = hi ^ lo;
    unsigned rot = static_cast<unsigned>(hi >> 58);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  uint32_t next32() {
    if (has32) { has32 = false; return buf32; }
    uint64_t v = next64();
    has32 = true;
    buf32 = static_cast<uint32_t>(v >> 32);
    return static_cast<uint32_t>(v);
  }
  double next_double() { return static_cast<double>(next64() >> 11) * (1.0 / 9007199254740992.0); }
};

Pcg64 substream(uint64_t seed, uint32_t name_crc, uint64_t t) {
  uint64_t key[3] = {seed, name_crc, t}, w[4];
  seed_sequence_state(key, 3, w);
  return Pcg64(w);
}

// random_bounded_uint64(off=0, rng, mask=0, use_masked=false): Lemire
uint64_t bounded(Pcg64& g, uint64_t rng) {
  if (rng == 0) return 0;
  if (rng <= 0xFFFFFFFFull) {
    if (rng == 0xFFFFFFFFull) return g.next32();
    const uint32_t r = static_cast<uint32_t>(rng), ex = r + 1;
    uint64_t m = static_cast<uint64_t>(g.next32()) * ex;
    uint32_t left = static_cast<uint32_t>(m);
    if (left < ex) {
      const uint32_t thr = (0xFFFFFFFFu - r) % ex;
      while (left < thr) {
        m = static_cast<uint64_t>(g.next32()) * ex;
        left = static_cast<uint32_t>(m);
      }
    }
    return m >> 32;
  }
  if (rng == ~0ull) return g.next64();
  const uint64_t ex = rng + 1;
  u128 m = static_cast<u128>(g.next64()) * ex;
  uint64_t left = static_cast<uint64_t>(m);
  if (left < ex) {
    const uint64_t thr = (~0ull - rng) % ex;
    while (left < thr) {
      m = static_cast<u128>(g.next64()) * ex;
      left = static_cast<uint64_t>(m);
    }
  }
  return static_cast<uint64_t>(m >> 64);
}

// Generator.choice(n, b, replace=False) as a sorted set (the shuffle that
// follows Floyd's loop permutes the set only, so it is not replayed)
void choice_sorted(Pcg64& g, int64_t n, int64_t b, int64_t* out, std::vector<uint64_t>& scratch) {
  if (n > 10000 && b > n / 50) {
    scratch.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) scratch[i] = static_cast<uint64_t>(i);
    const int64_t first = std::max<int64_t>(n - b, 1);
    for (int64_t i = n - 1; i >= first; --i) {
      uint64_t j = bounded(g, static_cast<uint64_t>(i));
      std::swap(scratch[i], scratch[j]);
    }
    for (int64_t k = 0; k < b; ++k) out[k] = static_cast<int64_t>(scratch[n - b + k]);
  } else {
    uint64_t want = static_cast<uint64_t>(1.2 * static_cast<double>(b)), mask = want;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
    mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
    const uint64_t empty = ~0ull;
    scratch.assign(static_cast<size_t>(mask + 1), empty);
    for (int64_t j = n - b; j < n; ++j) {
      uint64_t v = bounded(g, static_cast<uint64_t>(j)), loc = v & mask;
      while (scratch[loc] != empty && scratch[loc] != v) loc = (loc + 1) & mask;
      if (scratch[loc] == empty) {
        scratch[loc] = v;
        out[j - n + b] = static_cast<int64_t>(v);
      } else {
        loc = static_cast<uint64_t>(j) & mask;
        while (scratch[loc] != empty) loc = (loc + 1) & mask;
        scratch[loc] = static_cast<uint64_t>(j);
        out[j - n + b] = j;
      }
    }
  }
  std::sort(out, out + b);
}

// random_standard_normal (256-step ziggurat)
double standard_normal(Pcg64& g) {
  using namespace sap::zig;
  constexpr double kR = 3.6541528853610087963519472518;
  constexpr double kInvR = 0.27366123732975827203338247596;
  for (;;) {
    uint64_t r = g.next64();
    const int idx = static_cast<int>(r & 0xff);
    r >>= 8;
    const int sign = static_cast<int>(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = static_cast<double>(rabs) * wi[idx];
    if (sign) x = -x;
    if (rabs < ki[idx]) return x;
    if (idx == 0) {
      for (;;) {
        const double xx = -kInvR * std::log1p(-g.next_double());
        const double yy = -std::log1p(-g.next_double());
        if (yy + yy > xx * xx) return ((rabs >> 8) & 1) ? -(kR + xx) : kR + xx;
      }
    }
    if ((fi[idx - 1] - fi[idx]) * g.next_double() + fi[idx] < std::exp(-0.5 * x * x)) return x;
  }
}

// one iteration's draws; returns false when the power start vector is zero twice
bool draw_one(uint64_t seed, int64_t t, int64_t n, int64_t b, int64_t* block, uint32_t* crc,
              int64_t* omega, double* v0, std::vector<uint64_t>& scratch) {
  static const uint32_t kBlock = crc32("block", 5), kOmega = crc32("omega", 5),
                        kPower = crc32("power", 5);
  Pcg64 gb = substream(seed, kBlock, static_cast<uint64_t>(t));
  choice_sorted(gb, n, b, block, scratch);
  *crc = crc32(block, static_cast<size_t>(b) * sizeof(int64_t));
  if (omega) {  // (state_hi, state_lo, inc_hi, inc_lo) of the fresh generator
    Pcg64 go = substream(seed, kOmega, static_cast<uint64_t>(t));
    const uint64_t w[4] = {static_cast<uint64_t>(go.state >> 64), static_cast<uint64_t>(go.state),
                           static_cast<uint64_t>(go.inc >> 64), static_cast<uint64_t>(go.inc)};
    std::memcpy(omega, w, sizeof(w));
  }
  if (v0) {
    Pcg64 gp = substream(seed, kPower, static_cast<uint64_t>(t));
    for (int attempt = 0; attempt < 2; ++attempt) {
      double ss = 0.0;
      for (int64_t i = 0; i < b; ++i) {
        v0[i] = standard_normal(gp);
        ss += v0[i] * v0[i];
      }
      if (ss > 0.0) {
        const double nv = std::sqrt(ss);
        for (int64_t i = 0; i < b; ++i) v0[i] /= nv;
        return true;
      }
    }
    return false;
  }
  return true;
}

}  // namespace

extern "C" int sap_host_draws(uint64_t seed, int64_t t0, int count, int64_t n, int64_t b,
                              int64_t* blocks, uint32_t* crcs, int64_t* omega_states, double* v0,
                              int nthreads) {
  if (count < 0 || n < 1 || b < 1 || b > n || t0 < 0 || !blocks || !crcs)
    return sap::fail(SAP_ERR_CONTRACT, "sap_host_draws: need 0 <= t0, 1 <= b <= n, count >= 0");
  if (count == 0) return SAP_OK;
  int nt = std::max(1, std::min(nthreads, count));
  std::vector<int> ok(static_cast<size_t>(count), 1);
  auto work = [&](int w) {
    std::vector<uint64_t> scratch;
    for (int i = w; i < count; i += nt)
      ok[i] = draw_one(seed, t0 + i, n, b, blocks + static_cast<int64_t>(i) * b, crcs + i,
                       omega_states ? omega_states + 4 * i : nullptr,
                       v0 ? v0 + static_cast<int64_t>(i) * b : nullptr, scratch);
  };
  if (nt == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int w = 0; w < nt; ++w) th.emplace_back(work, w);
    for (auto& x : th) x.join();
  }
  for (int i = 0; i < count; ++i)
    if (!ok[i]) return sap::fail(SAP_ERR_NUMERICAL, "power iteration start vector is zero");
  return SAP_OK;
}
