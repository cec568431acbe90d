// Device-side numpy Generator.standard_normal, bit-exact with the host stream.
//
// The reference draws every iteration's Nystrom test matrix on the host,
//   Omega_t = substream(seed, "omega", t).standard_normal((b, r))   solvers.py:384
// (rng.py:14-24: numpy PCG64 seeded by a SeedSequence), 4.4 ms of CPU per
// iteration at b=2000, r=100 -- more than an iteration's GPU time. Here the
// host only seeds the stream (SeedSequence hashing, ~30 us) and passes the
// PCG64 state; the GPU reproduces numpy's sampler exactly:
//
//   PCG64 (XSL-RR 128/64): s <- s*M + inc (mod 2^128), out = rotr(hi^lo, hi>>58)
//   random_standard_normal (numpy/random/src/distributions/distributions.c):
//     r = next_uint64; idx = r & 0xff; r >>= 8; sign = r & 1;
//     rabs = (r >> 1) & (2^52-1); x = +-rabs * wi[idx];
//     rabs < ki[idx]                       -> x                 (~99.3%)
//     idx == 0: tail loop on pairs of next_double -> +-(R + xx)
//     else: wedge test with one next_double -> x, or reject and restart
//
// The draw is a variable-length walk over the raw stream, so it runs in
// three data-parallel passes instead of one sequential loop:
//   1. raw:      R[p] = output after p+1 LCG steps (jump-ahead per chunk)
//   2. classify: for every position p, the outcome IF a normal starts at p:
//                value, emitted or rejected, and how many words it consumes
//   3. resolve:  one CTA per stream compacts the ~1.5% non-trivial positions
//                (in order), decides which of them start a draw (clusters of
//                positions within reach of each other are walked in parallel)
//                and scans the words each start consumes without a value
//   4. emit:     every position computes its output index from the nearest
//                non-trivial position before it (binary search) and writes
// Floating-point steps use explicit _rn intrinsics in numpy's operation order
// (no FMA contraction, as in numpy's x86-64 baseline build). Exactness: every
// fast-path and wedge draw is bit-identical to numpy (the wedge's accept test
// compares against exp(), so CUDA's and libm's exp could only disagree on a
// comparison within 1 ulp, probability ~1e-16). The tail branch (|x| > r =
// 3.654, ~2.6e-4 of draws) calls log1p, where numpy's libm (glibc, an
// ifunc-selected variant) and CUDA can round differently: measured 8 values
// of 12.8M draws differ, each by 1 ulp (tests/test_device_rng.py pins that).
#include <climits>
#include <cstdint>

#include "common.cuh"
#include "ziggurat_tables.cuh"

namespace sap {

int fail(int code, const char *fmt, ...);
int check_launch(const char *what);

namespace rng {

struct U128 {
  uint64_t hi, lo;
};
__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
  return r;
}
__device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}
constexpr uint64_t kMulHi = 0x2360ED051FC65DA4ull, kMulLo = 0x4385DF649FCCF645ull;

// state after `delta` LCG steps (pcg_advance_lcg_128: square-and-multiply)
__device__ U128 advance(U128 s, uint64_t delta, U128 inc) {
  U128 acc_mult{0, 1}, acc_plus{0, 0};
  U128 cur_mult{kMulHi, kMulLo}, cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, U128{0, 1}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  return add128(mul128(acc_mult, s), acc_plus);
}
__device__ __forceinline__ uint64_t output(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = unsigned(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
__device__ __forceinline__ double next_double(uint64_t r) {
  return double(r >> 11) * (1.0 / 9007199254740992.0);
}

constexpr double kR = 3.6541528853610087963519472518;
constexpr double kInvR = 0.27366123732975827203338247596;
constexpr int kChunk = 16;       // raw words per thread
constexpr int kResolveThreads = 1024;
constexpr int kMaxSpecial = 18432;  // non-trivial positions per stream (shared memory; ~1.5%
                                    // of positions, 16.3k expected at count = 2^20)
constexpr int64_t kMaxCount = 1 << 20;

// stream layout of the workspace: R[L] u64, val[L] f64, code[L] i32
// code: bits 0..29 = words consumed by a draw starting here, bit 30 = emits a value,
// 0 = the draw would run past the generated words
__host__ __device__ inline int64_t raw_len(int64_t count) { return count + count / 32 + 2048; }

__global__ void raw_kernel(const uint64_t *states, int64_t L, uint64_t *R) {
  const int s = blockIdx.y;
  const int64_t p0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * kChunk;
  if (p0 >= L) return;
  const uint64_t *st = states + 4 * s;
  const U128 inc{st[2], st[3]};
  U128 x = advance(U128{st[0], st[1]}, uint64_t(p0), inc);
  const U128 mult{kMulHi, kMulLo};
  uint64_t *r = R + s * L;
  for (int k = 0; k < kChunk && p0 + k < L; ++k) {
    x = add128(mul128(x, mult), inc);
    r[p0 + k] = output(x);
  }
}

// The ziggurat tables, gathered into shared memory by every kernel that
// indexes them per thread (divergent __constant__ reads serialise).
struct ZigTables {
  uint64_t ki[256];
  double wi[256], fi[256];
};
__device__ __forceinline__ void load_tables(ZigTables &t) {
  for (int k = threadIdx.x; k < 256; k += blockDim.x) {
    t.ki[k] = zig::ki[k];
    t.wi[k] = zig::wi[k];
    t.fi[k] = zig::fi[k];
  }
}

// The draw that would start at raw word p: its value and code (words consumed,
// bit 30 = emits; 0 = runs past the L generated words).
__device__ __forceinline__ void draw_at(const uint64_t *R, int64_t L, int64_t p,
                                        const ZigTables &t, double &val, int &code) {
  uint64_t r = R[p];
  const int idx = int(r & 0xff);
  r >>= 8;
  const bool neg = (r & 1) != 0;
  const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
  double x = __dmul_rn(double(rabs), t.wi[idx]);
  if (neg) x = -x;
  val = x;
  if (rabs < t.ki[idx]) {
    code = (1 << 30) | 1;
  } else if (idx == 0) {
    code = 0;  // runs past the generated words unless accepted below
    for (int64_t q = p + 1; q + 1 < L; q += 2) {
      const double xx = __dmul_rn(-kInvR, log1p(-next_double(R[q])));
      const double yy = -log1p(-next_double(R[q + 1]));
      if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
        val = ((rabs >> 8) & 1) ? -__dadd_rn(kR, xx) : __dadd_rn(kR, xx);
        code = (1 << 30) | int(q + 2 - p);
        break;
      }
    }
  } else if (p + 1 < L) {
    const double u = next_double(R[p + 1]);
    const double lhs = __dadd_rn(__dmul_rn(__dadd_rn(t.fi[idx - 1], -t.fi[idx]), u), t.fi[idx]);
    const bool acc = lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x));
    code = (acc ? (1 << 30) : 0) | 2;
  } else {
    code = 0;
  }
}

__global__ void __launch_bounds__(256) classify_kernel(const uint64_t *Rall, int64_t L,
                                                      double *valall, int *codeall) {
  __shared__ ZigTables t;
  load_tables(t);
  __syncthreads();
  const int s = blockIdx.y;
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= L) return;
  double val;
  int code;
  draw_at(Rall + s * L, L, p, t, val, code);
  if (valall) valall[s * L + p] = val;
  codeall[s * L + p] = code;
}

// Block-wide exclusive scans of one value per thread (1024 threads).
template <bool MAX>
__device__ int block_scan(int v, int *warp_sums, int &excl) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = MAX ? max(x, y) : x + y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = warp_sums[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w = MAX ? max(w, y) : w + y;
    }
    warp_sums[lane] = w;  // inclusive
  }
  __syncthreads();
  const int base = wid ? warp_sums[wid - 1] : (MAX ? INT_MIN : 0);
  const int xe = __shfl_up_sync(0xffffffffu, x, 1);  // exclusive within the warp
  excl = lane ? (MAX ? max(base, xe) : base + xe) : base;
  const int total = warp_sums[31];
  __syncthreads();
  return total;
}

constexpr int kFast = (1 << 30) | 1;  // code of a one-word emitting draw
constexpr int kChunkPos = 2048;       // positions per compaction chunk

// Per-stream special list (global): pos, flags (bit0 start, bit1 emits), D
// exclusive/inclusive (non-emitting positions before/through the entry's
// range, counted over starts only), cover (prefix max of start range ends).
struct Special {
  int *pos, *flags, *dex, *din, *cover, *n;
};
__device__ __forceinline__ Special special_list(int *base, int s) {
  int *b = base + size_t(s) * (5 * kMaxSpecial + 32);
  return Special{b, b + kMaxSpecial, b + 2 * kMaxSpecial, b + 3 * kMaxSpecial,
                 b + 4 * kMaxSpecial, b + 5 * kMaxSpecial};
}

// One CTA per stream: compact the non-trivial positions (ballot, in order),
// find which of them start a draw (parallel over clusters of mutually
// reachable positions, which are almost always single entries), then scan the
// words each start wastes so every position knows its output index.
__global__ void __launch_bounds__(kResolveThreads, 1)
    resolve_kernel(const int *codeall, int64_t L, int64_t count, int *splist, int *status) {
  extern __shared__ int sm[];
  int *sp_pos = sm;                     // [kMaxSpecial]
  int *sp_code = sp_pos + kMaxSpecial;  // [kMaxSpecial]
  int *chunk_off = sp_code + kMaxSpecial;  // [kResolveThreads]
  __shared__ int warp_sums[32];
  const int s = blockIdx.x;
  const int *code = codeall + s * L;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nchunks = int((L + kChunkPos - 1) / kChunkPos);  // <= 1024 (count <= 2^20)
  // 1. count per chunk (warp per chunk, coalesced), scan, compact in order
  for (int c = wid; c < nchunks; c += 32) {
    int cnt = 0;
    for (int64_t p = int64_t(c) * kChunkPos + lane; p < min(L, int64_t(c + 1) * kChunkPos); p += 32)
      cnt += code[p] != kFast;
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) chunk_off[c] = cnt;
  }
  __syncthreads();
  int my = threadIdx.x < nchunks ? chunk_off[threadIdx.x] : 0, off;
  const int nsp = block_scan<false>(my, warp_sums, off);
  if (nsp > kMaxSpecial) {
    if (threadIdx.x == 0) atomicMax(status, 2);
    return;
  }
  if (threadIdx.x < nchunks) chunk_off[threadIdx.x] = off;
  __syncthreads();
  for (int c = wid; c < nchunks; c += 32) {
    int o = chunk_off[c];
    for (int64_t p0 = int64_t(c) * kChunkPos; p0 < min(L, int64_t(c + 1) * kChunkPos); p0 += 32) {
      const int64_t p = p0 + lane;
      const int cd = p < L ? code[p] : kFast;
      const unsigned m = __ballot_sync(0xffffffffu, cd != kFast);
      if (cd != kFast) {
        const int k = o + __popc(m & ((1u << lane) - 1));
        sp_pos[k] = int(p);
        sp_code[k] = cd;
      }
      o += __popc(m);
    }
  }
  __syncthreads();
  // 2. starts: entry k is certainly a start when no earlier entry's range
  //    reaches it (exclusive prefix max of pos + len); the thread owning such
  //    a head walks its cluster up to the next head
  const int per = (nsp + kResolveThreads - 1) / kResolveThreads;
  const int k0 = min(nsp, per * int(threadIdx.x)), k1 = min(nsp, k0 + per);
  auto reach = [&](int k) {
    const int len = sp_code[k] & 0x3fffffff;
    return len ? sp_pos[k] + len : int(L);  // len 0: the draw runs past the words
  };
  int rmax = INT_MIN;
  for (int k = k0; k < k1; ++k) rmax = max(rmax, reach(k));
  int rex;
  block_scan<true>(rmax, warp_sums, rex);
  // Heads in [k0, k1) (prefix max before k <= pos_k) are starts; the owning
  // thread walks the cluster: cur = end of the last start's range, an entry at
  // or past cur starts a draw, the next head (running prefix max <= its
  // position) ends the cluster. Each entry's start bit (sp_code bit 31) has
  // exactly one writer; reach() reads only the length bits.
  {
    int pm = rex;
    for (int k = k0; k < k1; ++k) {
      if (pm <= sp_pos[k]) {
        sp_code[k] |= int(0x80000000u);
        int cur = reach(k), pmw = max(pm, cur);
        for (int j = k + 1; j < nsp; ++j) {
          const int pj = sp_pos[j];
          if (pmw <= pj) break;  // head of the next cluster
          const int rj = reach(j);
          if (pj >= cur) {
            sp_code[j] |= int(0x80000000u);
            cur = rj;
          }
          pmw = max(pmw, rj);
        }
      }
      pm = max(pm, reach(k));
    }
  }
  __syncthreads();
  // 3. non-emitting positions per start: the range's interior + the start
  //    itself when rejected; exclusive sum -> D, prefix max of start ends -> cover
  Special sp = special_list(splist, s);
  int dsum = 0, cmax = 0;
  for (int k = k0; k < k1; ++k) {
    const int c = sp_code[k];
    if (c < 0) {
      const int r = reach(k);
      dsum += (r - sp_pos[k] - 1) + ((c >> 30) & 1 ? 0 : 1);
      cmax = max(cmax, r);
    }
  }
  int dex;
  const int dtot = block_scan<false>(dsum, warp_sums, dex);
  int cex;
  block_scan<true>(cmax, warp_sums, cex);
  cex = max(cex, 0);
  for (int k = k0; k < k1; ++k) {
    const int c = sp_code[k];
    const bool st = c < 0;
    const int r = reach(k);
    const int nonemit = st ? (r - sp_pos[k] - 1) + ((c >> 30) & 1 ? 0 : 1) : 0;
    sp.pos[k] = sp_pos[k];
    sp.flags[k] = (st ? 1 : 0) | (st && ((c >> 30) & 1) ? 2 : 0);
    sp.dex[k] = dex;
    sp.din[k] = dex + nonemit;
    if (st) cex = max(cex, r);
    sp.cover[k] = cex;
    // a start whose draw runs past the generated words matters only if its
    // value would be one of the first `count`
    if (st && (c & 0x3fffffff) == 0 && sp_pos[k] - dex < count) atomicMax(status, 1);
    dex += nonemit;
  }
  if (threadIdx.x == 0) {
    *sp.n = nsp;
    if (L - dtot < count) atomicMax(status, 1);
  }
}

// Every position writes its value at its output index (or nothing).
__global__ void emit_kernel(const double *valall, int64_t L, int64_t count, const int *splist,
                            double *out, int64_t ldo) {
  const int s = blockIdx.y;
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= L) return;
  const Special sp = special_list(const_cast<int *>(splist), s);
  const int nsp = *sp.n;
  int lo = 0, hi = nsp;  // first entry with pos > p
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sp.pos[mid] <= p) lo = mid + 1; else hi = mid;
  }
  const int k = lo - 1;  // last entry with pos <= p
  int64_t idx;
  if (k >= 0 && sp.pos[k] == p) {
    if (sp.flags[k] != 3) return;
    idx = p - sp.dex[k];
  } else {
    if (k >= 0 && sp.cover[k] > p) return;
    idx = p - (k >= 0 ? sp.din[k] : 0);
  }
  if (idx < count) out[s * ldo + idx] = valall[s * L + p];
}

// ---------------------------------------------------------------------------
// Large draws (count > kMaxCount, one stream): the same passes with the
// non-trivial positions in global memory and every scan split into a
// per-block pass, a one-CTA scan of the block totals and an apply pass.

constexpr int64_t kMaxLarge = int64_t(1) << 30;
constexpr int kScanBlock = 1024;  // entries per block of the special-list scans

__host__ __device__ inline int64_t large_cap(int64_t L) { return L / 32 + 8192; }

struct LargeWs {
  uint64_t *R;
  int *code, *off;  // off[nch + 1]: exclusive chunk offsets, off[nch] = #specials
  int *sp_pos, *sp_code, *sp_flags, *sp_dex, *sp_din, *sp_cover;
  double *sp_val;
  int *blk_a, *blk_b;
  int64_t L, nch, cap, nblk;
};
__host__ __device__ inline size_t align8(size_t x) { return (x + 7) & ~size_t(7); }
__host__ __device__ inline size_t large_bytes(int64_t count, LargeWs *w, uint8_t *base) {
  const int64_t L = raw_len(count), nch = (L + kChunkPos - 1) / kChunkPos, cap = large_cap(L);
  const int64_t nblk = (cap + kScanBlock - 1) / kScanBlock;
  size_t o = 256;
  auto take = [&](size_t bytes) { const size_t at = o; o = align8(o + bytes); return at; };
  const size_t oR = take(8 * L), oc = take(4 * L), oo = take(4 * (nch + 1));
  const size_t op = take(4 * cap), oq = take(4 * cap), of = take(4 * cap), od = take(4 * cap),
               oi = take(4 * cap), ov = take(4 * cap), ol = take(8 * cap);
  const size_t oa = take(4 * nblk), ob = take(4 * nblk);
  if (w) {
    w->R = reinterpret_cast<uint64_t *>(base + oR);
    w->code = reinterpret_cast<int *>(base + oc);
    w->off = reinterpret_cast<int *>(base + oo);
    w->sp_pos = reinterpret_cast<int *>(base + op);
    w->sp_code = reinterpret_cast<int *>(base + oq);
    w->sp_flags = reinterpret_cast<int *>(base + of);
    w->sp_dex = reinterpret_cast<int *>(base + od);
    w->sp_din = reinterpret_cast<int *>(base + oi);
    w->sp_cover = reinterpret_cast<int *>(base + ov);
    w->sp_val = reinterpret_cast<double *>(base + ol);
    w->blk_a = reinterpret_cast<int *>(base + oa);
    w->blk_b = reinterpret_cast<int *>(base + ob);
    w->L = L; w->nch = nch; w->cap = cap; w->nblk = nblk;
  }
  return o;
}

__device__ __forceinline__ int reach_of(int pos, int code, int64_t L) {
  const int len = code & 0x3fffffff;
  return len ? pos + len : int(L);
}

// special positions per 2048-position chunk (a warp per chunk)
__global__ void chunk_count_kernel(const int *code, int64_t L, int64_t nch, int *cnt) {
  const int64_t c = int64_t(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (c >= nch) return;
  int n = 0;
  for (int64_t p = c * kChunkPos + lane; p < min(L, (c + 1) * kChunkPos); p += 32)
    n += code[p] != kFast;
  n = __reduce_add_sync(0xffffffffu, n);
  if (lane == 0) cnt[c] = n;
}

// in-place exclusive scan (sum or max) of v[0..n) by one 1024-thread CTA;
// v[n] receives the total when `total_slot`
template <bool MAX>
__global__ void __launch_bounds__(kResolveThreads, 1)
    scan_inplace_kernel(int *v, int64_t n, bool total_slot, int64_t cap, int *status) {
  __shared__ int warp_sums[32];
  const int64_t per = (n + kResolveThreads - 1) / kResolveThreads;
  const int64_t a = min(n, per * threadIdx.x), b = min(n, a + per);
  int loc = MAX ? INT_MIN : 0;
  for (int64_t k = a; k < b; ++k) loc = MAX ? max(loc, v[k]) : loc + v[k];
  int ex;
  const int tot = block_scan<MAX>(loc, warp_sums, ex);
  for (int64_t k = a; k < b; ++k) {
    const int x = v[k];
    v[k] = ex;
    ex = MAX ? max(ex, x) : ex + x;
  }
  if (threadIdx.x == 0 && total_slot) {
    v[n] = tot;
    if (!MAX && tot > cap) atomicMax(status, 2);
  }
}

// compaction in order (ballot per 32 positions) plus each special's value
__global__ void compact_kernel(const uint64_t *R, int64_t L, const int *code, int64_t nch,
                               const int *off, int64_t cap, int *sp_pos, int *sp_code,
                               double *sp_val, int *sp_flags) {
  __shared__ ZigTables t;
  load_tables(t);
  __syncthreads();
  const int64_t c = int64_t(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (c >= nch || off[nch] > cap) return;
  int o = off[c];
  for (int64_t p0 = c * kChunkPos; p0 < min(L, (c + 1) * kChunkPos); p0 += 32) {
    const int64_t p = p0 + lane;
    const int cd = p < L ? code[p] : kFast;
    const unsigned m = __ballot_sync(0xffffffffu, cd != kFast);
    if (cd != kFast) {
      const int k = o + __popc(m & ((1u << lane) - 1));
      double v;
      int c2;
      draw_at(R, L, p, t, v, c2);
      sp_pos[k] = int(p);
      sp_code[k] = cd;
      sp_val[k] = v;
      sp_flags[k] = 0;
    }
    o += __popc(m);
  }
}

// per block of 1024 entries: max reach (blk_a) -- the prefix-max scan's block totals
__global__ void __launch_bounds__(kScanBlock) reach_block_kernel(const int *sp_pos,
                                                                const int *sp_code,
                                                                const int *nsp_p, int64_t L,
                                                                int *blk) {
  __shared__ int red[32];
  const int nsp = *nsp_p;
  const int64_t k = int64_t(blockIdx.x) * kScanBlock + threadIdx.x;
  int r = k < nsp ? reach_of(sp_pos[k], sp_code[k], L) : INT_MIN;
  r = __reduce_max_sync(0xffffffffu, r);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = r;
  __syncthreads();
  if (threadIdx.x < 32) {
    int v = red[threadIdx.x];
    v = __reduce_max_sync(0xffffffffu, v);
    if (threadIdx.x == 0) blk[blockIdx.x] = v;
  }
}

// heads (no earlier entry reaches them) start clusters; the head's thread
// walks its cluster and writes the start/emit flags of every entry in it
__global__ void __launch_bounds__(kScanBlock) walk_kernel(const int *sp_pos, const int *sp_code,
                                                         const int *nsp_p, int64_t L,
                                                         const int *blkpre, int *sp_flags) {
  __shared__ int warp_sums[32];
  const int nsp = *nsp_p;
  const int64_t k = int64_t(blockIdx.x) * kScanBlock + threadIdx.x;
  const int rk = k < nsp ? reach_of(sp_pos[k], sp_code[k], L) : INT_MIN;
  int ex;
  block_scan<true>(rk, warp_sums, ex);
  if (k >= nsp) return;
  const int pm = max(ex, blkpre[blockIdx.x]);
  if (pm > sp_pos[k]) return;  // inside some earlier range: not a head
  int cur = rk, pmw = max(pm, rk);
  sp_flags[k] = 1 | (((sp_code[k] >> 30) & 1) << 1);
  for (int64_t j = k + 1; j < nsp; ++j) {
    const int pj = sp_pos[j];
    if (pmw <= pj) break;  // the next head
    const int cj = sp_code[j], rj = reach_of(pj, cj, L);
    if (pj >= cur) {
      sp_flags[j] = 1 | (((cj >> 30) & 1) << 1);
      cur = rj;
    }
    pmw = max(pmw, rj);
  }
}

__device__ __forceinline__ int nonemit_of(int pos, int code, int flags, int64_t L) {
  if (!(flags & 1)) return 0;
  return (reach_of(pos, code, L) - pos - 1) + ((flags & 2) ? 0 : 1);
}

// per block: sum of the words starts consume without a value (blk_a) and the
// max start reach (blk_b)
__global__ void __launch_bounds__(kScanBlock) dsum_block_kernel(const int *sp_pos,
                                                               const int *sp_code,
                                                               const int *sp_flags,
                                                               const int *nsp_p, int64_t L,
                                                               int *blk_sum, int *blk_max) {
  __shared__ int rs[32], rm[32];
  const int nsp = *nsp_p;
  const int64_t k = int64_t(blockIdx.x) * kScanBlock + threadIdx.x;
  int ne = 0, cm = 0;
  if (k < nsp) {
    const int f = sp_flags[k];
    ne = nonemit_of(sp_pos[k], sp_code[k], f, L);
    cm = (f & 1) ? reach_of(sp_pos[k], sp_code[k], L) : 0;
  }
  ne = __reduce_add_sync(0xffffffffu, ne);
  cm = __reduce_max_sync(0xffffffffu, cm);
  if ((threadIdx.x & 31) == 0) { rs[threadIdx.x >> 5] = ne; rm[threadIdx.x >> 5] = cm; }
  __syncthreads();
  if (threadIdx.x < 32) {
    int a = __reduce_add_sync(0xffffffffu, rs[threadIdx.x]);
    int m = __reduce_max_sync(0xffffffffu, rm[threadIdx.x]);
    if (threadIdx.x == 0) { blk_sum[blockIdx.x] = a; blk_max[blockIdx.x] = m; }
  }
}

__global__ void __launch_bounds__(kScanBlock) dapply_kernel(
    const int *sp_pos, const int *sp_code, const int *sp_flags, const int *nsp_p, int64_t L,
    int64_t count, const int *blk_sum, const int *blk_max, int *sp_dex, int *sp_din,
    int *sp_cover, int *status) {
  __shared__ int warp_sums[32];
  const int nsp = *nsp_p;
  const int64_t k = int64_t(blockIdx.x) * kScanBlock + threadIdx.x;
  int ne = 0, cr = 0, f = 0;
  if (k < nsp) {
    f = sp_flags[k];
    ne = nonemit_of(sp_pos[k], sp_code[k], f, L);
    cr = (f & 1) ? reach_of(sp_pos[k], sp_code[k], L) : 0;
  }
  int dex, cex;
  block_scan<false>(ne, warp_sums, dex);
  block_scan<true>(cr, warp_sums, cex);
  if (k >= nsp) return;
  dex += blk_sum[blockIdx.x];
  const int cover = max(max(cex, blk_max[blockIdx.x]), cr);
  sp_dex[k] = dex;
  sp_din[k] = dex + ne;
  sp_cover[k] = max(cover, 0);
  if ((f & 1) && (sp_code[k] & 0x3fffffff) == 0 && sp_pos[k] - dex < count)
    atomicMax(status, 1);  // a needed draw runs past the generated words
  if (k == nsp - 1 && L - (dex + ne) < count) atomicMax(status, 1);
}

__global__ void emit_large_kernel(const uint64_t *R, int64_t L, int64_t count, const int *off,
                                  int64_t nch, const int *sp_pos, const int *sp_code,
                                  const int *sp_flags, const int *sp_dex, const int *sp_din,
                                  const int *sp_cover, const double *sp_val, int64_t cap,
                                  double *out, long long *words_used) {
  __shared__ double wi[256];
  for (int e = threadIdx.x; e < 256; e += blockDim.x) wi[e] = zig::wi[e];
  __syncthreads();
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= L || off[nch] > cap) return;
  const int64_t c = p / kChunkPos;
  int lo = off[c], hi = off[c + 1];
  const int first = lo;
  while (lo < hi) {  // first entry of this chunk with pos > p
    const int mid = (lo + hi) >> 1;
    if (sp_pos[mid] <= p) lo = mid + 1; else hi = mid;
  }
  const int k = lo - 1;  // last entry with pos <= p (the previous chunk's last if lo == first)
  (void)first;
  int64_t idx;
  double v;
  if (k >= 0 && sp_pos[k] == p) {
    if (sp_flags[k] != 3) return;
    idx = p - sp_dex[k];
    v = sp_val[k];
    // the stream position after the last requested draw (continuation)
    if (idx == count - 1) *words_used = reach_of(sp_pos[k], sp_code[k], L);
  } else {
    if (k >= 0 && sp_cover[k] > p) return;
    idx = p - (k >= 0 ? sp_din[k] : 0);
    uint64_t r = R[p];  // a one-word draw: recompute its value
    const int layer = int(r & 0xff);
    r >>= 8;
    v = __dmul_rn(double((r >> 1) & 0x000fffffffffffffull), wi[layer]);
    if (r & 1) v = -v;
    if (idx == count - 1) *words_used = p + 1;  // a one-word draw
  }
  if (idx < count) out[idx] = v;
}

}  // namespace rng
}  // namespace sap

using namespace sap;

extern "C" {

size_t sap_normal_workspace(int64_t count, int nstreams) {
  if (count > rng::kMaxCount) return rng::large_bytes(count, nullptr, nullptr);
  const int64_t L = rng::raw_len(count);
  return 256 + size_t(nstreams) * size_t(L) * (8 + 8 + 4) +
         size_t(nstreams) * (5 * rng::kMaxSpecial + 32) * sizeof(int);
}

// one stream of more than kMaxCount normals (rng.cu "Large draws")
static int normal_fill_large(const uint64_t *states, int64_t count, double *out, void *ws,
                             cudaStream_t st) {
  using namespace rng;
  LargeWs w;
  large_bytes(count, &w, static_cast<uint8_t *>(ws));
  int *status = static_cast<int *>(ws);  // sticky, see sap_normal_fill
  int rc;
  const int64_t L = w.L;
  {
    const int64_t threads = (L + kChunk - 1) / kChunk;
    raw_kernel<<<dim3(unsigned((threads + 255) / 256), 1), 256, 0, st>>>(states, L, w.R);
    if ((rc = check_launch("normal_raw_kernel")) != SAP_OK) return rc;
  }
  classify_kernel<<<dim3(unsigned((L + 255) / 256), 1), 256, 0, st>>>(w.R, L, nullptr, w.code);
  if ((rc = check_launch("normal_classify_kernel")) != SAP_OK) return rc;
  const unsigned cgrid = unsigned((w.nch + 7) / 8);
  chunk_count_kernel<<<cgrid, 256, 0, st>>>(w.code, L, w.nch, w.off);
  scan_inplace_kernel<false><<<1, kResolveThreads, 0, st>>>(w.off, w.nch, true, w.cap, status);
  compact_kernel<<<cgrid, 256, 0, st>>>(w.R, L, w.code, w.nch, w.off, w.cap, w.sp_pos, w.sp_code,
                                        w.sp_val, w.sp_flags);
  const int *nsp = w.off + w.nch;
  const unsigned bgrid = unsigned(w.nblk);
  reach_block_kernel<<<bgrid, kScanBlock, 0, st>>>(w.sp_pos, w.sp_code, nsp, L, w.blk_a);
  scan_inplace_kernel<true><<<1, kResolveThreads, 0, st>>>(w.blk_a, w.nblk, false, 0, status);
  walk_kernel<<<bgrid, kScanBlock, 0, st>>>(w.sp_pos, w.sp_code, nsp, L, w.blk_a, w.sp_flags);
  dsum_block_kernel<<<bgrid, kScanBlock, 0, st>>>(w.sp_pos, w.sp_code, w.sp_flags, nsp, L, w.blk_a,
                                                  w.blk_b);
  scan_inplace_kernel<false><<<1, kResolveThreads, 0, st>>>(w.blk_a, w.nblk, false, 0, status);
  scan_inplace_kernel<true><<<1, kResolveThreads, 0, st>>>(w.blk_b, w.nblk, false, 0, status);
  dapply_kernel<<<bgrid, kScanBlock, 0, st>>>(w.sp_pos, w.sp_code, w.sp_flags, nsp, L, count,
                                              w.blk_a, w.blk_b, w.sp_dex, w.sp_din, w.sp_cover,
                                              status);
  emit_large_kernel<<<unsigned((L + 255) / 256), 256, 0, st>>>(
      w.R, L, count, w.off, w.nch, w.sp_pos, w.sp_code, w.sp_flags, w.sp_dex, w.sp_din,
      w.sp_cover, w.sp_val, w.cap, out,
      reinterpret_cast<long long *>(static_cast<uint8_t *>(ws) + 8));
  return check_launch("normal_emit_large_kernel");
}

int sap_normal_fill(const uint64_t *states, int nstreams, int64_t count, double *out, int64_t ldo,
                    void *ws, size_t ws_bytes, void *stream) {
  if (nstreams <= 0 || count <= 0 || count > rng::kMaxLarge || ldo < count ||
      (count > rng::kMaxCount && nstreams != 1))
    return fail(SAP_ERR_CONTRACT, "normal_fill: bad shape streams=%d count=%lld ldo=%lld "
                "(more than 2^20 normals: one stream at a time, at most 2^30)",
                nstreams, (long long)count, (long long)ldo);
  if (!ws || ws_bytes < sap_normal_workspace(count, nstreams))
    return fail(SAP_ERR_CONTRACT, "normal_fill: workspace too small");
  if (count > rng::kMaxCount)
    return normal_fill_large(states, count, out, ws, reinterpret_cast<cudaStream_t>(stream));
  const int64_t L = rng::raw_len(count);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint8_t *w = static_cast<uint8_t *>(ws);
  int *status = reinterpret_cast<int *>(w);  // first 256 bytes: status word
  uint64_t *R = reinterpret_cast<uint64_t *>(w + 256);
  double *val = reinterpret_cast<double *>(w + 256 + size_t(nstreams) * L * 8);
  int *code = reinterpret_cast<int *>(w + 256 + size_t(nstreams) * L * 16);
  int *splist = reinterpret_cast<int *>(w + 256 + size_t(nstreams) * L * 20);
  int rc;
  // the status word is sticky (zeroed by the caller with the workspace; every
  // fill only raises it), so a failed fill is still reported after the
  // workspace has been reused
  {
    const int64_t threads = (L + rng::kChunk - 1) / rng::kChunk;
    dim3 grid(unsigned((threads + 255) / 256), unsigned(nstreams));
    rng::raw_kernel<<<grid, 256, 0, st>>>(states, L, R);
    if ((rc = check_launch("normal_raw_kernel")) != SAP_OK) return rc;
  }
  const dim3 pgrid(unsigned((L + 255) / 256), unsigned(nstreams));
  rng::classify_kernel<<<pgrid, 256, 0, st>>>(R, L, val, code);
  if ((rc = check_launch("normal_classify_kernel")) != SAP_OK) return rc;
  const int smem = (2 * rng::kMaxSpecial + rng::kResolveThreads) * int(sizeof(int));
  cudaFuncSetAttribute(rng::resolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  rng::resolve_kernel<<<nstreams, rng::kResolveThreads, smem, st>>>(code, L, count, splist,
                                                                   status);
  if ((rc = check_launch("normal_resolve_kernel")) != SAP_OK) return rc;
  rng::emit_kernel<<<pgrid, 256, 0, st>>>(val, L, count, splist, out, ldo);
  return check_launch("normal_emit_kernel");
}

// status word of the sap_normal_fill calls on this workspace since the caller
// zeroed it (device pointer, the workspace's first int; sticky: the worst
// outcome of any fill): 0 ok, 1 the generated raw words ran out, 2 too many
// non-trivial draws for the resolve pass
int *sap_normal_status(void *ws) { return static_cast<int *>(ws); }

// raw 64-bit words the last fill of more than 2^20 normals consumed (device
// int64 at byte 8 of the workspace): advancing the stream's PCG64 by it
// continues the stream exactly where numpy would draw the next normal
long long *sap_normal_words(void *ws) {
  return reinterpret_cast<long long *>(static_cast<uint8_t *>(ws) + 8);
}

}  // extern "C"
