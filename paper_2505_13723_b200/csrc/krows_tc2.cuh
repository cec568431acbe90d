// CTA-pair (cta_group::2) version of the tensor-core block-row product.
//
// Same math as krows_tc.cuh (GEMM1 tf32 3-term distances -> TMEM, epilogue
// P = 2^14 k(S) split fp16 hi/lo -> TMEM, GEMM2 f16 with A from TMEM), but
// every MMA spans the two SMs of a cluster pair: M = 256 block rows (128 per
// CTA's TMEM) and each CTA stages only HALF of the B operands (its 64 of the
// 128 points of a column tile for GEMM1, its nz/2 of the right-hand sides for
// GEMM2). Per SM this halves the shared-memory footprint and L2->SM traffic
// of the column tiles and halves the MMA instructions and barrier round trips
// the single issuing thread spends per kernel entry -- the per-tile
// synchronisation of the single-thread roles is what bounded the 1-CTA kernel
// (profiles/).
//
// Barrier ownership: full/p_full/g_empty/a_full live in the leader CTA (rank
// 0) and receive the peer's TMA bytes (peer bit cleared, cta_group::2 TMA)
// and remote epilogue arrivals (mapa + release.cluster); s_full/empty/
// a_empty/g_full are signalled in both CTAs by multicast tcgen05.commit.
#pragma once

#include "krows_tc.cuh"

// per-role cycle timers (SAP_TC_PROF=1 at run time needs a -DSAP_TC_TIMERS=1
// build); compiled out otherwise -- the clock reads cost epilogue issue slots
#ifndef SAP_TC_TIMERS
#define SAP_TC_TIMERS 0
#endif

namespace sap {
namespace tck2 {

using tck::BM;
using tck::kPScale;
using tck::kSmemCap;
using tck::Params;
using tck::poly_entry;
using tck::pvalue;
using tck::split2;
using tck::split_range;
using tck::kDescBase;

#ifndef SAP_EPI_SPIN
#define SAP_EPI_SPIN 0
#endif
__device__ __forceinline__ void epi_wait(uint32_t bar, uint32_t parity) {
#if SAP_EPI_SPIN
  tc::mbar_wait_spin(bar, parity);
#else
  tc::mbar_wait(bar, parity);
#endif
}

__device__ __forceinline__ unsigned long long prof_clock() {
#if SAP_TC_TIMERS
  return clock64();
#else
  return 0ull;
#endif
}

constexpr int NT = 128;     // points per column tile (64 staged per CTA)
constexpr int NB = 3;       // S/P tiles in flight in TMEM (columns 0..383)
#ifndef SAP_EPI_STAGGER
#define SAP_EPI_STAGGER -1  // cycles; -1: the per-family default (kStagger)
#endif
#ifndef SAP_KSEG
#define SAP_KSEG 16
#endif
constexpr int kSeg = SAP_KSEG;  // tiles per TMEM accumulator segment (2048 points)
constexpr uint32_t kGCol = NB * NT;  // the (single) accumulator, nz columns
constexpr int kEpiGroups = 4;                       // epilogue warpgroups
constexpr int kUR = 4;                              // unit ring entries (dynamic schedule)
// readers of a unit id that release it: the peer's producer, the MMA issuer
// and every epilogue warp of both CTAs
constexpr int kUnitReaders = 1 + 1 + 2 * 4 * kEpiGroups;
constexpr int kThreads = 128 * (1 + kEpiGroups);    // + the control warpgroup
// setmaxnreg split of the registers the launch holds (640 threads x 96): the
// increases can only draw what the control warpgroup's decrease released,
// otherwise setmaxnreg.inc spins forever
constexpr int kLaunchRegs = 65536 / kThreads / 8 * 8;
#ifndef SAP_CTL_REGS
#define SAP_CTL_REGS 64
#endif
constexpr int kCtlRegs = SAP_CTL_REGS;  // warps 2-3 stream the next operand (zop::next_pass)
constexpr int kEpiRegs = 104;
static_assert(128 * kCtlRegs + 128 * kEpiGroups * kEpiRegs <= kThreads * kLaunchRegs,
              "setmaxnreg budget exceeds the launch allocation");

// H: the augmented features in fp16 (GEMM1 kind::f16, 64-byte swizzled rows)
// instead of fp32 (kind::tf32, 128-byte rows): the same 11-bit significands
// (the features are tf32-rounded splits, exact in fp16), twice the tensor
// rate and half the bytes per point
template <int NZ, int KA, bool H = false>
struct Geometry2 {
  static constexpr uint32_t elem = H ? 2 : 4;
  static constexpr uint32_t a_bytes = BM * KA * elem;          // this CTA's 128 block rows
  static constexpr uint32_t x_bytes = (NT / 2) * KA * elem;    // this CTA's 64 points
  static constexpr uint32_t z_atom = (NZ / 2) * 128;           // 64 points x nz/2 columns
  static constexpr uint32_t z_bytes = 2 * z_atom;              // 128 points
  static constexpr uint32_t stage_bytes = x_bytes + 2 * z_bytes;
  static constexpr uint32_t fixed = 1024 + 2 * a_bytes + 512;
  static constexpr uint32_t stages_raw = (kSmemCap - fixed) / stage_bytes;
  static constexpr uint32_t STAGES = stages_raw > 8 ? 8 : stages_raw;
  static constexpr uint32_t smem = fixed + STAGES * stage_bytes;
  static constexpr bool fits = STAGES >= 3 && NZ % 16 == 0 && NZ >= 16 && kGCol + NZ <= 512 &&
                              (!H || KA == 32 || KA == 64);
};

// K-major SWIZZLE_64B descriptor (fp16 features: 64-byte rows, 8-row atoms of
// 512 bytes), start address added to the low bits
constexpr uint64_t kDescBase64 = (uint64_t(1) << 16) | (uint64_t(512 >> 4) << 32) |
                                 (uint64_t(1) << 46) | (uint64_t(4) << 61);

template <int FAM, int NZ, int KA, bool H = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    krows_tc2_kernel(const __grid_constant__ CUtensorMap tm_rows,
                     const __grid_constant__ CUtensorMap tm_cols,
                     const __grid_constant__ CUtensorMap tm_zhi,
                     const __grid_constant__ CUtensorMap tm_zlo, const Params p) {
  using Geo = Geometry2<NZ, KA, H>;
  constexpr uint32_t STAGES = Geo::STAGES;
  // 128-byte fp32 atoms, or one fp16 atom: 64-byte rows (32 features) or
  // 128-byte rows (64 features)
  constexpr int KATOMS = H ? 1 : KA / 32;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t cr = tc::cluster_ctarank();   // 0 = leader (issues the MMAs)
  const unsigned long long kstart = prof_clock();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  uint8_t *sA = smem;                          // [2][a_bytes]
  uint8_t *sStage = smem + 2 * Geo::a_bytes;   // [STAGES][stage_bytes]
  uint64_t *bars = reinterpret_cast<uint64_t *>(sStage + STAGES * Geo::stage_bytes);
  uint64_t *full = bars;                  // [STAGES]  leader: TMA bytes of both CTAs
  uint64_t *empty = full + STAGES;        // [STAGES]  both: multicast commit
  uint64_t *a_full = empty + STAGES;      // [2]       leader
  uint64_t *a_empty = a_full + 2;         // [2]       both
  uint64_t *s_full = a_empty + 2;         // [NB]      both
  uint64_t *p_full = s_full + NB;         // [NB]      leader: 16 warp arrivals
  uint64_t *g_full = p_full + NB;         // [1]       both
  uint64_t *g_empty = g_full + 1;         // [1]       leader: 16 warp arrivals
  uint64_t *u_full = g_empty + 1;         // [kUR]     both: the leader producer's unit id
  uint64_t *u_empty = u_full + kUR;       // [kUR]     leader: every consumer read it
  int *u_ring = reinterpret_cast<int *>(u_empty + kUR);  // [kUR] unit ids (-1: done)
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(u_ring + kUR);

  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < STAGES; ++s) {
      tc::mbar_init(tc::smem_u32(&full[s]), 1);
      tc::mbar_init(tc::smem_u32(&empty[s]), 1);
    }
    for (int k = 0; k < NB; ++k) {
      tc::mbar_init(tc::smem_u32(&s_full[k]), 1);
      tc::mbar_init(tc::smem_u32(&p_full[k]), 8 * kEpiGroups);
    }
    for (int k = 0; k < 2; ++k) {
      tc::mbar_init(tc::smem_u32(&a_full[k]), 1);
      tc::mbar_init(tc::smem_u32(&a_empty[k]), 1);
    }
    tc::mbar_init(tc::smem_u32(g_full), 1);
    tc::mbar_init(tc::smem_u32(g_empty), 8 * kEpiGroups);
    for (int k = 0; k < kUR; ++k) {
      tc::mbar_init(tc::smem_u32(&u_full[k]), 1);
      tc::mbar_init(tc::smem_u32(&u_empty[k]), kUnitReaders);
    }
    tc::fence_barrier_init();
  }
  if (p.sched && blockIdx.x == 0 && threadIdx.x == 0)  // arm the next launch's counter slot
    p.sched[(p.epoch + 1u) & 1u] = static_cast<unsigned long long>(p.epoch + 1u) << 32;
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tm_rows);
    tc::prefetch_tmap(&tm_cols);
    tc::prefetch_tmap(&tm_zhi);
    tc::prefetch_tmap(&tm_zlo);
  }
  if (warp == 2) {
    tc::tmem_alloc_pair(tc::smem_u32(tmem_slot), 512);
    tc::tmem_relinquish_pair();
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();  // barriers of both CTAs initialised before any remote signal
  tc::fence_after();
  // launched with programmatic stream serialization: the set-up above (barrier
  // init, TMEM allocation, descriptor prefetch, arming the NEXT launch's
  // counter slot) may overlap the previous kernel's tail; everything below
  // reads or writes what earlier kernels produce or consume (features, the
  // operand, the partials), so it waits for them (a no-op when not launched
  // as a dependent)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int units = p.row_tiles * p.splits;  // row_tiles counts 256-row pair tiles here
  // Units (256-row tile x column split) are handed out dynamically: the
  // leader's producer takes the next one from a global counter and publishes
  // it to every role of both CTAs through a small shared-memory ring, so a
  // pair that starts late (SMs still held by a concurrent kernel on another
  // stream) simply takes fewer units instead of stretching the launch. The
  // partial sums are indexed by unit, so the result does not depend on which
  // pair ran what. p.sched == NULL: static round-robin units.
  const bool dyn = p.sched != nullptr;
  auto unit_at = [&](int k) -> int {  // static schedule
    const int u = pair + k * npairs;
    return u < units ? u : -1;
  };
  // consumer side of the ring: wait for entry k, read it, release it to the leader
  auto take_unit = [&](int k, bool arrive) -> int {
    if (!dyn) return unit_at(k);
    const int slot = k % kUR;
    tc::mbar_wait_acquire_cluster(tc::smem_u32(&u_full[slot]), (k / kUR) & 1);
    const int u = *reinterpret_cast<volatile int *>(&u_ring[slot]);
    if (arrive) tc::mbar_arrive_cluster(tc::mapa(tc::smem_u32(&u_empty[slot]), 0));
    return u;
  };

  if (warp < 4) tc::setmaxnreg_dec<kCtlRegs>();
  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if (tc::elect_one()) {
      uint32_t s = 0, ph = 0;
      int uc = 0;
      const uint32_t full0 = tc::smem_u32(full), empty0 = tc::smem_u32(empty);
      const uint32_t stage0 = tc::smem_u32(sStage);
      unsigned long long tw = 0, ti = 0, c0;
      for (int k = 0;; ++k, ++uc) {
        int u;
        if (dyn && cr == 0) {  // the leader's producer fetches and publishes
          const int slot = k % kUR;
          tc::mbar_wait(tc::smem_u32(&u_empty[slot]), ((k / kUR) & 1) ^ 1);
          // u = this launch's next unit from its counter slot, tagged with the
          // launch's epoch. The previous launch on this workspace armed the
          // slot ((epoch << 32) | 0), so one atomicAdd is the whole fetch; a
          // stale tag (first launch on a workspace) falls back to re-arming it
          // by compare-and-swap. (A compare-and-swap loop for every fetch made
          // 74 leaders retry against each other: ~10 us per unit at config 2.)
          unsigned long long *slot_ctr = p.sched + (p.epoch & 1u);
          unsigned long long old = atomicAdd(slot_ctr, 1ull), prev;
          if (unsigned(old >> 32) == p.epoch) {
            u = int(old & 0xffffffffull);
          } else {
            old = *reinterpret_cast<volatile unsigned long long *>(slot_ctr);
            do {
              prev = old;
              const bool mine = unsigned(old >> 32) == p.epoch;
              const unsigned long long nxt = (static_cast<unsigned long long>(p.epoch) << 32) |
                                             ((mine ? (old & 0xffffffffull) : 0ull) + 1ull);
              u = mine ? int(old & 0xffffffffull) : 0;
              old = atomicCAS(slot_ctr, prev, nxt);
            } while (old != prev);
          }
          if (u >= units) u = -1;
          u_ring[slot] = u;
          tc::st_cluster_u32(tc::mapa(tc::smem_u32(&u_ring[slot]), 1), uint32_t(u));
          tc::mbar_arrive_release_cluster(tc::mapa(tc::smem_u32(&u_full[slot]), 0));
          tc::mbar_arrive_release_cluster(tc::mapa(tc::smem_u32(&u_full[slot]), 1));
        } else {
          u = take_unit(k, true);
        }
        if (u < 0) break;
        const int rt = u % p.row_tiles, split = u / p.row_tiles;
        int64_t t0, t1;
        split_range(p.tiles, p.splits, split, t0, t1);
        const int ab = uc & 1;
        tc::mbar_wait(tc::smem_u32(&a_empty[ab]), ((uc >> 1) & 1) ^ 1);
        const uint32_t abar = tc::smem_u32(&a_full[ab]);
        if (cr == 0) tc::mbar_expect_tx(abar, 2 * Geo::a_bytes);
#pragma unroll
        for (int ka = 0; ka < KATOMS; ++ka)
          tc::tma_load_2d_pair(tc::smem_u32(sA + ab * Geo::a_bytes + ka * BM * 128), &tm_rows,
                               abar, ka * 32, rt * 2 * BM + int(cr) * BM);
        for (int64_t t = t0; t < t1; ++t) {
          c0 = prof_clock();
          tc::mbar_wait(empty0 + 8 * s, ph ^ 1);
          const unsigned long long c1 = prof_clock();
          tw += c1 - c0;
          const uint32_t fbar = full0 + 8 * s;
          if (cr == 0) tc::mbar_expect_tx(fbar, 2 * Geo::stage_bytes);
          const uint32_t st = stage0 + s * Geo::stage_bytes;
          const int32_t col0 = int32_t(t * NT);
#pragma unroll
          for (int ka = 0; ka < KATOMS; ++ka)
            tc::tma_load_2d_pair(st + ka * (NT / 2) * 128, &tm_cols, fbar, ka * 32,
                                 col0 + int(cr) * (NT / 2));
#pragma unroll
          for (int za = 0; za < 2; ++za) {
            tc::tma_load_2d_pair(st + Geo::x_bytes + za * Geo::z_atom, &tm_zhi, fbar,
                                 col0 + za * 64, int(cr) * (NZ / 2));
            tc::tma_load_2d_pair(st + Geo::x_bytes + Geo::z_bytes + za * Geo::z_atom, &tm_zlo,
                                 fbar, col0 + za * 64, int(cr) * (NZ / 2));
          }
          ti += prof_clock() - c1;
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
      if (p.prof) {
        p.prof[blockIdx.x * 16 + 0] = tw;
        p.prof[blockIdx.x * 16 + 1] = ti;
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA only) =====================
    if (cr == 0 && tc::elect_one()) {
      constexpr uint32_t id1 = tc::idesc(H ? 0 : 2, 2 * BM, NT);  // tf32 / f16, M=256, N=128
      constexpr uint32_t id2 = tc::idesc(0, 2 * BM, NZ);  // f16,  M=256, N=nz
      const uint32_t full0 = tc::smem_u32(full), empty0 = tc::smem_u32(empty);
      const uint32_t sfull0 = tc::smem_u32(s_full), pfull0 = tc::smem_u32(p_full);
      const uint64_t stage_desc0 = kDescBase | (tc::smem_u32(sStage) >> 4);
      constexpr uint64_t kFDesc = (H && KA == 32) ? kDescBase64 : kDescBase;
      const uint64_t f_desc0 = kFDesc | (tc::smem_u32(sStage) >> 4);
      const uint64_t a_desc0 = kFDesc | (tc::smem_u32(sA) >> 4);
      uint32_t s1 = 0, ph1 = 0, r1 = 0;    // GEMM1 cursor (one tile ahead)
      uint32_t s2 = 0, r2 = 0, ph2 = 0;    // GEMM2 cursor
      uint32_t sc = 0;
      int uc = 0;
      unsigned long long wf = 0, wp = 0, wg = 0, i1 = 0, i2 = 0, cc;
      for (int k = 0;; ++k, ++uc) {
        const int u = take_unit(k, true);
        if (u < 0) break;
        const int split = u / p.row_tiles;
        int64_t t0, t1;
        split_range(p.tiles, p.splits, split, t0, t1);
        const int nt = int(t1 - t0);
        const int ab = uc & 1;
        tc::mbar_wait(tc::smem_u32(&a_full[ab]), (uc >> 1) & 1);
        tc::fence_after();
        const uint64_t a_desc = a_desc0 + ((ab * Geo::a_bytes) >> 4);
        int g1 = 0;  // GEMM1s issued in this unit
        auto gemm1 = [&]() {
          cc = prof_clock();
          tc::mbar_wait(full0 + 8 * s1, ph1);
          tc::fence_after();
          const unsigned long long cw = prof_clock();
          wf += cw - cc;
          const uint64_t x_desc = f_desc0 + ((s1 * Geo::stage_bytes) >> 4);
          const uint32_t d = tmem + r1 * NT;
          if constexpr (H) {
#pragma unroll
            for (int k = 0; k < KA / 16; ++k)  // K = 16 halves (32 bytes) per MMA
              tc::mma_f16_ss_pair(d, a_desc + 2 * k, x_desc + 2 * k, id1, k > 0);
          } else {
#pragma unroll
            for (int k = 0; k < KA / 8; ++k) {
              const uint32_t ko = ((k >> 2) * (BM * 128) + (k & 3) * 32) >> 4;
              const uint32_t kx = ((k >> 2) * ((NT / 2) * 128) + (k & 3) * 32) >> 4;
              tc::mma_tf32_ss_pair(d, a_desc + ko, x_desc + kx, id1, k > 0);
            }
          }
          tc::commit_pair(sfull0 + 8 * r1);
          i1 += prof_clock() - cw;
          if (++s1 == STAGES) { s1 = 0; ph1 ^= 1; }
          if (++r1 == NB) r1 = 0;
          if (++g1 == nt) tc::commit_pair(tc::smem_u32(&a_empty[ab]));
        };
        const uint32_t g_tmem = tmem + kGCol;
        int seg_j = 0;
        for (int j = 0; j < nt; ++j) {
          // GEMM1 runs up to NB-1 tiles ahead: GEMM1(j+NB-1) overwrites the
          // S/P slot of tile j-1, whose GEMM2 was issued earlier (in-order
          // tensor pipe), so the epilogue converts while GEMM2 streams
          while (g1 < nt && g1 <= j + NB - 1) gemm1();
          const bool seg_first = seg_j == 0;
          const bool seg_last = seg_j == kSeg - 1 || j + 1 == nt;
          cc = prof_clock();
          if (seg_first) tc::mbar_wait_cluster(tc::smem_u32(g_empty), (sc & 1) ^ 1);
          const unsigned long long cg = prof_clock();
          wg += cg - cc;
          tc::mbar_wait_cluster(pfull0 + 8 * r2, ph2);
          tc::fence_after();
          const unsigned long long cp = prof_clock();
          wp += cp - cg;
          const uint64_t zhi = stage_desc0 + ((s2 * Geo::stage_bytes + Geo::x_bytes) >> 4);
          const uint64_t zlo = zhi + (Geo::z_bytes >> 4);
          const uint32_t pbase = tmem + r2 * NT;
          if (p.debug < 4) {
#pragma unroll
            for (int kk = 0; kk < NT / 16; ++kk) {  // 16 points per MMA K step
              const uint32_t bo = ((kk >> 2) * Geo::z_atom + (kk & 3) * 32) >> 4;
              const uint32_t ahi = pbase + (kk >> 1) * 32 + (kk & 1) * 8;
              const uint32_t acc0 = (!seg_first || kk > 0) ? 1u : 0u;
              tc::mma_f16_ts_pair(g_tmem, ahi, zhi + bo, id2, acc0);
              tc::mma_f16_ts_pair(g_tmem, ahi, zlo + bo, id2, 1u);
              tc::mma_f16_ts_pair(g_tmem, ahi + 16, zhi + bo, id2, 1u);
            }
          }
          tc::commit_pair(empty0 + 8 * s2);
          if (seg_last) {
            tc::commit_pair(tc::smem_u32(g_full));
            ++sc;
            seg_j = 0;
          } else {
            ++seg_j;
          }
          i2 += prof_clock() - cp;
          if (++s2 == STAGES) s2 = 0;
          if (++r2 == NB) { r2 = 0; ph2 ^= 1; }
        }
      }
      if (p.prof) {
        p.prof[blockIdx.x * 16 + 2] = wf;
        p.prof[blockIdx.x * 16 + 3] = wp;
        p.prof[blockIdx.x * 16 + 4] = wg;
        p.prof[blockIdx.x * 16 + 5] = i1;
        p.prof[blockIdx.x * 16 + 6] = i2;
      }
    }
  } else if (warp < 4) {
    // ============ next iterate's operand (warps 2-3, otherwise idle) ============
    // Z_{t+1} = zp P + zq Q into the second operand buffer while this kernel
    // consumes Z_t: ~5 MB per CTA streamed over the kernel's lifetime (HBM is
    // <10% busy here), instead of a separate HBM-bound pass on the critical
    // path between two block-row products. The block rows are patched by
    // the Phase IV kernel after the update (phase4.cu).
    if (p.zn.Zhi) zop::next_pass(p.zn, blockIdx.x, gridDim.x, (warp - 2) * 32 + lane, 64);
    if (p.prof && warp == 2 && lane == 0) p.prof[blockIdx.x * 16 + 14] = prof_clock() - kstart;
  } else {
    // ===================== epilogue (both CTAs) =====================
    // Four warpgroups, i.e. four warps per SM sub-partition, so TMEM load/store
    // and dependency latencies hide behind the other warps' MUFU/FMA work:
    // warpgroup w converts S columns [32w, 32w+32) of every tile and drains the
    // accumulator's 8-column granules w, w+4, w+8, ... at every segment end.
    tc::setmaxnreg_inc<kEpiRegs>();
    const int q = warp & 3;
    const int w = (warp - 4) >> 2;
    const int row_in_tile = q * 32 + lane;
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    constexpr int NGRAN = NZ / 8;                           // 8-column accumulator granules
    constexpr int NMINE = (NGRAN + kEpiGroups - 1) / kEpiGroups;
    const int ngran = (NGRAN - w + kEpiGroups - 1) / kEpiGroups;  // granules of this warpgroup
    const uint32_t sfull0 = tc::smem_u32(s_full);
    const uint32_t pfull_leader = tc::mapa(tc::smem_u32(p_full), 0);
    const uint32_t gempty_leader = tc::mapa(tc::smem_u32(g_empty), 0);
    uint32_t r = 0, ph = 0, sc = 0;
    float acc[NMINE * 8];
#pragma unroll
    for (int c = 0; c < NMINE * 8; ++c) acc[c] = 0.0f;
    bool pend = false, pend_last = false, pend_live = false;
    float *pend_dst = nullptr;
    unsigned long long es = 0, ec = 0, ed = 0, ea = 0, ce, efirst = 0, eu = 0;
    auto drain = [&]() {  // add a finished TMEM segment, one tile late
      epi_wait(tc::smem_u32(g_full), sc & 1);
      tc::fence_after();
      const uint32_t gbase = tmem + lane_off + kGCol;
#pragma unroll
      for (int k = 0; k < NMINE; ++k) {
        if (k < ngran) {
          uint32_t v[8];
          tc::ld8(gbase + (w + k * kEpiGroups) * 8, v);
          tc::wait_ld();
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[k * 8 + e] += __uint_as_float(v[e]);
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(gempty_leader);
      ++sc;
      pend = false;
      if (pend_last) {
        if (pend_live) {
#pragma unroll
          for (int k = 0; k < NMINE; ++k)
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int c = (w + k * kEpiGroups) * 8 + e;
              if (k < ngran && c < p.m) pend_dst[int64_t(c) * p.b] = acc[k * 8 + e];
            }
        }
#pragma unroll
        for (int c = 0; c < NMINE * 8; ++c) acc[c] = 0.0f;
      }
    };
    // Matern: warpgroups 0-1 start ~0.4 tile later than 2-3, so the two
    // halves of every sub-partition's epilogue warps run out of phase: one
    // half's per-tile serial part (TMEM load/store waits, barrier arrive)
    // overlaps the other half's MUFU work instead of all four idling the
    // MUFU pipe together (config 3: -1.6%; RBF, whose epilogue is not
    // MUFU-bound, +0.4%, so 0 there; SAP_EPI_STAGGER overrides)
    constexpr long long kStagger =
        SAP_EPI_STAGGER >= 0 ? SAP_EPI_STAGGER
                             : ((FAM == SAP_MATERN32 || FAM == SAP_MATERN52) ? 1200 : 0);
    if (kStagger > 0 && w < 2) {
      const long long t0 = clock64();
      while (clock64() - t0 < kStagger) {
      }
    }
    for (int k = 0;; ++k) {
      const unsigned long long cu = prof_clock();
      const int u = take_unit(k, false);
      eu += prof_clock() - cu;
      if (dyn) {  // one arrival per warp
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster(tc::mapa(tc::smem_u32(&u_empty[k % kUR]), 0));
      }
      if (u < 0) break;
      const int rt = u % p.row_tiles, split = u / p.row_tiles;
      int64_t t0, t1;
      split_range(p.tiles, p.splits, split, t0, t1);
      const int64_t grow = int64_t(rt) * 2 * BM + int64_t(cr) * BM + row_in_tile;
      const bool live = grow < p.b;
      float *dst = p.part + int64_t(split) * p.m * p.b + (live ? grow : 0);
      const int64_t rid = (p.row_ids && live) ? p.row_ids[grow] : INT64_MIN;
      if (t1 == t0 && live) {
        for (int k = 0; k < ngran; ++k)
          for (int e = 0; e < 8; ++e) {
            const int c = (w + k * kEpiGroups) * 8 + e;
            if (c < p.m) dst[int64_t(c) * p.b] = 0.0f;
          }
      }
      int seg_j = 0;
      for (int64_t t = t0; t < t1; ++t) {
        ce = prof_clock();
        epi_wait(sfull0 + 8 * r, ph);
        tc::fence_after();
        const unsigned long long cs = prof_clock();
        es += cs - ce;
        if (!efirst) efirst = cs - kstart;
        const uint32_t taddr = tmem + lane_off + r * NT + w * 32;
        uint32_t v[32];
        tc::ld32(taddr, v);
        const int64_t dc64 = rid - (p.col_base + t * NT) - w * 32;
        const bool diag = dc64 >= 0 && dc64 < 32;
        const int dc = int(dc64);
        tc::wait_ld();
        uint32_t o[32];  // P_hi (16 packed words) then P_lo over the 32 columns
        if (p.debug == 1 || p.debug == 3 || p.debug == 4) {
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = v[e];
        } else if (__any_sync(0xffffffffu, diag)) {
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            float p0 = pvalue<FAM>(__uint_as_float(v[e]));
            float p1 = pvalue<FAM>(__uint_as_float(v[e + 1]));
            if (diag && dc == e) p0 = kPScale;
            if (diag && dc == e + 1) p1 = kPScale;
            split2(p0, p1, o[e / 2], o[16 + e / 2]);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const float x0 = __uint_as_float(v[e]), x1 = __uint_as_float(v[e + 1]);
            split2(poly_entry<FAM>(e) ? pvalue<FAM, true>(x0) : pvalue<FAM>(x0),
                   poly_entry<FAM>(e + 1) ? pvalue<FAM, true>(x1) : pvalue<FAM>(x1),
                   o[e / 2], o[16 + e / 2]);
          }
        }
        tc::st32(taddr, o);
        tc::wait_st();
        tc::fence_before();
        __syncwarp();
        const unsigned long long cw2 = prof_clock();
        ec += cw2 - cs;
        if (lane == 0) tc::mbar_arrive_cluster(pfull_leader + 8 * r);
        if (++r == NB) { r = 0; ph ^= 1; }
        const unsigned long long ca = prof_clock();
        ea += ca - cw2;
        if (pend) drain();
        ed += prof_clock() - ca;
        if (seg_j == kSeg - 1 || t + 1 == t1) {
          pend = true;
          pend_last = t + 1 == t1;
          pend_live = live;
          pend_dst = dst;
          seg_j = 0;
        } else {
          ++seg_j;
        }
      }
    }
    if (pend) drain();
    if (p.prof && warp == 4 && lane == 0) {
      p.prof[blockIdx.x * 16 + 12] = efirst;
      p.prof[blockIdx.x * 16 + 13] = prof_clock() - kstart;
      p.prof[blockIdx.x * 16 + 15] = eu;
      p.prof[blockIdx.x * 16 + 7] = es;
      p.prof[blockIdx.x * 16 + 8] = ec;
      p.prof[blockIdx.x * 16 + 9] = ea;
      p.prof[blockIdx.x * 16 + 10] = ed;
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();  // the peer's TMEM/barriers stay live until both CTAs are done
  tc::fence_after();

  if (p.prof && threadIdx.x == 0) p.prof[blockIdx.x * 16 + 11] = prof_clock() - kstart;
  if (warp == 2) tc::tmem_dealloc_pair(tmem, 512);
}

template <int FAM, int NZ, int KA, bool H>
bool launch_tc2_shape(const CUtensorMap &a, const CUtensorMap &c, const CUtensorMap &zh,
                      const CUtensorMap &zl, const Params &p, int grid, cudaStream_t st) {
  if constexpr (!Geometry2<NZ, KA, H>::fits) {
    return false;
  } else {
    constexpr uint32_t smem = Geometry2<NZ, KA, H>::smem;
    cudaFuncSetAttribute(krows_tc2_kernel<FAM, NZ, KA, H>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    // programmatic dependent launch (SAP_TC_PDL=0: plain stream order): the
    // grid is scheduled while the previous kernel (Phase IV's last stage)
    // drains, hiding the launch gap
    static const bool pdl = !(getenv("SAP_TC_PDL") && atoi(getenv("SAP_TC_PDL")) == 0);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, krows_tc2_kernel<FAM, NZ, KA, H>, a, c, zh, zl, p);
    return true;
  }
}

// ka: 32 / 64 fp32 features, or kKaF16 (32 fp16 features, include/sapgp_b200.h)
constexpr int kKaF16 = SAP_TC_KA_F16;
constexpr int kKaF16x64 = SAP_TC_KA_F16X64;
template <int FAM>
bool launch_tc2_family(const CUtensorMap &a, const CUtensorMap &c, const CUtensorMap &zh,
                       const CUtensorMap &zl, const Params &p, int nz, int ka, int grid,
                       cudaStream_t st) {
#define SAP_TC2_KA(NZV)                                                                   \
  return ka == 32     ? launch_tc2_shape<FAM, NZV, 32, false>(a, c, zh, zl, p, grid, st)  \
         : ka == 64   ? launch_tc2_shape<FAM, NZV, 64, false>(a, c, zh, zl, p, grid, st)  \
         : ka == kKaF16 ? launch_tc2_shape<FAM, NZV, 32, true>(a, c, zh, zl, p, grid, st) \
         : ka == kKaF16x64 ? launch_tc2_shape<FAM, NZV, 64, true>(a, c, zh, zl, p, grid, st) \
                        : false;
  switch (nz) {
    case 16: SAP_TC2_KA(16)
    case 32: SAP_TC2_KA(32)
    case 48: SAP_TC2_KA(48)
    case 64: SAP_TC2_KA(64)
    case 80: SAP_TC2_KA(80)
    case 96: SAP_TC2_KA(96)
    case 112: SAP_TC2_KA(112)
    case 128: SAP_TC2_KA(128)
    default: return false;
  }
#undef SAP_TC2_KA
}

inline bool tc2_fits(int nz, int ka) {
  const bool h = ka == kKaF16 || ka == kKaF16x64;
  if (h) ka = ka == kKaF16 ? 32 : 64;
  if (nz % 16 || nz < 16 || kGCol + nz > 512 || (ka != 32 && ka != 64)) return false;
  const uint32_t elem = h ? 2 : 4;
  const uint32_t stage = (NT / 2) * ka * elem + 2 * 2 * (nz / 2) * 128;
  const uint32_t fixed = 1024 + 2 * BM * ka * elem + 512;
  return (kSmemCap - fixed) / stage >= 3;
}

}  // namespace tck2
}  // namespace sap
