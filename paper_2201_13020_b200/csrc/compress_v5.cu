// compress_v5.cu -- SZx block encoder for sm_100a, bs == 128 (K1, variant 5: two teams).
//
// Replaces the reference's whole compress path in ONE launch per chunk:
//   block_stats           pipeline.py:54-81   (== blockcodec.summarize_block 87-112)
//   _encode_elements      pipeline.py:94-133  (== blockcodec.encode_nonconstant 123-141)
//   prefix_scan + scatter parallel.py:21-44,104-140 / pipeline.py:143-166
// Output pools use the UFZX container layout (container.py:3-21).
//
// The variant-1 pipeline (compress.cu: TMA input boxes, tagged per-group count words, one
// contiguous elastic staging ring, decoupled look-back, realigned write-out) with the 16
// compute warps split into TWO TEAMS of 8 that take alternate tiles of 32 blocks.  In
// variant 1 all 16 compute warps run each tile in lockstep, so the SM alternates between an
// issue-bound encode phase and a shared-memory-bound staging phase; here the
// ring-offset chain (tile k needs tile k-1's size) staggers the teams by half a tile, so one
// team encodes while the other stages.  Tiles are half as large, so two look-back warps
// (shared floor) keep the look-back rate, and one write-out warp serves both teams.
#include <cuda.h>

#include "k1_common.cuh"

namespace szx {

namespace {
using namespace k1;

#ifndef SZX_V5_SCAN
#define SZX_V5_SCAN 2
#endif
#ifndef SZX_V5_WRITERS
#define SZX_V5_WRITERS 1
#endif
#ifndef SZX_V5_IN
#define SZX_V5_IN 6
#endif
#ifndef SZX_V5_REC
#define SZX_V5_REC 12
#endif
#ifndef SZX_V5_RING_KB
#define SZX_V5_RING_KB 64
#endif
#ifndef SZX_V5_SPIN_NS
#define SZX_V5_SPIN_NS 300
#endif
constexpr int kTeams = SZX_V5_TEAMS;
constexpr int kTW = kCompWarps / kTeams;          // compute warps (groups) per tile
constexpr int kTB = kV5TileBlocks;                // blocks per tile (4 per group)
static_assert(kTB == 4 * kTW, "tile = 4 blocks per group");
constexpr int kTV = kTB * 128;                    // values per tile
constexpr int kTR = kTV / 32;                     // 128-byte rows per tile (TMA box)
constexpr int kScan = SZX_V5_SCAN;
constexpr int kScanPer5 = kScan > 1 ? 16 : 8;  // look-back window: 32 * kScanPer5 tiles
constexpr int kWrite = SZX_V5_WRITERS;
constexpr int kIn5 = SZX_V5_IN;
constexpr int kRec5 = SZX_V5_REC;
constexpr uint32_t kRing5 = SZX_V5_RING_KB * 1024;
constexpr int kScanW0 = 0, kWriteW0 = kScan, kCompW0 = kScan + kWrite;
constexpr int kProd5 = kCompW0 + kCompWarps;
constexpr int kThreads5 = (kProd5 + 1) * 32;
constexpr int kStop5 = kScan > kWrite ? kScan : kWrite;
static_assert(kTB % 8 == 0 && kTR <= 256, "whole map bytes per tile, one TMA box");
static_assert(kStop5 <= kRec5 && kTeams <= kIn5, "stop signals must fit the rings");
static_assert(kRing5 % 16 == 0 && kRing5 >= 8 * kTV, "ring must hold two worst-case tiles");
static_assert(kTeams == 1 || kTeams == 2, "one or two teams");

struct __align__(1024) Box5 {
  float v[kTV];
};
struct __align__(16) Rec5 {
  uint32_t codes[kTB][8];           // NC-rank-ordered 32-byte code rows
  uint8_t req[kTB];
  uint32_t tile;                    // producer -> look-back / write-out (~0u: stop)
  uint32_t mid_total, nc_total;     // compute -> look-back: tile totals
  uint32_t map_lo, map_hi;          // compute -> look-back: constant-block bits
  uint32_t vphys;                   // compute -> write-out: ring offset % kRing5
  uint32_t done;                    // write-out -> compute: local tile index + 1
  unsigned long long pre_nc, pre_mid;  // look-back -> write-out: exclusive prefixes
  unsigned long long lb_incl;       // look-back -> look-back: inclusive prefix of lb_tile,
  uint32_t lb_tile, lb_tag;         //   valid when lb_tag == local index + 1
};
struct Smem5 {
  Box5 in[kIn5];
  uint8_t ring[kRing5 + 64];
  Rec5 rec[kRec5];
  uint64_t full[kIn5];
  uint64_t in_free[kIn5];           // the tile's team (kTW warps) -> producer
  uint32_t tile[kIn5];
  uint64_t claimed[kRec5];
  uint64_t counted[kRec5];
  uint64_t prefix[kRec5];
  uint64_t staged[kRec5];           // the tile's team (kTW warps, after staging) -> write-out
  uint64_t written[kRec5];
  uint32_t xw[4][kTW];              // per-group counts of tile k in xw[k & 3] (tagged)
  // tile k's ring placement for the next tile (in slot k & 15): virtual offset, physical
  // offset, mid bytes | tag (k + 1) << 16 (release-stored last)
  uint32_t tvpos[16], tvphys[16], ttot[16];
};

__device__ __forceinline__ void write_out5(const CompressArgs& a, const Rec5& S, const uint8_t* ring,
                                           int lane) {
  const uint32_t nnc = S.nc_total;
  const uint64_t pre_nc = S.pre_nc;
  for (int r = lane; r < (int)nnc; r += 32) a.req[pre_nc + r] = S.req[r];
  for (int i = lane; i < (int)(2 * nnc); i += 32) {
    const int r = i >> 1, h = i & 1;
    const uint4 v = *reinterpret_cast<const uint4*>(&S.codes[r][4 * h]);
    uint8_t* dst = a.codes + 32 * (pre_nc + r) + 16 * h;
    if (((uintptr_t)a.codes & 15) == 0) {
      *reinterpret_cast<uint4*>(dst) = v;
    } else {
      uint32_t* d4 = reinterpret_cast<uint32_t*>(dst);
      d4[0] = v.x; d4[1] = v.y; d4[2] = v.z; d4[3] = v.w;
    }
  }
  copy_out(a.mid, S.pre_mid, ring + S.vphys, S.mid_total, lane, 32);
}

}  // namespace

__global__ void __launch_bounds__(kThreads5, 1)
    compress128v5_kernel(CompressArgs a, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem5& sm = *reinterpret_cast<Smem5*>(smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t n = a.n;
  const uint64_t nb = (n + 127) >> 7;

  if (tid == 0) {
    for (int s = 0; s < kIn5; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.in_free[s], kTW);
    }
    for (int r = 0; r < kRec5; ++r) {
      sm.rec[r].done = 0;
      sm.rec[r].lb_tag = 0;
      mbar_init(&sm.claimed[r], 1);
      mbar_init(&sm.counted[r], 1);
      mbar_init(&sm.prefix[r], 1);
      mbar_init(&sm.staged[r], kTW);
      mbar_init(&sm.written[r], 1);
    }
    for (int i = 0; i < 4 * kTW; ++i) (&sm.xw[0][0])[i] = 0;
    for (int i = 0; i < 16; ++i) sm.ttot[i] = 0;
    fence_barrier_init();
  }
  __syncthreads();

  // ---------------------------------------------------------------- producer warp
  if (warp == kProd5) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      uint32_t next = atomicAdd(a.counter, 1u);
      for (uint32_t k = 0;; ++k) {
        const int s = k % kIn5;
        mbar_wait_sleep(&sm.in_free[s], ((k / kIn5) & 1) ^ 1);
        const uint32_t tile = next;
        if (tile < a.ntiles) next = atomicAdd(a.counter, 1u);
        if (tile >= a.ntiles) {
          // stop each team at its next tile index and every look-back / write-out warp at
          // its next record index, each after the box / record it reuses is released
          for (uint32_t j = k; j < k + kTeams; ++j) {
            const int sj = j % kIn5;
            if (j > k) mbar_wait_sleep(&sm.in_free[sj], ((j / kIn5) & 1) ^ 1);
            sm.tile[sj] = ~0u;
            mbar_arrive(&sm.full[sj]);
          }
          for (uint32_t j = k; j < k + kStop5; ++j) {
            const int rj = j % kRec5;
            mbar_wait_sleep(&sm.written[rj], ((j / kRec5) & 1) ^ 1);
            sm.rec[rj].tile = ~0u;
            if (j < k + kScan) mbar_arrive(&sm.claimed[rj]);
            if (j < k + kWrite) mbar_arrive(&sm.prefix[rj]);
          }
          break;
        }
        sm.tile[s] = tile;
        mbar_wait_sleep(&sm.written[k % kRec5], ((k / kRec5) & 1) ^ 1);
        sm.rec[k % kRec5].tile = tile;
        mbar_arrive(&sm.claimed[k % kRec5]);
        if (((uint64_t)tile + 1) * kTV <= n) {
          mbar_arrive_expect_tx(&sm.full[s], kTV * 4);
          tma_load_2d(sm.in[s].v, &tmap, 0, (int)(tile * kTR), &sm.full[s]);
        } else {
          mbar_arrive(&sm.full[s]);
        }
      }
    }
    return;
  }

  // ---------------------------------------------------------------- look-back warps
  if (warp >= kScanW0 && warp < kScanW0 + kScan) {
    int64_t floor = -1;
    uint64_t floor_incl = 0;
    for (uint32_t k = warp - kScanW0;; k += kScan) {
      const int rk = k % kRec5;
      Rec5& S = sm.rec[rk];
      mbar_wait_sleep(&sm.claimed[rk], (k / kRec5) & 1);
      const uint32_t tile = S.tile;
      if (tile == ~0u) break;
      if (kScan > 1 && k >= 1) {  // the CTA's previous tile, if already resolved, is a closer floor
        const Rec5& P = sm.rec[(k - 1) % kRec5];
        if (ld_acquire_cta(&P.lb_tag) == k && (int64_t)P.lb_tile > floor) {
          floor = P.lb_tile;
          floor_incl = P.lb_incl;
        }
      }
      const uint64_t ex =
          tile == 0 ? 0 : lookback_excl<kScanPer5>(a.status, tile, 128, floor, floor_incl);
      mbar_wait_sleep(&sm.counted[rk], (k / kRec5) & 1);
      const uint64_t agg = pack2(S.nc_total, S.mid_total);
      if (lane == 0) {
        st_relaxed(a.status + tile, kFlagPre | (ex + agg));
        if (kScan > 1) {
          S.lb_tile = tile;
          S.lb_incl = ex + agg;
          st_release_cta(&S.lb_tag, k + 1);
        }
      }
      floor = tile;
      floor_incl = ex + agg;
      const uint64_t bnc = a.base ? a.base->n_nc : 0, bm = a.base ? a.base->m : 0;
      const uint64_t bmid = a.base ? a.base->mid_len : 0;
      if (lane == 0) {
        S.pre_nc = bnc + hi_of(ex);
        S.pre_mid = bmid + lo_of(ex);
        const uint64_t tb = (uint64_t)tile * kTB;
        const uint64_t bits = ((uint64_t)S.map_hi << 32) | S.map_lo;
        if (tile == a.ntiles - 1) {
          const uint64_t run = ex + agg;
          const uint64_t cnc = hi_of(run);
          a.totals->n_nc = bnc + cnc;
          const uint64_t lastb = nb - 1, nvb = n - 128 * lastb;
          const uint32_t lb = (uint32_t)(lastb - tb);
          const uint32_t madj = (nvb < 128 && !((bits >> lb) & 1)) ? 128 - (uint32_t)nvb : 0u;
          a.totals->m = bm + 128 * cnc - madj;
          a.totals->mid_len = bmid + lo_of(run);
          a.totals->pad = 0;
        }
        // constant map: kTB bits per tile, LSB-first (container.py:12-13,321)
        uint8_t* mp = a.map + (kTB / 8) * (uint64_t)tile;
        if (tb + kTB <= nb) {
          reinterpret_cast<uint32_t*>(mp)[0] = S.map_lo;
          if (kTB == 64) reinterpret_cast<uint32_t*>(mp)[1] = S.map_hi;
        } else {
          const uint32_t nbytes = (uint32_t)((nb - tb + 7) >> 3);
          for (uint32_t i = 0; i < nbytes; ++i) mp[i] = (uint8_t)(bits >> (8 * i));
        }
        mbar_arrive(&sm.prefix[rk]);
      }
      __syncwarp();
    }
    return;
  }

  // ---------------------------------------------------------------- write-out warps
  if (warp >= kWriteW0 && warp < kWriteW0 + kWrite) {
    for (uint32_t k = warp - kWriteW0;; k += kWrite) {
      const int r = k % kRec5;
      const Rec5& S = sm.rec[r];
      mbar_wait_sleep(&sm.prefix[r], (k / kRec5) & 1);
      if (S.tile == ~0u) break;
      mbar_wait(&sm.staged[r], (k / kRec5) & 1);
      write_out5(a, S, sm.ring, lane);
      __syncwarp();
      if (lane == 0) {
        st_release_cta(&sm.rec[r].done, k + 1);
        mbar_arrive(&sm.written[r]);
      }
    }
    return;
  }

  // ---------------------------------------------------------------- compute warps
  const int cw = warp - kCompW0;      // 0..15
  const int team = cw / kTW;          // tiles k with k % kTeams == team
  const int gw = cw % kTW;
  const int grp = kTW - 1 - gw;       // the team's highest-priority warp owns the first blocks
  const int jb = lane >> 3;
  const int g = lane & 7;
  uint32_t tail = 0;                  // oldest tile (any team) not known written out
  auto release = [&]() {
    if (ld_acquire_cta(&sm.rec[tail % kRec5].done) != tail + 1)
      mbar_wait(&sm.written[tail % kRec5], (tail / kRec5) & 1);
    ++tail;
  };
  auto wait_counts = [&](uint32_t kk, int upto) {
    const uint32_t tag = (kk + 1) & 0x1FFFu;
    uint32_t e, it = 0;
    while (true) {
      e = lane < upto ? ld_volatile_cta(&sm.xw[kk & 3][lane]) : tag << 19;
      if (__all_sync(kFull, (e >> 19) == tag)) break;
      __nanosleep(SZX_V5_SPIN_NS);
      if (++it > (1u << 24)) __trap();
    }
    return lane < upto ? e & 0x7FFFFu : 0u;
  };
  for (uint32_t k = team;; k += kTeams) {
    const int ik = k % kIn5, rk = k % kRec5;
    Rec5& R = sm.rec[rk];
    mbar_wait(&sm.full[ik], (k / kIn5) & 1);
    const uint32_t tile = sm.tile[ik];
    if (tile == ~0u) break;
    const uint64_t v0 = (uint64_t)tile * kTV;
    const bool full = v0 + kTV <= n;
    Cls c;
    Lane16 s;
    bool exists = true;
    if (full) encode_full(sm.in[ik].v, grp, lane, a, c, s);
    else encode_tail(grp, lane, a, v0, c, s, exists);
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.in_free[ik]);

    const uint64_t b0 = (uint64_t)tile * kTB + (uint64_t)grp * kFastBPW;
    if (g == 0 && exists) a.mu[b0 + jb] = c.mu;  // container.py:14
    const uint32_t ncb = __ballot_sync(kFull, c.nc) & 0x01010101u;
    const uint32_t csb = __ballot_sync(kFull, !c.nc && exists) & 0x01010101u;
    uint32_t incl = s.L;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += t;
    }
    const uint32_t wmid = __shfl_sync(kFull, incl, 31);
    if (lane == 0)
      st_volatile_cta(&sm.xw[k & 3][grp],
                      wmid | ((uint32_t)__popc(ncb) << 12) |
                          (((csb & 1) | ((csb >> 7) & 2) | ((csb >> 14) & 4) | ((csb >> 21) & 8)) << 15) |
                          (((k + 1) & 0x1FFFu) << 19));
    // this tile's ring offset: after tile k - 1 (the other team's), whose last group published
    // its placement and size; moved to the next lap when a worst-case tile would not fit
    uint32_t vpos = 0, vphys = 0;
    if (k > 0) {
      const uint32_t slot = (k - 1) & 15, tag = k & 0xFFFFu;
      uint32_t w, it = 0;
      while (((w = ld_acquire_cta(&sm.ttot[slot])) >> 16) != tag) {
        __nanosleep(SZX_V5_SPIN_NS);
        if (++it > (1u << 24)) __trap();
      }
      const uint32_t adv = ((w & 0xFFFFu) + 15) & ~15u;
      vpos = sm.tvpos[slot] + adv;
      vphys = sm.tvphys[slot] + adv;
      if (vphys >= kRing5) vphys -= kRing5;
      if (vphys > kRing5 - 4 * kTV) {
        vpos += kRing5 - vphys;
        vphys = 0;
      }
    }
    // records of tiles kRec5 back must be written out (the code rows of this tile go there)
    while (tail + kRec5 <= k) release();
    const int upto = grp == kTW - 1 ? kTW : grp;
    const uint32_t cnt = wait_counts(k, upto);
    const uint32_t pk = (cnt & 0xFFFu) | (((cnt >> 12) & 7u) << 16);
    const bool last_grp = grp == kTW - 1;
    const uint32_t sum_pk = __reduce_add_sync(kFull, last_grp || lane < grp ? pk : 0u);
    const uint32_t own_pk = wmid | ((uint32_t)__popc(ncb) << 16);
    const uint32_t pre_pk = last_grp ? sum_pk - own_pk : sum_pk;
    const uint32_t pre_mid = pre_pk & 0xFFFFu, pre_nc = pre_pk >> 16;
    if (last_grp && lane == 0) {  // the next tile's placement
      const uint32_t slot = k & 15;
      sm.tvpos[slot] = vpos;
      sm.tvphys[slot] = vphys;
      st_release_cta(&sm.ttot[slot], (sum_pk & 0xFFFFu) | (((k + 1) & 0xFFFFu) << 16));
    }
    // the tiles (in order, any team) whose ring bytes this group's region overlaps must be
    // written out; a pending tile t < k published its placement before tile k was placed
    const uint32_t my_end = vpos + pre_mid + wmid;
    while (tail < k && (int32_t)(my_end - sm.tvpos[tail & 15]) > (int32_t)kRing5) release();
    if (last_grp) {
      const uint32_t tmid = sum_pk & 0xFFFFu, tnc = sum_pk >> 16;
      const uint32_t cs = lane < kTW ? ((cnt >> 15) & 15u) << (kFastBPW * (lane & 7)) : 0u;
      const uint32_t lo = __reduce_or_sync(kFull, lane < 8 ? cs : 0u);
      const uint32_t hi = __reduce_or_sync(kFull, lane >= 8 ? cs : 0u);
      if (lane == 0) {
        if (tile != 0) st_relaxed(a.status + tile, kFlagAgg | pack2(tnc, tmid));
        R.mid_total = tmid;
        R.nc_total = tnc;
        R.map_lo = lo;
        R.map_hi = hi;
        R.vphys = vphys;
        mbar_arrive(&sm.counted[rk]);
      }
    }
    if (c.nc) {
      const uint32_t rank = pre_nc + __popc(ncb & ((1u << (8 * jb)) - 1));
      R.codes[rank][g] = s.cb;
      if (g == 0) {
        R.req[rank] = (uint8_t)c.req;
        if (c.req < 1) atomicOr(a.err, kErrBadReq);  // container.py:206-207
      }
    }
    const uint32_t qm = __reduce_max_sync(kFull, c.nc ? (uint32_t)c.q : 0u);
    const uint32_t base = smem_u32(sm.ring) + vphys + pre_mid + incl - s.L;
    switch (qm) {
      case 0: break;
      case 1: stage_lane<1>(s, base); break;
      case 2: stage_lane<2>(s, base); break;
      case 3: stage_lane<3>(s, base); break;
      default: stage_lane<4>(s, base); break;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.staged[rk]);
  }
}

cudaError_t launch_compress128v5(const CompressArgs& a, cudaStream_t s) {
  static bool configured = false;
  const size_t smem = sizeof(Smem5) + 1024;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(compress128v5_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  alignas(64) CUtensorMap map;
  const cudaError_t me = make_tile_tmap(a.x, a.n, &map, kTR);
  if (me != cudaSuccess) return me;
  const uint32_t cap = (uint32_t)sm_count();
  const uint32_t grid = a.ntiles < cap ? a.ntiles : cap;
  compress128v5_kernel<<<grid, kThreads5, smem, s>>>(a, map);
  return cudaGetLastError();
}

}  // namespace szx
