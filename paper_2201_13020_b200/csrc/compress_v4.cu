// compress_v4.cu -- SZx block encoder for sm_100a, bs == 128 (K1, variant 4: two-phase tiles).
//
// Replaces the reference's whole compress path in ONE launch per chunk:
//   block_stats           pipeline.py:54-81   (== blockcodec.summarize_block 87-112)
//   _encode_elements      pipeline.py:94-133  (== blockcodec.encode_nonconstant 123-141)
//   prefix_scan + scatter parallel.py:21-44,104-140 / pipeline.py:143-166
// Output pools use the UFZX container layout (container.py:3-21).
//
// Persistent, one CTA per SM: a producer warp, kLB4 look-back warps and 16 compute warps.
// A tile is 64 blocks (32 KiB) and stays in its shared-memory input box from the TMA load
// until it is written out, which lets every compute warp run each tile in two phases that
// never wait for another warp's progress on the SAME tile:
//   A(k)      classify + count the warp's 4-block group of tile k (mid bytes, NC blocks,
//             constant bits), publish the counts (one shared word + an mbarrier arrival;
//             the last warp to add its counts to the tile's shared accumulator publishes the
//             tile aggregate for the decoupled look-back at once);
//   B(k - D)  D tiles later: the tile's stream offsets are known by then (the look-back
//             warps turned its aggregate into an inclusive prefix and the group counts into
//             group offsets meanwhile), so the warp re-encodes its group from the resident
//             box, stages the mid bytes in a private buffer AT THE FINAL 16-BYTE PHASE and
//             writes them out with aligned 16-byte stores (bytes only at the two edges),
//             together with its code rows and req bytes, then releases the box.
// The compute warps' only waits are mbarrier phases (input full, tile prefix) that are
// normally complete already: no count polls, no shared staging ring, no write-out warps.
#include <cuda.h>

#include "k1_common.cuh"

namespace szx {

namespace {
using namespace k1;

#ifndef SZX_V4_BOXES
#define SZX_V4_BOXES 5
#endif
#ifndef SZX_V4_DEFER
#define SZX_V4_DEFER 2
#endif
#ifndef SZX_V4_LB
#define SZX_V4_LB 2
#endif
#ifndef SZX_V4_STATIC
#define SZX_V4_STATIC 1  // 1: CTA c encodes tiles c, c + G, ... (no claim counter)
#endif
#ifndef SZX_V4_AHEAD
#define SZX_V4_AHEAD 0   // 1: the producer claims one tile ahead of the free box
#endif
constexpr int kNB4 = SZX_V4_BOXES;   // input boxes = tile records: tile k in box k % kNB4
constexpr int kD4 = SZX_V4_DEFER;    // B(k) runs after A(k + kD4)
constexpr int kLB4 = SZX_V4_LB;      // look-back warps (tiles round robin)
static_assert(kD4 >= 1 && kNB4 >= kD4 + 2, "boxes: kD4 + 1 resident tiles and >= 1 prefetch");
static_assert(kLB4 >= 1 && kLB4 <= kNB4, "look-back warps");

constexpr int kW4 = kCompWarps;                // 16 compute warps = 4-block groups
constexpr int kLBW0 = 0;                       // look-back warps 0 .. kLB4-1
constexpr int kCW04 = kLB4;                    // compute warps
constexpr int kProd4 = kCW04 + kW4;            // producer: highest warp id
constexpr int kThreads4 = (kProd4 + 1) * 32;
constexpr uint32_t kStage4 = 4 * 128 * 4 + 32;  // a worst-case group + 16-byte phase + slack

struct __align__(1024) Box4 {
  float v[kTileVals];
};
struct __align__(16) Rec4 {
  unsigned long long acc;          // compute (shared atomics): mid | nc << 20 | arrivals << 32
  unsigned long long pre_mid;      // look-back -> compute: stream offsets of the tile
  unsigned long long pre_nc;
  uint32_t tile;                   // producer -> everyone (~0u: stop)
  uint32_t cnt[kW4];               // compute -> look-back: mid | nc << 12 | cst bits << 15
  uint32_t gpre[kW4];              // look-back -> compute: group prefix mid | nc << 16
};
struct V4Smem {
  Box4 in[kNB4];
  uint8_t stage[kW4][kStage4];     // per compute warp, 16-byte aligned
  Rec4 rec[kNB4];
  uint64_t full[kNB4];             // producer -> compute (TMA transaction bytes)
  uint64_t claimed[kNB4];          // producer -> look-back (tile id set)
  uint64_t counted[kNB4];          // compute (16 arrivals, after A) -> look-back
  uint64_t prefix[kNB4];           // look-back -> compute (offsets ready)
  uint64_t in_free[kNB4];          // compute (16 arrivals, after B) -> producer
};
static_assert(kStage4 % 16 == 0, "stage buffers stay 16-byte aligned");

// Phase-B write-out of one group: staged bytes [a16, a16 + len) of `st` (the string sits at
// its final 16-byte phase) go to global mid bytes [gmid, gmid + len); dst16 = gmid - a16.
__device__ __forceinline__ void group_out(uint8_t* dst16, const uint8_t* st, uint32_t a16,
                                          uint32_t len, int lane) {
  if (len == 0) return;
  const uint32_t end = a16 + len;
  const uint32_t nchunk = (end + 15) >> 4;
  const uint32_t c0 = a16 ? 1u : 0u;                       // first whole chunk
  const uint32_t c1 = (end & 15) ? nchunk - 1 : nchunk;    // one past the last whole chunk
  for (uint32_t c = c0 + lane; c < c1; c += 32)
    *reinterpret_cast<uint4*>(dst16 + 16 * c) = *reinterpret_cast<const uint4*>(st + 16 * c);
  // edges: lanes 0-15 the head chunk, lanes 16-31 the tail chunk, one byte each
  const uint32_t c = lane < 16 ? 0u : nchunk - 1;
  const bool part = lane < 16 ? a16 != 0 : ((end & 15) != 0 && !(nchunk == 1 && a16 != 0));
  const uint32_t x = 16 * c + (lane & 15);
  if (part && x >= a16 && x < end) dst16[x] = st[x];
}

}  // namespace

__global__ void __launch_bounds__(kThreads4, 1)
    compress128v4_kernel(CompressArgs a, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  V4Smem& sm = *reinterpret_cast<V4Smem*>(smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t n = a.n;
  const uint64_t nb = (n + 127) >> 7;

  if (tid == 0) {
    for (int s = 0; s < kNB4; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.claimed[s], 1);
      mbar_init(&sm.counted[s], kW4);
      mbar_init(&sm.prefix[s], 1);
      mbar_init(&sm.in_free[s], kW4);
    }
    fence_barrier_init();
  }
  __syncthreads();

  // ---------------------------------------------------------------- producer warp
  if (warp == kProd4) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      // Claims are made as late as possible: a tile claimed now is counted (phase A) only
      // after the tiles already in this CTA's boxes, and every tile's prefix waits for the
      // counts of all lower tiles -- so the claim-to-count depth must stay below kD4.
      uint32_t next = SZX_V4_AHEAD ? atomicAdd(a.counter, 1u) : 0u;
      for (uint32_t k = 0;; ++k) {
        const int s = k % kNB4;
        // box / record s is free once B(k - kNB4) is done (the look-back finished it earlier)
        mbar_wait_sleep(&sm.in_free[s], ((k / kNB4) & 1) ^ 1);
        uint32_t tile;
        if (SZX_V4_STATIC) {  // round robin: a tile's look-back waits only for its round
          const uint64_t t = blockIdx.x + (uint64_t)k * gridDim.x;
          tile = t < a.ntiles ? (uint32_t)t : a.ntiles;
        } else if (SZX_V4_AHEAD) {
          tile = next;
          if (tile < a.ntiles) next = atomicAdd(a.counter, 1u);
        } else {
          tile = atomicAdd(a.counter, 1u);
        }
        Rec4& R = sm.rec[s];
        if (tile >= a.ntiles) {
          // stop the compute warps at k and every look-back warp at its next index k + i
          R.tile = ~0u;
          mbar_arrive(&sm.full[s]);
          mbar_arrive(&sm.claimed[s]);
          for (uint32_t j = k + 1; j < k + kLB4; ++j) {
            const int sj = j % kNB4;
            mbar_wait_sleep(&sm.in_free[sj], ((j / kNB4) & 1) ^ 1);
            sm.rec[sj].tile = ~0u;
            mbar_arrive(&sm.claimed[sj]);
          }
          break;
        }
        R.tile = tile;
        R.acc = 0;
        mbar_arrive(&sm.claimed[s]);
        if (((uint64_t)tile + 1) * kTileVals <= n) {
          mbar_arrive_expect_tx(&sm.full[s], kTileVals * 4);
          tma_load_2d(sm.in[s].v, &tmap, 0, (int)(tile * kTileRows), &sm.full[s]);
        } else {
          mbar_arrive(&sm.full[s]);  // partial tile: the compute warps read global memory
        }
      }
    }
    return;
  }

  // ---------------------------------------------------------------- look-back warps
  if (warp < kLBW0 + kLB4) {
    int64_t floor = -1;       // this warp's previous tile and its inclusive prefix: the
    uint64_t floor_incl = 0;  // look-back never scans past it
    const uint64_t bnc = a.base ? a.base->n_nc : 0, bm = a.base ? a.base->m : 0;
    const uint64_t bmid = a.base ? a.base->mid_len : 0;
    for (uint32_t k = warp - kLBW0;; k += kLB4) {
      const int s = k % kNB4;
      Rec4& R = sm.rec[s];
      mbar_wait_sleep(&sm.claimed[s], (k / kNB4) & 1);
      const uint32_t tile = R.tile;
      if (tile == ~0u) break;
      // the scan needs only the other tiles' status words: it runs while this tile is counted
      const uint64_t ex = tile == 0 ? 0
                                    : lookback_excl<8>(a.status, tile, /*backoff_ns=*/128, floor,
                                                       floor_incl);
      mbar_wait_sleep(&sm.counted[s], (k / kNB4) & 1);
      const unsigned long long acc = R.acc;
      const uint64_t tmid = acc & 0xFFFFFull, tnc = (acc >> 20) & 0xFFFull;
      const uint64_t incl = ex + pack2(tnc, tmid);
      if (lane == 0) st_relaxed(a.status + tile, kFlagPre | incl);
      floor = tile;
      floor_incl = incl;
      // group prefixes (mid | nc << 16) and constant bits from the 16 count words
      const uint32_t w = lane < kW4 ? R.cnt[lane] : 0u;
      const uint32_t pk = (w & 0xFFFu) | (((w >> 12) & 7u) << 16);
      const uint32_t inc = warp_incl_scan(pk);
      if (lane < kW4) R.gpre[lane] = inc - pk;
      const uint32_t cs = lane < kW4 ? ((w >> 15) & 15u) << (4 * (lane & 7)) : 0u;
      const uint32_t lo = __reduce_or_sync(kFull, lane < 8 ? cs : 0u);
      const uint32_t hi = __reduce_or_sync(kFull, lane >= 8 ? cs : 0u);
      if (lane == 0) {
        R.pre_nc = bnc + hi_of(ex);
        R.pre_mid = bmid + lo_of(ex);
        // constant map: 64 bits = 8 bytes per tile, LSB-first (container.py:12-13,321)
        const uint64_t tb = (uint64_t)tile * kTileBlocks;
        uint8_t* mp = a.map + 8 * (uint64_t)tile;
        const uint64_t bits = ((uint64_t)hi << 32) | lo;
        if (tb + kTileBlocks <= nb) {
          reinterpret_cast<uint32_t*>(mp)[0] = lo;
          reinterpret_cast<uint32_t*>(mp)[1] = hi;
        } else {
          const uint32_t nbytes = (uint32_t)((nb - tb + 7) >> 3);
          for (uint32_t i = 0; i < nbytes; ++i) mp[i] = (uint8_t)(bits >> (8 * i));
        }
        if (tile == a.ntiles - 1) {  // chunk totals for the host / the next chunk
          const uint64_t cnc = hi_of(incl);
          a.totals->n_nc = bnc + cnc;
          // the field's short last block counts only its live values when it is NC
          // (container.py:241-244)
          const uint64_t lastb = nb - 1, nvb = n - 128 * lastb;
          const uint32_t lb = (uint32_t)(lastb - tb);
          const uint32_t madj = (nvb < 128 && !((bits >> lb) & 1)) ? 128 - (uint32_t)nvb : 0u;
          a.totals->m = bm + 128 * cnc - madj;
          a.totals->mid_len = bmid + lo_of(incl);
          a.totals->pad = 0;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.prefix[s]);
    }
    return;
  }

  // ---------------------------------------------------------------- compute warps
  const int g = warp - kCW04;        // group: blocks 4g..4g+3 of every tile
  const int jb = lane >> 3;          // block of the group this lane works on
  const int g8 = lane & 7;           // 16-value slice within the block
  uint8_t* const stage = sm.stage[g];

  // Phase B of the tile in box s (local index k): re-encode, stage at the final phase,
  // write out the mid bytes, code rows and req bytes, release the box.
  auto phase_b = [&](uint32_t k) {
    const int s = k % kNB4;
    Rec4& R = sm.rec[s];
    mbar_wait(&sm.prefix[s], (k / kNB4) & 1);
    const uint32_t tile = R.tile;
    const uint64_t v0 = (uint64_t)tile * kTileVals;
    Cls c;
    Lane16 ls;
    bool exists = true;
    if (v0 + kTileVals <= n) encode_full(sm.in[s].v, g, lane, a, c, ls);
    else encode_tail(g, lane, a, v0, c, ls, exists);
    const uint32_t gp = R.gpre[g];
    const uint64_t gmid = R.pre_mid + (gp & 0xFFFFu);
    const uint64_t gnc = R.pre_nc + (gp >> 16);
    const uint32_t incl = warp_incl_scan(ls.L);
    const uint32_t wmid = __shfl_sync(kFull, incl, 31);
    const uint32_t a16 = (uint32_t)(gmid & 15);
    const uint32_t qm = __reduce_max_sync(kFull, c.nc ? (uint32_t)c.q : 0u);
    const uint32_t base = smem_u32(stage) + a16 + incl - ls.L;
    switch (qm) {  // warp-uniform: largest q among the group's NC blocks
      case 0: break;
      case 1: stage_lane<1>(ls, base); break;
      case 2: stage_lane<2>(ls, base); break;
      case 3: stage_lane<3>(ls, base); break;
      default: stage_lane<4>(ls, base); break;
    }
    // code rows (32 bytes per NC block, lane g8 owns word g8) and req bytes
    const uint32_t ncb = __ballot_sync(kFull, c.nc) & 0x01010101u;
    if (c.nc) {
      const uint64_t rank = gnc + __popc(ncb & ((1u << (8 * jb)) - 1));
      reinterpret_cast<uint32_t*>(a.codes + 32 * rank)[g8] = ls.cb;
      if (g8 == 0) a.req[rank] = (uint8_t)c.req;
    }
    __syncwarp();
    group_out(a.mid + (gmid - a16), stage, a16, wmid, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.in_free[s]);
  };

  uint32_t k = 0;
  for (;; ++k) {
    const int s = k % kNB4;
    Rec4& R = sm.rec[s];
    mbar_wait(&sm.full[s], (k / kNB4) & 1);
    const uint32_t tile = R.tile;
    if (tile == ~0u) break;
    // ---- phase A(k): classify + count
    const uint64_t v0 = (uint64_t)tile * kTileVals;
    Cls c;
    Lane16 ls;
    bool exists = true;
    if (v0 + kTileVals <= n) encode_full(sm.in[s].v, g, lane, a, c, ls);
    else encode_tail(g, lane, a, v0, c, ls, exists);
    const uint64_t b0 = (uint64_t)tile * kTileBlocks + (uint64_t)g * kFastBPW;
    if (g8 == 0 && exists) a.mu[b0 + jb] = c.mu;  // container.py:14 -- mu of every block
    if (g8 == 0 && c.nc && c.req < 1) atomicOr(a.err, kErrBadReq);  // container.py:206-207
    const uint32_t wmid = __reduce_add_sync(kFull, ls.L);
    const uint32_t ncb = __ballot_sync(kFull, c.nc) & 0x01010101u;
    const uint32_t csb = __ballot_sync(kFull, !c.nc && exists) & 0x01010101u;
    if (lane == 0) {
      const uint32_t nnc = __popc(ncb);
      R.cnt[g] = wmid | (nnc << 12) |
                 (((csb & 1) | ((csb >> 7) & 2) | ((csb >> 14) & 4) | ((csb >> 21) & 8)) << 15);
      const unsigned long long mine =
          (unsigned long long)wmid | ((unsigned long long)nnc << 20) | (1ull << 32);
      const unsigned long long old = atomicAdd(&R.acc, mine);
      if ((old >> 32) == kW4 - 1 && tile != 0) {  // last group: publish the tile aggregate now
        const unsigned long long t = old + mine;
        st_relaxed(a.status + tile, kFlagAgg | pack2((t >> 20) & 0xFFFull, t & 0xFFFFFull));
      }
      mbar_arrive(&sm.counted[s]);
    }
    // ---- phase B(k - D)
    if (k >= (uint32_t)kD4) phase_b(k - kD4);
  }
  // drain: the last kD4 tiles' phase B
  for (uint32_t j = k > (uint32_t)kD4 ? k - kD4 : 0; j < k; ++j) phase_b(j);
}

cudaError_t launch_compress128v4(const CompressArgs& a, cudaStream_t s) {
  static bool configured = false;
  const size_t smem = sizeof(V4Smem) + 1024;  // + alignment slack for the TMA boxes
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(compress128v4_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  alignas(64) CUtensorMap map;
  const cudaError_t me = make_tile_tmap(a.x, a.n, &map);
  if (me != cudaSuccess) return me;
  const uint32_t cap = (uint32_t)sm_count();
  const uint32_t grid = a.ntiles < cap ? a.ntiles : cap;
  compress128v4_kernel<<<grid, kThreads4, smem, s>>>(a, map);
  return cudaGetLastError();
}

}  // namespace szx
