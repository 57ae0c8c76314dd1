// compress.cu -- SZx block encoder for sm_100a, bs == 128 fast path (K1 in DESIGN.md).
//
// Replaces the reference's whole compress path in ONE launch per chunk:
//   block_stats           pipeline.py:54-81   (== blockcodec.summarize_block 87-112)
//   _encode_elements      pipeline.py:94-133  (== blockcodec.encode_nonconstant 123-141)
//   prefix_scan + scatter parallel.py:21-44,104-140 / pipeline.py:143-166
// Output pools use the UFZX container layout (container.py:3-21).
//
// Persistent, warp-specialised CTAs (1 per SM), 20 warps:
//   warp 19 (producer): claims tiles (64 blocks = 32 KiB of input) in order from a global
//          counter, one claim ahead, and streams them into 4 input boxes with 2-D TMA tensor
//          copies (128-byte swizzle, so every lane's LDS.128 is conflict free).  A box is
//          free again as soon as the compute warps hold the tile in registers;
//   warps 3-18 (compute): compute warp w owns blocks 4w..4w+3 of the tile, lane l owns the 16
//          consecutive values 16(l&7).. of block l>>3.  An 8-lane group reduces its block's
//          min/max and classifies it; the XOR-with-previous chain runs inside the lane.
//          The tile's mid bytes are staged CONTIGUOUSLY in an elastic shared-memory ring,
//          its code rows and req bytes in a tile record, so the write-out is a single
//          realigned copy per tile.  No tile-wide barrier: each warp publishes its group's
//          counts (a tagged word) and needs only its predecessors' -- the groups are mapped
//          so that the highest-priority warp owns the first blocks;
//   warp 0 (look-back): decoupled look-back (256-tile windows) over packed (NC blocks, mid
//          bytes) tile counts, started when the tile is claimed and bounded below by the
//          warp's previous tile;
//   warps 1-2 (write-out): alternate tiles, each writes a staged tile out once its prefix is
//          known (req, code rows, one realigned mid copy) and releases its record and ring
//          space.  Neither the look-back lag nor the write-out holds up the input stream or
//          the encoders: they only fill the ring (about 8 tiles of NYX-like data).
//
// Per element the encoder issues FADD, SHF, LOP3, FLO, LEA.HI, IMAD (pass 1: sizes and
// codes) and, per kept byte column, ISETP + STS.U8 at [reg+imm] (pass 2: staging).
#include <cuda.h>

#include "k1_common.cuh"

namespace szx {

// Per-launch timing counters (cycles), read by szx_debug_stats(); only accumulated in
// profiling builds (-DSZX_STATS), compute counters from compute warp 0 (the last group):
// [0] look-back scan, [1] encode (load..counts), [2] wait for the other groups' counts,
// [3] tiles, [4] ring / record release, [5] wait for input, [6] staging (including [4]),
// [7] write-out.
__device__ unsigned long long g_compress_stats[8];
#ifdef SZX_STATS
#define SZX_STAT_T0(v) const long long v = clock64()
#define SZX_STAT_ADD(i, v) atomicAdd(&g_compress_stats[i], (unsigned long long)(clock64() - (v)))
#define SZX_STAT_INC(i) atomicAdd(&g_compress_stats[i], 1ull)
#else
#define SZX_STAT_T0(v)
#define SZX_STAT_ADD(i, v)
#define SZX_STAT_INC(i)
#endif

// Per-tile event timeline (profiling builds, -DSZX_TRACE): g_k1_trace[8 * tile + e] =
// %globaltimer (ns) at event e: 0 claimed, 1 TMA issued, 2 input seen by the compute warps,
// 3 aggregate published, 4 look-back scan done, 5 inclusive prefix published, 6 staged
// (write-out starts), 7 written out.  szx_k1_trace_buffer() installs the buffer.
__device__ unsigned long long* g_k1_trace;
#ifdef SZX_TRACE
#define SZX_TR(tile, e)                                                              \
  do {                                                                               \
    if (g_k1_trace) {                                                                \
      unsigned long long t_;                                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                         \
      g_k1_trace[8ull * (tile) + (e)] = t_;                                          \
    }                                                                                \
  } while (0)
#else
#define SZX_TR(tile, e)
#endif

namespace {
using namespace k1;

// Warp roles.  The issue arbiter favours the highest warp id: the producer (a few
// latency-critical instructions per tile) gets the top id, the compute warps the next ones,
// and the polling look-back warps the lowest, so they only issue when nobody else can.
#ifndef SZX_K1_WRITERS
#define SZX_K1_WRITERS 2
#endif
#ifndef SZX_K1_SCAN
#define SZX_K1_SCAN 1
#endif
constexpr int kScanWarps = SZX_K1_SCAN;
constexpr int kScanPer = kScanWarps > 1 ? 16 : 8;  // look-back window: 32 * kScanPer tiles
constexpr int kWriteWarps = SZX_K1_WRITERS;
// warp ids: [look-back][write-out][compute][producer] (the issue arbiter favours high ids)
constexpr int kScanWarp = 0;
constexpr int kWriteWarp0 = kScanWarps;
constexpr int kCompWarp0 = kScanWarps + kWriteWarps;
constexpr int kProdWarp = kCompWarps + kWriteWarps + kScanWarps;
constexpr int kCThreads = (kProdWarp + 1) * 32;
constexpr int kStopWarps = kScanWarps > kWriteWarps ? kScanWarps : kWriteWarps;
#ifndef SZX_K1_SPIN_NS
#define SZX_K1_SPIN_NS 300  // poll interval of a group waiting for its predecessors' counts
#endif
#ifndef SZX_K1_STATIC
#define SZX_K1_STATIC 0  // 1: CTA c encodes tiles c, c + G, c + 2G, ... (G = grid size)
#endif
#ifndef SZX_K1_MBX
#define SZX_K1_MBX 0  // 1: count exchange through an mbarrier (all 16 words), no tagged-word polls
#endif
#ifndef SZX_K1_ABL
#define SZX_K1_ABL 0  // timing ablations (wrong output): 1 no staging stores, 2 no count wait, 4 no ttot wait
#endif
#ifndef SZX_K1_IN
#define SZX_K1_IN 4
#endif
#ifndef SZX_K1_REC
#define SZX_K1_REC 8
#endif
#ifndef SZX_K1_RING_KB
#define SZX_K1_RING_KB 72
#endif
constexpr bool kStatic = SZX_K1_STATIC != 0;
constexpr bool kMbx = SZX_K1_MBX != 0;
constexpr int kIn = SZX_K1_IN;    // input boxes: tile k in box k % kIn until it is encoded
constexpr int kRec = SZX_K1_REC;  // tile records: tile k in record k % kRec until written out
constexpr uint32_t kRing = SZX_K1_RING_KB * 1024;  // elastic mid-byte ring
static_assert(kStopWarps <= kIn && kStopWarps <= kRec, "stop signals must fit the rings");
static_assert(kRing % 16 == 0 && kRing >= 8 * kTileVals, "ring must hold two worst-case tiles");

// A tile's input box (128B-swizzled TMA destination), released as soon as every compute warp
// holds its values in registers: the producer refills it while the tile is staged, looked
// back and written out, so input keeps streaming whatever the look-back lag.
struct __align__(1024) InBox {
  float v[kTileVals];
};

// A tile's hand-over record: code rows and req bytes in NC-rank order and the fields passed
// between the roles.  Its mid bytes are staged in the elastic ring at [vpos, vpos + mid_total)
// (virtual offsets: physical vpos % kRing; a tile never straddles the ring end).
// Block sizes BS = 64, 128, 256, 512 share the tile of 8192 values: BS / 16 lanes per block,
// 512 / BS blocks per compute warp, 8192 / BS blocks per tile.
template <int BS>
struct BsGeom {
  static constexpr int kLPB = BS / 16;            // lanes per block
  static constexpr int kBPW = 32 / kLPB;          // blocks per compute warp (group)
  static constexpr int kTB = 16 * kBPW;           // blocks per tile
  static constexpr int kMapW = (kTB + 31) / 32;   // constant-map words per tile
  // bit of each block's first lane: lanes 0, kLPB, 2 kLPB, ...
  static constexpr uint32_t kLead = kLPB == 4    ? 0x11111111u
                                    : kLPB == 8  ? 0x01010101u
                                    : kLPB == 16 ? 0x00010001u
                                                 : 0x00000001u;
  static_assert(BS == 64 || BS == 128 || BS == 256 || BS == 512, "fast-path block sizes");
};

template <int BS>
struct __align__(16) RecT {
  uint32_t codes[2048 / 4];                 // NC-rank-ordered code rows of BS/4 bytes
  uint8_t req[BsGeom<BS>::kTB];
  uint32_t tile;                            // producer -> look-back / write-out (~0u: stop)
  uint32_t mid_total, nc_total;             // compute -> look-back: tile totals
  uint32_t map_w[BsGeom<BS>::kMapW];        // compute -> look-back: constant-block bits
  uint32_t vpos;                            // compute -> compute: ring offset (virtual)
  uint32_t vphys;                           // compute -> write-out: vpos % kRing
  uint32_t done;                            // write-out -> compute: local tile index + 1
  unsigned long long pre_nc, pre_mid;       // look-back -> write-out: exclusive prefixes
  uint16_t goff[kCompWarps];                // compute -> write-out: group mid offsets (index)
  unsigned long long lb_incl;               // look-back -> look-back: inclusive prefix of
  uint32_t lb_tile, lb_tag;                 //   lb_tile, valid when lb_tag == local index + 1
};


// Ring allocation is FIFO in tile order, so a new region is free iff it ends within kRing of
// the start of the OLDEST tile not yet written out.
template <int BS>
struct CompSmem {
  InBox in[kIn];
  uint8_t ring[kRing + 64];                 // staged mid bytes (+ the realignment over-read)
  RecT<BS> rec[kRec];
  uint64_t full[kIn];                       // producer -> compute (TMA transaction bytes)
  uint64_t in_free[kIn];                    // compute (16 warps) -> producer
  uint32_t tile[kIn];                       // producer -> compute: claimed tile id
  uint64_t claimed[kRec];                   // producer (record's tile id set) -> look-back
  uint64_t counted[kRec];                   // compute (warp 0) -> look-back warp
  uint64_t prefix[kRec];                    // look-back warp -> write-out warp
  uint64_t staged[kRec];                    // compute (16 warps, after staging) -> write-out
  uint64_t written[kRec];                   // write-out warp -> compute (record + ring free)
  uint32_t xw[4][kCompWarps];               // per-group counts of tile k in xw[k & 3] (tagged)
  uint32_t ttot[4];                         // tile k's mid bytes | tag (k + 1) << 16, in ttot[k & 3]
  uint64_t xbar[4];                         // SZX_K1_MBX: all 16 count words of tile k published
  uint32_t vhist[kCompWarps][kRec];         // per compute warp: ring offset of tile k (own copy)
};

// Write out a staged tile whose prefix is known (one warp: tid = lane, nthr = 32).
template <int BS>
__device__ __forceinline__ void write_out(const CompressArgs& a, const RecT<BS>& S,
                                          const uint8_t* ring, uint64_t pre_nc,
                                          uint64_t pre_mid, int tid, int nthr) {
  const uint32_t nnc = S.nc_total;
  // req: one byte per NC block (container.py:15,323)
  for (int r = tid; r < (int)nnc; r += nthr) a.req[pre_nc + r] = S.req[r];
  // codes: NC block r owns bytes [BS/4 r, BS/4 (r+1)) of the pool (every NC block but the
  // field's last is full; the short last block's unused codes are zero and lie inside the
  // capacity); the rows are contiguous, so the tile's rows are one 16-byte-chunked copy
  for (int i = tid; i < (int)(nnc * (BS / 64)); i += nthr) {
    const uint4 v = reinterpret_cast<const uint4*>(S.codes)[i];
    uint8_t* dst = a.codes + (uint64_t)(BS / 4) * pre_nc + 16 * i;
    if (((uintptr_t)a.codes & 15) == 0) {
      *reinterpret_cast<uint4*>(dst) = v;
    } else {
      uint32_t* d4 = reinterpret_cast<uint32_t*>(dst);
      d4[0] = v.x; d4[1] = v.y; d4[2] = v.z; d4[3] = v.w;
    }
  }
  copy_out(a.mid, pre_mid, ring + S.vphys, S.mid_total, tid, nthr);
}

}  // namespace

template <int BS>
__global__ void __launch_bounds__(kCThreads, 1)
    compress128_kernel(CompressArgs a, const __grid_constant__ CUtensorMap tmap) {
  using Geo = BsGeom<BS>;
  constexpr int kLPB = Geo::kLPB, kBPW = Geo::kBPW, kTB = Geo::kTB, kMapW = Geo::kMapW;
  constexpr uint32_t kLead = Geo::kLead;
  // count word: mid bytes (<= 2048, 12 bits) | NC blocks << 12 | constant bits << kCstSh |
  // tag (k + 1) << kTagSh: bs 128 (4 blocks per group) 3 + 4 bits and a 13-bit tag, the
  // others 4 + 8 bits and an 8-bit tag
  constexpr int kCstSh = kBPW <= 4 ? 15 : 16, kTagSh = kBPW <= 4 ? 19 : 24;
  constexpr uint32_t kTagMask = (1u << (32 - kTagSh)) - 1, kDataMask = (1u << kTagSh) - 1;
  constexpr uint32_t kNcMask = kBPW <= 4 ? 7u : 15u;
  using Rec = RecT<BS>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  CompSmem<BS>& sm = *reinterpret_cast<CompSmem<BS>*>(
      smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t n = a.n;
  const uint64_t nb = (n + BS - 1) / BS;

  if (tid == 0) {
    for (int s = 0; s < kIn; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.in_free[s], kCompWarps);
    }
    for (int r = 0; r < kRec; ++r) {
      sm.rec[r].done = 0;
      sm.rec[r].lb_tag = 0;
      mbar_init(&sm.claimed[r], 1);
      mbar_init(&sm.counted[r], 1);
      mbar_init(&sm.prefix[r], 1);
      mbar_init(&sm.staged[r], kCompWarps);
      mbar_init(&sm.written[r], 1);
    }
    for (int i = 0; i < 4 * kCompWarps; ++i) (&sm.xw[0][0])[i] = 0;
    for (int i = 0; i < 4; ++i) {
      sm.ttot[i] = 0;
      mbar_init(&sm.xbar[i], kCompWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  // ---------------------------------------------------------------- producer warp
  if (warp == kProdWarp) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      if (kStatic) {
        // Static round-robin tiles: a tile's look-back waits only for the tiles below it,
        // which the other CTAs encode in the same round, so prefetching deep delays no
        // prefix, and the producer never waits for a record (only the staging needs one).
        for (uint32_t k = 0;; ++k) {
          const int s = k % kIn;
          const uint64_t tile = blockIdx.x + (uint64_t)k * gridDim.x;
          mbar_wait_sleep(&sm.in_free[s], ((k / kIn) & 1) ^ 1);
          if (tile >= a.ntiles) {
            sm.tile[s] = ~0u;  // stops the compute warps (the other roles count their tiles)
            mbar_arrive(&sm.full[s]);
            break;
          }
          sm.tile[s] = (uint32_t)tile;
          if ((tile + 1) * kTileVals <= n) {
            mbar_arrive_expect_tx(&sm.full[s], kTileVals * 4);
            SZX_TR(tile, 1);
            tma_load_2d(sm.in[s].v, &tmap, 0, (int)(tile * kTileRows), &sm.full[s]);
          } else {
            mbar_arrive(&sm.full[s]);  // partial tile: the compute warps read global memory
          }
        }
        return;
      }
      uint32_t next = atomicAdd(a.counter, 1u);  // dynamic: slow CTAs simply claim fewer
      if (next < a.ntiles) SZX_TR(next, 0);
      for (uint32_t k = 0;; ++k) {
        const int s = k % kIn;
        mbar_wait_sleep(&sm.in_free[s], ((k / kIn) & 1) ^ 1);
        const uint32_t tile = next;  // claimed one tile ahead: the atomic's latency is hidden
        if (tile < a.ntiles) {
          next = atomicAdd(a.counter, 1u);
          if (next < a.ntiles) SZX_TR(next, 0);
        }
        if (tile >= a.ntiles) {
          // stop every role at its next tile index j = k, k+1, ...: box / record j may still
          // hold tile j - kIn / j - kRec, so wait until it is released, as for a real tile
          sm.tile[s] = ~0u;
          mbar_arrive(&sm.full[s]);                                  // compute warps
          for (uint32_t j = k; j < k + kStopWarps; ++j) {
            const int rj = j % kRec;
            mbar_wait_sleep(&sm.written[rj], ((j / kRec) & 1) ^ 1);
            sm.rec[rj].tile = ~0u;
            if (j < k + kScanWarps) mbar_arrive(&sm.claimed[rj]);    // look-back warps
            if (j < k + kWriteWarps) mbar_arrive(&sm.prefix[rj]);    // write-out warps
          }
          break;
        }
        sm.tile[s] = tile;
        // the look-back can start before the tile is encoded; its record is free once the
        // tile kRec earlier is written out (the look-back lag never holds up the input)
        mbar_wait_sleep(&sm.written[k % kRec], ((k / kRec) & 1) ^ 1);
        sm.rec[k % kRec].tile = tile;
        mbar_arrive(&sm.claimed[k % kRec]);
        if (((uint64_t)tile + 1) * kTileVals <= n) {
          mbar_arrive_expect_tx(&sm.full[s], kTileVals * 4);
          SZX_TR(tile, 1);
          tma_load_2d(sm.in[s].v, &tmap, 0, (int)(tile * kTileRows), &sm.full[s]);
        } else {
          mbar_arrive(&sm.full[s]);  // partial tile: the compute warps read global memory
        }
      }
    }
    return;
  }

  // ---------------------------------------------------------------- look-back warps
  // Decoupled look-back (256-tile windows) for this CTA's tiles, started as soon as the
  // producer has claimed a tile and bounded below by the warp's previous tile (whose
  // inclusive prefix it knows).  The compute warps publish each tile's aggregate as soon as
  // its counts are known and never wait for a prefix: the look-back latency and the
  // write-out run beside the encoding of the following tiles.
  if (SZX_K1_ABL & 8) {  // ablation: input pipeline only (static tiles, no encode / output)
    if (warp < kCompWarp0 || warp >= kCompWarp0 + kCompWarps) return;
    for (uint32_t k = 0;; ++k) {
      const int ik = k % kIn;
      mbar_wait(&sm.full[ik], (k / kIn) & 1);
      if (sm.tile[ik] == ~0u) break;
      const float4 x = *reinterpret_cast<const float4*>(
          reinterpret_cast<const uint8_t*>(sm.in[ik].v) + swz_off(warp - kCompWarp0, lane, 0));
      if (x.x == 12345.f) atomicOr(a.err, 64u);  // keep the load
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.in_free[ik]);
    }
    return;
  }
  if (warp >= kScanWarp && warp < kScanWarp + kScanWarps) {
    int64_t floor = -1;       // this warp's previous tile and its inclusive prefix: the
    uint64_t floor_incl = 0;  // look-back never scans past it
    for (uint32_t k = warp - kScanWarp;; k += kScanWarps) {
      const int rk = k % kRec;
      Rec& S = sm.rec[rk];
      uint32_t tile;
      if (kStatic) {
        const uint64_t t = blockIdx.x + (uint64_t)k * gridDim.x;
        if (t >= a.ntiles) break;
        tile = (uint32_t)t;
      } else {
        mbar_wait_sleep(&sm.claimed[rk], (k / kRec) & 1);
        tile = S.tile;
        if (tile == ~0u) break;
      }
      if (lane == 0) { SZX_STAT_INC(3); }
      // the scan needs only the other tiles' status words: it runs while this tile is encoded
      SZX_STAT_T0(t_lb);
      if (kStatic && lane == 0) SZX_TR(tile, 0);  // static: event 0 = look-back scan start
      if (kScanWarps > 1 && k >= 1) {
        // the CTA's previous tile, if another look-back warp has resolved it already, is a
        // closer floor than this warp's own previous tile
        const Rec& P = sm.rec[(k - 1) % kRec];
        if (ld_acquire_cta(&P.lb_tag) == k && (int64_t)P.lb_tile > floor) {
          floor = P.lb_tile;
          floor_incl = P.lb_incl;
        }
      }
      const uint64_t ex = tile == 0 ? 0
                                    : lookback_excl<kScanPer>(a.status, tile, /*backoff_ns=*/128,
                                                              floor, floor_incl);
      if (lane == 0) { SZX_STAT_ADD(0, t_lb); SZX_TR(tile, 4); }
      mbar_wait_sleep(&sm.counted[rk], (k / kRec) & 1);
      const uint64_t agg = pack2(S.nc_total, S.mid_total);
      if (lane == 0) {
        if (kStatic) S.tile = tile;  // (the record is this tile's once `counted` completed)
        st_relaxed(a.status + tile, kFlagPre | (ex + agg));
        SZX_TR(tile, 5);
        if (kScanWarps > 1) {
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
        if (tile == a.ntiles - 1) {  // chunk totals for the host / the next chunk
          const uint64_t run = ex + agg;  // inclusive
          const uint64_t cnc = hi_of(run);
          a.totals->n_nc = bnc + cnc;
          // the field's short last block counts only its live values when it is NC
          // (container.py:241-244)
          const uint64_t lastb = nb - 1, nvb = n - (uint64_t)BS * lastb;
          const uint32_t lb = (uint32_t)(lastb - (uint64_t)tile * kTB);
          const uint32_t lbit = (S.map_w[lb >> 5] >> (lb & 31)) & 1u;
          const uint32_t madj = (nvb < (uint64_t)BS && !lbit) ? BS - (uint32_t)nvb : 0u;
          a.totals->m = bm + (uint64_t)BS * cnc - madj;
          a.totals->mid_len = bmid + lo_of(run);
          a.totals->pad = 0;
          if (a.index && a.idx_last) {  // closing entry (totals, range 0) + base table {0}
            uint64_t* ce = a.index + 8 * a.idx_ntiles;
            ce[0] = bnc + cnc;
            ce[1] = bmid + lo_of(run);
            for (int i = 2; i < 8; ++i) ce[i] = 0;
            ce[8] = 0;
          }
        }
        // constant map: 64 bits = 8 bytes per tile, LSB-first (container.py:12-13,321)
        const uint64_t tb = (uint64_t)tile * kTB;
        uint8_t* mp = a.map + (kTB / 8) * (uint64_t)tile;
        if (tb + kTB <= nb) {
          if constexpr (kTB >= 32) {
#pragma unroll
            for (int w = 0; w < kMapW; ++w) reinterpret_cast<uint32_t*>(mp)[w] = S.map_w[w];
          } else {
            *reinterpret_cast<uint16_t*>(mp) = (uint16_t)S.map_w[0];
          }
        } else {
          const uint32_t nbytes = (uint32_t)((nb - tb + 7) >> 3);
          for (uint32_t i = 0; i < nbytes; ++i) mp[i] = (uint8_t)(S.map_w[i >> 2] >> (8 * (i & 3)));
        }
        mbar_arrive(&sm.prefix[rk]);
      }
      __syncwarp();
    }
    return;
  }

  // ---------------------------------------------------------------- write-out warps
  // Tile k (round robin) once its prefix is known and the compute warps have staged it; its
  // record and ring space then go back to the compute warps.
  if (warp >= kWriteWarp0 && warp < kWriteWarp0 + kWriteWarps) {
    for (uint32_t k = warp - kWriteWarp0;; k += kWriteWarps) {
      const int r = k % kRec;
      const Rec& S = sm.rec[r];
      if (kStatic && blockIdx.x + (uint64_t)k * gridDim.x >= a.ntiles) break;
      mbar_wait_sleep(&sm.prefix[r], (k / kRec) & 1);
      if (!kStatic && S.tile == ~0u) break;
      mbar_wait(&sm.staged[r], (k / kRec) & 1);
      SZX_STAT_T0(t_wo);
      if (lane == 0) SZX_TR(S.tile, 6);
      write_out(a, S, sm.ring, S.pre_nc, S.pre_mid, lane, 32);
      if (a.index && lane < 8) {
        // the decode index entry K3 would compute (decompress.cu IndexArgs): NC blocks and mid
        // bytes before the tile (absolute: one range, base 0), the group offsets, range 0
        const uint16_t* go = S.goff;
        const uint64_t w = lane == 0   ? S.pre_nc
                           : lane == 1 ? S.pre_mid
                           : lane < 6  ? (uint64_t)go[4 * (lane - 2)] |
                                            ((uint64_t)go[4 * (lane - 2) + 1] << 16) |
                                            ((uint64_t)go[4 * (lane - 2) + 2] << 32) |
                                            ((uint64_t)go[4 * (lane - 2) + 3] << 48)
                                       : 0ull;
        a.index[8 * (a.idx_tile0 + S.tile) + lane] = w;
      }
      if (lane == 0) SZX_TR(S.tile, 7);
      if (lane == 0) { SZX_STAT_ADD(7, t_wo); }
      __syncwarp();
      if (lane == 0) {
        st_release_cta(&sm.rec[r].done, k + 1);  // fast path for the compute warps
        mbar_arrive(&sm.written[r]);             // the producer (and slow path) waits here
      }
    }
    return;
  }

  // ---------------------------------------------------------------- compute warps
  const int cw = warp - kCompWarp0;  // compute warp index 0..15
  const int ctid = cw * 32 + lane;
  const int jb = lane / kLPB;       // block of the warp this lane works on
  const int g = lane % kLPB;        // 16-value group within the block
  // Group g = 15 - cw: the highest-priority warp encodes the tile's first four blocks, so the
  // per-group prefix below usually finds its predecessors' counts already published and no
  // warp waits on a tile-wide barrier.
  const int grp = kCompWarps - 1 - cw;
  // identical in every compute warp: oldest tile not known written out, ring offsets
  uint32_t tail = 0, vpos = 0, vphys = 0;  // vphys == vpos % kRing
  uint32_t tail_v = 0;                     // ring offset of tile `tail` (from the warp's history)
  uint32_t prev_tot = 0;                   // SZX_K1_MBX: the previous tile's mid bytes
  uint32_t* vhist = sm.vhist[cw];
  auto release = [&]() {  // wait until tile `tail` is written out
    // an acquire load of the record's flag (~an LDS) instead of an mbarrier try_wait; the
    // barrier only when the write-out is really still pending
    if (ld_acquire_cta(&sm.rec[tail % kRec].done) != tail + 1)
      mbar_wait(&sm.written[tail % kRec], (tail / kRec) & 1);
    ++tail;
    tail_v = vhist[tail % kRec];  // tail <= k: this warp stored it when it placed that tile
  };
  // counts word: mid bytes (<= 2048, 12 bits) | NC blocks << 12 | constant bits << 15 |
  // tag (k + 1, 13 bits) << 19; lanes >= `upto` get a dummy ready word
  auto wait_counts = [&](uint32_t kk, int upto) {
    const uint32_t tag = (kk + 1) & kTagMask;
    uint32_t e, it = 0;
    while (true) {
      e = lane < upto ? ld_volatile_cta(&sm.xw[kk & 3][lane]) : tag << kTagSh;
      if (__all_sync(kFull, (e >> kTagSh) == tag)) break;
      __nanosleep(SZX_K1_SPIN_NS);
      if (++it > (1u << 24)) __trap();  // watchdog: a lost count word must not hang the GPU
    }
    return lane < upto ? e & kDataMask : 0u;
  };
  for (uint32_t k = 0;; ++k) {
    const int ik = k % kIn, rk = k % kRec;
    Rec& R = sm.rec[rk];
    SZX_STAT_T0(t_loop);
    mbar_wait(&sm.full[ik], (k / kIn) & 1);
    if (ctid == 0) { SZX_STAT_ADD(5, t_loop); }
    SZX_STAT_T0(t_enc);
    const uint32_t tile = sm.tile[ik];
    if (tile == ~0u) break;  // the producer stops the other roles
    if (ctid == 0) SZX_TR(tile, 2);
    const uint64_t v0 = (uint64_t)tile * kTileVals;
    const bool full = v0 + kTileVals <= n;
    Cls c;
    Lane16 s;
    bool exists = true;
    if (full) encode_full<kLPB>(sm.in[ik].v, grp, lane, a, c, s);
    else encode_tail<kLPB>(grp, lane, a, v0, c, s, exists);
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.in_free[ik]);  // the warp's values are in registers

    const uint64_t b0 = (uint64_t)tile * kTB + (uint64_t)grp * kBPW;
    if (g == 0 && exists) a.mu[b0 + jb] = c.mu;  // container.py:14 -- mu of every block
    const uint32_t ncb = __ballot_sync(kFull, c.nc) & kLead;   // bit kLPB j: block j NC
    const uint32_t csb = __ballot_sync(kFull, !c.nc && exists) & kLead;
    uint32_t cbits = 0;  // constant bits of the group's blocks, block j at bit j
    if constexpr (kLPB == 8) {
      cbits = (csb & 1) | ((csb >> 7) & 2) | ((csb >> 14) & 4) | ((csb >> 21) & 8);
    } else {
#pragma unroll
      for (int j = 0; j < kBPW; ++j) cbits |= ((csb >> (j * kLPB)) & 1u) << j;
    }
    // mid-byte offsets of the lanes within the warp (stream order = lane order)
    uint32_t incl, wmid;
    incl = s.L;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += t;
    }
    wmid = __shfl_sync(kFull, incl, 31);
    if (lane == 0)  // relaxed: the word itself is the data (no MEMBAR behind the mu store)
      st_volatile_cta(&sm.xw[k & 3][grp],
                     wmid | ((uint32_t)__popc(ncb) << 12) | (cbits << kCstSh) |
                         (((k + 1) & kTagMask) << kTagSh));
    if (kMbx && lane == 0) mbar_arrive(&sm.xbar[k & 3]);  // (release: the word is visible)
    if (ctid == 0) { SZX_STAT_ADD(1, t_enc); }
    SZX_STAT_T0(t_x);
    // this tile's ring offset: after the previous tile (all groups' counts), moved to the
    // next lap when a worst-case tile would not fit before the ring end
    if (kMbx && k > 0) {
      // every group summed the previous tile's counts itself
      const uint32_t adv = (prev_tot + 15) & ~15u;  // vpos stays 16-byte aligned
      vpos += adv;
      vphys += adv;
      if (vphys >= kRing) vphys -= kRing;
      if (vphys > kRing - 4 * kTileVals) {  // a worst-case tile would not fit: next lap
        vpos += kRing - vphys;
        vphys = 0;
      }
    } else if (k > 0) {
      // the previous tile's mid total, published by its last group as one tagged word
      const uint32_t tag = k & 0xFFFFu;  // (k - 1) + 1
      uint32_t w = SZX_K1_ABL & 4 ? 8192u : 0u, it = 0;
      while (!(SZX_K1_ABL & 4) && ((w = ld_volatile_cta(&sm.ttot[(k - 1) & 3])) >> 16) != tag) {
        __nanosleep(SZX_K1_SPIN_NS);
        if (++it > (1u << 24)) __trap();  // watchdog
      }
      const uint32_t prev_mid = w & 0xFFFFu;
      const uint32_t adv = (prev_mid + 15) & ~15u;  // vpos stays 16-byte aligned
      vpos += adv;
      vphys += adv;
      if (vphys >= kRing) vphys -= kRing;
      if (vphys > kRing - 4 * kTileVals) {  // a worst-case tile would not fit: next lap
        vpos += kRing - vphys;
        vphys = 0;
      }
    }
    if (lane == 0) vhist[k % kRec] = vpos;
    __syncwarp();
    // the record's previous tile (kRec back) must be written out; checked here, while the
    // other groups' counts are still coming in
    while (tail + kRec <= k) release();
    // this group's offsets: counts of the groups before it (all 16 for the last group)
    const int upto = grp == kCompWarps - 1 ? kCompWarps : grp;
    uint32_t cnt;
    if (kMbx) {  // all 16 count words: one hardware-suspending barrier wait, no polls
      mbar_wait(&sm.xbar[k & 3], (k >> 2) & 1);
      cnt = lane < kCompWarps ? ld_volatile_cta(&sm.xw[k & 3][lane]) & kDataMask : 0u;
    } else {
      cnt = SZX_K1_ABL & 2 ? (lane < upto ? ld_volatile_cta(&sm.xw[k & 3][lane]) & kDataMask : 0u)
                           : wait_counts(k, upto);
    }
    if (ctid == 0) { SZX_STAT_ADD(2, t_x); }
    SZX_STAT_T0(t_stg);
    // one reduction for both: mid bytes (<= 32768 per tile) | NC blocks << 16
    const uint32_t pk = (cnt & 0xFFFu) | (((cnt >> 12) & kNcMask) << 16);
    const bool last_grp = grp == kCompWarps - 1;
    uint32_t sum_pk, pre_pk;
    if (kMbx) {
      sum_pk = __reduce_add_sync(kFull, pk);
      pre_pk = __reduce_add_sync(kFull, lane < grp ? pk : 0u);
      prev_tot = sum_pk & 0xFFFFu;
    } else {
      sum_pk = __reduce_add_sync(kFull, last_grp || lane < grp ? pk : 0u);
      // the last group summed every group: its prefix is the total minus its own counts
      const uint32_t own_pk = wmid | ((uint32_t)__popc(ncb) << 16);
      pre_pk = last_grp ? sum_pk - own_pk : sum_pk;
    }
    const uint32_t pre_mid = pre_pk & 0xFFFFu, pre_nc = pre_pk >> 16;
    if (a.index && lane == 0) R.goff[grp] = (uint16_t)pre_mid;  // (before `staged`)
    if (!kMbx && last_grp && lane == 0)  // the next tile's ring offset needs only this word
      st_volatile_cta(&sm.ttot[k & 3], (sum_pk & 0xFFFFu) | (((k + 1) & 0xFFFFu) << 16));
    // the tiles (in order) whose ring bytes this group's region overlaps must be written out
    SZX_STAT_T0(t_rel);
    const uint32_t my_end = vpos + pre_mid + wmid;
    // wrap-safe: virtual offsets are compared by their signed difference
    while (tail < k && (int32_t)(my_end - tail_v) > (int32_t)kRing) release();
    if (ctid == 0) { SZX_STAT_ADD(4, t_rel); }
    if (last_grp) {  // the last group has every count: tile totals + hand-over
      const uint32_t tmid = sum_pk & 0xFFFFu, tnc = sum_pk >> 16;
      // the tile's constant map: group l's kBPW bits at bit kBPW l (map word kBPW l / 32)
      const uint32_t cs =
          lane < kCompWarps ? ((cnt >> kCstSh) & ((1u << kBPW) - 1u)) << ((kBPW * lane) & 31) : 0u;
      uint32_t mw[kMapW];
      if constexpr (kMapW == 2 && kBPW == 4) {  // bs 128: groups 0-7 / 8-15
        mw[0] = __reduce_or_sync(kFull, lane < 8 ? cs : 0u);
        mw[1] = __reduce_or_sync(kFull, lane >= 8 ? cs : 0u);
      } else {
#pragma unroll
        for (int w = 0; w < kMapW; ++w) {
          const int l0 = w * 32 / kBPW, l1 = l0 + 32 / kBPW;
          mw[w] = __reduce_or_sync(kFull, lane >= l0 && lane < l1 ? cs : 0u);
        }
      }
      if (lane == 0) {
        // publish the tile aggregate at once; the look-back warp's inclusive-prefix store
        // is ordered after it by the counted barrier
        if (tile != 0) st_relaxed(a.status + tile, kFlagAgg | pack2(tnc, tmid));
        SZX_TR(tile, 3);
        R.mid_total = tmid;
        R.nc_total = tnc;
#pragma unroll
        for (int w = 0; w < kMapW; ++w) R.map_w[w] = mw[w];
        R.vpos = vpos;
        R.vphys = vphys;
        mbar_arrive(&sm.counted[rk]);
      }
    }
    if (c.nc) {
      const uint32_t rank = pre_nc + __popc(ncb & ((1u << (kLPB * jb)) - 1));
      R.codes[rank * kLPB + g] = s.cb;
      if (g == 0) {
        R.req[rank] = (uint8_t)c.req;
        if (c.req < 1) atomicOr(a.err, kErrBadReq);  // container.py:206-207
      }
    }
    const uint32_t qm = __reduce_max_sync(kFull, c.nc ? (uint32_t)c.q : 0u);
    const uint32_t base = smem_u32(sm.ring) + vphys + pre_mid + incl - s.L;
    switch (SZX_K1_ABL & 1 ? 0u : qm) {  // warp-uniform: largest q among the warp's NC blocks
      case 0: break;
      case 1: stage_lane<1>(s, base); break;
      case 2: stage_lane<2>(s, base); break;
      case 3: stage_lane<3>(s, base); break;
      default: stage_lane<4>(s, base); break;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.staged[rk]);  // the write-out warp may copy it out
    if (ctid == 0) { SZX_STAT_ADD(6, t_stg); }
  }
}

cudaError_t k1_trace_buffer(unsigned long long* d_buf) {
  return cudaMemcpyToSymbol(g_k1_trace, &d_buf, sizeof d_buf);
}

cudaError_t compress_stats(unsigned long long* out8, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out8, g_compress_stats, 8 * sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    e = cudaMemcpyToSymbol(g_compress_stats, z, sizeof z);
  }
  return e;
}

namespace k1 {
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda needed).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D view of a chunk: rows of 32 floats (128 bytes), boxes of one tile (kTileRows rows),
// 128-byte swizzle.  Only whole rows are mapped; partial tiles are read from global memory.
cudaError_t make_tile_tmap(const float* x, uint64_t n, CUtensorMap* map, uint32_t box_rows) {
  memset(map, 0, sizeof *map);
  const uint64_t rows = n / 32;
  if (rows < box_rows) return cudaSuccess;
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {32, rows};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {32, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  if (fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(x), dims, strides, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  return cudaSuccess;
}

int sm_count() {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  return nsm;
}
}  // namespace k1

namespace {
template <int BS>
cudaError_t launch_fast(const CompressArgs& a, cudaStream_t s) {
  static bool configured = false;
  static int per_sm = 1;
  const size_t smem = sizeof(CompSmem<BS>) + 1024;  // + alignment slack for the TMA boxes
  if (!configured) {
    cudaFuncSetAttribute(compress128_kernel<BS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, compress128_kernel<BS>, kCThreads, smem);
    if (per_sm < 1) per_sm = 1;
    configured = true;
  }
  const int nsm = sm_count();
  alignas(64) CUtensorMap map;
  const cudaError_t me = make_tile_tmap(a.x, a.n, &map);
  if (me != cudaSuccess) return me;
  const uint32_t cap = (uint32_t)(per_sm * nsm);
  const uint32_t grid = a.ntiles < cap ? a.ntiles : cap;
  compress128_kernel<BS><<<grid, kCThreads, smem, s>>>(a, map);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_compress128(const CompressArgs& a, cudaStream_t s) {
  return launch_fast<128>(a, s);
}

cudaError_t launch_compress_fast(const CompressArgs& a, cudaStream_t s) {
  switch (a.bs) {
    case 64: return launch_fast<64>(a, s);
    case 128: return launch_fast<128>(a, s);
    case 256: return launch_fast<256>(a, s);
    case 512: return launch_fast<512>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace szx
