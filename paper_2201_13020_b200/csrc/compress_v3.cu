// compress_v3.cu -- SZx block encoder for sm_100a, bs == 128 (K1, variant 3).
//
// Replaces the reference's whole compress path in ONE launch per chunk:
//   block_stats           pipeline.py:54-81   (== blockcodec.summarize_block 87-112)
//   _encode_elements      pipeline.py:94-133  (== blockcodec.encode_nonconstant 123-141)
//   prefix_scan + scatter parallel.py:21-44,104-140 / pipeline.py:143-166
// Output pools use the UFZX container layout (container.py:3-21).
//
// Persistent, one CTA per SM, 18 warps: a producer, a look-back warp and 16 compute warps.
// A tile is 64 blocks (32 KiB); compute warp g owns blocks 4g..4g+3 and lane l the 16
// consecutive values 16(l&7).. of block 4g + (l>>3) (the k1_common.cuh encoder).
//
// The compute warps never wait for each other.  Each warp stages its group's mid bytes in a
// PRIVATE 4 KiB shared-memory ring at an offset only it knows (group-relative offsets from
// its own lane scan): no count exchange, no shared ring offset.  Its counts go to the
// look-back warp (one word + an mbarrier arrival; the last warp to count a tile publishes
// the tile aggregate for the decoupled look-back) and, once the look-back warp has turned
// the tile prefix and the group prefixes into stream offsets, the SAME warp writes its
// group out: the mid string as realigned 16-byte stores, its code-row words and req bytes.
// Write-outs are adaptive: after every tile a warp writes out whatever of its pending tiles
// already has a prefix (a non-blocking mbarrier test), and waits only when its ring or the
// tile records run out -- so the look-back lag (a few tiles) never stalls the encoders.
// The input box is released as soon as the warp holds its values in registers.
#include "k1_common.cuh"

namespace szx {

namespace {
using namespace k1;

#ifndef SZX_V3_IN
#define SZX_V3_IN 3
#endif
#ifndef SZX_V3_REC
#define SZX_V3_REC 12
#endif
#ifndef SZX_V3_RING
#define SZX_V3_RING 4096
#endif
constexpr int kIn3 = SZX_V3_IN;     // input boxes: tile k in box k % kIn3 until encoded
constexpr int kRec3 = SZX_V3_REC;   // tile records: tile k in record k % kRec3 until written out
constexpr uint32_t kWRing = SZX_V3_RING;  // private staging ring per compute warp
constexpr uint32_t kGroupMax = 4 * 128 * 4;  // a group's worst-case mid bytes
static_assert(kWRing >= kGroupMax && kWRing % 16 == 0, "a ring must hold a worst-case group");
static_assert(kRec3 >= 2, "records");

constexpr int kW = kV3Warps;                     // compute warps (groups of 4 blocks) per tile
constexpr int kTB = kV3TileBlocks;               // blocks per tile (4 kW)
constexpr int kTV = kTB * 128;                   // values per tile
constexpr int kTRows = kTV / 32;                 // 128-byte rows per tile
constexpr int kBoxRows = kTRows <= 256 ? kTRows : kTRows / 2;  // TMA boxes are <= 256 rows
static_assert(kTRows % kBoxRows == 0 && kBoxRows <= 256 && (kBoxRows * 128) % 1024 == 0,
              "tile = whole 1024-byte-aligned TMA boxes (the swizzle phase restarts per box)");
static_assert(kW <= 32 && kTB % 8 == 0, "one look-back lane per group; whole map bytes per tile");
constexpr int kLBWarp3 = 0;
constexpr int kCW0 = 1;                          // compute warps 1..kW
constexpr int kProd3 = kCW0 + kW;                // producer: highest warp id
constexpr int kThreads3 = (kProd3 + 1) * 32;

struct __align__(1024) Box3 {
  float v[kTV];
};
struct __align__(16) Side3 {       // one compute warp's pending write-out of one tile
  uint32_t cb[32];                 // lane words: word (l & 7) of block (l >> 3)'s code row
  uint32_t req;                    // req byte of block j in bits 8j..8j+7
  uint32_t ncb;                    // bit 8j: block j is non-constant
  uint32_t mid;                    // staged mid bytes
  uint32_t voff;                   // their virtual offset in the warp's ring
};
struct __align__(16) Rec3 {
  unsigned long long acc;          // compute (relaxed shared atomics): mid | nc << 20 | n << 32
  unsigned long long pre_nc, pre_mid;  // look-back -> compute: stream offsets of the tile
  uint32_t tile;                   // producer -> everyone (~0u: stop); global tile id
  uint32_t field;                  // producer -> everyone: field of the tile (batched)
  uint32_t lt;                     // producer -> everyone: tile index within its field
  uint32_t cnt[kW];                // compute -> look-back: mid | nc << 12 | cst bits << 15
  uint32_t gpre[kW];               // look-back -> compute: group prefix mid | nc << 16
};
struct V3Smem {
  Box3 in[kIn3];
  Side3 side[kRec3][kW];   // (rings after the records: the realigned copy may read
  Rec3 rec[kRec3];                 //  16 bytes before / after a staged string)
  uint8_t ring[kW][kWRing];
  uint8_t slack[64];
  uint64_t full[kIn3];             // producer (TMA tx) -> compute
  uint64_t in_free[kIn3];          // compute (16, values in registers) -> producer
  uint64_t claimed[kRec3];         // producer -> look-back
  uint64_t counted[kRec3];         // compute (16) -> look-back
  uint64_t prefix[kRec3];          // look-back -> compute
  uint64_t freed[kRec3];           // compute (16, after write-out) -> producer
};

__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// The per-field view of the launch arguments: a single-field launch uses `a` as is; a batched
// one takes the field's values, bound and pools from its descriptor.
template <bool kBatch>
__device__ __forceinline__ CompressArgs field_args(const CompressArgs& a, const FieldDesc* fds,
                                                   uint32_t f) {
  if constexpr (!kBatch) {
    return a;
  } else {
    CompressArgs r = a;
    const FieldDesc& d = fds[f];
    r.x = d.x;
    r.n = d.n;
    r.e = d.e;
    r.pe = d.pe;
    r.map = d.map;
    r.mu = d.mu;
    r.req = d.req;
    r.codes = d.codes;
    r.mid = d.mid;
    r.totals = d.totals;
    r.base = nullptr;
    r.ntiles = d.ntiles;
    r.index = d.groups;  // per-group offsets for the decode index (null: none)
    return r;
  }
}

__device__ __forceinline__ void fence_tensormap_acquire(const void* p) {
  asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(p) : "memory");
}

}  // namespace

// Profiling builds (-DSZX_STATS): per-phase cycle / event counters, accumulated per warp in
// registers and added to the globals once at the end (szx_debug_stats selector 4).
//  compute warps: [0] input wait [1] encode..counts [2] ring-room write-outs [3] staging
//  [4] record-forced write-outs [5] opportunistic write-outs [6] warp-tiles [7] blocking
//  write-outs [8] opportunistic write-outs [9] sum of pending tiles at each write-out
//  look-back warp: [10] look-back scan [11] counts wait [12] tiles
__device__ unsigned long long g_v3_stats[16];
#ifdef SZX_STATS
#define V3_T0(v) const long long v = clock64()
#define V3_ADD(i, v) stacc[i] += (unsigned long long)(clock64() - (v))
#define V3_INC(i, d) stacc[i] += (unsigned long long)(d)
#define V3_FLUSH() \
  if (lane == 0)   \
    for (int i_ = 0; i_ < 16; ++i_) atomicAdd(&g_v3_stats[i_], stacc[i_])
#define V3_DECL() unsigned long long stacc[16] = {}
#else
#define V3_T0(v)
#define V3_ADD(i, v)
#define V3_INC(i, d)
#define V3_FLUSH()
#define V3_DECL()
#endif
cudaError_t v3_stats(unsigned long long* out16, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out16, g_v3_stats, 16 * sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    const unsigned long long z[16] = {};
    e = cudaMemcpyToSymbol(g_v3_stats, z, sizeof z);
  }
  return e;
}

template <bool kBatch>
__global__ void __launch_bounds__(kThreads3, 1)
    compress128v3_kernel(CompressArgs a, const __grid_constant__ CUtensorMap tmap,
                         const FieldDesc* __restrict__ fds, uint32_t nfields,
                         const CUtensorMap* tmaps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  V3Smem& sm = *reinterpret_cast<V3Smem*>(smem_raw +
                                          ((1024 - (smem_u32(smem_raw) & 1023)) & 1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t n = a.n;

  if (tid == 0) {
    for (int s = 0; s < kIn3; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.in_free[s], kW);
    }
    for (int r = 0; r < kRec3; ++r) {
      mbar_init(&sm.claimed[r], 1);
      mbar_init(&sm.counted[r], kW);
      mbar_init(&sm.prefix[r], 1);
      mbar_init(&sm.freed[r], kW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  // ---------------------------------------------------------------- producer
  if (warp == kProd3) {
    if (lane == 0) {
      if (!kBatch)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      uint32_t next = atomicAdd(a.counter, 1u);  // claimed one ahead: the atomic is hidden
      uint32_t f = 0;                            // field of the last claim (claims increase)
      int32_t fenced = -1;                       // last field whose tensor map was acquired
      for (uint32_t k = 0;; ++k) {
        const int s = k % kIn3, r = k % kRec3;
        mbar_wait_sleep(&sm.in_free[s], ((k / kIn3) & 1) ^ 1);  // tile k - kIn3 encoded
        mbar_wait_sleep(&sm.freed[r], ((k / kRec3) & 1) ^ 1);   // tile k - kRec3 written out
        const uint32_t tile = next;
        if (tile < a.ntiles) next = atomicAdd(a.counter, 1u);
        Rec3& R = sm.rec[r];
        if (tile >= a.ntiles) {
          R.tile = ~0u;
          mbar_arrive(&sm.claimed[r]);
          mbar_arrive(&sm.full[s]);
          break;
        }
        uint32_t lt = tile;
        uint64_t nf = n;
        const CUtensorMap* map = &tmap;
        if constexpr (kBatch) {
          while (f + 1 < nfields && tile >= fds[f + 1].tile0) ++f;
          lt = tile - (uint32_t)fds[f].tile0;
          nf = fds[f].n;
          map = tmaps + f;
          if ((int32_t)f != fenced) {  // written by a host copy: acquire for the TMA proxy
            fence_tensormap_acquire(map);
            fenced = (int32_t)f;
          }
        }
        R.tile = tile;
        R.field = f;
        R.lt = lt;
        R.acc = 0;
        mbar_arrive(&sm.claimed[r]);  // the look-back can start before the tile is encoded
        if (((uint64_t)lt + 1) * kTV <= nf) {
          mbar_arrive_expect_tx(&sm.full[s], kTV * 4);
          for (int bx = 0; bx < kTRows / kBoxRows; ++bx)
            tma_load_2d(sm.in[s].v + bx * kBoxRows * 32, map, 0, (int)(lt * kTRows + bx * kBoxRows),
                        &sm.full[s]);
        } else {
          mbar_arrive(&sm.full[s]);  // partial tile: the compute warps read global memory
        }
      }
    }
    return;
  }

  // ---------------------------------------------------------------- look-back warp
  if (warp == kLBWarp3) {
    V3_DECL();
    int64_t floor = -1;       // this warp's previous tile and its inclusive prefix: the
    uint64_t floor_incl = 0;  // look-back never scans past it
    for (uint32_t k = 0;; ++k) {
      const int r = k % kRec3;
      const uint32_t ph = (k / kRec3) & 1;
      Rec3& R = sm.rec[r];
      mbar_wait_sleep(&sm.claimed[r], ph);
      const uint32_t tile = R.tile;
      if (tile == ~0u) break;
      const uint32_t lt = R.lt;
      const CompressArgs fa = field_args<kBatch>(a, fds, R.field);
      const uint64_t fnb = (fa.n + 127) >> 7;
      if (kBatch && (int64_t)tile - (int64_t)lt > floor) {  // first tile of a new field here
        floor = (int64_t)tile - (int64_t)lt - 1;  // the field starts at a zero prefix
        floor_incl = 0;
      }
      // the scan needs only the other tiles' status words: it runs while this tile is encoded
      V3_T0(t_lb);
      const uint64_t ex = lt == 0 ? 0
                                  : lookback_excl<8>(a.status, tile, /*backoff_ns=*/128, floor,
                                                     floor_incl);
      V3_ADD(10, t_lb);
      V3_T0(t_cw);
      mbar_wait(&sm.counted[r], ph);
      V3_ADD(11, t_cw);
      V3_INC(12, 1);
      // group prefixes inside the tile (lanes 0..kW-1 = groups), packed mid | nc << 16
      const uint32_t c = lane < kW ? R.cnt[lane] : 0u;
      const uint32_t pk = (c & 0xFFFu) | (((c >> 12) & 7u) << 16);
      const uint32_t incl = warp_incl_scan(pk);
      const uint32_t tot = __shfl_sync(kFull, incl, 31);
      if (lane < kW) R.gpre[lane] = incl - pk;
      const uint32_t tmid = tot & 0xFFFFu, tnc = tot >> 16;
      const uint64_t agg = pack2(tnc, tmid);
      // constant map: 4 bits per group, kTB / 8 bytes per tile, LSB-first (container.py:12-13);
      // lane b assembles byte b from groups 2b, 2b+1
      const uint32_t cs = (c >> 15) & 15u;
      const uint32_t cs_lo = __shfl_sync(kFull, cs, (2 * lane) & 31);
      const uint32_t cs_hi = __shfl_sync(kFull, cs, (2 * lane + 1) & 31);
      const uint64_t tb = (uint64_t)lt * kTB;
      const uint32_t nbytes = (uint32_t)((umin64(kTB, fnb - tb) + 7) >> 3);
      if (lane < (int)nbytes) fa.map[tb / 8 + lane] = (uint8_t)(cs_lo | (cs_hi << 4));
      const uint64_t lastb = fnb - 1;
      const uint32_t lb = (uint32_t)(lastb - tb);  // (meaningful in the field's last tile)
      const uint32_t lastcs = __shfl_sync(kFull, cs, (lb >> 2) & 31);
      if (lane == 0) {
        st_relaxed(a.status + tile, kFlagPre | (ex + agg));
        const uint64_t bnc = fa.base ? fa.base->n_nc : 0, bm = fa.base ? fa.base->m : 0;
        const uint64_t bmid = fa.base ? fa.base->mid_len : 0;
        R.pre_nc = bnc + hi_of(ex);
        R.pre_mid = bmid + lo_of(ex);
        if (lt == fa.ntiles - 1) {  // chunk totals for the host / the next chunk
          const uint64_t run = ex + agg;  // inclusive
          const uint64_t cnc = hi_of(run);
          fa.totals->n_nc = bnc + cnc;
          // the field's short last block counts only its live values when it is NC
          // (container.py:241-244)
          const uint64_t nvb = fa.n - 128 * lastb;
          const uint32_t madj = (nvb < 128 && !((lastcs >> (lb & 3)) & 1)) ? 128 - (uint32_t)nvb : 0u;
          fa.totals->m = bm + 128 * cnc - madj;
          fa.totals->mid_len = bmid + lo_of(run);
          fa.totals->pad = 0;
        }
      }
      floor = tile;
      floor_incl = ex + agg;
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.prefix[r]);
    }
    V3_FLUSH();
    return;
  }

  // ---------------------------------------------------------------- compute warps
  const int cw = warp - kCW0;  // compute warp == group 0..15
  const int g = cw;
  const int jb = lane >> 3;    // block of the group this lane works on
  const int gl = lane & 7;     // 16-value slice within the block
  uint8_t* ring = sm.ring[cw];
  uint32_t vpos = 0;           // next free virtual offset of this warp's ring (16-aligned)
  uint32_t tailj = 0;          // oldest tile this warp has not written out yet
  V3_DECL();
  // write out this warp's group of tile j (its prefix is known), then free its record share
  auto write_out = [&](uint32_t j) {
    const int r = j % kRec3;
    const Rec3& R = sm.rec[r];
    const Side3& S = sm.side[r][cw];
    const CompressArgs fa = field_args<kBatch>(a, fds, R.field);
    const uint32_t gp = R.gpre[g];
    const uint64_t pre_nc = R.pre_nc + (gp >> 16);
    const uint64_t pre_mid = R.pre_mid + (gp & 0xFFFFu);
    if constexpr (kBatch) {
      if (fa.index && lane == 0) {  // the group's stream offsets, for the decode index
        const uint64_t G = (uint64_t)R.lt * kW + g;
        fa.index[2 * G] = pre_nc;
        fa.index[2 * G + 1] = pre_mid;
      }
    }
    const uint32_t ncb = S.ncb;
    if ((ncb >> (8 * jb)) & 1) {
      // NC block r owns code bytes [32r, 32r + 32) (container.py:286-294 packing, bs 128)
      const uint32_t rank = __popc(ncb & ((1u << (8 * jb)) - 1));
      reinterpret_cast<uint32_t*>(fa.codes + 32 * (pre_nc + rank))[gl] = S.cb[lane];
      if (gl == 0) fa.req[pre_nc + rank] = (uint8_t)(S.req >> (8 * jb));  // container.py:15
    }
    copy_out(fa.mid, pre_mid, ring + (S.voff % kWRing), S.mid, lane, 32);
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.freed[r]);
  };
  auto write_next = [&]() {  // blocking
    mbar_wait(&sm.prefix[tailj % kRec3], (tailj / kRec3) & 1);
    write_out(tailj);
    ++tailj;
  };
  uint32_t k = 0;
  for (;; ++k) {
    const int s = k % kIn3, r = k % kRec3;
    Rec3& R = sm.rec[r];
    V3_T0(t_in);
    mbar_wait(&sm.full[s], (k / kIn3) & 1);
    V3_ADD(0, t_in);
    V3_INC(6, 1);
    const uint32_t tile = R.tile;
    if (tile == ~0u) break;
    V3_T0(t_enc);
    const uint32_t lt = R.lt;
    const CompressArgs fa = field_args<kBatch>(a, fds, R.field);
    const uint64_t v0 = (uint64_t)lt * kTV;
    Cls c;
    Lane16 ls;
    bool exists = true;
    if (v0 + kTV <= fa.n) encode_full(sm.in[s].v, g, lane, fa, c, ls);
    else encode_tail(g, lane, fa, v0, c, ls, exists);
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.in_free[s]);  // the warp's values are in registers

    const uint64_t b0 = (uint64_t)lt * kTB + (uint64_t)g * kFastBPW;
    if (gl == 0 && exists) fa.mu[b0 + jb] = c.mu;  // container.py:14 -- mu of every block
    if (c.nc && gl == 0 && c.req < 1) atomicOr(a.err, kErrBadReq);  // container.py:206-207
    const uint32_t ncb = __ballot_sync(kFull, c.nc) & 0x01010101u;   // bit 8j: block j NC
    const uint32_t csb = __ballot_sync(kFull, !c.nc && exists) & 0x01010101u;
    // mid-byte offsets of the lanes within the group (stream order = lane order)
    const uint32_t incl = warp_incl_scan(ls.L);
    const uint32_t wmid = __shfl_sync(kFull, incl, 31);
    const uint32_t nnc = __popc(ncb);
    if (lane == 0) {
      R.cnt[g] = wmid | (nnc << 12) |
                 (((csb & 1) | ((csb >> 7) & 2) | ((csb >> 14) & 4) | ((csb >> 21) & 8)) << 15);
      // the last group to count the tile publishes its aggregate for the look-back at once
      const unsigned long long mine = (unsigned long long)wmid |
                                      ((unsigned long long)nnc << 20) | (1ull << 32);
      const unsigned long long old = atomicAdd(&R.acc, mine);
      if ((old >> 32) == kW - 1 && lt != 0) {
        const unsigned long long t = old + mine;
        st_relaxed(a.status + tile, kFlagAgg | pack2((t >> 20) & 0xFFFu, t & 0xFFFFFu));
      }
      mbar_arrive(&sm.counted[r]);
    }
    V3_ADD(1, t_enc);
    V3_T0(t_room);
    // ring room: a group never straddles the ring end; free the oldest tiles if needed
    if ((vpos % kWRing) + wmid > kWRing) vpos += kWRing - (vpos % kWRing);
    while (tailj < k && (int32_t)(vpos + wmid - sm.side[tailj % kRec3][cw].voff) > (int32_t)kWRing) {
      V3_INC(7, 1);
      V3_INC(9, k - tailj);
      write_next();
    }
    V3_ADD(2, t_room);
    V3_T0(t_stg);
    const uint32_t reqw = __reduce_or_sync(kFull, (gl == 0 && c.nc) ? c.req << (8 * jb) : 0u);
    Side3& S = sm.side[r][cw];
    S.cb[lane] = ls.cb;
    if (lane == 0) {
      S.req = reqw;
      S.ncb = ncb;
      S.mid = wmid;
      S.voff = vpos;
    }
    const uint32_t qm = __reduce_max_sync(kFull, c.nc ? (uint32_t)c.q : 0u);
    const uint32_t base = smem_u32(ring) + (vpos % kWRing) + incl - ls.L;
    switch (qm) {  // warp-uniform: largest q among the group's NC blocks
      case 0: break;
      case 1: stage_lane<1>(ls, base); break;
      case 2: stage_lane<2>(ls, base); break;
      case 3: stage_lane<3>(ls, base); break;
      default: stage_lane<4>(ls, base); break;
    }
    vpos += (wmid + 15) & ~15u;
    __syncwarp();
    V3_ADD(3, t_stg);
    // adaptive write-out: everything whose prefix is already there, and (blocking) whatever
    // record the producer needs next (tile k + 1 reuses the record of tile k + 1 - kRec3)
    V3_T0(t_forced);
    while (tailj + kRec3 <= k + 1) {
      V3_INC(7, 1);
      V3_INC(9, k - tailj);
      write_next();
    }
    V3_ADD(4, t_forced);
    V3_T0(t_opp);
    while (tailj < k && mbar_test_wait(&sm.prefix[tailj % kRec3], (tailj / kRec3) & 1)) {
      V3_INC(8, 1);
      V3_INC(9, k - tailj);
      write_out(tailj);
      ++tailj;
    }
    V3_ADD(5, t_opp);
  }
  // drain: the tiles still waiting for their prefixes
  while (tailj < k) write_next();
  V3_FLUSH();
}

cudaError_t launch_compress128v3(const CompressArgs& a, cudaStream_t s) {
  static bool configured = false;
  const size_t smem = sizeof(V3Smem) + 1024;  // + alignment slack for the TMA boxes
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(compress128v3_kernel<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  alignas(64) CUtensorMap map;
  const cudaError_t me = make_tile_tmap(a.x, a.n, &map, kBoxRows);
  if (me != cudaSuccess) return me;
  const uint32_t cap = (uint32_t)sm_count();
  const uint32_t grid = a.ntiles < cap ? a.ntiles : cap;
  compress128v3_kernel<false><<<grid, kThreads3, smem, s>>>(a, map, nullptr, 1, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_compress128v3_batch(const CompressArgs& a, FieldDesc* d_fields,
                                       const FieldDesc* h_fields, uint32_t nfields,
                                       void* d_tmaps, void* h_tmaps, cudaStream_t s) {
  static bool configured = false;
  const size_t smem = sizeof(V3Smem) + 1024;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(compress128v3_kernel<true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  CUtensorMap* hm = static_cast<CUtensorMap*>(h_tmaps);
  for (uint32_t f = 0; f < nfields; ++f) {
    const cudaError_t me = make_tile_tmap(h_fields[f].x, h_fields[f].n, hm + f, kBoxRows);
    if (me != cudaSuccess) return me;
  }
  cudaError_t e = cudaMemcpyAsync(d_tmaps, h_tmaps, sizeof(CUtensorMap) * nfields,
                                  cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(d_fields, h_fields, sizeof(FieldDesc) * nfields, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  alignas(64) CUtensorMap dummy;
  memset(&dummy, 0, sizeof dummy);
  const uint32_t cap = (uint32_t)sm_count();
  const uint32_t grid = a.ntiles < cap ? a.ntiles : cap;
  compress128v3_kernel<true><<<grid, kThreads3, smem, s>>>(a, dummy, d_fields, nfields,
                                                           static_cast<const CUtensorMap*>(d_tmaps));
  return cudaGetLastError();
}

// Decode index entries from the compress kernel's per-group offsets, one warp per entry
// (blockIdx.y = field): entry t = (NC blocks, mid bytes) before group 16 t, the 16 groups' mid
// offsets relative to it, range 0; groups past the field's end sit at its end.  Entry
// ntiles closes with the totals, then the base table {0} -- what K3 (index128_kernel)
// computes, with one range.  Lane i < 16 reads group 16 t + i (one coalesced 256-byte row).
__global__ void groups_to_index_kernel(const FieldDesc* __restrict__ fds) {
  const FieldDesc& d = fds[blockIdx.y];
  if (!d.index) return;
  const int lane = threadIdx.x & 31;
  const uint64_t nb = (d.n + 127) >> 7, ng = (nb + 3) >> 2;
  const uint64_t nt = (nb + 63) >> 6;  // 64-block decode tiles
  const uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t > nt) return;
  const uint64_t tnc = d.totals->n_nc, tmid = d.totals->mid_len;
  uint64_t* e = d.index + 8 * t;
  if (t == nt) {
    if (lane < 9) e[lane] = lane == 0 ? tnc : lane == 1 ? tmid : 0ull;  // + base[0] = 0
    return;
  }
  const uint64_t G = 16 * t + (lane & 15);
  const uint64_t mid = G < ng ? d.groups[2 * G + 1] : tmid;
  const uint64_t mid0 = __shfl_sync(0xFFFFFFFFu, mid, 0);
  const uint64_t off = (mid - mid0) & 0xFFFFu;
  // lane q < 4 packs groups 4q .. 4q + 3
  uint64_t w = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) w |= __shfl_sync(0xFFFFFFFFu, off, (4 * lane + i) & 15) << (16 * i);
  const uint64_t wq = __shfl_sync(0xFFFFFFFFu, w, (lane + 2) & 3);  // lane 2 + q: word of q
  if (lane < 8) {
    const uint64_t g0 = 16 * t;
    e[lane] = lane == 0 ? (g0 < ng ? d.groups[2 * g0] : tnc)
              : lane == 1 ? mid0
              : lane < 6  ? wq
                          : 0ull;
  }
}

cudaError_t launch_groups_to_index(const FieldDesc* d_fields, const FieldDesc* h_fields,
                                   uint32_t nfields, cudaStream_t s) {
  uint64_t most = 0;
  for (uint32_t f = 0; f < nfields; ++f) {
    if (!h_fields[f].index) continue;
    const uint64_t nt = ((h_fields[f].n + 127) / 128 + 63) / 64;
    most = nt + 1 > most ? nt + 1 : most;
  }
  if (!most) return cudaSuccess;
  const dim3 grid((unsigned)((most + 7) / 8), nfields);  // 8 entries (warps) per block
  groups_to_index_kernel<<<grid, 256, 0, s>>>(d_fields);
  return cudaGetLastError();
}

}  // namespace szx
