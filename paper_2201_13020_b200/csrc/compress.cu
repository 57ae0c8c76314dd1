// compress.cu -- SZx block encoder for sm_100a, bs == 128 fast path (K1 in DESIGN.md).
//
// Replaces the reference's whole compress path in ONE launch per chunk:
//   block_stats           pipeline.py:54-81   (== blockcodec.summarize_block 87-112)
//   _encode_elements      pipeline.py:94-133  (== blockcodec.encode_nonconstant 123-141)
//   prefix_scan + scatter parallel.py:21-44,104-140 / pipeline.py:143-166
// Output pools use the UFZX container layout (container.py:3-21).
//
// Persistent, warp-specialised CTAs (2 per SM), 10 warps:
//   warp 8 (producer): claims tiles (32 blocks = 16 KiB of input) in order from a global
//          counter and streams them into a 3-deep shared-memory ring with 1-D bulk copies
//          (TMA engine, mbarrier transaction counts);
//   warps 0-7 (compute): one warp = 4 blocks, lane l owns values 4l..4l+3 of each block.
//          Tile k is classified, encoded and STAGED (mid bytes, codes, req) in shared memory
//          and its counts published; only then is tile k-1 written out, so a tile's
//          aggregate never waits for an earlier tile's prefix (no look-back convoys);
//   warp 9 (scan): decoupled look-back (256-tile windows) over packed (NC blocks, mid
//          bytes) tile counts, overlapped with the compute warps' next tile.
#include "szx_device.cuh"
#include "szx_kernels.h"

namespace szx {

// Per-launch timing counters (cycles), read by szx_debug_stats(): [0] scan-warp look-back,
// [1] look-back windows, [2] compute-warp wait for the prefix, [3] tiles, [4] compute-warp
// encode, [5] compute-warp write-out, [6] producer wait for a free slot, [7] compute-warp
// wait for input.
__device__ unsigned long long g_compress_stats[8];

namespace {

constexpr int kCompWarps = 8;
constexpr int kProdWarp = 8;
constexpr int kScanWarp = 9;     // scan warps 9 and 10 take alternate tiles
constexpr int kScanWarps = 2;
constexpr int kCThreads = (kCompWarps + 1 + kScanWarps) * 32;
constexpr int kDefer = 2;        // tile k is written out after tile k+kDefer is staged
constexpr int kTileBufs = kDefer + 1;
constexpr int kInStages = 3;
constexpr int kTileVals = kFastTileBlocks * 128;   // 4096
constexpr int kWarpMidBytes = kFastBPW * 512;       // worst case per compute warp
constexpr int kWarpMidStride = kWarpMidBytes + 32;  // room for the realignment window
constexpr uint32_t kBarThreads = (kCompWarps + 1) * 32;

// Everything a tile needs between "staged" and "written out" (double-buffered by parity).
struct __align__(16) TileBuf {
  uint8_t mid[kCompWarps][kWarpMidStride];
  uint8_t codes[kCompWarps][kFastBPW][32];
  uint8_t req[kCompWarps][kFastBPW];
  uint32_t wnc[kCompWarps], wmid[kCompWarps], wcst[kCompWarps], wncm[kCompWarps];
  uint32_t wnc_ex[kCompWarps], wmid_ex[kCompWarps];
  uint32_t cur_tile;
  uint32_t pad;
  unsigned long long pre_nc, pre_mid;
  unsigned long long agg;  // per-tile aggregate being accumulated by the compute warps
};

struct CompSmem {
  float in[kInStages][kTileVals];
  TileBuf tb[kTileBufs];
  uint64_t full[kInStages];
  uint64_t empty[kInStages];
  uint32_t tile[kInStages];
  uint32_t madj;
};

__device__ __forceinline__ void bar_arrive(uint32_t id) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(kBarThreads) : "memory");
}
__device__ __forceinline__ void bar_sync(uint32_t id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kBarThreads) : "memory");
}
// barrier ids: counts ready (compute -> scan) and prefix ready (scan -> compute), by parity
__device__ __forceinline__ uint32_t bar_counts(uint32_t buf) { return 1 + buf; }
__device__ __forceinline__ uint32_t bar_prefix(uint32_t buf) { return 1 + kTileBufs + buf; }

// Copy `len` staged bytes (16-byte aligned shared source) to global byte offset `pos` of
// `dst` (16-byte aligned base), one 16-byte aligned global chunk per lane-iteration: the
// source window is re-aligned with funnel shifts (the shift is warp-uniform).
__device__ __forceinline__ void copy_out_realigned(uint8_t* dst, uint64_t pos,
                                                   const uint8_t* src, uint32_t len, int lane) {
  if (len == 0) return;
  const uint32_t a = (uint32_t)(pos & 15);
  uint8_t* g = dst + (pos - a);
  const uint32_t nchunk = (a + len + 15) >> 4;
  // the source window of global chunk c starts at staged byte 16c - a; the staging region
  // is read as 16-byte rows starting one row early (the region keeps 16 bytes of slack on
  // each side), so every chunk is rows j, j+1 funnel-shifted by a warp-uniform amount
  const uint32_t d = (16 - a) & 15;
  const uint32_t k = d >> 2, b = 8 * (d & 3);
  const uint4* s128 = reinterpret_cast<const uint4*>(src);
  for (uint32_t c = lane; c < nchunk; c += 32) {
    const int lo = 16 * (int)c - (int)a;  // first staged byte of this chunk (may be < 0)
    const int j = (lo + 16) >> 4;         // row index relative to one row before src
    const uint4 q0 = s128[j - 1], q1 = s128[j];
    const uint32_t w[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
    uint4 o;
    switch (k) {  // warp-uniform
      case 0: o = make_uint4(__funnelshift_r(w[0], w[1], b), __funnelshift_r(w[1], w[2], b),
                             __funnelshift_r(w[2], w[3], b), __funnelshift_r(w[3], w[4], b)); break;
      case 1: o = make_uint4(__funnelshift_r(w[1], w[2], b), __funnelshift_r(w[2], w[3], b),
                             __funnelshift_r(w[3], w[4], b), __funnelshift_r(w[4], w[5], b)); break;
      case 2: o = make_uint4(__funnelshift_r(w[2], w[3], b), __funnelshift_r(w[3], w[4], b),
                             __funnelshift_r(w[4], w[5], b), __funnelshift_r(w[5], w[6], b)); break;
      default: o = make_uint4(__funnelshift_r(w[3], w[4], b), __funnelshift_r(w[4], w[5], b),
                              __funnelshift_r(w[5], w[6], b), __funnelshift_r(w[6], w[7], b)); break;
    }
    uint8_t* gc = g + 16 * c;
    if (lo >= 0 && lo + 16 <= (int)len) {
      *reinterpret_cast<uint4*>(gc) = o;
    } else {
      // chunk shared with a neighbour: whole words where all 4 bytes are ours, bytes else
      const uint32_t ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
      for (int wi = 0; wi < 4; ++wi) {
        const int b0 = lo + 4 * wi;  // staged index of the word's first byte
        if (b0 >= 0 && b0 + 4 <= (int)len) {
          *reinterpret_cast<uint32_t*>(gc + 4 * wi) = ow[wi];
        } else {
#pragma unroll
          for (int bi = 0; bi < 4; ++bi)
            if (b0 + bi >= 0 && b0 + bi < (int)len) gc[4 * wi + bi] = (uint8_t)(ow[wi] >> (8 * bi));
        }
      }
    }
  }
}

// Stage the mid bytes of one element: big-endian bytes [c, Q) of sh at d[0..Q-c)
// (pipeline.py:114-116,151).  `d` is already offset by -c, so byte k lands at d[k].
template <int Q>
__device__ __forceinline__ void stage_bytes(uint8_t* d, uint32_t sh, int c) {
#pragma unroll
  for (int k = 0; k < Q; ++k)
    if (c <= k) d[k] = (uint8_t)(sh >> (24 - 8 * k));
}

// Write out a staged tile (its prefix is known): req, codes, mid bytes.
__device__ __forceinline__ void write_out(const CompressArgs& a, const TileBuf& T, uint32_t tile,
                                          int warp, int lane, uint64_t n) {
  const uint32_t nnc = T.wnc[warp];
  const uint64_t pre_nc = T.pre_nc + T.wnc_ex[warp];
  // req and codes were staged in NC-rank order (compacted), so row r goes to NC block
  // pre_nc + r.  req: one byte per NC block (container.py:15,323)
  if (lane < (int)nnc) a.req[pre_nc + lane] = T.req[warp][lane];
  // codes: NC block r owns bytes [32r, 32r+32) of the pool (earlier NC blocks are full; a
  // short last block is written with its exact byte count -- its padding codes are zero)
  if (lane < (int)(2 * nnc)) {
    const int r = lane >> 1, h = 16 * (lane & 1);
    const uint4 v = *reinterpret_cast<const uint4*>(&T.codes[warp][r][h]);
    uint8_t* dst = a.codes + 32 * (pre_nc + r) + h;
    const uint64_t v_end = ((uint64_t)tile * kFastTileBlocks + warp * kFastBPW) * 128 + 512;
    if (v_end <= n) {
      *reinterpret_cast<uint4*>(dst) = v;
    } else {  // the field's short last block: the last NC row of this warp
      const uint64_t b = (uint64_t)tile * kFastTileBlocks + warp * kFastBPW +
                         __fns(T.wncm[warp], 0, r + 1);
      const uint64_t rem = n - b * 128;
      const int used = rem >= 128 ? 32 : (int)((rem + 3) >> 2);  // code bytes of the block
      const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (h + i < used) dst[i] = (uint8_t)(vw[i >> 2] >> (8 * (i & 3)));
    }
  }
  copy_out_realigned(a.mid, T.pre_mid + T.wmid_ex[warp], T.mid[warp] + 16, T.wmid[warp], lane);
}


// Classify, encode and stage one tile for one compute warp (4 blocks).  FULL: every block
// of the tile holds 128 values (all tiles but possibly the last), so no tail logic at all.
template <bool FULL>
__device__ __forceinline__ void encode_tile(const CompressArgs& a, CompSmem& sm, TileBuf& T,
                                            const float* in, uint32_t tile, int warp, int lane,
                                            uint64_t n, uint64_t nb) {
  const uint64_t b0 = (uint64_t)tile * kFastTileBlocks + (uint64_t)warp * kFastBPW;

  // ---- values to registers ---------------------------------------------------------------
  float4 v[kFastBPW];
#pragma unroll
  for (int j = 0; j < kFastBPW; ++j)
    v[j] = *reinterpret_cast<const float4*>(&in[(warp * kFastBPW + j) * 128 + lane * 4]);

  int cnt[kFastBPW], nv[kFastBPW];
#pragma unroll
  for (int j = 0; j < kFastBPW; ++j) {
    if (FULL) {
      cnt[j] = 128;
      nv[j] = 4;
    } else {
      const uint64_t b = b0 + j;
      cnt[j] = b < nb ? (int)umin64(128, n - (b << 7)) : 0;
      nv[j] = max(0, min(4, cnt[j] - lane * 4));
    }
  }

  // ---- block min / max: reduce-scatter so lanes 8j..8j+7 end up owning block j --------
  float mn[kFastBPW], mx[kFastBPW];
#pragma unroll
  for (int j = 0; j < kFastBPW; ++j) {
    if (FULL) {
      mn[j] = fminf(fminf(v[j].x, v[j].y), fminf(v[j].z, v[j].w));
      mx[j] = fmaxf(fmaxf(v[j].x, v[j].y), fmaxf(v[j].z, v[j].w));
    } else {
      float lo = INFINITY, hi = -INFINITY;
      if (nv[j] > 0) { lo = v[j].x; hi = v[j].x; }
      if (nv[j] > 1) { lo = fminf(lo, v[j].y); hi = fmaxf(hi, v[j].y); }
      if (nv[j] > 2) { lo = fminf(lo, v[j].z); hi = fmaxf(hi, v[j].z); }
      if (nv[j] > 3) { lo = fminf(lo, v[j].w); hi = fmaxf(hi, v[j].w); }
      mn[j] = lo;
      mx[j] = hi;
    }
  }
  const bool h16 = lane & 16, h8 = lane & 8;
  float k0 = h16 ? mn[2] : mn[0], k1 = h16 ? mx[2] : mx[0];
  float k2 = h16 ? mn[3] : mn[1], k3 = h16 ? mx[3] : mx[1];
  {
    const float s0 = h16 ? mn[0] : mn[2], s1 = h16 ? mx[0] : mx[2];
    const float s2 = h16 ? mn[1] : mn[3], s3 = h16 ? mx[1] : mx[3];
    k0 = fminf(k0, __shfl_xor_sync(kFull, s0, 16));
    k1 = fmaxf(k1, __shfl_xor_sync(kFull, s1, 16));
    k2 = fminf(k2, __shfl_xor_sync(kFull, s2, 16));
    k3 = fmaxf(k3, __shfl_xor_sync(kFull, s3, 16));
  }
  float bmn = h8 ? k2 : k0, bmx = h8 ? k3 : k1;
  bmn = fminf(bmn, __shfl_xor_sync(kFull, h8 ? k0 : k2, 8));
  bmx = fmaxf(bmx, __shfl_xor_sync(kFull, h8 ? k1 : k3, 8));
#pragma unroll
  for (int d = 4; d > 0; d >>= 1) {
    bmn = fminf(bmn, __shfl_xor_sync(kFull, bmn, d));
    bmx = fmaxf(bmx, __shfl_xor_sync(kFull, bmx, d));
  }
  // ---- classify once per block (lane group 8j..8j+7 holds block j), then broadcast ----
  const BlockClass mine = classify(bmn, bmx, a.e, a.pe);
  const uint32_t pk = (uint32_t)mine.req | ((uint32_t)mine.s << 6) | ((uint32_t)mine.q << 9) |
                      ((uint32_t)mine.cst << 12);
  float mu[kFastBPW];
  int req[kFastBPW], sft[kFastBPW], q[kFastBPW];
  uint32_t w_cst = 0, w_ncm = 0;
#pragma unroll
  for (int j = 0; j < kFastBPW; ++j) {
    mu[j] = __shfl_sync(kFull, mine.mu, 8 * j);
    const uint32_t p = __shfl_sync(kFull, pk, 8 * j);
    req[j] = p & 63;
    sft[j] = (p >> 6) & 7;
    q[j] = (p >> 9) & 7;
    if (FULL || cnt[j] > 0) {
      if (p >> 12) w_cst |= 1u << j;
      else w_ncm |= 1u << j;
    }
  }
  // container.py:14 -- mu for every block (4 consecutive floats per warp)
  if (lane < kFastBPW && (FULL || cnt[lane] > 0)) {
    const float m = lane == 0 ? mu[0] : lane == 1 ? mu[1] : lane == 2 ? mu[2] : mu[3];
    a.mu[b0 + lane] = m;
  }

  // ---- encode: shifted words, XOR-with-previous leading-byte codes ---------------------
  uint32_t sh[kFastBPW][4];
  uint32_t codeb[kFastBPW], lcnt[kFastBPW];
#pragma unroll
  for (int j = 0; j < kFastBPW; ++j) {
    codeb[j] = 0;
    lcnt[j] = 0;
    sh[j][0] = sh[j][1] = sh[j][2] = sh[j][3] = 0;
    if (!((w_ncm >> j) & 1)) continue;  // warp-uniform
    const int s = sft[j], qq = q[j];
    // pipeline.py:102-106 -- float32 subtraction (RN, no FTZ), byte-aligning shift
    sh[j][0] = __float_as_uint(__fsub_rn(v[j].x, mu[j])) >> s;
    sh[j][1] = __float_as_uint(__fsub_rn(v[j].y, mu[j])) >> s;
    sh[j][2] = __float_as_uint(__fsub_rn(v[j].z, mu[j])) >> s;
    sh[j][3] = __float_as_uint(__fsub_rn(v[j].w, mu[j])) >> s;
    // pipeline.py:108-111 -- previous word, zero at the block start
    uint32_t prev = __shfl_up_sync(kFull, sh[j][3], 1);
    if (lane == 0) prev = 0;
    uint32_t cb = 0, cm = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      // pipeline.py:112 -- code = min(3, leading zero bytes of sh ^ prev, q)
      int c = min(min(3, __clz(sh[j][i] ^ prev) >> 3), qq);
      prev = sh[j][i];
      if (!FULL && i >= nv[j]) {
        c = qq;  // past the tail: no mid bytes, and a zero (padding) code
        cm += 0;
      } else {
        cm += (uint32_t)(qq - c);
        cb |= (uint32_t)c << (2 * i);
      }
    }
    codeb[j] = cb;
    lcnt[j] = cm;
  }
  // ---- mid-byte offsets: two packed (16-bit field) warp scans cover the 4 blocks -------
  const uint32_t pa = lcnt[0] | (lcnt[1] << 16), pb = lcnt[2] | (lcnt[3] << 16);
  const uint32_t ia = warp_incl_scan(pa), ib = warp_incl_scan(pb);
  const uint32_t ta = __shfl_sync(kFull, ia, 31), tb_ = __shfl_sync(kFull, ib, 31);
  const uint32_t ea = ia - pa, eb = ib - pb;
  const uint32_t btot[kFastBPW] = {ta & 0xFFFF, ta >> 16, tb_ & 0xFFFF, tb_ >> 16};
  const uint32_t loff[kFastBPW] = {ea & 0xFFFF, ea >> 16, eb & 0xFFFF, eb >> 16};

  // ---- stage: codes, req, mid bytes (warp-private region, warp-local offsets) ------------
  uint8_t* my_mid = T.mid[warp] + 16;  // 16 bytes of slack before (copy_out_realigned)
  uint32_t bpos = 0;
  int rank = 0;  // codes and req are staged in NC-rank order
#pragma unroll
  for (int j = 0; j < kFastBPW; ++j) {
    if (!((w_ncm >> j) & 1)) continue;
    T.codes[warp][rank][lane] = (uint8_t)codeb[j];
    if (lane == 0) T.req[warp][rank] = (uint8_t)req[j];
    ++rank;
    uint8_t* d = my_mid + bpos + loff[j];
    // dead (past-the-tail) elements stage nothing: treat them as fully reused
    int cc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      cc[i] = (!FULL && i >= nv[j]) ? q[j] : (int)((codeb[j] >> (2 * i)) & 3);
    switch (q[j]) {  // warp-uniform, hoisted out of the element loop
      case 2:
#pragma unroll
        for (int i = 0; i < 4; ++i) { stage_bytes<2>(d - cc[i], sh[j][i], cc[i]); d += 2 - cc[i]; }
        break;
      case 3:
#pragma unroll
        for (int i = 0; i < 4; ++i) { stage_bytes<3>(d - cc[i], sh[j][i], cc[i]); d += 3 - cc[i]; }
        break;
      case 4:
#pragma unroll
        for (int i = 0; i < 4; ++i) { stage_bytes<4>(d - cc[i], sh[j][i], cc[i]); d += 4 - cc[i]; }
        break;
      default: {  // q == 1 (never produced for req >= 9, kept for completeness)
        const int qq = q[j];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int c = cc[i] > qq ? qq : cc[i];
          stage_bytes<1>(d - c, sh[j][i], c);
          d += qq - c;
        }
        break;
      }
    }
    bpos += btot[j];
    if (lane == 0) {
      if (req[j] < 1) atomicOr(a.err, kErrBadReq);  // container.py:206-207
      if (!FULL && b0 + j == nb - 1 && cnt[j] < 128) sm.madj = 128 - cnt[j];
    }
  }
  if (lane == 0) {
    T.wnc[warp] = __popc(w_ncm);
    T.wmid[warp] = bpos;
    T.wcst[warp] = w_cst;
    T.wncm[warp] = w_ncm;
    // the last compute warp to finish publishes the tile aggregate at once, so no tile's
    // aggregate ever waits behind this CTA's previous look-back
    // shared accumulator: [63:56] warps arrived, [55:32] NC blocks, [31:0] mid bytes
    const unsigned long long mine = (1ull << 56) | ((unsigned long long)__popc(w_ncm) << 32) | bpos;
    const unsigned long long prior = atomicAdd(&T.agg, mine);
    if ((prior >> 56) == kCompWarps - 1) {
      const unsigned long long tot = prior + mine;
      st_relaxed(a.status + tile, kFlagAgg | pack2((tot >> 32) & 0xFFFFFF, tot & 0xFFFFFFFFu));
      T.agg = 0;  // this parity buffer is next used two tiles later
    }
  }
}

}  // namespace

__global__ void __launch_bounds__(kCThreads, 2) compress128_kernel(CompressArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  CompSmem& sm = *reinterpret_cast<CompSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t n = a.n;
  const uint64_t nb = (n + 127) >> 7;
  const uint32_t G = gridDim.x;

  if (tid == 0) {
    for (int s = 0; s < kInStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kCompWarps);
    }
    sm.madj = 0;
    for (int b = 0; b < kTileBufs; ++b) sm.tb[b].agg = 0;
    fence_barrier_init();
  }
  __syncthreads();

  // ---------------------------------------------------------------- producer warp
  // Tiles are claimed dynamically in order; a claimed tile waits at most kInStages-1 tiles
  // in the ring, which the deferred write-out absorbs.
  if (warp == kProdWarp) {
    if (lane == 0) {
      unsigned long long c_prod = 0;
      for (uint32_t k = 0;; ++k) {
        const int s = k % kInStages;
        const long long tw = clock64();
        mbar_wait_sleep(&sm.empty[s], ((k / kInStages) & 1) ^ 1);
        c_prod += clock64() - tw;
        uint32_t tile = atomicAdd(a.counter, 1u);  // dynamic: slow CTAs simply claim fewer
        if (tile >= a.ntiles) tile = ~0u;
        sm.tile[s] = tile;
        if (tile == ~0u) {
          mbar_arrive(&sm.full[s]);
          atomicAdd(&g_compress_stats[6], c_prod);
          break;
        }
        const uint64_t v0 = (uint64_t)tile * kTileVals;
        const uint32_t vals = (uint32_t)umin64(kTileVals, n - v0);
        const uint32_t bulk = (vals * 4) & ~15u;
        for (uint32_t i = bulk / 4; i < vals; ++i) sm.in[s][i] = a.x[v0 + i];  // <= 3 values
        mbar_arrive_expect_tx(&sm.full[s], bulk);
        if (bulk) bulk_g2s(sm.in[s], a.x + v0, bulk, &sm.full[s]);
      }
    }
    return;
  }

  // ---------------------------------------------------------------- scan warps
  // Decoupled look-back (lookback_wide: 256-tile coalesced windows).  Two scan warps take
  // alternate tiles, and the compute warps only need a tile's prefix kDefer tiles later,
  // so both the latency and the throughput of the look-back are hidden.
  if (warp >= kScanWarp) {
    unsigned long long st_lookback = 0;
    for (uint32_t k = warp - kScanWarp;; k += kScanWarps) {
      const uint32_t buf = k % kTileBufs;
      TileBuf& T = sm.tb[buf];
      bar_sync(bar_counts(buf));
      const uint32_t tile = T.cur_tile;  // handed over with the counts
      if (tile == ~0u) break;
      const uint32_t wn = lane < kCompWarps ? T.wnc[lane] : 0;
      const uint32_t wm = lane < kCompWarps ? T.wmid[lane] : 0;
      const uint32_t in_n = warp_incl_scan(wn), in_m = warp_incl_scan(wm);
      if (lane < kCompWarps) {
        T.wnc_ex[lane] = in_n - wn;
        T.wmid_ex[lane] = in_m - wm;
      }
      const uint32_t t_nc = __shfl_sync(kFull, in_n, 31), t_mid = __shfl_sync(kFull, in_m, 31);
      const uint64_t agg = pack2(t_nc, t_mid);
      const long long tl0 = clock64();
      const uint64_t ex = lookback_wide<8>(a.status, tile, agg, /*published=*/true);
      st_lookback += clock64() - tl0;
      const uint64_t run = ex + agg;  // inclusive
      if (lane == 0) {
        const uint64_t bnc = a.base ? a.base->n_nc : 0, bm = a.base ? a.base->m : 0;
        const uint64_t bmid = a.base ? a.base->mid_len : 0;
        T.pre_nc = bnc + hi_of(ex);
        T.pre_mid = bmid + lo_of(ex);
        if (tile == a.ntiles - 1) {  // chunk totals for the host / the next chunk
          const uint64_t cnc = hi_of(run);
          a.totals->n_nc = bnc + cnc;
          a.totals->m = bm + 128 * cnc - sm.madj;
          a.totals->mid_len = bmid + lo_of(run);
          a.totals->pad = 0;
        }
        // constant map: 32 bits = 4 bytes per tile, LSB-first (container.py:12-13,321)
        uint32_t bits = 0;
#pragma unroll
        for (int w = 0; w < kCompWarps; ++w) bits |= T.wcst[w] << (kFastBPW * w);
        const uint64_t tb = (uint64_t)tile * kFastTileBlocks;
        if (tb + kFastTileBlocks <= nb) {
          *reinterpret_cast<uint32_t*>(a.map + 4 * (uint64_t)tile) = bits;
        } else {
          const uint32_t nbytes = (uint32_t)((nb - tb + 7) >> 3);
          for (uint32_t i = 0; i < nbytes; ++i) a.map[4 * (uint64_t)tile + i] = (uint8_t)(bits >> (8 * i));
        }
      }
      __syncwarp();
      __threadfence_block();
      bar_arrive(bar_prefix(buf));
    }
    if (lane == 0) atomicAdd(&g_compress_stats[0], st_lookback);
    return;
  }

  // ---------------------------------------------------------------- compute warps
  unsigned long long c_in = 0, c_enc = 0, c_wait = 0, c_wo = 0, c_tiles = 0;
  auto flush = [&](uint32_t j) {  // write out tile j (its prefix is published)
    const uint32_t b = j % kTileBufs;
    bar_sync(bar_prefix(b));
    write_out(a, sm.tb[b], sm.tb[b].cur_tile, warp, lane, n);
    __syncwarp();
  };
  for (uint32_t k = 0;; ++k) {
    const int st = k % kInStages;
    const uint32_t buf = k % kTileBufs;
    TileBuf& T = sm.tb[buf];
    long long t0 = clock64();
    mbar_wait(&sm.full[st], (k / kInStages) & 1);
    long long t1 = clock64();
    c_in += t1 - t0;
    const uint32_t tile = sm.tile[st];
    if (tile == ~0u) {
      // release the scan warp that owns tile k, flush the staged tiles, then release the
      // other scan warp (its barrier instance for tile k+1 is free only after the flush)
      if (warp == 0 && lane == 0) T.cur_tile = ~0u;
      __syncwarp();
      __threadfence_block();
      bar_arrive(bar_counts(buf));
      for (uint32_t j = k >= kDefer ? k - kDefer : 0; j < k; ++j) flush(j);
      TileBuf& T1 = sm.tb[(k + 1) % kTileBufs];
      if (warp == 0 && lane == 0) T1.cur_tile = ~0u;
      __syncwarp();
      __threadfence_block();
      bar_arrive(bar_counts((k + 1) % kTileBufs));
      break;
    }
    if (warp == 0 && lane == 0) T.cur_tile = tile;
    const bool full = ((uint64_t)tile + 1) * kTileVals <= n;
    if (full) encode_tile<true>(a, sm, T, sm.in[st], tile, warp, lane, n, nb);
    else encode_tile<false>(a, sm, T, sm.in[st], tile, warp, lane, n, nb);
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[st]);  // input slot free
    __threadfence_block();
    bar_arrive(bar_counts(buf));
    t0 = clock64();
    c_enc += t0 - t1;
    ++c_tiles;

    // ---- tile k-kDefer's prefix is known by now: write it out ----------------------------
    if (k >= kDefer) {
      flush(k - kDefer);
      c_wo += clock64() - t0;
    }
  }
  if (warp == 0 && lane == 0) {
    atomicAdd(&g_compress_stats[2], c_wait);
    atomicAdd(&g_compress_stats[3], c_tiles);
    atomicAdd(&g_compress_stats[4], c_enc);
    atomicAdd(&g_compress_stats[5], c_wo);
    atomicAdd(&g_compress_stats[7], c_in);
  }
}

cudaError_t compress_stats(unsigned long long* out8, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out8, g_compress_stats, 8 * sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    e = cudaMemcpyToSymbol(g_compress_stats, z, sizeof z);
  }
  return e;
}

void launch_compress128(const CompressArgs& a, cudaStream_t s) {
  static bool configured = false;
  static int per_sm = 1;
  if (!configured) {
    cudaFuncSetAttribute(compress128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(CompSmem));
    // the round-synchronous prefix needs every CTA of the grid co-resident
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, compress128_kernel, kCThreads,
                                                  sizeof(CompSmem));
    if (per_sm < 1) per_sm = 1;
    configured = true;
  }
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  const uint32_t cap = (uint32_t)(per_sm * nsm);
  const uint32_t grid = a.ntiles < cap ? a.ntiles : cap;
  compress128_kernel<<<grid, kCThreads, sizeof(CompSmem), s>>>(a);
}

}  // namespace szx
