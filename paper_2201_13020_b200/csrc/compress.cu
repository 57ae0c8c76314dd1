// compress.cu -- SZx block encoder for sm_100a, bs == 128 fast path (K1 in DESIGN.md).
//
// Replaces the reference's whole compress path in ONE launch per chunk:
//   block_stats           pipeline.py:54-81   (== blockcodec.summarize_block 87-112)
//   _encode_elements      pipeline.py:94-133  (== blockcodec.encode_nonconstant 123-141)
//   prefix_scan + scatter parallel.py:21-44,104-140 / pipeline.py:143-166
// Output pools use the UFZX container layout (container.py:3-21).
//
// Persistent, warp-specialised CTAs (2 per SM):
//   warp 8 (producer): claims tiles in order and streams each tile's 16 KiB of input into
//          a 3-deep shared-memory ring with 1-D bulk copies (TMA engine, mbarrier tx count);
//   warps 0-7 (compute): one warp = 4 blocks = 4 x 128 values, lane l owns values 4l..4l+3;
//          classify, encode, publish per-warp counts, stage mid bytes in a private
//          shared-memory region, then write the pools once the tile's offsets are known;
//   warp 9 (scan): decoupled look-back over the packed (NC blocks, mid bytes) tile counts,
//          overlapped with the compute warps' mid-byte staging.
// A tile's input slot is released as soon as its values are in registers, so the next
// tiles' loads are always in flight while a tile waits for its prefix.
#include "szx_device.cuh"
#include "szx_kernels.h"

namespace szx {

namespace {

constexpr int kCompWarps = 8;
constexpr int kProdWarp = 8;
constexpr int kScanWarp = 9;
constexpr int kCThreads = 320;
constexpr int kInStages = 3;
constexpr int kTileVals = kFastTileBlocks * 128;  // 4096
constexpr int kWarpMidBytes = kFastBPW * 512;      // worst case per compute warp
constexpr int kWarpMidStride = kWarpMidBytes + 32; // room for the realignment window

struct CompSmem {
  float in[kInStages][kTileVals];
  uint8_t mid[kCompWarps][kWarpMidStride];
  uint64_t full[kInStages];
  uint64_t empty[kInStages];
  uint32_t tile[kInStages];
  uint32_t wnc[kCompWarps], wmid[kCompWarps], wcst[kCompWarps];
  uint32_t wnc_ex[kCompWarps], wmid_ex[kCompWarps];
  uint32_t madj;
  unsigned long long pre_nc, pre_mid;
};

// Copy `len` staged bytes (16-byte aligned shared source) to global byte offset `pos` of
// `dst` (16-byte aligned base), one 16-byte aligned global chunk per lane-iteration: the
// source window is re-aligned with funnel shifts (the shift is warp-uniform).
__device__ __forceinline__ void copy_out_realigned(uint8_t* dst, uint64_t pos,
                                                   const uint8_t* src, uint32_t len, int lane) {
  if (len == 0) return;
  const uint32_t a = (uint32_t)(pos & 15);
  uint8_t* g = dst + (pos - a);
  const uint32_t nchunk = (a + len + 15) >> 4;
  const uint32_t d = (16 - a) & 15;  // source offset of every full chunk, mod 16
  const uint32_t k = d >> 2, b = 8 * (d & 3);
  const uint4* s128 = reinterpret_cast<const uint4*>(src);
  for (uint32_t c = lane; c < nchunk; c += 32) {
    const int64_t lo = 16 * (int64_t)c - a;
    if (lo >= 0 && lo + 16 <= (int64_t)len) {
      const uint32_t j = (uint32_t)lo >> 4;
      const uint4 q0 = s128[j], q1 = s128[j + 1];
      uint32_t w[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
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
      *reinterpret_cast<uint4*>(g + 16 * (uint64_t)c) = o;
    } else {  // partial chunk shared with a neighbour: byte stores on our bytes only
      const int64_t i0 = lo < 0 ? 0 : lo, i1 = lo + 16 < (int64_t)len ? lo + 16 : len;
      for (int64_t i = i0; i < i1; ++i) g[16 * (uint64_t)c + (i - lo)] = src[i];
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

  if (tid == 0) {
    for (int s = 0; s < kInStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kCompWarps);
    }
    sm.madj = 0;
    fence_barrier_init();
  }
  __syncthreads();

  // ---------------------------------------------------------------- producer warp
  if (warp == kProdWarp) {
    if (lane == 0) {
      for (uint32_t k = 0;; ++k) {
        const int s = k % kInStages;
        const uint32_t ph = (k / kInStages) & 1;
        mbar_wait(&sm.empty[s], ph ^ 1);
        const uint32_t tile = atomicAdd(a.counter, 1u);
        sm.tile[s] = tile;
        if (tile >= a.ntiles) {
          mbar_arrive(&sm.full[s]);
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

  // ---------------------------------------------------------------- scan warp
  if (warp == kScanWarp) {
    for (uint32_t k = 0;; ++k) {
      const int s = k % kInStages;
      mbar_wait(&sm.full[s], (k / kInStages) & 1);
      const uint32_t tile = sm.tile[s];
      if (tile >= a.ntiles) break;
      named_bar(1, (kCompWarps + 1) * 32);  // per-warp counts are in shared memory
      const uint32_t wn = lane < kCompWarps ? sm.wnc[lane] : 0;
      const uint32_t wm = lane < kCompWarps ? sm.wmid[lane] : 0;
      const uint32_t in_n = warp_incl_scan(wn), in_m = warp_incl_scan(wm);
      if (lane < kCompWarps) {
        sm.wnc_ex[lane] = in_n - wn;
        sm.wmid_ex[lane] = in_m - wm;
      }
      const uint32_t t_nc = __shfl_sync(kFull, in_n, 31), t_mid = __shfl_sync(kFull, in_m, 31);
      const uint64_t ex = lookback(a.status, tile, pack2(t_nc, t_mid));
      if (lane == 0) {
        const uint64_t bnc = a.base ? a.base->n_nc : 0, bm = a.base ? a.base->m : 0;
        const uint64_t bmid = a.base ? a.base->mid_len : 0;
        sm.pre_nc = bnc + hi_of(ex);
        sm.pre_mid = bmid + lo_of(ex);
        if (tile == a.ntiles - 1) {  // chunk totals for the host / the next chunk
          const uint64_t cnc = hi_of(ex) + t_nc;
          a.totals->n_nc = bnc + cnc;
          a.totals->m = bm + 128 * cnc - sm.madj;
          a.totals->mid_len = bmid + lo_of(ex) + t_mid;
          a.totals->pad = 0;
        }
        // constant map: 32 bits = 4 bytes per tile, LSB-first (container.py:12-13,321)
        uint32_t bits = 0;
#pragma unroll
        for (int w = 0; w < kCompWarps; ++w) bits |= sm.wcst[w] << (kFastBPW * w);
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
      named_bar(2, (kCompWarps + 1) * 32);  // prefix published to the compute warps
    }
    return;
  }

  // ---------------------------------------------------------------- compute warps
  uint8_t* my_mid = sm.mid[warp];
  for (uint32_t k = 0;; ++k) {
    const int st = k % kInStages;
    mbar_wait(&sm.full[st], (k / kInStages) & 1);
    const uint32_t tile = sm.tile[st];
    if (tile >= a.ntiles) break;
    const uint64_t b0 = (uint64_t)tile * kFastTileBlocks + (uint64_t)warp * kFastBPW;

    // ---- values to registers; release the input slot at once ------------------------------
    float4 v[kFastBPW];
#pragma unroll
    for (int j = 0; j < kFastBPW; ++j)
      v[j] = *reinterpret_cast<const float4*>(&sm.in[st][(warp * kFastBPW + j) * 128 + lane * 4]);
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[st]);

    // ---- classify (warp-uniform results) -----------------------------------------------------
    int cnt[kFastBPW];
    BlockClass bc[kFastBPW];
#pragma unroll
    for (int j = 0; j < kFastBPW; ++j) {
      const uint64_t b = b0 + j;
      cnt[j] = b < nb ? (int)umin64(128, n - (b << 7)) : 0;
      const int nv = max(0, min(4, cnt[j] - lane * 4));
      float mn = INFINITY, mx = -INFINITY;
      if (nv > 0) { mn = fminf(mn, v[j].x); mx = fmaxf(mx, v[j].x); }
      if (nv > 1) { mn = fminf(mn, v[j].y); mx = fmaxf(mx, v[j].y); }
      if (nv > 2) { mn = fminf(mn, v[j].z); mx = fmaxf(mx, v[j].z); }
      if (nv > 3) { mn = fminf(mn, v[j].w); mx = fmaxf(mx, v[j].w); }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(kFull, mn, d));
        mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, d));
      }
      bc[j] = classify(mn, mx, a.e, a.pe);
    }

    // ---- encode: shifted words, XOR-with-previous leading-byte codes ---------------------
    uint32_t sh[kFastBPW][4];
    uint32_t codeb[kFastBPW], loff[kFastBPW], btot[kFastBPW];
    uint32_t w_nc = 0, w_mid = 0, w_cst = 0;
#pragma unroll
    for (int j = 0; j < kFastBPW; ++j) {
      codeb[j] = 0; loff[j] = 0; btot[j] = 0;
      sh[j][0] = sh[j][1] = sh[j][2] = sh[j][3] = 0;
      if (cnt[j] == 0) continue;
      if (bc[j].cst) { w_cst |= 1u << j; continue; }
      const int s = bc[j].s, q = bc[j].q;
      const float mu = bc[j].mu;
      // pipeline.py:102-106 -- float32 subtraction (RN, no FTZ), byte-aligning shift
      sh[j][0] = __float_as_uint(__fsub_rn(v[j].x, mu)) >> s;
      sh[j][1] = __float_as_uint(__fsub_rn(v[j].y, mu)) >> s;
      sh[j][2] = __float_as_uint(__fsub_rn(v[j].z, mu)) >> s;
      sh[j][3] = __float_as_uint(__fsub_rn(v[j].w, mu)) >> s;
      // pipeline.py:108-111 -- previous word, zero at the block start
      uint32_t prev = __shfl_up_sync(kFull, sh[j][3], 1);
      if (lane == 0) prev = 0;
      const int nv = max(0, min(4, cnt[j] - lane * 4));
      uint32_t cb = 0, cntm = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        // pipeline.py:112 -- code = min(3, leading zero bytes of sh ^ prev, q)
        int c = min(min(3, __clz(sh[j][i] ^ prev) >> 3), q);
        prev = sh[j][i];
        if (i >= nv) c = q;  // past the tail: no code bits, no mid bytes
        cntm += (uint32_t)(q - c);
        cb |= (uint32_t)(i < nv ? c : 0) << (2 * i);
      }
      codeb[j] = cb;
      const uint32_t incl = warp_incl_scan(cntm);
      loff[j] = incl - cntm;
      btot[j] = __shfl_sync(kFull, incl, 31);
      w_nc += 1;
      w_mid += btot[j];
      if (lane == 0) {
        if (bc[j].req < 1) atomicOr(a.err, kErrBadReq);
        if (b0 + j == nb - 1 && cnt[j] < 128) sm.madj = 128 - cnt[j];
      }
    }
    if (lane == 0) {
      sm.wnc[warp] = w_nc;
      sm.wmid[warp] = w_mid;
      sm.wcst[warp] = w_cst;
    }
    __syncwarp();
    __threadfence_block();
    asm volatile("bar.arrive 1, %0;" ::"r"((kCompWarps + 1) * 32) : "memory");

    // ---- while the scan warp looks back: mu, and mid bytes staged at warp-local offsets ---
#pragma unroll
    for (int j = 0; j < kFastBPW; ++j)
      if (lane == j && cnt[j] > 0) a.mu[b0 + j] = bc[j].mu;  // container.py:14
    uint32_t bpos = 0;
#pragma unroll
    for (int j = 0; j < kFastBPW; ++j) {
      if (cnt[j] == 0 || bc[j].cst) continue;
      const int q = bc[j].q;
      uint32_t p = bpos + loff[j];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int c = (codeb[j] >> (2 * i)) & 3;
        const bool live = lane * 4 + i < cnt[j];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          if (live && kk >= c && kk < q) my_mid[p++] = (uint8_t)(sh[j][i] >> (24 - 8 * kk));
      }
      bpos += btot[j];
    }
    __syncwarp();

    named_bar(2, (kCompWarps + 1) * 32);  // tile prefix is known
    const uint64_t pre_mid = sm.pre_mid + sm.wmid_ex[warp];
    uint64_t r = sm.pre_nc + sm.wnc_ex[warp];
#pragma unroll
    for (int j = 0; j < kFastBPW; ++j) {
      if (cnt[j] == 0 || bc[j].cst) continue;
      if (lane == 0) a.req[r] = (uint8_t)bc[j].req;
      // NC block r owns code bytes [32r, 32r + ceil(cnt/4)) (earlier NC blocks are full)
      if (lane * 4 < cnt[j]) a.codes[32 * r + lane] = (uint8_t)codeb[j];
      ++r;
    }
    copy_out_realigned(a.mid, pre_mid, my_mid, w_mid, lane);
    __syncwarp();  // staging region is reused by the next tile
  }
}

void launch_compress128(const CompressArgs& a, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(compress128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(CompSmem));
    configured = true;
  }
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  const uint32_t grid = a.ntiles < (uint32_t)(2 * nsm) ? a.ntiles : (uint32_t)(2 * nsm);
  compress128_kernel<<<grid, kCThreads, sizeof(CompSmem), s>>>(a);
}

}  // namespace szx
