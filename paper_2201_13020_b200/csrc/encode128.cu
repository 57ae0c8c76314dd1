// encode128.cu -- SZx block encoder for sm_100a, bs == 128 (K1 in DESIGN.md).
//
// Replaces the reference's whole compress path in ONE launch per chunk:
//   block_stats           pipeline.py:54-81   (== blockcodec.summarize_block 87-112)
//   _encode_elements      pipeline.py:94-133  (== blockcodec.encode_nonconstant 123-141)
//   prefix_scan + scatter parallel.py:21-44,104-140 / pipeline.py:143-166
// Output pools use the UFZX container layout (container.py:3-21).
//
// Warp-autonomous design: every warp of a persistent grid runs the whole pipeline for its
// own tiles of 8 blocks (1024 values, 4 KiB) with no intra-CTA coordination at all:
//   claim  -- a tile id from the chunk's counter (one tile ahead), and a 4 KiB bulk copy
//             (TMA engine) of its values into one of the warp's two shared-memory buffers;
//   encode -- lane l owns values 4l..4l+3 of each block (one block = one warp row, so every
//             per-block quantity is warp-uniform): CREDUX min/max, the fp64 classification
//             computed once per block (lane j classifies block j & 3 of the half-tile, then
//             broadcast), the XOR-with-previous chain (one shuffle per block), codes and kept
//             bytes; the kept bytes are staged IN PLACE over the tile's input bytes (a half
//             tile's output never exceeds its input), lanes 4 bytes apart on average so the
//             byte stores are bank-conflict free;
//   scan   -- decoupled look-back over (NC blocks, mid bytes) per tile, bounded below by the
//             warp's previous tile;
//   write  -- mid bytes as realigned 16-byte chunks (bytewise only at the two partial edge
//             chunks), code rows, req bytes, mu, one constant-map byte per tile.
// Latency (look-back, loads) is hidden by the other warps of the SM instead of by role
// hand-offs.
#include "szx_device.cuh"
#include "szx_kernels.h"

namespace szx {

namespace {

#ifndef SZX_K1V2_WARPS
#define SZX_K1V2_WARPS 24
#endif
constexpr int kEW = SZX_K1V2_WARPS;       // warps per CTA (one CTA per SM)
constexpr int kTB = 8;                    // blocks per warp tile (one constant-map byte)
constexpr int kTV = kTB * 128;            // values per tile
constexpr int kTileBytes = kTV * 4;       // 4 KiB

struct __align__(16) WarpBuf {
  uint8_t pre[16];                        // realignment over-read slack before the staging
  float v[kTV];                           // the tile's values, then its staged mid bytes
  uint8_t post[48];                       // over-read slack after it
};
struct __align__(16) WarpSide {
  uint8_t codes[kTB * 32];                // code rows of the tile's NC blocks, NC-rank order
  uint8_t req[16];                        // req bytes, NC-rank order
};
struct EncSmem {
  WarpBuf buf[kEW][2];
  WarpSide side[kEW];
  uint64_t full[kEW][2];
};

__device__ __forceinline__ uint32_t shr_clamp(uint32_t x, uint32_t s) {  // 0 for s >= 32
  uint32_t r;
  asm("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
  return r;
}
__device__ __forceinline__ int flo32(uint32_t x) {  // index of the highest set bit, -1 for 0
  int r;
  asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}
__device__ __forceinline__ float redux_min(float v) {
  float r;
  asm volatile("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float redux_max(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}
// Stage byte (v & 0xFF) at shared address a + OFF iff f >= LIM (the element keeps more than
// LIM / 8 bytes).  [reg+imm] addressing: no address arithmetic per byte.
template <int LIM, int OFF>
__device__ __forceinline__ void sts_u8_if(uint32_t a, uint32_t v, int f) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ge.s32 p, %2, %3;\n @p st.shared.u8 [%0+%4], %1;\n}\n" ::"r"(a),
      "r"(v), "r"(f), "n"(LIM), "n"(OFF)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Stage the kept bytes of a lane's 4 elements of one block (Q = the block's q, uniform).
// Element i keeps n_i = (f_i >> 3) + 1 bytes (0 when f_i < 0), big-endian (pipeline.py:
// 114-116,151); with u accumulating sum_{j<=i} (f_j >> 3), element i's last byte lands at
// base + u + i, and its kept byte c (counted from the last) at base + u + i - c.
template <int Q>
__device__ __forceinline__ void stage4(uint32_t base, const uint32_t (&t)[4], const int (&f)[4]) {
  uint32_t u = base - 3;  // immediate offsets i - c + 3 >= 0
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    u += (uint32_t)(f[i] >> 3);
    switch (i) {  // compile-time
      case 0:
        sts_u8_if<0, 3>(u, t[0], f[0]);
        if (Q >= 2) sts_u8_if<8, 2>(u, t[0] >> 8, f[0]);
        if (Q >= 3) sts_u8_if<16, 1>(u, t[0] >> 16, f[0]);
        if (Q >= 4) sts_u8_if<24, 0>(u, t[0] >> 24, f[0]);
        break;
      case 1:
        sts_u8_if<0, 4>(u, t[1], f[1]);
        if (Q >= 2) sts_u8_if<8, 3>(u, t[1] >> 8, f[1]);
        if (Q >= 3) sts_u8_if<16, 2>(u, t[1] >> 16, f[1]);
        if (Q >= 4) sts_u8_if<24, 1>(u, t[1] >> 24, f[1]);
        break;
      case 2:
        sts_u8_if<0, 5>(u, t[2], f[2]);
        if (Q >= 2) sts_u8_if<8, 4>(u, t[2] >> 8, f[2]);
        if (Q >= 3) sts_u8_if<16, 3>(u, t[2] >> 16, f[2]);
        if (Q >= 4) sts_u8_if<24, 2>(u, t[2] >> 24, f[2]);
        break;
      default:
        sts_u8_if<0, 6>(u, t[3], f[3]);
        if (Q >= 2) sts_u8_if<8, 5>(u, t[3] >> 8, f[3]);
        if (Q >= 3) sts_u8_if<16, 4>(u, t[3] >> 16, f[3]);
        if (Q >= 4) sts_u8_if<24, 3>(u, t[3] >> 24, f[3]);
        break;
    }
  }
}

// Interior chunks [c0, c1) of copy_out with a uniform word offset K and bit shift b.
template <int K>
__device__ __forceinline__ void copy_chunks(uint8_t* g, const uint4* s128, uint32_t a, uint32_t b,
                                            uint32_t c0, uint32_t c1, int lane) {
#pragma unroll 2
  for (uint32_t c = c0 + lane; c < c1; c += 32) {
    // staged window of chunk c starts at byte 16c - a; rows j-1, j relative to src
    const int j = (int)((16 * c - a + 16) >> 4);
    const uint4 q0 = s128[j - 1], q1 = s128[j];
    const uint32_t w[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
    *reinterpret_cast<uint4*>(g + 16 * c) =
        make_uint4(__funnelshift_r(w[K], w[K + 1], b), __funnelshift_r(w[K + 1], w[K + 2], b),
                   __funnelshift_r(w[K + 2], w[K + 3], b), __funnelshift_r(w[K + 3], w[K + 4], b));
  }
}

// Copy `len` staged bytes (shared, 16-byte aligned, 16 bytes of readable slack on both sides)
// to byte offset `pos` of `dst` (16-byte aligned base), one warp.  Interior 16-byte chunks
// are realigned with funnel shifts (the shift is uniform); the two partial edge chunks are
// written bytewise (16 lanes each) -- the neighbouring tiles own their other bytes.
__device__ __forceinline__ void copy_out(uint8_t* dst, uint64_t pos, const uint8_t* src,
                                         uint32_t len, int lane) {
  if (len == 0) return;
  const uint32_t a = (uint32_t)(pos & 15);
  uint8_t* g = dst + (pos - a);
  const uint32_t nchunk = (a + len + 15) >> 4;
  const bool head_partial = a != 0;
  const bool tail_partial = ((a + len) & 15) != 0;
  const uint32_t d = (16 - a) & 15;
  const uint32_t b = 8 * (d & 3);
  const uint4* s128 = reinterpret_cast<const uint4*>(src);
  const uint32_t c0 = head_partial ? 1 : 0;
  const uint32_t c1 = tail_partial ? nchunk - 1 : nchunk;
  switch (d >> 2) {  // uniform
    case 0: copy_chunks<0>(g, s128, a, b, c0, c1, lane); break;
    case 1: copy_chunks<1>(g, s128, a, b, c0, c1, lane); break;
    case 2: copy_chunks<2>(g, s128, a, b, c0, c1, lane); break;
    default: copy_chunks<3>(g, s128, a, b, c0, c1, lane); break;
  }
  const bool head = lane < 16;
  const uint32_t c = head ? 0 : nchunk - 1;
  const bool part = head ? head_partial : tail_partial;
  const int x = 16 * (int)c + (lane & 15) - (int)a;  // staged index of this byte
  if (part && x >= 0 && x < (int)len) g[16 * c + (lane & 15)] = src[x];
}

// Classification of one block (pipeline.py:54-81), packed for the broadcast:
// info = shift (6 bits) | q << 8 | K << 12 | nc << 13 | req << 16.
__device__ __forceinline__ void classify_pack(float mn, float mx, double e, int pe, float& mu,
                                              uint32_t& info) {
  const BlockClass c = classify(mn, mx, e, pe);
  mu = c.mu;
  const uint32_t nc = !c.cst;
  // constant blocks: shift 32 makes every t zero, so they stage nothing (L = 0)
  const uint32_t shift = nc ? (uint32_t)(c.s + 32 - 8 * c.q) : 32u;
  const uint32_t K = (nc && c.q == 4) ? 1u : 0u;
  info = shift | ((uint32_t)c.q << 8) | (K << 12) | (nc << 13) | ((uint32_t)c.req << 16);
}

}  // namespace

__global__ void __launch_bounds__(kEW * 32, 1) encode128_kernel(CompressArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  EncSmem& sm = *reinterpret_cast<EncSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpBuf* B = sm.buf[warp];
  WarpSide& SD = sm.side[warp];
  uint64_t* full = sm.full[warp];
  const uint64_t n = a.n;
  const uint64_t nb = (n + 127) >> 7;
  const uint64_t bnc = a.base ? a.base->n_nc : 0, bm = a.base ? a.base->m : 0;
  const uint64_t bmid = a.base ? a.base->mid_len : 0;

  if (lane == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_barrier_init();
  }
  __syncwarp();

  // claim a tile and start its input copy into buffer b (lane 0); every lane gets the id
  auto claim = [&](int b) -> uint32_t {
    uint32_t t = 0;
    if (lane == 0) {
      t = atomicAdd(a.counter, 1u);
      if (t < a.ntiles) {
        const uint64_t v0 = (uint64_t)t * kTV;
        if (v0 + kTV <= n) {
          fence_proxy_async_smem();  // the buffer's generic reads/writes before the copy
          mbar_arrive_expect_tx(&full[b], kTileBytes);
          bulk_g2s(B[b].v, a.x + v0, kTileBytes, &full[b]);
        } else {
          mbar_arrive(&full[b]);  // partial tile: the lanes read global memory
        }
      }
    }
    return __shfl_sync(kFull, t, 0);
  };

  uint32_t t0 = claim(0), t1 = claim(1);  // the tiles in buffers 0 and 1
  int64_t floor = -1;       // this warp's previous tile and its inclusive prefix: the
  uint64_t floor_incl = 0;  // look-back never scans past it
  const double e = a.e;
  const int pe = a.pe;

  for (uint32_t k = 0;; ++k) {
    const int b = k & 1;
    const uint32_t tile = b ? t1 : t0;
    if (tile >= a.ntiles) break;  // claims grow monotonically: the other buffer is later
    mbar_wait(&full[b], (k >> 1) & 1);
    const uint64_t v0 = (uint64_t)tile * kTV;
    const bool full_tile = v0 + kTV <= n;
    const uint64_t tb = (uint64_t)tile * kTB;
    const int nbt = (int)umin64(kTB, nb - tb);  // blocks of this tile
    const uint32_t stage = smem_u32(B[b].v);
    uint32_t mid_off = 0, nc_cnt = 0, cmap = 0;

#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      // ---- values: lane l holds values 4l..4l+3 of blocks 4h..4h+3 of the tile
      float v[4][4];
      int nlive[4];
      if (full_tile) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 x = reinterpret_cast<const float4*>(B[b].v)[(4 * h + j) * 32 + lane];
          v[j][0] = x.x; v[j][1] = x.y; v[j][2] = x.z; v[j][3] = x.w;
          nlive[j] = 4;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t first = v0 + (uint64_t)(4 * h + j) * 128 + 4 * lane;
          nlive[j] = first >= n ? 0 : (int)umin64(4, n - first);
#pragma unroll
          for (int i = 0; i < 4; ++i) v[j][i] = i < nlive[j] ? a.x[first + i] : 0.f;
        }
      }
      __syncwarp();  // every lane holds its values before the half's bytes are overwritten
      // ---- per-block min / max (pipeline.py:67-69); dead values excluded
      float mn[4], mx[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float lo = INFINITY, hi = -INFINITY;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (full_tile || i < nlive[j]) {
            lo = fminf(lo, v[j][i]);
            hi = fmaxf(hi, v[j][i]);
          }
        }
        mn[j] = redux_min(lo);
        mx[j] = redux_max(hi);
      }
      // ---- classification: lane l classifies block l & 3, then a broadcast per block
      float cmu;
      uint32_t cinfo;
      {
        const int j = lane & 3;
        const float lo = j == 0 ? mn[0] : j == 1 ? mn[1] : j == 2 ? mn[2] : mn[3];
        const float hi = j == 0 ? mx[0] : j == 1 ? mx[1] : j == 2 ? mx[2] : mx[3];
        classify_pack(lo, hi, e, pe, cmu, cinfo);
        // mu of every existing block (container.py:14), lanes 0-3 store blocks 4h..4h+3
        if (lane < 4 && 4 * h + lane < nbt) a.mu[tb + 4 * h + lane] = cmu;
      }
      // ---- encode + stage block by block (stream order = block order, lane order)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int jb = 4 * h + j;  // block in the tile
        const float mu = __shfl_sync(kFull, cmu, j);
        const uint32_t info = __shfl_sync(kFull, cinfo, j);
        const bool exists = jb < nbt;
        const bool nc = exists && ((info >> 13) & 1);
        const uint32_t shift = exists ? (info & 0xFF) : 32u;
        const uint32_t K = (info >> 12) & 1;
        const int q = (int)((info >> 8) & 7);
        uint32_t t[4];
        int f[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)  // pipeline.py:102-106
          t[i] = shr_clamp(__float_as_uint(__fsub_rn(v[j][i], mu)), shift);
        // predecessor of the lane's first value: the previous lane's last (0 at block start,
        // pipeline.py:108-111)
        uint32_t p = __shfl_up_sync(kFull, t[3], 1);
        if (lane == 0) p = 0;
        int us = 0;
        uint32_t acc = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          // code = min(3, lzb(t ^ prev), q) = q - n, n = (f >> 3) + 1; the q == 4 sentinel
          // K caps the code at 3 (pipeline.py:84-91,112)
          f[i] = flo32((t[i] ^ (i ? t[i - 1] : p)) | K);
          if (!full_tile && i >= nlive[j]) f[i] = -1;  // dead values keep nothing
          us += f[i] >> 3;
          acc += (uint32_t)(f[i] >> 3) << (2 * i);
        }
        const uint32_t L = (uint32_t)(us + 4);  // kept bytes of the lane (0 when constant)
        // 4 codes of the lane = one byte of the block's code row (container.py:286-294)
        uint32_t cb = ((uint32_t)(q - 1) * 0x55u - acc) & 0xFFu;
        if (!full_tile) cb &= (1u << (2 * nlive[j])) - 1;  // zero padding codes
        // lane offsets within the block (stream order = lane order)
        uint32_t incl = L;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, incl, d);
          if (lane >= d) incl += y;
        }
        const uint32_t tot = __shfl_sync(kFull, incl, 31);
        if (nc) {  // warp-uniform
          const uint32_t base = stage + mid_off + incl - L;
          switch (q) {
            case 1: stage4<1>(base, t, f); break;
            case 2: stage4<2>(base, t, f); break;
            case 3: stage4<3>(base, t, f); break;
            default: stage4<4>(base, t, f); break;
          }
          SD.codes[nc_cnt * 32 + lane] = (uint8_t)cb;
          if (lane == 0) {
            const uint32_t req = info >> 16;
            SD.req[nc_cnt] = (uint8_t)req;
            if (req < 1) atomicOr(a.err, kErrBadReq);  // container.py:206-207
          }
          ++nc_cnt;
        } else if (exists) {
          cmap |= 1u << jb;  // constant block (container.py:12-13)
        }
        mid_off += tot;
      }
    }

    // ---- decoupled look-back over (NC blocks, mid bytes) per tile
    const uint64_t agg = pack2(nc_cnt, mid_off);
    uint64_t ex = 0;
    if (tile == 0) {
      if (lane == 0) st_relaxed(a.status, kFlagPre | agg);
    } else {
      if (lane == 0) st_relaxed(a.status + tile, kFlagAgg | agg);
      ex = lookback_excl<4>(a.status, tile, /*backoff_ns=*/64, floor, floor_incl);
      if (lane == 0) st_relaxed(a.status + tile, kFlagPre | (ex + agg));
    }
    floor = tile;
    floor_incl = ex + agg;
    const uint64_t pre_nc = bnc + hi_of(ex), pre_mid = bmid + lo_of(ex);
    __syncwarp();  // staged bytes / side rows visible to every lane

    // ---- write-out
    if (lane == 0) a.map[tile] = (uint8_t)cmap;  // one map byte per tile, LSB-first
    if (lane < (int)nc_cnt) a.req[pre_nc + lane] = SD.req[lane];
    if (lane < 2 * (int)nc_cnt) {
      // NC block r owns bytes [32r, 32r+32) of the code pool (every NC block but the field's
      // last is full; the short last block's unused codes are zero and inside the capacity)
      const uint4 cv = reinterpret_cast<const uint4*>(SD.codes)[lane];
      uint8_t* dst = a.codes + 32 * pre_nc + 16 * lane;
      if (((uintptr_t)a.codes & 15) == 0) {
        *reinterpret_cast<uint4*>(dst) = cv;
      } else {
        uint32_t* d4 = reinterpret_cast<uint32_t*>(dst);
        d4[0] = cv.x; d4[1] = cv.y; d4[2] = cv.z; d4[3] = cv.w;
      }
    }
    copy_out(a.mid, pre_mid, reinterpret_cast<const uint8_t*>(B[b].v), mid_off, lane);
    if (tile == a.ntiles - 1 && lane == 0) {  // chunk totals for the host / the next chunk
      const uint64_t run = ex + agg;
      const uint64_t cnc = hi_of(run);
      a.totals->n_nc = bnc + cnc;
      // the field's short last block counts only its live values when it is NC
      // (container.py:241-244)
      const uint64_t lastb = nb - 1, nvb = n - 128 * lastb;
      const uint32_t lb = (uint32_t)(lastb - tb);
      const uint64_t madj = (nvb < 128 && !((cmap >> lb) & 1)) ? 128 - nvb : 0;
      a.totals->m = bm + 128 * cnc - madj;
      a.totals->mid_len = bmid + lo_of(run);
      a.totals->pad = 0;
    }
    __syncwarp();  // every lane is done with buffer b before it is refilled
    const uint32_t tn = claim(b);
    if (b) t1 = tn;
    else t0 = tn;
  }
}

cudaError_t launch_encode128(const CompressArgs& a, cudaStream_t s) {
  static bool configured = false;
  static int per_sm = 1;
  const size_t smem = sizeof(EncSmem);
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(encode128_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, encode128_kernel, kEW * 32, smem);
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
  // enough CTAs for every tile to have a warp, at most one wave of resident CTAs (the
  // look-back needs every claimed tile's warp to be resident)
  const uint64_t want = (a.ntiles + kEW - 1) / kEW;
  const uint64_t cap = (uint64_t)per_sm * nsm;
  const uint32_t grid = (uint32_t)(want < cap ? want : cap);
  encode128_kernel<<<grid, kEW * 32, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace szx
