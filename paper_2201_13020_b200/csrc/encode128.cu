// encode128.cu -- SZx block encoder for sm_100a, bs == 128 (K1 in DESIGN.md).
//
// Replaces the reference's whole compress path in ONE launch per chunk:
//   block_stats           pipeline.py:54-81   (== blockcodec.summarize_block 87-112)
//   _encode_elements      pipeline.py:94-133  (== blockcodec.encode_nonconstant 123-141)
//   prefix_scan + scatter parallel.py:21-44,104-140 / pipeline.py:143-166
// Output pools use the UFZX container layout (container.py:3-21).
//
// Persistent grid, one CTA per SM: kEW compute warps + 1 look-back warp.  A CTA encodes one
// super-tile of kEW warp tiles (4 blocks each) per step; super-tiles are claimed in order
// from the chunk's counter a few steps ahead (a slow CTA simply claims fewer).  Compute warp
// w owns blocks 4w..4w+3 of the super-tile and never waits for another warp while encoding:
//   input  -- each warp streams its 2 KiB tiles with 1-D bulk copies (TMA engine) into
//             buffers of its own (tile k+2 is in flight while tile k is encoded);
//   encode -- lane l owns values 4l..4l+3 of each block (one block = one warp row, so every
//             per-block quantity is warp-uniform): CREDUX min/max, the fp64 classification
//             computed once per block (lane j classifies block j & 3, then a broadcast), the
//             XOR-with-previous chain (one shuffle per block), codes and kept bytes.  Kept
//             bytes are staged IN PLACE over the tile's own input (a tile's output never
//             exceeds its input) at tile-relative offsets, so staging needs no prefix; lanes
//             are ~4 bytes apart, so the byte stores are bank-conflict free.  The warp then
//             publishes its (NC blocks, mid bytes) counts; the last warp of the super-tile
//             publishes the super-tile aggregate for the decoupled look-back;
//   look-back warp -- warp prefixes inside the super-tile, the look-back over super-tiles
//             (bounded below by the CTA's previous super-tile), the constant-map bytes;
//   write  -- kDefer steps later (so the look-back latency hides behind later encodes) each
//             warp writes its staged tile out: mid bytes as realigned 16-byte chunks
//             (bytewise only at the two partial edge chunks), code rows, req bytes.
// Every wait is an mbarrier try_wait with nanosleep back-off (few issue slots).
#include "szx_device.cuh"
#include "szx_kernels.h"

namespace szx {

namespace {

#ifndef SZX_K1V2_DEFER
#define SZX_K1V2_DEFER 2
#endif
constexpr int kEW = kEncWarps;            // compute warps per CTA
constexpr int kLBWarp = kEW;              // the look-back warp
constexpr int kThreads1 = (kEW + 1) * 32;
constexpr int kWB = kEncWarpBlocks;       // blocks per warp tile (4)
constexpr int kWV = kWB * 128;            // values per warp tile
constexpr int kTileBytes = kWV * 4;       // 2 KiB
constexpr int kSB = kEncTileBlocks;       // blocks per super-tile
constexpr int kDefer = SZX_K1V2_DEFER;    // a tile is written out kDefer steps after its encode
constexpr int kBufs = kDefer + 2;         // buffers per warp: one encoding, kDefer staged, one
                                          // loading
constexpr int kSides = kDefer + 1;        // code / req staging per warp
constexpr int kAhead = kDefer + 2;        // super-tiles are claimed this many steps ahead
constexpr int kSlots = 8;                 // super-tile steps in flight
constexpr int kSidRing = 16;              // claimed super-tile ids, sid[m % kSidRing]
static_assert(kDefer + 2 <= kSlots, "count slots");
static_assert(kAhead + 2 <= kSidRing, "claim ring");
static_assert((2 + kDefer) % kBufs == 0, "the buffer written out is the one refilled");

struct __align__(16) WarpBuf {
  uint8_t pre[16];                        // realignment over-read slack before the staging
  float v[kWV];                           // the tile's values, then its staged mid bytes
  uint8_t post[48];                       // over-read slack after it
};
struct __align__(16) WarpSide {
  uint8_t codes[kWB * 32];                // code rows of the tile's NC blocks, NC-rank order
  uint8_t req[16];                        // req bytes, NC-rank order
};
struct __align__(16) SuperPre {           // look-back warp -> compute warps, per step slot
  unsigned long long nc, mid;             // stream offsets of the super-tile
  uint32_t wpre[kEW];                     // tile prefixes inside it: nc << 16 | mid
};
struct EncSmem {
  WarpBuf buf[kEW][kBufs];
  WarpSide side[kEW][kSides];
  SuperPre pre[kSlots];
  uint64_t full[kEW][kBufs];              // bulk copy -> compute warp
  uint64_t counted[kSlots];               // compute warps (kEW arrivals) -> look-back warp
  uint64_t offsets[kSlots];               // look-back warp -> compute warps
  uint32_t cnt[kSlots][kEW];              // per warp tile: nc << 16 | mid bytes
  uint32_t nib[kSlots][kEW];              // per warp tile: constant bits (4)
  uint32_t order[kSlots];                 // arrival order (the last warp publishes the aggregate)
  uint32_t sid[kSidRing];                 // super-tile claimed for step m
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
template <int OFF>
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u8 [%0+%2], %1;" ::"r"(a), "r"(v), "n"(OFF) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint32_t atom_acq_rel_add_cta(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;"
               : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
}
// mbarrier wait: one check, then sleeps with exponential back-off from NS0 to NS1 between
// checks, so a waiting warp issues a handful of instructions (a suspending try_wait wakes up
// on every barrier event of the SM, and 20+ warps make those frequent); watchdog: trap
template <uint32_t NS0, uint32_t NS1>
__device__ __forceinline__ void wait_phase(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  uint32_t ns = NS0, it = 0;
  while (!mbar_try_wait(bar, parity)) {
    __nanosleep(ns);
    ns = ns < NS1 ? 2 * ns : NS1;
    if (++it > (1u << 24)) __trap();
  }
}

// Stage the kept bytes of a lane's 4 elements of one block (Q = the block's q, uniform).
// Element i keeps n_i = (f_i >> 3) + 1 bytes, big-endian (pipeline.py:114-116,151); with u
// accumulating sum_{j<=i} (f_j >> 3), element i's last byte lands at u + 3 + i and its kept
// byte c (counted from the last) at u + 3 + i - c.
// Column 0 is stored unconditionally: an element that keeps no byte equals its predecessor
// in all q bytes, so its "last byte" position is the last byte written before it, which holds
// the same value -- except when every element from the block start is zero, where it is the
// byte before the block: blocks are staged last-to-first, so that byte is rewritten afterwards
// (and before the first block lies the buffer's slack).  DEAD: the tile has dead values (past
// the field's end, f = -1 but t arbitrary), whose column 0 must not be stored.
template <int Q, bool DEAD>
__device__ __forceinline__ void stage4(uint32_t base, const uint32_t (&t)[4], const int (&f)[4]) {
  uint32_t u = base - 3;  // immediate offsets i - c + 3 >= 0
  u += (uint32_t)(f[0] >> 3);
  if (DEAD) sts_u8_if<0, 3>(u, t[0], f[0]);
  else sts_u8<3>(u, t[0]);
  if (Q >= 2) sts_u8_if<8, 2>(u, t[0] >> 8, f[0]);
  if (Q >= 3) sts_u8_if<16, 1>(u, t[0] >> 16, f[0]);
  if (Q >= 4) sts_u8_if<24, 0>(u, t[0] >> 24, f[0]);
  u += (uint32_t)(f[1] >> 3);
  if (DEAD) sts_u8_if<0, 4>(u, t[1], f[1]);
  else sts_u8<4>(u, t[1]);
  if (Q >= 2) sts_u8_if<8, 3>(u, t[1] >> 8, f[1]);
  if (Q >= 3) sts_u8_if<16, 2>(u, t[1] >> 16, f[1]);
  if (Q >= 4) sts_u8_if<24, 1>(u, t[1] >> 24, f[1]);
  u += (uint32_t)(f[2] >> 3);
  if (DEAD) sts_u8_if<0, 5>(u, t[2], f[2]);
  else sts_u8<5>(u, t[2]);
  if (Q >= 2) sts_u8_if<8, 4>(u, t[2] >> 8, f[2]);
  if (Q >= 3) sts_u8_if<16, 3>(u, t[2] >> 16, f[2]);
  if (Q >= 4) sts_u8_if<24, 2>(u, t[2] >> 24, f[2]);
  u += (uint32_t)(f[3] >> 3);
  if (DEAD) sts_u8_if<0, 6>(u, t[3], f[3]);
  else sts_u8<6>(u, t[3]);
  if (Q >= 2) sts_u8_if<8, 5>(u, t[3] >> 8, f[3]);
  if (Q >= 3) sts_u8_if<16, 4>(u, t[3] >> 16, f[3]);
  if (Q >= 4) sts_u8_if<24, 3>(u, t[3] >> 24, f[3]);
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

// Encode one warp tile (4 blocks): values from the warp's buffer (FULL) or global memory
// (the chunk's last, partial tile), kept bytes staged in place, code rows and req bytes into
// the side record.  Returns the tile's NC blocks, mid bytes and constant bits.
template <bool FULL>
__device__ __forceinline__ void encode_tile(const CompressArgs& a, const float* buf,
                                            uint32_t stage, WarpSide& SD, uint64_t v0,
                                            uint64_t tb, int nbt, int lane, uint32_t& nc_out,
                                            uint32_t& mid_out, uint32_t& cmap_out) {
  const uint64_t n = a.n;
  // ---- values: lane l holds values 4l..4l+3 of the tile's 4 blocks
  float v[4][4];
  int nlive[4];
  if (FULL) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 x = reinterpret_cast<const float4*>(buf)[j * 32 + lane];
      v[j][0] = x.x; v[j][1] = x.y; v[j][2] = x.z; v[j][3] = x.w;
      nlive[j] = 4;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t first = v0 + (uint64_t)j * 128 + 4 * lane;
      nlive[j] = first >= n ? 0 : (int)umin64(4, n - first);
#pragma unroll
      for (int i = 0; i < 4; ++i) v[j][i] = i < nlive[j] ? a.x[first + i] : 0.f;
    }
  }
  __syncwarp();  // every lane holds its values before the buffer is overwritten
  // ---- per-block min / max (pipeline.py:67-69); dead values excluded
  float mn[4], mx[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float lo, hi;
    if (FULL) {
      lo = fminf(fminf(v[j][0], v[j][1]), fminf(v[j][2], v[j][3]));
      hi = fmaxf(fmaxf(v[j][0], v[j][1]), fmaxf(v[j][2], v[j][3]));
    } else {
      lo = INFINITY;
      hi = -INFINITY;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i < nlive[j]) {
          lo = fminf(lo, v[j][i]);
          hi = fmaxf(hi, v[j][i]);
        }
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
    classify_pack(lo, hi, a.e, a.pe, cmu, cinfo);
    // mu of every existing block (container.py:14): lanes 0-3 store the 4 blocks
    if (lane < nbt) a.mu[tb + lane] = cmu;
  }
  // ---- per block: t (kept bytes, right-aligned), f (highest changed bit), lane byte count
  uint32_t tv[4][4];
  int f[4][4];
  uint32_t L[4], cb[4], info[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float mu = __shfl_sync(kFull, cmu, j);
    info[j] = __shfl_sync(kFull, cinfo, j);
    if (!FULL && j >= nbt) info[j] = 32u;  // absent block: constant-like, nothing kept
    const uint32_t shift = info[j] & 0xFF;
    const uint32_t K = (info[j] >> 12) & 1;
#pragma unroll
    for (int i = 0; i < 4; ++i)  // pipeline.py:102-106
      tv[j][i] = shr_clamp(__float_as_uint(__fsub_rn(v[j][i], mu)), shift);
    // predecessor of the lane's first value: the previous lane's last (0 at block start,
    // pipeline.py:108-111)
    uint32_t p = __shfl_up_sync(kFull, tv[j][3], 1);
    if (lane == 0) p = 0;
    // acc = sum_i n_i (4^i + 2^16), n_i = (f_i >> 3) + 1 kept bytes: the code byte and the
    // lane's byte count in one IMAD per element
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      // code = min(3, lzb(t ^ prev), q) = q - n; the q == 4 sentinel K caps the code at 3
      // (pipeline.py:84-91,112)
      f[j][i] = flo32((tv[j][i] ^ (i ? tv[j][i - 1] : p)) | K);
      if (!FULL && i >= nlive[j]) f[j][i] = -1;  // dead values keep nothing
      acc += (uint32_t)((f[j][i] >> 3) + 1) * ((1u << (2 * i)) | (1u << 16));
    }
    L[j] = acc >> 16;  // kept bytes of the lane (0 for constant blocks: t = 0, f = -1)
    // 4 codes of the lane = one byte of the block's code row (container.py:286-294)
    const uint32_t q = (info[j] >> 8) & 7;
    cb[j] = (q * 0x55u - (acc & 0xFFFFu)) & 0xFFu;
    if (!FULL) cb[j] &= (1u << (2 * nlive[j])) - 1;  // zero padding codes
  }
  // ---- lane offsets (stream order = block order, lane order): two packed 16-bit scans
  uint32_t s01 = L[0] | (L[1] << 16), s23 = L[2] | (L[3] << 16);
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y01 = __shfl_up_sync(kFull, s01, d);
    const uint32_t y23 = __shfl_up_sync(kFull, s23, d);
    if (lane >= d) {
      s01 += y01;
      s23 += y23;
    }
  }
  const uint32_t t01 = __shfl_sync(kFull, s01, 31), t23 = __shfl_sync(kFull, s23, 31);
  const uint32_t T0 = t01 & 0xFFFFu, T1 = t01 >> 16, T2 = t23 & 0xFFFFu, T3 = t23 >> 16;
  const uint32_t off[4] = {(s01 & 0xFFFFu) - L[0], T0 + (s01 >> 16) - L[1],
                           T0 + T1 + (s23 & 0xFFFFu) - L[2], T0 + T1 + T2 + (s23 >> 16) - L[3]};
  // ---- NC blocks
  uint32_t ncm = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) ncm |= ((info[j] >> 13) & 1) << j;
  if (!FULL) ncm &= (1u << nbt) - 1;
  // ---- stage, last block first (see stage4)
#pragma unroll
  for (int j = 3; j >= 0; --j) {
    if ((ncm >> j) & 1) {  // warp-uniform
      const uint32_t base = stage + off[j];
      switch ((info[j] >> 8) & 7) {
        case 1: stage4<1, !FULL>(base, tv[j], f[j]); break;
        case 2: stage4<2, !FULL>(base, tv[j], f[j]); break;
        case 3: stage4<3, !FULL>(base, tv[j], f[j]); break;
        default: stage4<4, !FULL>(base, tv[j], f[j]); break;
      }
      const uint32_t rank = __popc(ncm & ((1u << j) - 1));
      SD.codes[rank * 32 + lane] = (uint8_t)cb[j];
      if (lane == 0) {
        const uint32_t req = info[j] >> 16;
        SD.req[rank] = (uint8_t)req;
        if (req < 1) atomicOr(a.err, kErrBadReq);  // container.py:206-207
      }
    }
  }
  nc_out = __popc(ncm);
  mid_out = T0 + T1 + T2 + T3;
  cmap_out = ~ncm & (FULL ? 0xFu : ((1u << nbt) - 1));  // constant blocks (container.py:12-13)
}

}  // namespace

// Profiling builds (-DSZX_STATS) only, cycles summed over warps: compute warps [0] input
// wait, [1] encode, [2] offsets wait, [3] write-out, [4] warp steps; look-back warp [5]
// counts wait, [6] look-back, [7] steps.
__device__ unsigned long long g_encode_stats[16];
#ifdef SZX_STATS
// accumulated per warp in registers (stacc, constant indices), added to the globals once at
// the end of the kernel, so the counters do not perturb what they measure
#define ENC_T0(v) const long long v = clock64()
#define ENC_ADD(i, v) stacc[i] += (unsigned long long)(clock64() - (v))
#define ENC_INC(i) stacc[i] += 1ull
#define ENC_FLUSH() \
  if (lane == 0)    \
    for (int i_ = 0; i_ < 16; ++i_) atomicAdd(&g_encode_stats[i_], stacc[i_])
#else
#define ENC_FLUSH()
#define ENC_T0(v)
#define ENC_ADD(i, v)
#define ENC_INC(i)
#endif
cudaError_t encode_stats(unsigned long long* out8, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out8, g_encode_stats, 16 * sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    const unsigned long long z[16] = {};
    e = cudaMemcpyToSymbol(g_encode_stats, z, sizeof z);
  }
  return e;
}

// lookback_excl (szx_device.cuh) with counters in profiling builds: [8] windows, [9] polls,
// [10] summed distance to the nearest inclusive prefix, [11] polls that found a missing entry
template <int PER>
__device__ __forceinline__ uint64_t lookback_sup(const uint64_t* status, uint64_t tile,
                                                 int backoff_ns, int64_t floor,
                                                 uint64_t floor_incl,
                                                 unsigned long long (&stacc)[16]) {
  const int lane = threadIdx.x & 31;
  uint64_t excl = 0;
  int64_t look = (int64_t)tile - 1;
  while (true) {
    ENC_INC(8);
    uint64_t s[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int64_t idx = look - lane - 32 * j;
      s[j] = idx > floor ? ld_relaxed(status + idx) : kFlagPre | (idx == floor ? floor_incl : 0);
    }
    const long long t0 = clock64();
    int dmin;
    while (true) {
      ENC_INC(9);
      dmin = 32 * PER;
#pragma unroll
      for (int j = PER - 1; j >= 0; --j) {
        const uint32_t b = __ballot_sync(kFull, (s[j] & kFlagMask) == kFlagPre);
        if (b) dmin = 32 * j + __ffs(b) - 1;
      }
      bool missing = false;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        if (lane + 32 * j < dmin && (s[j] & kFlagMask) == 0) {
          s[j] = ld_relaxed(status + (look - lane - 32 * j));
          missing = true;
        }
      }
      if (!__any_sync(kFull, missing)) break;
      ENC_INC(11);
      if (backoff_ns) __nanosleep(backoff_ns);
      spin_guard(t0);
    }
#ifdef SZX_STATS
    stacc[10] += (unsigned long long)dmin;
#endif
    uint64_t v = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j)
      if (lane + 32 * j <= dmin) v += s[j] & kPayload;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
    excl += v;
    if (dmin < 32 * PER) break;
    look -= 32 * PER;
  }
  return excl;
}

// What a warp keeps about its staged tile until its write-out.
struct Staged {
  uint32_t nc, mid;   // NC blocks, mid bytes of the tile
  int exists;         // the tile has at least one block
};

// registers: a warp's registers come from its SM sub-partition's quarter of the file, so with
// kEW + 1 warps the fullest quarter holds ceil((kEW + 1) / 4) warps
constexpr int kRegs = (65536 / 4) / (((kEW + 1 + 3) / 4) * 32) / 8 * 8;
__global__ void __maxnreg__(kRegs > 255 ? 255 : kRegs) encode128_kernel(CompressArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  EncSmem& sm = *reinterpret_cast<EncSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t n = a.n;
  const uint64_t nb = (n + 127) >> 7;
  unsigned long long stacc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) stacc[i] = 0;

  if (threadIdx.x < kSlots) {
    sm.order[threadIdx.x] = 0;
    mbar_init(&sm.counted[threadIdx.x], kEW);
    mbar_init(&sm.offsets[threadIdx.x], 1);
  }
  // the first kAhead steps are assigned statically in grid order; later super-tiles are
  // claimed in order, kAhead steps ahead, so a super-tile's look-back only waits for OLDER
  // claims
  if (threadIdx.x < kAhead) sm.sid[threadIdx.x] = blockIdx.x + threadIdx.x * gridDim.x;
  if (warp < kEW && lane < kBufs) mbar_init(&sm.full[warp][lane], 1);
  fence_barrier_init();
  __syncthreads();

  // ------------------------------------------------------------------ look-back warp
  if (warp == kLBWarp) {
    int64_t floor = -1;       // this CTA's previous super-tile and its inclusive prefix: the
    uint64_t floor_incl = 0;  // look-back never scans past it
    const uint64_t bnc = a.base ? a.base->n_nc : 0, bm = a.base ? a.base->m : 0;
    const uint64_t bmid = a.base ? a.base->mid_len : 0;
    for (uint32_t k = 0;; ++k) {
      const uint32_t S = sm.sid[k % kSidRing];
      if (S >= a.ntiles) break;  // claims grow monotonically
      const int slot = k % kSlots;
      uint32_t next = 0;  // the claim for step k + kAhead, published with this step's offsets
      if (lane == 0) next = kAhead * gridDim.x + atomicAdd(a.counter, 1u);
      ENC_T0(t_w);
      wait_phase<64, 256>(&sm.counted[slot], (k / kSlots) & 1);
      ENC_ADD(5, t_w);
      ENC_INC(7);
      const uint32_t c = lane < kEW ? sm.cnt[slot][lane] : 0u;
      const uint32_t nib = lane < kEW ? sm.nib[slot][lane] : 0u;
      uint32_t incl = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += y;
      }
      const uint32_t tot = __shfl_sync(kFull, incl, 31);
      if (lane < kEW) sm.pre[slot].wpre[lane] = incl - c;
      const uint64_t agg = pack2(tot >> 16, tot & 0xFFFFu);
      uint64_t ex = 0;
      if (S == 0) {
        if (lane == 0) st_relaxed(a.status, kFlagPre | agg);
      } else {
        // (the aggregate was published by the last compute warp to count the super-tile)
        ENC_T0(t_lb);
        ex = lookback_sup<8>(a.status, S, /*backoff_ns=*/32, floor, floor_incl, stacc);
        ENC_ADD(6, t_lb);
        if (lane == 0) st_relaxed(a.status + S, kFlagPre | (ex + agg));
      }
      floor = S;
      floor_incl = ex + agg;
      if (lane == 0) {
        sm.pre[slot].nc = bnc + hi_of(ex);
        sm.pre[slot].mid = bmid + lo_of(ex);
        sm.sid[(k + kAhead) % kSidRing] = next;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.offsets[slot]);  // release: prefixes + the next claim
      // constant map: warp tiles 2i, 2i+1 -> byte i of the super-tile (LSB-first,
      // container.py:12-13,321); bits of blocks past the field are zero
      const uint64_t sb = (uint64_t)S * kSB;
      const uint32_t nib_lo = __shfl_sync(kFull, nib, (2 * lane) & 31);
      const uint32_t nib_hi = __shfl_sync(kFull, nib, (2 * lane + 1) & 31);
      if (lane < kSB / 8 && 2 * lane * kWB + sb < nb)
        a.map[sb / 8 + lane] = (uint8_t)(nib_lo | (nib_hi << 4));
      if (S == a.ntiles - 1 && lane == 0) {  // chunk totals for the host / the next chunk
        const uint64_t run = ex + agg;
        const uint64_t cnc = hi_of(run);
        a.totals->n_nc = bnc + cnc;
        // the field's short last block counts only its live values when it is NC
        // (container.py:241-244)
        const uint64_t lastb = nb - 1, nvb = n - 128 * lastb;
        const uint32_t lw = (uint32_t)((lastb - sb) / kWB), lb = (uint32_t)((lastb - sb) % kWB);
        const bool last_const = (sm.nib[slot][lw] >> lb) & 1;
        const uint64_t madj = (nvb < 128 && !last_const) ? 128 - nvb : 0;
        a.totals->m = bm + 128 * cnc - madj;
        a.totals->mid_len = bmid + lo_of(run);
        a.totals->pad = 0;
      }
    }
    ENC_FLUSH();
    return;
  }

  // ------------------------------------------------------------------ compute warps
  WarpBuf* B = sm.buf[warp];
  uint64_t* full = sm.full[warp];
  const uint64_t nwt = (nb + kWB - 1) / kWB;  // warp tiles of the chunk
  // start the input copy of step k's tile into buffer k % kBufs (lane 0); the super-tile of
  // step k was published with the offsets of step k - kAhead (acquired by this warp before
  // it issues) or statically
  auto issue = [&](uint32_t k) {
    if (lane == 0 && sm.sid[k % kSidRing] < a.ntiles) {
      const uint64_t t = (uint64_t)sm.sid[k % kSidRing] * kEW + warp;
      const int bi = k % kBufs;
      if (t < nwt) {
        const uint64_t v0 = t * kWV;
        if (v0 + kWV <= n) {
          fence_proxy_async_smem();  // the buffer's generic reads/writes before the copy
          mbar_arrive_expect_tx(&full[bi], kTileBytes);
          bulk_g2s(B[bi].v, a.x + v0, kTileBytes, &full[bi]);
        } else {
          mbar_arrive(&full[bi]);  // partial tile: the lanes read global memory
        }
      }
    }
  };
  // write out the tile staged at step k (buffer k % kBufs, side k % kSides) once its offsets
  // are known
  auto write_out = [&](uint32_t k, const Staged& st) {
    const int slot = k % kSlots;
    ENC_T0(t_t);
    wait_phase<64, 512>(&sm.offsets[slot], (k / kSlots) & 1);
    ENC_ADD(2, t_t);
    if (!st.exists) return;
    ENC_T0(t_wo);
    const uint32_t wp = sm.pre[slot].wpre[warp];
    const uint64_t pre_nc = sm.pre[slot].nc + (wp >> 16);
    const uint64_t pre_mid = sm.pre[slot].mid + (wp & 0xFFFFu);
    const WarpSide& SD = sm.side[warp][k % kSides];
    if (lane < (int)st.nc) a.req[pre_nc + lane] = SD.req[lane];
    if (lane < 2 * (int)st.nc) {
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
    copy_out(a.mid, pre_mid, reinterpret_cast<const uint8_t*>(B[k % kBufs].v), st.mid, lane);
    ENC_ADD(3, t_wo);
  };

  issue(0);
  issue(1);
  Staged prev[kDefer];  // the staged tiles of steps k - kDefer .. k - 1 (oldest first)
#pragma unroll
  for (int d = 0; d < kDefer; ++d) prev[d] = Staged{0, 0, 0};

  uint32_t k = 0;
  for (;; ++k) {
    const uint32_t S = sm.sid[k % kSidRing];
    if (S >= a.ntiles) break;
    const int bi = k % kBufs;
    const int slot = k % kSlots;
    const uint64_t t = (uint64_t)S * kEW + warp;
    const uint64_t tb = t * kWB;  // first block of the tile (chunk-relative)
    Staged cur{0, 0, 0};
    uint32_t cmap = 0;
    if (t < nwt) {
      cur.exists = 1;
      ENC_T0(t_in);
      wait_phase<32, 256>(&full[bi], (k / kBufs) & 1);
      ENC_ADD(0, t_in);
      ENC_INC(4);
      ENC_T0(t_enc);
      const uint64_t v0 = t * kWV;
      const int nbt = (int)umin64(kWB, nb - tb);
      WarpSide& SD = sm.side[warp][k % kSides];
      if (v0 + kWV <= n)
        encode_tile<true>(a, B[bi].v, smem_u32(B[bi].v), SD, v0, tb, nbt, lane, cur.nc, cur.mid,
                          cmap);
      else
        encode_tile<false>(a, B[bi].v, smem_u32(B[bi].v), SD, v0, tb, nbt, lane, cur.nc,
                           cur.mid, cmap);
      ENC_ADD(1, t_enc);
    }
    // ---- publish the tile's counts; the last warp to count the super-tile publishes its
    // aggregate at once (the look-back warp may still be busy with an earlier step, and a
    // late aggregate would hold up every later super-tile's look-back)
    uint32_t order = 0;
    if (lane == 0) {
      sm.cnt[slot][warp] = (cur.nc << 16) | cur.mid;
      sm.nib[slot][warp] = cmap;
      order = atom_acq_rel_add_cta(&sm.order[slot], 1);
      mbar_arrive(&sm.counted[slot]);
    }
    order = __shfl_sync(kFull, order, 0);
    if (order == kEW - 1) {
      if (S != 0) {
        const uint32_t c = lane < kEW ? sm.cnt[slot][lane] : 0u;
        const uint32_t tot = __reduce_add_sync(kFull, c);
        if (lane == 0) st_relaxed(a.status + S, kFlagAgg | pack2(tot >> 16, tot & 0xFFFFu));
      }
      if (lane == 0) sm.order[slot] = 0;  // every warp has counted: reusable next round
    }
    // ---- write out the tile of step k - kDefer (its look-back ran during the encodes since)
    if (k >= kDefer) write_out(k - kDefer, prev[0]);
    __syncwarp();  // every lane is done with that buffer before it is refilled
    issue(k + 2);  // into buffer (k + 2) % kBufs == (k - kDefer) % kBufs, just written out
#pragma unroll
    for (int d = 0; d + 1 < kDefer; ++d) prev[d] = prev[d + 1];
    prev[kDefer - 1] = cur;
  }
#pragma unroll
  for (int d = 0; d < kDefer; ++d)
    if (k + d >= kDefer) write_out(k + d - kDefer, prev[d]);
  ENC_FLUSH();
}

cudaError_t launch_encode128(const CompressArgs& a, cudaStream_t s) {
  static bool configured = false;
  static int per_sm = 1;
  const size_t smem = sizeof(EncSmem);
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(encode128_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, encode128_kernel, kThreads1, smem);
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
  // every CTA resident at once (a look-back waits on other CTAs' super-tiles)
  const uint64_t cap = (uint64_t)per_sm * nsm;
  const uint32_t grid = (uint32_t)(a.ntiles < cap ? a.ntiles : cap);
  if (grid) encode128_kernel<<<grid, kThreads1, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace szx
