// szx_device.cuh -- shared device helpers for the sm_100a SZx kernels.
//
// Numerics contract: every float32 / float64 op that
// decides a stream byte is an explicit round-to-nearest intrinsic, and the library is built
// WITHOUT --use_fast_math and with -ftz=false, so subnormals are kept exactly as the
// reference's NumPy arithmetic keeps them (blockcodec.py:38-48, test_blockcodec.py:294-307).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace szx {

constexpr uint32_t kFull = 0xFFFFFFFFu;

// ---- decoupled look-back status words ------------------------------------------------
// One 64-bit word per tile: [63:62] flag, [61:0] payload.  Payload packs two counters
// (high field, low field) so ONE chain carries both prefix sums the stream layout needs.
constexpr uint64_t kFlagAgg = 1ull << 62;    // tile aggregate published
constexpr uint64_t kFlagPre = 2ull << 62;    // inclusive prefix published
constexpr uint64_t kFlagMask = 3ull << 62;
constexpr uint64_t kPayload = ~kFlagMask;
constexpr int kLowBits = 36;                 // low field: byte counts (< 64 GiB / launch)
constexpr uint64_t kLowMask = (1ull << kLowBits) - 1;

__device__ __forceinline__ uint64_t pack2(uint64_t hi, uint64_t lo) {
  return (hi << kLowBits) | lo;
}
__device__ __forceinline__ uint64_t hi_of(uint64_t p) { return (p & kPayload) >> kLowBits; }
__device__ __forceinline__ uint64_t lo_of(uint64_t p) { return p & kLowMask; }

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Watchdog for every spin-wait: a wait that outlives ~2^33 cycles (seconds) means a broken
// protocol or a corrupt input; trap so the launch fails loudly instead of hanging the GPU.
__device__ __forceinline__ void spin_guard(long long t0) {
  if (clock64() - t0 > (1ll << 33)) __trap();
}

// Warp-cooperative decoupled look-back (run by ONE full warp).  Publishes `agg` for
// `tile`, returns the exclusive prefix (payload sum over tiles < tile) in every lane, and
// publishes the inclusive prefix.  Payload sums never carry across the field boundary
// because callers bound the per-launch totals (see abi.cu chunking).
__device__ __forceinline__ uint64_t lookback(uint64_t* status, uint32_t tile, uint64_t agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_relaxed(status, kFlagPre | agg);
    return 0;
  }
  if (lane == 0) st_relaxed(status + tile, kFlagAgg | agg);
  uint64_t excl = 0;
  int64_t look = (int64_t)tile - 1;
  while (true) {
    const int64_t idx = look - lane;
    // tiles before 0 read as a ready zero prefix
    uint64_t s = idx >= 0 ? ld_relaxed(status + idx) : kFlagPre;
    // every lane must hold a ready word before the window is summed
    const long long t0 = clock64();
    while (!__all_sync(kFull, (s & kFlagMask) != 0)) {
      if ((s & kFlagMask) == 0) s = ld_relaxed(status + idx);
      spin_guard(t0);
    }
    const uint32_t pre = __ballot_sync(kFull, (s & kFlagMask) == kFlagPre);
    uint64_t v = s & kPayload;
    if (pre) {
      const int first = __ffs(pre) - 1;  // nearest tile holding an inclusive prefix
      if (lane > first) v = 0;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
    excl += v;
    if (pre) break;
    look -= 32;
  }
  if (lane == 0) st_relaxed(status + tile, kFlagPre | (excl + agg));
  return excl;
}

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// Wide decoupled look-back, scan part: the exclusive prefix of `tile` (> 0) from the status
// words of its predecessors -- a window of 32*PER per step, read as PER warp-coalesced rows
// of 32 consecutive words (entry at distance d = lane + 32*j), so the inclusive-prefix front
// advances faster than a persistent grid retires tiles while each window costs PER coalesced
// 256-byte reads.  Publishes nothing (the caller may not know its aggregate yet).
// `backoff_ns`: sleep between polls (0: spin), for warps that share an SM with compute warps.
// `floor` / `floor_incl`: a tile below this one whose inclusive prefix the caller already
// knows (-1 / 0: none) -- the scan never reads at or below it, so its length is bounded by
// tile - floor however far the other tiles' look-backs lag.
template <int PER = 8>
__device__ __forceinline__ uint64_t lookback_excl(const uint64_t* status, uint64_t tile,
                                                  int backoff_ns = 0, int64_t floor = -1,
                                                  uint64_t floor_incl = 0) {
  const int lane = threadIdx.x & 31;
  uint64_t excl = 0;
  int64_t look = (int64_t)tile - 1;
  while (true) {
    uint64_t s[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int64_t idx = look - lane - 32 * j;
      // before tile 0: zero prefix; at the floor: its known inclusive prefix
      s[j] = idx > floor ? ld_relaxed(status + idx) : kFlagPre | (idx == floor ? floor_incl : 0);
    }
    // Wait only for the entries between this tile and the nearest inclusive prefix: older
    // stragglers beyond it are irrelevant (waiting on them would couple every tile to the
    // slowest tile in flight).
    const long long t0 = clock64();
    int dmin;  // distance (lane + 32 j) of the nearest inclusive prefix, 32*PER if none
    while (true) {
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
      if (backoff_ns) __nanosleep(backoff_ns);
      spin_guard(t0);
    }
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

// Wide decoupled look-back (whole warp): publishes the aggregate (unless `published`: another
// warp of this CTA stored it), scans, publishes the inclusive prefix, returns the exclusive
// one.  Same contract as lookback().
template <int PER = 8>
__device__ __forceinline__ uint64_t lookback_wide(uint64_t* status, uint64_t tile, uint64_t agg,
                                                  bool published = false, int backoff_ns = 0) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_relaxed(status, kFlagPre | agg);
    return 0;
  }
  if (lane == 0 && !published) st_relaxed(status + tile, kFlagAgg | agg);
  const uint64_t excl = lookback_excl<PER>(status, tile, backoff_ns);
  if (lane == 0) st_relaxed(status + tile, kFlagPre | (excl + agg));
  return excl;
}

// ---- float bit helpers ----------------------------------------------------------------
// blockcodec.py:38-48: exponent field - 127; subnormal -> -126; zero -> -127
__device__ __forceinline__ int exponent_of(float x) {
  const uint32_t w = __float_as_uint(x);
  const int field = (int)((w >> 23) & 0xFFu);
  return field ? field - 127 : ((w & 0x7FFFFFu) ? -126 : -127);
}

__device__ __forceinline__ bool nonfinite(float x) {
  return (__float_as_uint(x) & 0x7F800000u) == 0x7F800000u;
}

// Byte-column masks on a big-endian-read u32: columns [c,4) = 0xFFFFFFFF >> 8c.
__device__ __forceinline__ uint32_t tail_mask(int c) {
  return c >= 4 ? 0u : (kFull >> (8 * c));
}

// Per-block classification (pipeline.py:54-81 == blockcodec.summarize_block 87-112).
struct BlockClass {
  float mu;
  int cst;   // 1 = constant block
  int req;   // kept bits (NC only)
  int s;     // byte-aligning shift
  int q;     // kept bytes
};

__device__ __forceinline__ BlockClass classify(float mn, float mx, double e, int pe) {
  BlockClass b;
  // pipeline.py:71 -- float64 midrange, one rounding to float32
  const double sum = __dadd_rn((double)mn, (double)mx);
  b.mu = __double2float_rn(__dmul_rn(sum, 0.5));
  const double mu64 = (double)b.mu;
  // pipeline.py:72-74 -- constant iff max endpoint deviation <= e (float64)
  const double d1 = __dsub_rn((double)mx, mu64);
  const double d2 = __dsub_rn(mu64, (double)mn);
  const double maxdev = d1 > d2 ? d1 : d2;
  b.cst = maxdev <= e;
  // pipeline.py:76-80 -- r_v in float32, req = clip(9 + p(r_v) - p(e), 0, 32)
  const float a = fabsf(__fsub_rn(mx, b.mu));
  const float c = fabsf(__fsub_rn(mn, b.mu));
  const float rv = a > c ? a : c;
  int req = 9 + exponent_of(rv) - pe;
  req = req < 0 ? 0 : (req > 32 ? 32 : req);
  b.req = req;
  b.s = (8 - (req & 7)) & 7;
  b.q = (req + b.s) >> 3;
  return b;
}

// q and s from a stored req byte (container.py:156-157,241-244)
__device__ __forceinline__ void q_s_of(int req, int& q, int& s) {
  s = (8 - (req & 7)) & 7;
  q = (req + s) >> 3;
}

// ---- memory helpers ---------------------------------------------------------------------
__device__ __forceinline__ float4 ld_stream_f4(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_stream_f4(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

// 32-byte store (sm_100: STG.256): a lane writes a whole sector, so a lane-strided pattern
// of 32-byte runs costs no partial-sector writes.  p must be 32-byte aligned.
__device__ __forceinline__ void st_stream_v8(float* p, const float* v) {
  asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]),
               "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}

// ---- mbarrier + bulk-copy (TMA engine) helpers -------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// try_wait with a suspend-time hint: the thread sleeps in hardware until the phase
// completes (or the hint expires), instead of burning issue slots in a spin loop.
#ifndef SZX_SLEEP_NS0
#define SZX_SLEEP_NS0 64     // helper-warp waits: first back-off (ns)
#endif
#ifndef SZX_SLEEP_NSMAX
#define SZX_SLEEP_NSMAX 512  // helper-warp waits: longest back-off (ns)
#endif
#ifndef SZX_WAIT_HINT
#define SZX_WAIT_HINT 0   // 1: compute-warp waits suspend in hardware; 2: helper warps too
#endif
__device__ __forceinline__ bool mbar_try_wait_hint(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
// Wait for an mbarrier phase: one (hardware-suspending) try_wait, then exponential
// back-off with nanosleep, so a waiting warp issues a handful of instructions instead of a
// spin loop that competes with the working warps for issue slots.  Watchdog by iteration
// count: 2^24 sleeps of >= 256 ns are seconds -> trap instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity,
                                                  uint32_t ns0, uint32_t ns_max) {
  if (mbar_try_wait(bar, parity)) return;
  uint32_t ns = ns0, it = 0;
  while (!mbar_try_wait(bar, parity)) {
    __nanosleep(ns);
    ns = ns < ns_max ? 2 * ns : ns_max;
    if (++it > (1u << 24)) __trap();
  }
}
// latency-critical consumers (compute warps)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if SZX_WAIT_HINT
  uint32_t it = 0;
  while (!mbar_try_wait_hint(bar, parity))
    if (++it > (1u << 24)) __trap();
#else
  mbar_wait_backoff(bar, parity, 32, 128);
#endif
}
// helper warps (producers, look-back) that are idle most of the time: sleep longer between
// polls so their waiting costs the compute warps few issue slots (the ring depth covers it)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
#if SZX_WAIT_HINT >= 2
  uint32_t it = 0;
  while (!mbar_try_wait_hint(bar, parity))
    if (++it > (1u << 24)) __trap();
#else
  mbar_wait_backoff(bar, parity, SZX_SLEEP_NS0, SZX_SLEEP_NSMAX);
#endif
}
// 1-D bulk copy global -> shared through the TMA engine; completes `bytes` on `bar`.
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                        uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Named barrier over a subset of warps (ids 1..15; 0 is __syncthreads).
__device__ __forceinline__ void named_bar(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Warp inclusive scan (u32).
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v += t;
  }
  return v;
}

}  // namespace szx
