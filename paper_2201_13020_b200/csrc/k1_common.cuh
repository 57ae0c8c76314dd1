// k1_common.cuh -- device helpers shared by the bs == 128 compress kernels (K1): TMA input,
// the 16-values-per-lane encoder (classification, pass 1) and the byte staging / realigned
// write-out primitives.  See compress.cu for the kernels and DESIGN.md section 4.
#pragma once
#include <cuda.h>

#include "szx_device.cuh"
#include "szx_kernels.h"

#ifndef SZX_K1_F2
#define SZX_K1_F2 1  // pass 1's x - mu as packed f32x2 subtracts (FADD2)
#endif

namespace szx {
namespace k1 {

constexpr int kCompWarps = 16;                      // compute warps per CTA (4 blocks each)
constexpr int kTileBlocks = kCompTileBlocks;        // 64 blocks per tile
constexpr int kTileVals = kTileBlocks * 128;        // 8192 values = 32 KiB
constexpr int kTileRows = kTileVals / 32;           // 256 rows of 128 bytes (TMA box)

__device__ __forceinline__ void st_release_cta(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void st_volatile_cta(uint32_t* p, uint32_t v) {
  asm volatile("st.volatile.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_volatile_cta(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_cta(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

#ifndef SZX_K1_EVICT
#define SZX_K1_EVICT 0  // 1: input boxes loaded with an L2 evict-first policy (read once)
#endif
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
#if SZX_K1_EVICT
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
#else
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
#endif
}

// Shared-memory byte offset (within a 1024-aligned TMA box with 128-byte swizzle) of the
// 16-byte chunk k (0..3) of lane l's 16 values in compute warp w.
__device__ __forceinline__ uint32_t swz_off(int w, int l, int k) {
  const uint32_t row = 16 * w + (l >> 1);
  const uint32_t chunk = (4 * (l & 1) + k) ^ (row & 7);
  return row * 128 + chunk * 16;
}

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
// Stage byte (v & 0xFF) at shared address a + OFF iff f >= LIM (the element keeps > LIM/8
// bytes).  [reg+imm] addressing, no address arithmetic per byte.
template <int LIM, int OFF>
__device__ __forceinline__ void sts_u8_if(uint32_t a, uint32_t v, int f) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ge.s32 p, %2, %3;\n @p st.shared.u8 [%0+%4], %1;\n}\n" ::"r"(a),
      "r"(v), "r"(f), "n"(LIM), "n"(OFF));
}

// Everything pass 2 needs about one lane (16 values of one block).
struct Lane16 {
  uint32_t t[16];   // kept bytes of (x - mu) >> s, right-aligned (pipeline.py:102-106)
  int f[16];        // bit index of the highest set bit of t ^ prev (| 1 for q == 4), -1: none
  uint32_t L;       // mid bytes of the lane
  uint32_t cb;      // the lane's 16 2-bit codes (one code-pool word, container.py:286-294)
};

// Pass 2: stage the mid bytes of one lane.  Element i keeps n_i = (f_i >> 3) + 1 bytes
// (0 when f_i < 0); its last byte lands at base + u_i + i where u_i = sum_{i'<=i} f_i' >> 3,
// and kept byte k (counted from the last) is (t_i >> 8k) & 0xFF (big-endian order,
// pipeline.py:114-116,151).  QM = the largest q in the warp; lanes with smaller q simply
// never satisfy the higher predicates.
template <int QM, int I>
__device__ __forceinline__ void stage_elem(const Lane16& s, uint32_t& u) {
  if constexpr (I < 16) {
    u += (uint32_t)(s.f[I] >> 3);
    sts_u8_if<0, 3 + I>(u, s.t[I], s.f[I]);
    if constexpr (QM >= 2) sts_u8_if<8, 2 + I>(u, s.t[I] >> 8, s.f[I]);
    if constexpr (QM >= 3) sts_u8_if<16, 1 + I>(u, s.t[I] >> 16, s.f[I]);
    if constexpr (QM >= 4) sts_u8_if<24, 0 + I>(u, s.t[I] >> 24, s.f[I]);
    stage_elem<QM, I + 1>(s, u);
  }
}
template <int QM>
__device__ __forceinline__ void stage_lane(const Lane16& s, uint32_t base) {
  uint32_t u = base - 3;  // immediate offsets i - k + 3 >= 0
  stage_elem<QM, 0>(s, u);
}

// Interior chunks [c0, c1) of copy_out with a uniform word offset K and bit shift b.
template <int K>
__device__ __forceinline__ void copy_chunks(uint8_t* g, const uint4* s128, uint32_t a, uint32_t b,
                                            uint32_t c0, uint32_t c1, int tid, int nthr) {
#pragma unroll 4
  for (uint32_t c = c0 + tid; c < c1; c += nthr) {
    // staged window of chunk c starts at byte 16c - a; rows j-1, j relative to src
    const int j = (int)((16 * c - a + 16) >> 4);
    const uint4 q0 = s128[j - 1], q1 = s128[j];
    const uint32_t w[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
    *reinterpret_cast<uint4*>(g + 16 * c) =
        make_uint4(__funnelshift_r(w[K], w[K + 1], b), __funnelshift_r(w[K + 1], w[K + 2], b),
                   __funnelshift_r(w[K + 2], w[K + 3], b), __funnelshift_r(w[K + 3], w[K + 4], b));
  }
}

// Copy `len` staged bytes (shared, 16-byte aligned source with 16 bytes of slack on both
// sides) to global byte offset `pos` of `dst` (16-byte aligned base) by `nthr` threads.
// Interior 16-byte chunks are realigned with funnel shifts (the shift is uniform); the two
// partial edge chunks are written bytewise by 16 lanes each of the last warp.
__device__ __forceinline__ void copy_out(uint8_t* dst, uint64_t pos, const uint8_t* src,
                                         uint32_t len, int tid, int nthr) {
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
    case 0: copy_chunks<0>(g, s128, a, b, c0, c1, tid, nthr); break;
    case 1: copy_chunks<1>(g, s128, a, b, c0, c1, tid, nthr); break;
    case 2: copy_chunks<2>(g, s128, a, b, c0, c1, tid, nthr); break;
    default: copy_chunks<3>(g, s128, a, b, c0, c1, tid, nthr); break;
  }
  // edges: threads nthr-32 .. nthr-1 (the last warp): 16 lanes per partial chunk
  const int e = tid - (nthr - 32);
  if (e >= 0) {
    const bool head = e < 16;
    const uint32_t c = head ? 0 : nchunk - 1;
    const bool part = head ? head_partial : tail_partial;
    const int x = 16 * (int)c + (e & 15) - (int)a;  // staged index of this byte
    if (part && x >= 0 && x < (int)len) g[16 * c + (e & 15)] = src[x];
  }
}

// ------------------------------------------------------------------------------------------
// Pass 1 for one lane: classification already done.  Computes t, f, L, cb.
//   shift = s + 32 - 8q keeps the q high bytes of (x - mu) >> s right-aligned;
//   f = bfind((t ^ prev) | (q == 4)): code = min(3, lzb, q) = q - n with n = (f >> 3) + 1
//   (pipeline.py:84-91,112); the q == 4 sentinel caps the code at 3.
// cb = sum_i code_i 4^i = (q-1) * 0x55555555 - sum_i (f_i >> 3) 4^i, and with the running
// sums u_i the last sum telescopes to u_15 * 4^15 - 3 * sum_{i<15} u_i 4^i (one IMAD/elt).
__device__ __forceinline__ void pass1(Lane16& s, const float (&v)[16], float mu, uint32_t shift,
                                      uint32_t K, uint32_t prev, int q) {
#if SZX_K1_F2
  // two values per packed subtract: each lane of sub.rn.f32x2 is the IEEE RN float32
  // x - mu of pipeline.py:102
  uint64_t mu2;
  asm("mov.b64 %0, {%1, %1};" : "=l"(mu2) : "r"(__float_as_uint(mu)));
#pragma unroll
  for (int i = 0; i < 16; i += 2) {
    uint64_t x2, d2;
    uint32_t d0, d1;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x2) : "r"(__float_as_uint(v[i])), "r"(__float_as_uint(v[i + 1])));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d2) : "l"(x2), "l"(mu2));
    asm("mov.b64 {%0, %1}, %2;" : "=r"(d0), "=r"(d1) : "l"(d2));
    s.t[i] = shr_clamp(d0, shift);  // pipeline.py:102-106
    s.t[i + 1] = shr_clamp(d1, shift);
  }
#else
#pragma unroll
  for (int i = 0; i < 16; ++i)
    s.t[i] = shr_clamp(__float_as_uint(__fsub_rn(v[i], mu)), shift);  // pipeline.py:102-106
#endif
  int u = 0;
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t p = i ? s.t[i - 1] : prev;
    s.f[i] = flo32((s.t[i] ^ p) | K);
    u += s.f[i] >> 3;
    if (i < 15) acc += (uint32_t)u << (2 * i);
  }
  s.L = (uint32_t)(u + 16);
  const uint32_t sum_x = ((uint32_t)u << 30) - 3u * acc;
  s.cb = (uint32_t)(q - 1) * 0x55555555u - sum_x;
}

struct Cls {
  float mu;
  uint32_t req, shift, K;
  int q;
  bool nc;
};

// LPB-lane min/max + classification (pipeline.py:54-81); every lane of the group gets it.
// LPB = lanes per block = block size / 16 (8 for bs == 128).
template <int LPB = 8>
__device__ __forceinline__ Cls classify_group(float mn, float mx, const CompressArgs& a) {
#pragma unroll
  for (int d = 1; d < LPB; d <<= 1) {
    mn = fminf(mn, __shfl_xor_sync(kFull, mn, d));
    mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, d));
  }
  const BlockClass c = classify(mn, mx, a.e, a.pe);
  Cls r;
  r.mu = c.mu;
  r.req = (uint32_t)c.req;
  r.q = c.q;
  r.nc = !c.cst;
  // constant blocks: shift 32 makes every t zero, so they stage nothing (L = 0)
  r.shift = r.nc ? (uint32_t)(c.s + 32 - 8 * c.q) : 32u;
  r.K = (r.nc && c.q == 4) ? 1u : 0u;
  return r;
}

// Classify + pass 1 for one lane of a FULL tile (lane l of group w owns the 16 values
// 512 w + 16 l .. of the tile, i.e. of block (32 w + l) / LPB).
template <int LPB = 8>
__device__ __forceinline__ void encode_full(const float* in, int warp, int lane,
                                            const CompressArgs& a, Cls& c, Lane16& s) {
  float v[16];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float4 x = *reinterpret_cast<const float4*>(
        reinterpret_cast<const uint8_t*>(in) + swz_off(warp, lane, k));
    v[4 * k] = x.x; v[4 * k + 1] = x.y; v[4 * k + 2] = x.z; v[4 * k + 3] = x.w;
  }
  float mn = v[0], mx = v[0];
#pragma unroll
  for (int i = 1; i < 16; ++i) {
    mn = fminf(mn, v[i]);
    mx = fmaxf(mx, v[i]);
  }
  c = classify_group<LPB>(mn, mx, a);
  // predecessor of the lane's first value: the previous lane's last value in the same
  // block; the first value of a block has a zero predecessor (pipeline.py:108-111)
  const float pv = __shfl_up_sync(kFull, v[15], 1);
  if (!__any_sync(kFull, c.nc)) {  // the warp's blocks are all constant: nothing to encode
    s.L = 0;
    s.cb = 0;
    return;
  }
  const uint32_t pt =
      (lane & (LPB - 1)) ? shr_clamp(__float_as_uint(__fsub_rn(pv, c.mu)), c.shift) : 0u;
  pass1(s, v, c.mu, c.shift, c.K, pt, c.q);
}

// Classify + pass 1 for one lane of the chunk's last (partial) tile: values past n are
// excluded from min/max, keep no bytes and get zero codes.  Values of the last partial
// 32-value row are read from global memory (the TMA box only covers whole rows).
template <int LPB = 8>
__device__ __forceinline__ void encode_tail(int warp, int lane, const CompressArgs& a,
                                            uint64_t v0, Cls& c, Lane16& s, bool& exists) {
  const uint64_t n = a.n;
  const uint64_t first = v0 + (uint64_t)(warp * 32 + lane) * 16;  // this lane's first value
  const uint64_t bfirst = v0 + (uint64_t)((warp * 32 + lane) / LPB) * (16 * LPB);
  exists = bfirst < n;
  const int nlive = first >= n ? 0 : (int)umin64(16, n - first);
  float v[16];
  float mn = INFINITY, mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    v[i] = i < nlive ? a.x[first + i] : 0.f;
    if (i < nlive) {
      mn = fminf(mn, v[i]);
      mx = fmaxf(mx, v[i]);
    }
  }
  c = classify_group<LPB>(mn, mx, a);
  if (!exists) {
    c.nc = false;
    c.shift = 32;
    c.K = 0;
  }
  const float pv = __shfl_up_sync(kFull, v[15], 1);
  const uint32_t pt =
      (lane & (LPB - 1)) ? shr_clamp(__float_as_uint(__fsub_rn(pv, c.mu)), c.shift) : 0u;
  pass1(s, v, c.mu, c.shift, c.K, pt, c.q);
  // dead values: no bytes, zero codes (container.py:304-305 padding)
  uint32_t cb = 0;
  int L = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (i >= nlive) s.f[i] = -1;
    const int nkeep = (s.f[i] >> 3) + 1;
    L += nkeep;
    if (i < nlive && c.nc) cb |= (uint32_t)(c.q - nkeep) << (2 * i);
  }
  s.L = (uint32_t)L;
  s.cb = cb;
}

// host: the TMA tensor map of a chunk (compress.cu) and the SM count
cudaError_t make_tile_tmap(const float* x, uint64_t n, CUtensorMap* map,
                           uint32_t box_rows = kTileRows);
int sm_count();

}  // namespace k1
}  // namespace szx
