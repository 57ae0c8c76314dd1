// decompress.cu -- SZx block decoder for sm_100a (K2 in DESIGN.md).
//
// Replaces, in one launch per chunk:
//   decode_layout (q/s/codes/mid offsets)   pipeline.py:193-214
//   leading-byte resolution                 pipeline.py:227-260 / parallel.py:143-180
//                                           (index propagation, parallel.py:79-101)
//   _assemble                               pipeline.py:217-224
// Two decoupled look-back chains per tile: non-constant block count (from the map, ready
// immediately) and mid-byte count (needs the tile's codes, which need the first chain).
//
// Leading-byte resolution is a warp scan: element i owns byte columns [min(code,q), 4) of
// its word (own bytes from the mid pool, zeros past q); a word is the last owner of each
// column at or before i, with the zero word before the block start.  The operator
//   (w_a, m_a) . (w_b, m_b) = ((w_b & m_b) | (w_a & ~m_b), m_a | m_b)
// is associative, so the stride-doubling propagation of parallel.py:79-101 becomes five
// shuffle steps instead of ceil(log2 m) passes over memory.
#include "szx_device.cuh"
#include "szx_kernels.h"

namespace szx {

constexpr int kMidStageD = kFastTileBlocks * 512 + 48;

__device__ __forceinline__ uint32_t read_be4(const uint8_t* s, uint32_t p) {
  // 4 bytes starting at s[p] (unaligned), returned big-endian (s[p] in bits 31..24)
  const uint32_t* w = reinterpret_cast<const uint32_t*>(s);
  const uint32_t lo = w[p >> 2], hi = w[(p >> 2) + 1];
  const uint32_t le = __funnelshift_r(lo, hi, 8 * (p & 3));
  return __byte_perm(le, 0, 0x0123);
}

__global__ void __launch_bounds__(kThreads, 3) decompress128_kernel(DecompressArgs a) {
  __shared__ uint32_t s_tile, s_cbits;
  __shared__ uint32_t s_wmid[kWarps], s_wmid_ex[kWarps];
  __shared__ unsigned long long s_pre_nc, s_pre_mid;
  __shared__ __align__(16) uint8_t s_mid[kMidStageD];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(a.counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t n = a.n;
  const uint64_t nb = (n + 127) >> 7;
  const uint64_t tb = (uint64_t)tile * kFastTileBlocks;
  const int nvalid = (int)umin64(kFastTileBlocks, nb - tb);
  const uint32_t vmask = nvalid >= 32 ? kFull : ((1u << nvalid) - 1);

  // ---- chain 1: non-constant block count from the map ---------------------------------
  if (warp == 0) {
    uint32_t bits;
    if (nvalid == kFastTileBlocks) {
      bits = *reinterpret_cast<const uint32_t*>(a.map + 4 * (uint64_t)tile);
    } else {
      bits = 0;
      const int nbytes = (nvalid + 7) >> 3;
      for (int i = 0; i < nbytes; ++i) bits |= (uint32_t)a.map[4 * (uint64_t)tile + i] << (8 * i);
    }
    bits &= vmask;
    const uint32_t t_nc = __popc(~bits & vmask);
    const uint64_t ex = lookback(a.status_nc, tile, t_nc);
    if (lane == 0) {
      s_pre_nc = (a.base ? a.base->n_nc : 0) + ex;
      s_cbits = bits;
    }
  }
  __syncthreads();

  const uint32_t cbits = s_cbits;
  const uint64_t b0 = tb + (uint64_t)warp * kFastBPW;
  int cnt[kFastBPW], q[kFastBPW], s[kFastBPW];
  uint32_t codeb[kFastBPW], loff[kFastBPW], btot[kFastBPW];
  uint64_t rr[kFastBPW];
  uint32_t w_mid = 0;
#pragma unroll
  for (int j = 0; j < kFastBPW; ++j) {
    const int lb = warp * kFastBPW + j;
    cnt[j] = lb < nvalid ? (int)umin64(128, n - ((b0 + j) << 7)) : 0;
    q[j] = 0; s[j] = 0; codeb[j] = 0; loff[j] = 0; btot[j] = 0; rr[j] = 0;
    if (cnt[j] == 0 || ((cbits >> lb) & 1)) continue;
    const uint64_t r = s_pre_nc + __popc(~cbits & vmask & ((1u << lb) - 1));
    rr[j] = r;
    q_s_of(a.req[r], q[j], s[j]);
    const int nv = max(0, min(4, cnt[j] - lane * 4));
    const uint32_t cb = nv > 0 ? a.codes[32 * r + lane] : 0;
    codeb[j] = cb;
    uint32_t k = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = min((int)((cb >> (2 * i)) & 3), q[j]);  // pipeline.py:208
      k += i < nv ? (uint32_t)(q[j] - c) : 0;
    }
    const uint32_t incl = warp_incl_scan(k);
    loff[j] = incl - k;
    btot[j] = __shfl_sync(kFull, incl, 31);
    w_mid += btot[j];
  }
  if (lane == 0) s_wmid[warp] = w_mid;
  __syncthreads();

  // ---- chain 2: mid-byte count ---------------------------------------------------------
  if (warp == 0) {
    const uint32_t wm = lane < kWarps ? s_wmid[lane] : 0;
    const uint32_t in_m = warp_incl_scan(wm);
    if (lane < kWarps) s_wmid_ex[lane] = in_m - wm;
    const uint32_t t_mid = __shfl_sync(kFull, in_m, 31);
    const uint64_t ex = lookback(a.status_mid, tile, t_mid);
    if (lane == 0) {
      const uint64_t bmid = a.base ? a.base->mid_len : 0;
      s_pre_mid = bmid + ex;
      if (bmid + ex + t_mid > a.mid_len) atomicOr(a.err, kErrUnderrun);
      if (tile == a.ntiles - 1) {
        a.totals->n_nc = s_pre_nc + __popc(~cbits & vmask);
        a.totals->m = 0;
        a.totals->mid_len = bmid + ex + t_mid;
        a.totals->pad = 0;
      }
    }
  }
  __syncthreads();

  // ---- stage the tile's mid bytes (16-byte vectors, alignment-preserving) ----------------
  const uint64_t pre_mid = s_pre_mid;
  const uint32_t shift = (uint32_t)(pre_mid & 15);
  const uint32_t t_mid = s_wmid_ex[kWarps - 1] + s_wmid[kWarps - 1];
  const uint8_t* src = a.mid + (pre_mid - shift);
  const uint32_t nchunk = (shift + t_mid + 15) >> 4;
  const uint64_t cap = (a.mid_len + 15) & ~15ull;  // readable bytes (padded)
  for (uint32_t t = tid; t < nchunk; t += kThreads) {
    uint4 val = make_uint4(0, 0, 0, 0);
    if (pre_mid - shift + 16ull * t + 16 <= cap)
      val = __ldg(reinterpret_cast<const uint4*>(src + 16 * t));
    *reinterpret_cast<uint4*>(s_mid + 16 * t) = val;
  }
  __syncthreads();

  // ---- reconstruct ---------------------------------------------------------------------
  uint32_t mpos = shift + s_wmid_ex[warp];
#pragma unroll
  for (int j = 0; j < kFastBPW; ++j) {
    if (cnt[j] == 0) continue;
    const uint64_t b = b0 + j;
    const float mu = a.mu[b];
    if (lane == 0 && nonfinite(mu)) atomicOr(a.err, kErrMuNonFinite);  // container.py:198
    const uint64_t off = (b << 7) + (uint64_t)lane * 4;
    const int nv = max(0, min(4, cnt[j] - lane * 4));
    float4 o;
    if (q[j] == 0) {  // constant block: every value is mu (pipeline.py:219-220)
      o = make_float4(mu, mu, mu, mu);
    } else {
      const int qq = q[j];
      const uint32_t qmask = ~tail_mask(qq);  // columns [0, q)
      uint32_t p = mpos + loff[j];
      uint32_t w[4], m[4];
      uint32_t W = 0, M = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int c = min((int)((codeb[j] >> (2 * i)) & 3), qq);
        m[i] = tail_mask(c);
        w[i] = (read_be4(s_mid, p) >> (8 * c)) & m[i] & qmask;
        p += (uint32_t)(qq - c);
        W = (w[i] & m[i]) | (W & ~m[i]);
        M |= m[i];
      }
      // inclusive warp scan of (W, M) -- the index propagation
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t wu = __shfl_up_sync(kFull, W, d), mu_ = __shfl_up_sync(kFull, M, d);
        if (lane >= d) {
          W = (W & M) | (wu & ~M);
          M |= mu_;
        }
      }
      uint32_t P = __shfl_up_sync(kFull, W, 1);
      if (lane == 0) P = 0;  // the zero word before the block start
      float r[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        P = (w[i] & m[i]) | (P & ~m[i]);
        // pipeline.py:222-223 -- (w << s) as float32, + mu in float32
        r[i] = __fadd_rn(__uint_as_float(P << s[j]), mu);
      }
      o = make_float4(r[0], r[1], r[2], r[3]);
      mpos += btot[j];
      // the reference re-validates the output as a DataField (pipeline.py:224 ->
      // container.py:84-85); a corrupt stream can decode to inf / nan
      const bool bad = (nv > 0 && nonfinite(r[0])) || (nv > 1 && nonfinite(r[1])) ||
                       (nv > 2 && nonfinite(r[2])) || (nv > 3 && nonfinite(r[3]));
      if (__any_sync(kFull, bad) && lane == 0) atomicOr(a.err, kErrNonFinite);
    }
    if (nv == 4) {
      st_stream_f4(a.out + off, o);
    } else {
      if (nv > 0) a.out[off + 0] = o.x;
      if (nv > 1) a.out[off + 1] = o.y;
      if (nv > 2) a.out[off + 2] = o.z;
    }
  }
}

// ----------------------------------------------------------------------------------------
// Generic path, any bs in 8..65535: one warp per block, 32 elements per step.
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ int code_at(const uint8_t* codes, uint64_t g) {
  return (codes[g >> 2] >> (2 * (g & 3))) & 3;
}

__global__ void __launch_bounds__(kThreads) decompress_generic_kernel(DecompressArgs a) {
  __shared__ uint32_t s_tile, s_cbits;
  __shared__ uint32_t s_wmid[kWarps], s_wmid_ex[kWarps];
  __shared__ unsigned long long s_pre_nc, s_pre_mid;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(a.counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t n = a.n, bs = a.bs;
  const uint64_t nb = (n + bs - 1) / bs;
  const uint64_t tb = (uint64_t)tile * kGenTileBlocks;
  const int nvalid = (int)umin64(kGenTileBlocks, nb - tb);
  const uint32_t vmask = (1u << nvalid) - 1;

  if (warp == 0) {
    const uint32_t bits = a.map[tile] & vmask;
    const uint64_t ex = lookback(a.status_nc, tile, __popc(~bits & vmask));
    if (lane == 0) {
      s_pre_nc = (a.base ? a.base->n_nc : 0) + ex;
      s_cbits = bits;
    }
  }
  __syncthreads();
  const uint32_t cbits = s_cbits;
  const uint64_t b = tb + warp;
  const int cnt = warp < nvalid ? (int)umin64(bs, n - b * bs) : 0;
  const bool nc = cnt > 0 && !((cbits >> warp) & 1);
  int q = 0, s = 0;
  uint64_t g0 = 0;
  uint32_t btot = 0;
  if (nc) {
    const uint64_t r = s_pre_nc + __popc(~cbits & vmask & ((1u << warp) - 1));
    q_s_of(a.req[r], q, s);
    g0 = r * bs;
    for (int base = 0; base < cnt; base += 32) {
      const int i = base + lane;
      const uint32_t k = i < cnt ? (uint32_t)(q - min(code_at(a.codes, g0 + i), q)) : 0;
      btot += __reduce_add_sync(kFull, k);
    }
  }
  if (lane == 0) s_wmid[warp] = btot;
  __syncthreads();
  if (warp == 0) {
    const uint32_t wm = lane < kWarps ? s_wmid[lane] : 0;
    const uint32_t in_m = warp_incl_scan(wm);
    if (lane < kWarps) s_wmid_ex[lane] = in_m - wm;
    const uint32_t t_mid = __shfl_sync(kFull, in_m, 31);
    const uint64_t ex = lookback(a.status_mid, tile, t_mid);
    if (lane == 0) {
      const uint64_t bmid = a.base ? a.base->mid_len : 0;
      s_pre_mid = bmid + ex;
      if (bmid + ex + t_mid > a.mid_len) atomicOr(a.err, kErrUnderrun);
      if (tile == a.ntiles - 1) {
        a.totals->n_nc = s_pre_nc + __popc(~cbits & vmask);
        a.totals->m = 0;
        a.totals->mid_len = bmid + ex + t_mid;
        a.totals->pad = 0;
      }
    }
  }
  __syncthreads();
  if (cnt == 0) return;
  const float mu = a.mu[b];
  if (lane == 0 && nonfinite(mu)) atomicOr(a.err, kErrMuNonFinite);  // container.py:198
  float* ob = a.out + b * bs;
  if (!nc) {
    for (int i = lane; i < cnt; i += 32) ob[i] = mu;
    return;
  }
  uint64_t mpos = s_pre_mid + s_wmid_ex[warp];
  const uint32_t qmask = ~tail_mask(q);
  uint32_t carry = 0;  // resolved word of the previous element (zero word at block start)
  for (int base = 0; base < cnt; base += 32) {
    const int i = base + lane;
    const bool live = i < cnt;
    const int c = live ? min(code_at(a.codes, g0 + i), q) : q;
    const uint32_t k = (uint32_t)(q - c);
    const uint32_t incl = warp_incl_scan(k);
    uint64_t p = mpos + incl - k;
    uint32_t w = 0;
    for (int kk = c; kk < q; ++kk) {
      const uint32_t byte = p < a.mid_len ? a.mid[p] : 0;
      w |= byte << (24 - 8 * kk);
      ++p;
    }
    w &= qmask;
    uint32_t M = tail_mask(c), W = w & M;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t wu = __shfl_up_sync(kFull, W, d), mu_ = __shfl_up_sync(kFull, M, d);
      if (lane >= d) {
        W = (W & M) | (wu & ~M);
        M |= mu_;
      }
    }
    W = (W & M) | (carry & ~M);
    carry = __shfl_sync(kFull, W, 31);
    const float val = __fadd_rn(__uint_as_float(W << s), mu);
    if (live) ob[i] = val;
    if (__any_sync(kFull, live && nonfinite(val)) && lane == 0) atomicOr(a.err, kErrNonFinite);
    mpos += __shfl_sync(kFull, incl, 31);
  }
}

void launch_decompress128(const DecompressArgs& a, cudaStream_t s) {
  decompress128_kernel<<<a.ntiles, kThreads, 0, s>>>(a);
}
void launch_decompress_generic(const DecompressArgs& a, cudaStream_t s) {
  decompress_generic_kernel<<<a.ntiles, kThreads, 0, s>>>(a);
}

}  // namespace szx
