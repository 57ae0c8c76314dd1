// decompress_generic.cu -- SZx block decoder for any block size 8..65535 (K2, generic path).
//
// One warp per block, 32 elements per step, with two decoupled look-back chains per tile
// (non-constant block count, mid-byte count).  Same reference lines as decompress.cu
// (pipeline.py:193-260, parallel.py:79-180).
#include "szx_device.cuh"
#include "szx_kernels.h"

namespace szx {

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


void launch_decompress_generic(const DecompressArgs& a, cudaStream_t s) {
  decompress_generic_kernel<<<a.ntiles, kThreads, 0, s>>>(a);
}

}  // namespace szx
