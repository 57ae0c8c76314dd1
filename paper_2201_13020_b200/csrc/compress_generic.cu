// compress_generic.cu -- SZx block encoder for any block size 8..65535 (K1, generic path).
//
// One warp per block, 32 elements per step; three passes over the block (stats, counts,
// emit) with a decoupled look-back between counts and emit.  Codes are OR-ed into a
// zero-initialised pool because blocks need not start on a code byte when bs % 4 != 0.
// Same reference lines as compress.cu (pipeline.py:54-174, blockcodec.py:87-141).
#include "szx_device.cuh"
#include "szx_kernels.h"

namespace szx {

// ----------------------------------------------------------------------------------------
__device__ __forceinline__ int gen_code(uint32_t sh, uint32_t prev, int q) {
  return min(min(3, __clz(sh ^ prev) >> 3), q);
}

__global__ void __launch_bounds__(kThreads) compress_generic_kernel(CompressArgs a) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_wnc[kWarps], s_wmid[kWarps], s_wcst[kWarps];
  __shared__ uint32_t s_wnc_ex[kWarps], s_wmid_ex[kWarps];
  __shared__ uint32_t s_madj;
  __shared__ unsigned long long s_pre_nc, s_pre_mid;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    s_tile = atomicAdd(a.counter, 1u);
    s_madj = 0;
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t n = a.n, bs = a.bs;
  const uint64_t nb = (n + bs - 1) / bs;
  const uint64_t b = (uint64_t)tile * kGenTileBlocks + warp;
  const int cnt = b < nb ? (int)umin64(bs, n - b * bs) : 0;
  const float* xb = a.x + b * bs;

  // pass 1: block min / max
  BlockClass bc{};
  if (cnt > 0) {
    float mn = INFINITY, mx = -INFINITY;
    for (int i = lane; i < cnt; i += 32) {
      const float x = xb[i];
      mn = fminf(mn, x);
      mx = fmaxf(mx, x);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(kFull, mn, d));
      mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, d));
    }
    bc = classify(mn, mx, a.e, a.pe);
  }
  const bool nc = cnt > 0 && !bc.cst;

  // pass 2: mid-byte count of the block
  uint32_t btot = 0;
  if (nc) {
    uint32_t carry = 0;
    for (int base = 0; base < cnt; base += 32) {
      const int i = base + lane;
      const bool live = i < cnt;
      const uint32_t sh = live ? __float_as_uint(__fsub_rn(xb[i], bc.mu)) >> bc.s : 0;
      uint32_t prev = __shfl_up_sync(kFull, sh, 1);
      if (lane == 0) prev = carry;
      carry = __shfl_sync(kFull, sh, 31);
      const uint32_t k = live ? (uint32_t)(bc.q - gen_code(sh, prev, bc.q)) : 0;
      btot += __reduce_add_sync(kFull, k);
    }
    if (lane == 0) {
      if (bc.req < 1) atomicOr(a.err, kErrBadReq);
      if (b == nb - 1 && (uint64_t)cnt < bs) s_madj = (uint32_t)(bs - cnt);
    }
  }
  if (lane == 0) {
    s_wnc[warp] = nc ? 1 : 0;
    s_wmid[warp] = btot;
    s_wcst[warp] = (cnt > 0 && bc.cst) ? 1 : 0;
  }
  __syncthreads();

  if (warp == 0) {
    const uint32_t wn = lane < kWarps ? s_wnc[lane] : 0;
    const uint32_t wm = lane < kWarps ? s_wmid[lane] : 0;
    const uint32_t in_n = warp_incl_scan(wn), in_m = warp_incl_scan(wm);
    if (lane < kWarps) {
      s_wnc_ex[lane] = in_n - wn;
      s_wmid_ex[lane] = in_m - wm;
    }
    const uint32_t t_nc = __shfl_sync(kFull, in_n, 31), t_mid = __shfl_sync(kFull, in_m, 31);
    const uint64_t ex = lookback(a.status, tile, pack2(t_nc, t_mid));
    if (lane == 0) {
      const uint64_t bnc = a.base ? a.base->n_nc : 0, bm = a.base ? a.base->m : 0;
      const uint64_t bmid = a.base ? a.base->mid_len : 0;
      s_pre_nc = bnc + hi_of(ex);
      s_pre_mid = bmid + lo_of(ex);
      if (tile == a.ntiles - 1) {
        const uint64_t cnc = hi_of(ex) + t_nc;
        a.totals->n_nc = bnc + cnc;
        a.totals->m = bm + bs * cnc - s_madj;
        a.totals->mid_len = bmid + lo_of(ex) + t_mid;
        a.totals->pad = 0;
      }
    }
    if (lane == 0) {
      // one map byte per tile (8 blocks), padding bits zero
      const uint64_t tb = (uint64_t)tile * kGenTileBlocks;
      if (tb < nb) {
        uint32_t bits = 0;
        for (int w = 0; w < kWarps; ++w) bits |= s_wcst[w] << w;
        a.map[tile] = (uint8_t)bits;
      }
    }
  }
  __syncthreads();

  if (cnt == 0) return;
  if (lane == 0) a.mu[b] = bc.mu;
  if (!nc) return;
  const uint64_t r = s_pre_nc + s_wnc_ex[warp];
  if (lane == 0) a.req[r] = (uint8_t)bc.req;
  const uint64_t g0 = r * bs;  // first NC element index of this block
  uint64_t mpos = s_pre_mid + s_wmid_ex[warp];
  uint32_t* codes32 = reinterpret_cast<uint32_t*>(a.codes);

  // pass 3: emit codes and mid bytes
  uint32_t carry = 0;
  for (int base = 0; base < cnt; base += 32) {
    const int i = base + lane;
    const bool live = i < cnt;
    const uint32_t sh = live ? __float_as_uint(__fsub_rn(xb[i], bc.mu)) >> bc.s : 0;
    uint32_t prev = __shfl_up_sync(kFull, sh, 1);
    if (lane == 0) prev = carry;
    carry = __shfl_sync(kFull, sh, 31);
    const int c = gen_code(sh, prev, bc.q);
    const uint32_t k = live ? (uint32_t)(bc.q - c) : 0;
    const uint32_t incl = warp_incl_scan(k);
    if (live) {
      const uint64_t g = g0 + i;
      if (c) atomicOr(codes32 + (g >> 4), (uint32_t)c << (2 * (g & 15)));
      uint64_t p = mpos + incl - k;
      for (int kk = c; kk < bc.q; ++kk) a.mid[p++] = (uint8_t)(sh >> (24 - 8 * kk));
    }
    mpos += __shfl_sync(kFull, incl, 31);
  }
}

void launch_compress_generic(const CompressArgs& a, cudaStream_t s) {
  compress_generic_kernel<<<a.ntiles, kThreads, 0, s>>>(a);
}

}  // namespace szx
