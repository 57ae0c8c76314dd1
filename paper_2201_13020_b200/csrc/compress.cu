// compress.cu -- SZx block encoder for sm_100a (K1 in DESIGN.md).
//
// Replaces the reference's whole compress path in ONE launch per chunk:
//   block_stats           pipeline.py:54-81   (== blockcodec.summarize_block 87-112)
//   _encode_elements      pipeline.py:94-133  (== blockcodec.encode_nonconstant 123-141)
//   prefix_scan + scatter parallel.py:21-44,104-140 / pipeline.py:143-166
// Output pools use the UFZX container layout (container.py:3-21): LSB-first constant map,
// mu per block, req per NC block, 2-bit codes packed LSB-first, mid bytes.
#include "szx_device.cuh"
#include "szx_kernels.h"

namespace szx {

// ----------------------------------------------------------------------------------------
// Fast path, bs == 128.  One CTA = 8 warps = 32 blocks = 4096 values (16 KiB of input).
// Lane l of a warp owns values 4l..4l+3 of a block, loaded as one 16-byte vector.
// ----------------------------------------------------------------------------------------
constexpr int kMidStage = kFastTileBlocks * 512 + 32;

__global__ void __launch_bounds__(kThreads, 3) compress128_kernel(CompressArgs a) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_wnc[kWarps], s_wmid[kWarps], s_wcst[kWarps];
  __shared__ uint32_t s_wnc_ex[kWarps], s_wmid_ex[kWarps];
  __shared__ uint32_t s_madj;
  __shared__ unsigned long long s_pre_nc, s_pre_mid;
  __shared__ __align__(16) uint8_t s_mid[kMidStage];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    s_tile = atomicAdd(a.counter, 1u);
    s_madj = 0;
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t n = a.n;
  const uint64_t nb = (n + 127) >> 7;
  const uint64_t b0 = (uint64_t)tile * kFastTileBlocks + (uint64_t)warp * kFastBPW;

  // ---- 1. loads: 4 x 16 B per lane in flight --------------------------------------------
  float4 v[kFastBPW];
#pragma unroll
  for (int j = 0; j < kFastBPW; ++j) {
    const uint64_t off = ((b0 + j) << 7) + (uint64_t)lane * 4;
    if (off + 4 <= n) {
      v[j] = ld_stream_f4(a.x + off);
    } else {
      v[j].x = off + 0 < n ? a.x[off + 0] : 0.f;
      v[j].y = off + 1 < n ? a.x[off + 1] : 0.f;
      v[j].z = off + 2 < n ? a.x[off + 2] : 0.f;
      v[j].w = off + 3 < n ? a.x[off + 3] : 0.f;
    }
  }

  // ---- 2. per-block classification (warp-uniform results) -------------------------------
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

  // ---- 3. encode: shifted words, XOR-with-previous leading-byte codes ---------------------
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
    // pipeline.py:102-106 -- float32 subtraction (RN, no FTZ), then the byte-aligning shift
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
      if (b0 + j == nb - 1 && cnt[j] < 128) s_madj = 128 - cnt[j];
    }
  }
  if (lane == 0) {
    s_wnc[warp] = w_nc;
    s_wmid[warp] = w_mid;
    s_wcst[warp] = w_cst;
  }
  __syncthreads();

  // ---- 4. tile aggregate + decoupled look-back (warp 0) --------------------------------
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
      if (tile == a.ntiles - 1) {  // chunk totals for the host / the next chunk
        const uint64_t cnc = hi_of(ex) + t_nc;
        a.totals->n_nc = bnc + cnc;
        a.totals->m = bm + 128 * cnc - s_madj;
        a.totals->mid_len = bmid + lo_of(ex) + t_mid;
        a.totals->pad = 0;
      }
    }
  }
  __syncthreads();

  // ---- 5. pool writes --------------------------------------------------------------------
  const uint64_t pre_mid = s_pre_mid;
  const uint32_t shift = (uint32_t)(pre_mid & 15);
  uint64_t r = s_pre_nc + s_wnc_ex[warp];
  uint32_t mpos = shift + s_wmid_ex[warp];
#pragma unroll
  for (int j = 0; j < kFastBPW; ++j) {
    if (cnt[j] == 0) continue;
    if (lane == j) a.mu[b0 + j] = bc[j].mu;  // container.py:14 -- mu for every block
    if (bc[j].cst) continue;
    if (lane == 0) a.req[r] = (uint8_t)bc[j].req;
    // 2-bit codes: NC block r owns bytes [32r, 32r + ceil(cnt/4)) (all earlier NC blocks
    // are full, so the pool stays byte-aligned block by block)
    if (lane * 4 < cnt[j]) a.codes[32 * r + lane] = (uint8_t)codeb[j];
    // mid bytes: big-endian bytes [c, q) of each shifted word, staged in shared memory
    const int q = bc[j].q;
    uint32_t p = mpos + loff[j];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = (codeb[j] >> (2 * i)) & 3;
      const bool live = lane * 4 + i < cnt[j];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (live && k >= c && k < q) s_mid[p++] = (uint8_t)(sh[j][i] >> (24 - 8 * k));
      }
    }
    mpos += btot[j];
    ++r;
  }
  __syncthreads();

  // constant map: 32 bits = 4 bytes per tile, LSB-first (container.py:12-13,321)
  if (tid == 0) {
    uint32_t bits = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) bits |= s_wcst[w] << (kFastBPW * w);
    const uint64_t tb = (uint64_t)tile * kFastTileBlocks;
    if (tb + kFastTileBlocks <= nb) {
      *reinterpret_cast<uint32_t*>(a.map + 4 * (uint64_t)tile) = bits;
    } else {
      const uint32_t nbytes = (uint32_t)((nb - tb + 7) >> 3);
      for (uint32_t i = 0; i < nbytes; ++i) a.map[4 * (uint64_t)tile + i] = (uint8_t)(bits >> (8 * i));
    }
  }

  // ---- 6. coalesced copy of the staged mid bytes --------------------------------------
  const uint32_t t_mid = s_wmid_ex[kWarps - 1] + s_wmid[kWarps - 1];
  const uint32_t end = shift + t_mid;
  uint8_t* dst = a.mid + (pre_mid - shift);
  const uint32_t nchunk = (end + 15) >> 4;
  for (uint32_t t = tid; t < nchunk; t += kThreads) {
    const uint32_t lo = t << 4, hi = lo + 16;
    if (lo >= shift && hi <= end) {
      *reinterpret_cast<uint4*>(dst + lo) = *reinterpret_cast<const uint4*>(s_mid + lo);
    } else {
      for (uint32_t i = max(lo, shift); i < min(hi, end); ++i) dst[i] = s_mid[i];
    }
  }
}

// ----------------------------------------------------------------------------------------
// Generic path, any bs in 8..65535.  One warp per block, 32 elements per step; three passes
// over the block (stats, counts, emit) with a look-back between counts and emit.
// Codes are OR-ed into a zero-initialised pool (blocks need not start on a code byte).
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

void launch_compress128(const CompressArgs& a, cudaStream_t s) {
  compress128_kernel<<<a.ntiles, kThreads, 0, s>>>(a);
}
void launch_compress_generic(const CompressArgs& a, cudaStream_t s) {
  compress_generic_kernel<<<a.ntiles, kThreads, 0, s>>>(a);
}

}  // namespace szx
