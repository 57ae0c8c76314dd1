// decompress.cu -- SZx decoder for sm_100a, bs == 128 fast path (K3 index + K2 decode).
//
// Replaces:
//   decode_layout (q/s/codes/mid offsets, cumsum)  pipeline.py:193-214, container.py:246-253
//   leading-byte resolution                        pipeline.py:227-260, parallel.py:143-180
//                                                  (index propagation, parallel.py:79-101)
//   _assemble                                      pipeline.py:217-224
// in two launches -- "a scan of the stored sizes, then unpack and reconstruct":
//
// K3 index128_kernel: one CTA per 1024 blocks.  Map popcounts give the non-constant (NC)
//   block count per 32-block decode tile; a first decoupled look-back over those counts
//   locates the group's codes, whose per-block mid-byte counts (popcount algebra on packed
//   codes, one 32-byte code row per thread-step) feed a second look-back.  Output:
//   (NC blocks before, mid bytes before) for every decode tile, the mid-pool length, and
//   the container checks that need the pools.
//
// K2 decode128_kernel: persistent, warp-specialised, NO look-back.  A producer warp streams
//   each tile's mid bytes, codes, req, mu and map word into a 3-deep shared-memory ring with
//   1-D bulk copies (TMA engine); 8 compute warps (4 blocks each) rebuild the words.  A
//   word's leading bytes are resolved by a warp scan: element i owns byte columns
//   [min(code,q), 4) of its word; the operator
//     (w_a, m_a) . (w_b, m_b) = ((w_b & m_b) | (w_a & ~m_b), m_a | m_b)
//   is associative, so parallel.py:79-101's stride-doubling propagation becomes 5 shuffles.
#include "szx_device.cuh"
#include "szx_kernels.h"

namespace szx {

// =========================================================================================
// K3: tile index
// =========================================================================================
namespace {
constexpr int kIdxTiles = kIndexGroupTiles;              // decode tiles per group (32)
constexpr int kIdxBlocks = kIdxTiles * kFastTileBlocks;  // 1024 blocks per group
constexpr int kIdxThreads = 256;
constexpr int kIdxRowsPerThread = kIdxBlocks / kIdxThreads;  // 4

// sum over the 16 codes of a 32-bit code word of min(code, q)   (pipeline.py:208)
__device__ __forceinline__ uint32_t sum_min_codes(uint32_t w, int q) {
  const uint32_t lo = w & 0x55555555u, hi = (w >> 1) & 0x55555555u;
  if (q >= 3) return __popc(lo) + 2 * __popc(hi);
  if (q == 2) return __popc(lo) + 2 * __popc(hi) - __popc(lo & hi);
  return __popc(lo | hi);
}
}  // namespace

__global__ void __launch_bounds__(kIdxThreads) index128_kernel(IndexArgs a) {
  __shared__ uint32_t s_group, s_flags;
  __shared__ uint32_t s_cbits[kIdxTiles];
  __shared__ uint32_t s_ncpre[kIdxTiles + 1];
  __shared__ uint32_t s_blkmid[kIdxBlocks];
  __shared__ uint32_t s_tmid[kIdxTiles];
  __shared__ unsigned long long s_pre_nc;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    s_group = atomicAdd(a.counter, 1u);
    s_flags = 0;
  }
  __syncthreads();
  const uint32_t g = s_group;
  const uint64_t n = a.n, nb = (n + 127) >> 7;
  const uint64_t ntiles = (nb + kFastTileBlocks - 1) / kFastTileBlocks;
  const uint64_t t0 = (uint64_t)g * kIdxTiles;
  const int nt = (int)umin64(kIdxTiles, ntiles - t0);

  // ---- chain 1: NC blocks per decode tile, from the constant map -------------------------
  if (warp == 0) {
    uint32_t cb = 0, nc = 0;
    if (lane < nt) {
      const uint64_t t = t0 + lane;
      const uint64_t tb = t * kFastTileBlocks;
      const int nv = (int)umin64(kFastTileBlocks, nb - tb);
      const uint32_t vm = nv >= 32 ? kFull : ((1u << nv) - 1);
      const uint8_t* mp = a.map + 4 * t;
      if (nv == 32 && ((uintptr_t)mp & 3) == 0) {
        cb = *reinterpret_cast<const uint32_t*>(mp);
      } else {
        const int nbytes = (nv + 7) >> 3;
        for (int i = 0; i < nbytes; ++i) cb |= (uint32_t)mp[i] << (8 * i);
      }
      cb &= vm;
      nc = __popc(~cb & vm);
    }
    const uint32_t incl = warp_incl_scan(nc);
    s_cbits[lane] = cb;
    s_ncpre[lane] = incl - nc;
    if (lane == 31) s_ncpre[kIdxTiles] = incl;
    const uint64_t ex = lookback_wide<4>(a.status_nc, g, __shfl_sync(kFull, incl, 31));
    if (lane == 0) s_pre_nc = ex;
  }
  __syncthreads();

  const uint32_t nc_g = s_ncpre[kIdxTiles];
  const uint64_t pre_nc = s_pre_nc;
  // the field's last block may be short; it is the group's last NC block when it is NC
  uint32_t tail_rank = ~0u, tail_cnt = 128;
  if (t0 + nt == ntiles) {
    const uint64_t lastb = nb - 1;
    const uint32_t lb = (uint32_t)(lastb - t0 * kFastTileBlocks);
    if (!((s_cbits[lb >> 5] >> (lb & 31)) & 1)) {
      tail_rank = nc_g - 1;
      tail_cnt = (uint32_t)(n - lastb * 128);
    }
  }

  // ---- mid bytes per NC block: one 32-byte code row per thread, 4 rows in flight ---------
  uint32_t flags = 0;
  const uint8_t* crow0 = a.codes + 32 * pre_nc;
  const bool al16 = ((uintptr_t)crow0 & 15) == 0;
  uint4 rows[kIdxRowsPerThread][2];
  int rq[kIdxRowsPerThread];
#pragma unroll
  for (int u = 0; u < kIdxRowsPerThread; ++u) {
    const uint32_t r = tid + kIdxThreads * u;
    rows[u][0] = rows[u][1] = make_uint4(0, 0, 0, 0);
    rq[u] = 1;
    if (r < nc_g) {
      rq[u] = a.req[pre_nc + r];
      const uint8_t* p = crow0 + 32 * r;
      const uint32_t ncodes = r == tail_rank ? tail_cnt : 128;
      const uint32_t nbytes = (ncodes + 3) >> 2;  // code bytes present in the pool
      if (al16 && nbytes == 32) {
        rows[u][0] = *reinterpret_cast<const uint4*>(p);
        rows[u][1] = *reinterpret_cast<const uint4*>(p + 16);
      } else {
        uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (uint32_t i = 0; i < nbytes; ++i) w[i >> 2] |= (uint32_t)p[i] << (8 * (i & 3));
        rows[u][0] = make_uint4(w[0], w[1], w[2], w[3]);
        rows[u][1] = make_uint4(w[4], w[5], w[6], w[7]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kIdxRowsPerThread; ++u) {
    const uint32_t r = tid + kIdxThreads * u;
    if (r >= nc_g) continue;
    if (rq[u] < 1 || rq[u] > 32) flags |= kErrBadReq;  // container.py:206-207
    int q, s;
    q_s_of(rq[u], q, s);
    const uint32_t ncodes = r == tail_rank ? tail_cnt : 128;
    const uint32_t w[8] = {rows[u][0].x, rows[u][0].y, rows[u][0].z, rows[u][0].w,
                           rows[u][1].x, rows[u][1].y, rows[u][1].z, rows[u][1].w};
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t base = 16 * i;
      const uint32_t valid = ncodes <= base ? 0 : (ncodes - base >= 16 ? 16 : ncodes - base);
      const uint32_t live = valid >= 16 ? kFull : ((1u << (2 * valid)) - 1);
      if (w[i] & ~live) flags |= kErrCodePadding;  // container.py:304-305
      cnt += valid * q - sum_min_codes(w[i] & live, q);
    }
    s_blkmid[r] = cnt;
  }
  // mu of every block in the group must be finite (container.py:198-199)
  {
    const uint64_t gb0 = t0 * kFastTileBlocks;
    const uint64_t gbn = umin64(nb, gb0 + kIdxBlocks);
    for (uint64_t b = gb0 + tid; b < gbn; b += kIdxThreads)
      if (nonfinite(a.mu[b])) flags |= kErrMuNonFinite;
  }
  __syncthreads();

  // ---- per decode tile mid totals --------------------------------------------------------
  for (int t = warp; t < nt; t += kIdxThreads / 32) {
    const uint32_t r0 = s_ncpre[t], r1 = s_ncpre[t + 1];
    uint32_t v = lane < (int)(r1 - r0) ? s_blkmid[r0 + lane] : 0;
    v = __reduce_add_sync(kFull, v);
    if (lane == 0) s_tmid[t] = v;
  }
  flags = __reduce_or_sync(kFull, flags);
  if (lane == 0 && flags) atomicOr(&s_flags, flags);
  __syncthreads();

  // ---- chain 2: mid bytes; write the tile index -------------------------------------------
  if (warp == 0) {
    const uint32_t v = lane < nt ? s_tmid[lane] : 0;
    const uint32_t incl = warp_incl_scan(v);
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    const uint64_t ex = lookback_wide<4>(a.status_mid, g, total);
    if (lane < nt) {
      uint64_t* e = a.index + 2 * (t0 + lane);
      e[0] = pre_nc + s_ncpre[lane];
      e[1] = ex + incl - v;
    }
    if (lane == 0) {
      if (s_flags) atomicOr(a.err, s_flags);
      if (t0 + nt == ntiles) {  // closing entry + stream totals
        a.index[2 * ntiles] = pre_nc + nc_g;
        a.index[2 * ntiles + 1] = ex + total;
        *a.mid_total = ex + total;
        *a.nc_total = pre_nc + nc_g;
      }
    }
  }
}

void launch_index128(const IndexArgs& a, cudaStream_t s) {
  index128_kernel<<<a.ngroups, kIdxThreads, 0, s>>>(a);
}

// =========================================================================================
// K2: persistent decoder
// =========================================================================================
namespace {
constexpr int kDecWarps = 8;
constexpr int kDecThreads = (kDecWarps + 1) * 32;
constexpr int kDecStages = 3;

struct __align__(16) DecStage {
  uint8_t mid[kFastTileBlocks * 512 + 32];
  uint8_t codes[kFastTileBlocks * 32 + 32];
  uint8_t mu[kFastTileBlocks * 4 + 32];
  uint8_t req[kFastTileBlocks + 32];
  uint8_t map[32];
  uint32_t tile, mid_sh, codes_sh, mu_sh, req_sh, map_sh, pad0, pad1;
};

struct DecSmem {
  DecStage st[kDecStages];
  uint64_t full[kDecStages];
  uint64_t empty[kDecStages];
  uint32_t wmid[2][kDecWarps];
};

struct BulkPlan {
  const uint8_t* src;
  uint32_t bytes;
  uint32_t shift;
};

__device__ __forceinline__ BulkPlan plan(const uint8_t* base, uint64_t off, uint64_t len) {
  BulkPlan p;
  const uintptr_t s = (uintptr_t)(base + off);
  const uintptr_t a0 = s & ~(uintptr_t)15;
  p.src = reinterpret_cast<const uint8_t*>(a0);
  p.shift = (uint32_t)(s - a0);
  p.bytes = len ? (uint32_t)(((s + len + 15) & ~(uintptr_t)15) - a0) : 0;
  return p;
}

__device__ __forceinline__ uint32_t read_be4(const uint8_t* s, uint32_t p) {
  // 4 bytes starting at s[p] (unaligned), returned big-endian (s[p] in bits 31..24)
  const uint32_t* w = reinterpret_cast<const uint32_t*>(s);
  const uint32_t lo = w[p >> 2], hi = w[(p >> 2) + 1];
  return __byte_perm(__funnelshift_r(lo, hi, 8 * (p & 3)), 0, 0x0123);
}

// Rebuild the 4 values of one lane in one NC block with q == Q kept bytes.
// p: shared-memory offset of this lane's first mid byte.  Returns 4 floats.
template <int Q, bool FULL>
__device__ __forceinline__ float4 decode_lane(const uint8_t* mid, uint32_t p, uint32_t codeb,
                                              int s, float mu, int nv, int lane, bool& bad) {
  constexpr uint32_t kQMask = Q >= 4 ? 0xFFFFFFFFu : ~(0xFFFFFFFFu >> (8 * Q));  // columns [0,Q)
  uint32_t w[4], mk[4];
  uint32_t W = 0, M = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int c = (int)((codeb >> (2 * i)) & 3);
    if (Q < 3) c = c > Q ? Q : c;                 // pipeline.py:208 -- min(code, q)
    if (!FULL && i >= nv) {                       // past the tail: owns nothing
      mk[i] = 0;
      w[i] = 0;
    } else {
      mk[i] = 0xFFFFFFFFu >> (8 * c);               // own columns [c, 4); c <= 3
      w[i] = (read_be4(mid, p) >> (8 * c)) & kQMask;  // own bytes [c, Q), zeros past Q
      p += (uint32_t)(Q - c);
    }
    W = w[i] | (W & ~mk[i]);
    M |= mk[i];
  }
  // inclusive warp scan of (W, M): the index propagation of parallel.py:79-101.  Lanes
  // below d get their own values back from shfl_up, and combining a pair with itself is the
  // identity (W | (W & ~M) == W, M | M == M), so no lane predicate is needed.
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t wu = __shfl_up_sync(kFull, W, d), mu_ = __shfl_up_sync(kFull, M, d);
    W = W | (wu & ~M);
    M |= mu_;
  }
  uint32_t P = __shfl_up_sync(kFull, W, 1);
  if (lane == 0) P = 0;  // the zero word before the block start
  float r[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    P = w[i] | (P & ~mk[i]);
    // pipeline.py:222-223 -- (w << s) as float32, + mu in float32
    r[i] = __fadd_rn(__uint_as_float(P << s), mu);
    if (FULL || i < nv) bad |= !(fabsf(r[i]) <= 3.402823466e+38f);
  }
  return make_float4(r[0], r[1], r[2], r[3]);
}

template <bool FULL>
__device__ __forceinline__ void decode_tile(const Decode128Args& a, DecSmem& sm,
                                            const DecStage& S, uint32_t k, int warp, int lane,
                                            uint64_t n, uint64_t nb, uint64_t* st_slot) {
  const uint64_t tb = (uint64_t)S.tile * kFastTileBlocks;
  const int nvalid = FULL ? kFastTileBlocks : (int)umin64(kFastTileBlocks, nb - tb);
  const uint32_t vmask = nvalid >= 32 ? kFull : ((1u << nvalid) - 1);
  uint32_t cbits = 0;
  if (FULL && (S.map_sh & 3) == 0) {
    cbits = *reinterpret_cast<const uint32_t*>(&S.map[S.map_sh]);
  } else {
    const int nbytes = (nvalid + 7) >> 3;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i < nbytes) cbits |= (uint32_t)S.map[S.map_sh + i] << (8 * i);
    cbits &= vmask;
  }
  const uint64_t b0 = tb + (uint64_t)warp * kFastBPW;

  int cnt[kFastBPW], nv[kFastBPW], q[kFastBPW], sft[kFastBPW];
  uint32_t codeb[kFastBPW], lcnt[kFastBPW];
  float mu[kFastBPW];
#pragma unroll
  for (int j = 0; j < kFastBPW; ++j) {
    const int lb = warp * kFastBPW + j;
    if (FULL) {
      cnt[j] = 128;
      nv[j] = 4;
    } else {
      cnt[j] = lb < nvalid ? (int)umin64(128, n - ((b0 + j) << 7)) : 0;
      nv[j] = max(0, min(4, cnt[j] - lane * 4));
    }
    q[j] = 0; sft[j] = 0; codeb[j] = 0; lcnt[j] = 0;
    mu[j] = (FULL || cnt[j]) ? *reinterpret_cast<const float*>(&S.mu[S.mu_sh + 4 * lb]) : 0.f;
    if ((!FULL && cnt[j] == 0) || ((cbits >> lb) & 1)) continue;
    const uint32_t r = __popc(~cbits & vmask & ((1u << lb) - 1));
    q_s_of(S.req[S.req_sh + r], q[j], sft[j]);
    const uint32_t cb = (FULL || nv[j] > 0) ? S.codes[S.codes_sh + 32 * r + lane] : 0;
    codeb[j] = cb;
    uint32_t kk = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = min((int)((cb >> (2 * i)) & 3), q[j]);  // pipeline.py:208
      kk += (FULL || i < nv[j]) ? (uint32_t)(q[j] - c) : 0;
    }
    lcnt[j] = kk;
  }
  // mid-byte offsets: two packed (16-bit field) warp scans cover the 4 blocks
  const uint32_t pa = lcnt[0] | (lcnt[1] << 16), pb = lcnt[2] | (lcnt[3] << 16);
  const uint32_t ia = warp_incl_scan(pa), ib = warp_incl_scan(pb);
  const uint32_t ta = __shfl_sync(kFull, ia, 31), tb_ = __shfl_sync(kFull, ib, 31);
  const uint32_t ea = ia - pa, eb = ib - pb;
  const uint32_t btot[kFastBPW] = {ta & 0xFFFF, ta >> 16, tb_ & 0xFFFF, tb_ >> 16};
  const uint32_t loff[kFastBPW] = {ea & 0xFFFF, ea >> 16, eb & 0xFFFF, eb >> 16};
  // per-warp mid offsets inside the tile (double-buffered by tile parity)
  if (lane == 0) sm.wmid[k & 1][warp] = btot[0] + btot[1] + btot[2] + btot[3];
  named_bar(1, kDecWarps * 32);
  uint32_t mpos = S.mid_sh;
#pragma unroll
  for (int w = 0; w < kDecWarps; ++w)
    if (w < warp) mpos += sm.wmid[k & 1][w];

  float4 o[kFastBPW];
  bool bad = false, badmu = false;
#pragma unroll
  for (int j = 0; j < kFastBPW; ++j) {
    const float m = mu[j];
    badmu |= (FULL || cnt[j] > 0) && nonfinite(m);
    const uint32_t p = mpos + loff[j];
    switch (q[j]) {  // warp-uniform
      case 0: o[j] = make_float4(m, m, m, m); break;  // constant block (pipeline.py:219-220)
      case 2: o[j] = decode_lane<2, FULL>(S.mid, p, codeb[j], sft[j], m, nv[j], lane, bad); break;
      case 3: o[j] = decode_lane<3, FULL>(S.mid, p, codeb[j], sft[j], m, nv[j], lane, bad); break;
      case 4: o[j] = decode_lane<4, FULL>(S.mid, p, codeb[j], sft[j], m, nv[j], lane, bad); break;
      default: o[j] = decode_lane<1, FULL>(S.mid, p, codeb[j], sft[j], m, nv[j], lane, bad); break;
    }
    mpos += btot[j];
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(&sm.empty[k % kDecStages]);  // all reads of this stage done

  if (__any_sync(kFull, bad) && lane == 0) atomicOr(a.err, kErrNonFinite);
  if (__any_sync(kFull, badmu) && lane == 0) atomicOr(a.err, kErrMuNonFinite);
#pragma unroll
  for (int j = 0; j < kFastBPW; ++j) {
    if (!FULL && cnt[j] == 0) continue;
    float* dst = a.out + ((b0 + j) << 7) + lane * 4;
    if (FULL || nv[j] == 4) {
      st_stream_f4(dst, o[j]);
    } else {
      if (nv[j] > 0) dst[0] = o[j].x;
      if (nv[j] > 1) dst[1] = o[j].y;
      if (nv[j] > 2) dst[2] = o[j].z;
    }
  }
}
}  // namespace

__global__ void __launch_bounds__(kDecThreads, 2) decode128_kernel(Decode128Args a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  DecSmem& sm = *reinterpret_cast<DecSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t n = a.n, nb = (n + 127) >> 7;

  if (tid == 0) {
    for (int s = 0; s < kDecStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kDecWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  // ---------------------------------------------------------------- producer warp
  if (warp == kDecWarps) {
    if (lane == 0) {
      // the tile index entries are loaded one tile ahead, so their latency overlaps the
      // wait for a free slot instead of delaying the bulk copies
      auto load_idx = [&](uint64_t t, ulonglong2& x0, ulonglong2& x1) {
        if (t < a.ntiles) {
          x0 = *reinterpret_cast<const ulonglong2*>(a.index + 2 * t);
          x1 = *reinterpret_cast<const ulonglong2*>(a.index + 2 * t + 2);
        }
      };
      ulonglong2 n0 = make_ulonglong2(0, 0), n1 = make_ulonglong2(0, 0);
      load_idx(blockIdx.x, n0, n1);
      for (uint32_t k = 0;; ++k) {
        const int s = k % kDecStages;
        const uint64_t tile = (uint64_t)blockIdx.x + (uint64_t)k * gridDim.x;
        const ulonglong2 e0 = n0, e1 = n1;
        load_idx(tile + gridDim.x, n0, n1);
        mbar_wait(&sm.empty[s], ((k / kDecStages) & 1) ^ 1);
        DecStage& S = sm.st[s];
        if (tile >= a.ntiles) {
          S.tile = ~0u;
          mbar_arrive(&sm.full[s]);
          break;
        }
        const uint32_t nv = (uint32_t)umin64(kFastTileBlocks, nb - tile * kFastTileBlocks);
        uint64_t m0 = e0.y, m1 = e1.y;
        if (m1 > a.mid_len) {  // codes imply more mid bytes than present: never read past
          atomicOr(a.err, kErrUnderrun);
          m1 = a.mid_len;
          m0 = m0 < m1 ? m0 : m1;
        }
        const BulkPlan pm = plan(a.mid, m0, m1 - m0);
        const BulkPlan pc = plan(a.codes, 32 * e0.x, 32 * (e1.x - e0.x));
        const BulkPlan pu = plan(reinterpret_cast<const uint8_t*>(a.mu), 4 * tile * kFastTileBlocks, 4 * nv);
        const BulkPlan pr = plan(a.req, e0.x, e1.x - e0.x);
        const BulkPlan pp = plan(a.map, 4 * tile, (nv + 7) >> 3);
        S.tile = (uint32_t)tile;
        S.mid_sh = pm.shift;
        S.codes_sh = pc.shift;
        S.mu_sh = pu.shift;
        S.req_sh = pr.shift;
        S.map_sh = pp.shift;
        mbar_arrive_expect_tx(&sm.full[s], pm.bytes + pc.bytes + pu.bytes + pr.bytes + pp.bytes);
        if (pm.bytes) bulk_g2s(S.mid, pm.src, pm.bytes, &sm.full[s]);
        if (pc.bytes) bulk_g2s(S.codes, pc.src, pc.bytes, &sm.full[s]);
        bulk_g2s(S.mu, pu.src, pu.bytes, &sm.full[s]);
        if (pr.bytes) bulk_g2s(S.req, pr.src, pr.bytes, &sm.full[s]);
        bulk_g2s(S.map, pp.src, pp.bytes, &sm.full[s]);
      }
    }
    return;
  }

  // ---------------------------------------------------------------- compute warps
  for (uint32_t k = 0;; ++k) {
    const int st = k % kDecStages;
    mbar_wait(&sm.full[st], (k / kDecStages) & 1);
    const DecStage& S = sm.st[st];
    if (S.tile == ~0u) break;
    const bool full = ((uint64_t)S.tile + 1) * kFastTileBlocks * 128 <= n;
    if (full) decode_tile<true>(a, sm, S, k, warp, lane, n, nb, nullptr);
    else decode_tile<false>(a, sm, S, k, warp, lane, n, nb, nullptr);
  }
}

void launch_decode128(const Decode128Args& a, cudaStream_t s) {
  static bool configured = false;
  static int per_sm = 2;
  if (!configured) {
    cudaFuncSetAttribute(decode128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(DecSmem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode128_kernel, kDecThreads,
                                                  sizeof(DecSmem));
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
  const uint64_t want = (uint64_t)per_sm * nsm;
  const uint32_t grid = (uint32_t)(a.ntiles < want ? a.ntiles : want);
  decode128_kernel<<<grid, kDecThreads, sizeof(DecSmem), s>>>(a);
}

}  // namespace szx
