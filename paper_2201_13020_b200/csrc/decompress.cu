// decompress.cu -- SZx decoder for sm_100a, bs == 128 fast path (K3 index + K2 decode).
//
// Replaces:
//   decode_layout (q/s/codes/mid offsets, cumsum)  pipeline.py:193-214, container.py:246-253
//   leading-byte resolution                        pipeline.py:227-260, parallel.py:143-180
//                                                  (index propagation, parallel.py:79-101)
//   _assemble                                      pipeline.py:217-224
// in two launches -- "a scan of the stored sizes, then unpack and reconstruct":
//
// K3 index128_kernel: one CTA per 1024 blocks (16 decode tiles of 64 blocks).  Map
//   popcounts give the non-constant (NC) block count per tile; a first decoupled look-back
//   over those counts locates the group's codes, whose per-block mid-byte counts (popcount
//   algebra on packed codes, one 32-byte code row per thread-step) feed a second look-back.
//   Output per tile (64-byte entry): NC blocks before, mid bytes before, and the
//   tile-relative mid offset of each 4-block group; plus the mid-pool length and the
//   container checks that need the pools.
//
// K2 decode128_kernel: persistent, warp-specialised, NO look-back.  A producer warp streams
//   each tile's mid bytes, codes, req, mu, map and index entry into a 3-deep shared-memory
//   ring with 1-D bulk copies (TMA engine); 2 CTAs per SM, 16 compute warps each decoding 4
//   blocks, lane l
//   owning the 16 consecutive values 16(l&7).. of block l>>3 (the encoder's layout).  The
//   leading-byte reuse crosses lanes through an associative (K, V) scan over the block's 8
//   lanes -- K: byte columns the lane never writes, V: the columns' last written bytes --
//   the closed form of parallel.py:79-101's index propagation.  Each element then reads its
//   kept bytes column by column (predicated LDS.U8 into per-column registers that keep the
//   reused bytes), so no word is ever reassembled from shifted halves.
#include "szx_device.cuh"
#include "szx_kernels.h"

namespace szx {

// =========================================================================================
// K3: tile index
// =========================================================================================
namespace {
constexpr int kIdxTiles = kIndexGroupTiles;              // decode tiles per group (16)
constexpr int kIdxBlocks = kIdxTiles * kDecTileBlocks;   // 1024 blocks per group
constexpr int kIdxThreads = 256;
constexpr int kIdxRowsPerThread = kIdxBlocks / kIdxThreads;  // 4
constexpr int kIdxGroups = kIdxBlocks / kFastBPW;        // 4-block groups per CTA (256)

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
  __shared__ unsigned long long s_cbits[kIdxTiles];
  __shared__ uint32_t s_ncpre[kIdxTiles + 1];
  __shared__ uint32_t s_blkmid[kIdxBlocks];
  __shared__ uint32_t s_goff[kIdxGroups];
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
  const uint64_t ntiles = (nb + kDecTileBlocks - 1) / kDecTileBlocks;
  const uint64_t t0 = (uint64_t)g * kIdxTiles;
  const int nt = (int)umin64(kIdxTiles, ntiles - t0);

  // ---- chain 1: NC blocks per decode tile, from the constant map -------------------------
  if (warp == 0) {
    unsigned long long cb = 0;
    uint32_t nc = 0;
    if (lane < nt) {
      const uint64_t t = t0 + lane;
      const uint64_t tb = t * kDecTileBlocks;
      const int nv = (int)umin64(kDecTileBlocks, nb - tb);
      const unsigned long long vm = nv >= 64 ? ~0ull : ((1ull << nv) - 1);
      const uint8_t* mp = a.map + 8 * t;
      const int nbytes = (nv + 7) >> 3;
      if (nbytes == 8 && ((uintptr_t)mp & 3) == 0) {
        cb = (unsigned long long)reinterpret_cast<const uint32_t*>(mp)[0] |
             ((unsigned long long)reinterpret_cast<const uint32_t*>(mp)[1] << 32);
      } else {
        for (int i = 0; i < nbytes; ++i) cb |= (unsigned long long)mp[i] << (8 * i);
      }
      cb &= vm;
      nc = __popcll(~cb & vm);
      s_cbits[lane] = cb;
    }
    const uint32_t incl = warp_incl_scan(nc);
    if (lane < kIdxTiles) s_ncpre[lane] = incl - nc;
    if (lane == kIdxTiles - 1) s_ncpre[kIdxTiles] = incl;
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
    const uint32_t lb = (uint32_t)(lastb - t0 * kDecTileBlocks);
    if (!((s_cbits[lb >> 6] >> (lb & 63)) & 1)) {
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
    q_s_of(rq[u] > 32 ? 32 : rq[u], q, s);
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
    const uint64_t gb0 = t0 * kDecTileBlocks;
    const uint64_t gbn = umin64(nb, gb0 + kIdxBlocks);
    for (uint64_t b = gb0 + tid; b < gbn; b += kIdxThreads)
      if (nonfinite(a.mu[b])) flags |= kErrMuNonFinite;
  }
  __syncthreads();

  // ---- per 4-block group: mid bytes, tile-relative exclusive offsets, tile totals --------
  {
    const int t = tid / (kDecTileBlocks / kFastBPW);       // tile of this group (16 per tile)
    uint32_t gs = 0;
    if (t < nt) {
      const unsigned long long cb = s_cbits[t];
      const uint64_t tb = (t0 + t) * kDecTileBlocks;
      const int nv = (int)umin64(kDecTileBlocks, nb - tb);
      const unsigned long long ncm = ~cb & (nv >= 64 ? ~0ull : ((1ull << nv) - 1));
#pragma unroll
      for (int j = 0; j < kFastBPW; ++j) {
        const int lb = (tid % (kDecTileBlocks / kFastBPW)) * kFastBPW + j;  // block in tile
        if ((ncm >> lb) & 1) gs += s_blkmid[s_ncpre[t] + __popcll(ncm & ((1ull << lb) - 1))];
      }
    }
    // segmented (16-lane) inclusive scan: lanes 0-15 and 16-31 of a warp are two tiles
    uint32_t incl = gs;
#pragma unroll
    for (int d = 1; d < 16; d <<= 1) {
      const uint32_t v = __shfl_up_sync(kFull, incl, d);
      if ((lane & 15) >= d) incl += v;
    }
    s_goff[tid] = incl - gs;
    if ((lane & 15) == 15 && t < kIdxTiles) s_tmid[t] = incl;
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
      uint64_t* e = a.index + (kIndexEntryBytes / 8) * (t0 + lane);
      uint64_t wo[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t* o = &s_goff[16 * lane + 4 * i];
        wo[i] = (uint64_t)o[0] | ((uint64_t)o[1] << 16) | ((uint64_t)o[2] << 32) |
                ((uint64_t)o[3] << 48);
      }
      reinterpret_cast<ulonglong2*>(e)[0] = make_ulonglong2(pre_nc + s_ncpre[lane], ex + incl - v);
      reinterpret_cast<ulonglong2*>(e)[1] = make_ulonglong2(wo[0], wo[1]);
      reinterpret_cast<ulonglong2*>(e)[2] = make_ulonglong2(wo[2], wo[3]);
      reinterpret_cast<ulonglong2*>(e)[3] = make_ulonglong2(0, 0);
    }
    if (lane == 0) {
      if (s_flags) atomicOr(a.err, s_flags);
      if (t0 + nt == ntiles) {  // closing entry + stream totals
        uint64_t* e = a.index + (kIndexEntryBytes / 8) * ntiles;
        reinterpret_cast<ulonglong2*>(e)[0] = make_ulonglong2(pre_nc + nc_g, ex + total);
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
constexpr int kDecWarps = 16;                        // compute warps 0..15, producer warp 16
constexpr int kDecThreads = (kDecWarps + 1) * 32;
constexpr int kDecStages = 3;

struct __align__(16) DecStage {
  uint8_t slack[16];                                  // column loads may look 4 bytes back
  uint8_t mid[kDecTileBlocks * 512 + 32];
  uint8_t codes[kDecTileBlocks * 32 + 32];
  uint8_t mu[kDecTileBlocks * 4 + 32];
  uint8_t req[kDecTileBlocks + 32];
  uint8_t map[32];
  uint8_t idx[kIndexEntryBytes];                      // this tile's index entry (group offsets)
  uint32_t tile, mid_sh, codes_sh, mu_sh, req_sh, map_sh, pad0, pad1;
};

struct DecSmem {
  DecStage st[kDecStages];
  uint64_t full[kDecStages];
  uint64_t empty[kDecStages];
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

// 4 bytes at shared byte address `p` (any alignment), little-endian
__device__ __forceinline__ uint32_t lds_u32_any(const uint8_t* p) {
  const uintptr_t a = (uintptr_t)p;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
  return __funnelshift_r(w[0], w[1], 8 * (uint32_t)(a & 3));
}

// Unconditional byte load (inline asm, so it is never if-converted into a predicated load
// that would serialise the column chain).
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

template <int QM>
__device__ __forceinline__ uint32_t join_cols(uint32_t T0, uint32_t T1, uint32_t T2, uint32_t T3) {
  if (QM == 1) return T0;
  const uint32_t t01 = __byte_perm(T0, T1, 0x1140);
  if (QM == 2) return t01;
  if (QM == 3) return __byte_perm(t01, T2, 0x3410);
  return __byte_perm(t01, __byte_perm(T2, T3, 0x1140), 0x5410);
}

// Decode the 16 values of one lane.  m[k]: bit 2i set iff element i keeps > k bytes;
// tin: the kept-byte word of the element before the lane (previous lane's last, or 0);
// e: shared address of the lane's first mid byte; sh = 32 - 8q + s.
// Element i's kept bytes are [e_i - n_i, e_i) in big-endian order, so column k (0 = last
// kept byte) sits at e_i - 1 - k (pipeline.py:193-214, blockcodec.py:150-158); a column
// register keeps the reused byte when the element does not load it.
template <int QM>
__device__ __forceinline__ void decode16(float (&r)[16], const uint32_t (&m)[4], uint32_t tin,
                                         uint32_t e, uint32_t sh, float mu, float& amax) {
  uint32_t T0 = tin & 0xFF, T1 = (tin >> 8) & 0xFF, T2 = (tin >> 16) & 0xFF, T3 = tin >> 24;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t bit = 1u << (2 * i);
    const bool p0 = m[0] & bit, p1 = QM >= 2 && (m[1] & bit), p2 = QM >= 3 && (m[2] & bit),
               p3 = QM >= 4 && (m[3] & bit);
    if (p0) ++e;
    if (p1) ++e;
    if (p2) ++e;
    if (p3) ++e;
    const uint32_t l0 = lds_u8(e - 1);
    const uint32_t l1 = QM >= 2 ? lds_u8(e - 2) : 0u;
    const uint32_t l2 = QM >= 3 ? lds_u8(e - 3) : 0u;
    const uint32_t l3 = QM >= 4 ? lds_u8(e - 4) : 0u;
    T0 = p0 ? l0 : T0;
    if (QM >= 2) T1 = p1 ? l1 : T1;
    if (QM >= 3) T2 = p2 ? l2 : T2;
    if (QM >= 4) T3 = p3 ? l3 : T3;
    const uint32_t t = join_cols<QM>(T0, T1, T2, T3);
    // pipeline.py:222-223 -- (w << s) as float32, + mu in float32
    r[i] = __fadd_rn(__uint_as_float(t << sh), mu);
    float x;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(x) : "f"(amax), "f"(fabsf(r[i])));
    amax = x;
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

  // ---------------------------------------------------------------- producer warp (16)
  // (the issue arbiter favours the highest warp id: the producer's few instructions are
  // never starved by the compute warps)
  if (warp == kDecWarps) {
    if (lane == 0) {
      // the index entries are loaded one tile ahead, so their latency overlaps the wait for
      // a free slot instead of delaying the bulk copies
      const uint32_t ew = kIndexEntryBytes / 8;
      auto load_idx = [&](uint64_t t, ulonglong2& x0, ulonglong2& x1) {
        if (t < a.ntiles) {
          x0 = *reinterpret_cast<const ulonglong2*>(a.index + ew * t);
          x1 = *reinterpret_cast<const ulonglong2*>(a.index + ew * (t + 1));
        }
      };
      ulonglong2 n0 = make_ulonglong2(0, 0), n1 = make_ulonglong2(0, 0);
      load_idx(blockIdx.x, n0, n1);
      for (uint32_t k = 0;; ++k) {
        const int s = k % kDecStages;
        const uint64_t tile = (uint64_t)blockIdx.x + (uint64_t)k * gridDim.x;
        const ulonglong2 e0 = n0, e1 = n1;
        load_idx(tile + gridDim.x, n0, n1);
        mbar_wait_sleep(&sm.empty[s], ((k / kDecStages) & 1) ^ 1);
        DecStage& S = sm.st[s];
        if (tile >= a.ntiles) {
          S.tile = ~0u;
          mbar_arrive(&sm.full[s]);
          break;
        }
        const uint32_t nv = (uint32_t)umin64(kDecTileBlocks, nb - tile * kDecTileBlocks);
        uint64_t m0 = e0.y, m1 = e1.y;
        if (m1 > a.mid_len) {  // codes imply more mid bytes than present: never read past
          atomicOr(a.err, kErrUnderrun);
          m1 = a.mid_len;
          m0 = m0 < m1 ? m0 : m1;
        }
        if (m1 - m0 > kDecTileBlocks * 512) m1 = m0 + kDecTileBlocks * 512;  // corrupt index
        const BulkPlan pm = plan(a.mid, m0, m1 - m0);
        const BulkPlan pc = plan(a.codes, 32 * e0.x, 32 * (e1.x - e0.x));
        const BulkPlan pu = plan(reinterpret_cast<const uint8_t*>(a.mu), 4 * tile * kDecTileBlocks, 4 * nv);
        const BulkPlan pr = plan(a.req, e0.x, e1.x - e0.x);
        const BulkPlan pp = plan(a.map, 8 * tile, (nv + 7) >> 3);
        S.tile = (uint32_t)tile;
        S.mid_sh = pm.shift;
        S.codes_sh = pc.shift;
        S.mu_sh = pu.shift;
        S.req_sh = pr.shift;
        S.map_sh = pp.shift;
        mbar_arrive_expect_tx(&sm.full[s], pm.bytes + pc.bytes + pu.bytes + pr.bytes + pp.bytes +
                                               kIndexEntryBytes);
        if (pm.bytes) bulk_g2s(S.mid, pm.src, pm.bytes, &sm.full[s]);
        if (pc.bytes) bulk_g2s(S.codes, pc.src, pc.bytes, &sm.full[s]);
        bulk_g2s(S.mu, pu.src, pu.bytes, &sm.full[s]);
        if (pr.bytes) bulk_g2s(S.req, pr.src, pr.bytes, &sm.full[s]);
        bulk_g2s(S.map, pp.src, pp.bytes, &sm.full[s]);
        bulk_g2s(S.idx, a.index + ew * tile, kIndexEntryBytes, &sm.full[s]);
      }
    }
    return;
  }

  // ---------------------------------------------------------------- compute warps (0..15)
  const int cw = warp;
  const int jl = cw * kFastBPW + (lane >> 3);  // block of the tile this lane decodes
  const int g = lane & 7;                      // 16-value group within the block
  bool bad = false, badmu = false;
  const bool out32 = ((uintptr_t)a.out & 31) == 0;
  for (uint32_t k = 0;; ++k) {
    const int st = k % kDecStages;
    mbar_wait(&sm.full[st], (k / kDecStages) & 1);
    const DecStage& S = sm.st[st];
    if (S.tile == ~0u) break;
    const uint64_t tb = (uint64_t)S.tile * kDecTileBlocks;
    const int nvalid = (int)umin64(kDecTileBlocks, nb - tb);
    const unsigned long long vmask = nvalid >= 64 ? ~0ull : ((1ull << nvalid) - 1);
    unsigned long long cbits;
    {
      const uint8_t* mp = S.map + S.map_sh;
      cbits = (unsigned long long)lds_u32_any(mp) | ((unsigned long long)lds_u32_any(mp + 4) << 32);
      cbits &= vmask;
    }
    const bool exists = jl < nvalid;
    const bool nc = exists && !((cbits >> jl) & 1);
    const uint64_t b = tb + jl;
    const float mu = exists ? __uint_as_float(lds_u32_any(S.mu + S.mu_sh + 4 * jl)) : 0.f;
    // live values of this lane (the field's last block may be short)
    const int nlive = !exists ? 0 : (int)umin64(16, umin64(n - (b << 7), 128) > 16u * g
                                                        ? umin64(n - (b << 7), 128) - 16u * g : 0);
    uint32_t m[4] = {0, 0, 0, 0};
    int q = 0, sft = 0;
    uint32_t L = 0;
    if (nc) {
      const unsigned long long ncm = ~cbits & vmask;
      const uint32_t r = __popcll(ncm & ((1ull << jl) - 1));
      uint32_t cwd = lds_u32_any(S.codes + S.codes_sh + 32 * r + 4 * g);
      const uint32_t live = nlive >= 16 ? kFull : ((1u << (2 * nlive)) - 1);
      cwd &= live;
      int rq = S.req[S.req_sh + r];
      rq = rq < 1 ? 1 : (rq > 32 ? 32 : rq);  // K3 flags bad req; keep the decode in bounds
      q_s_of(rq, q, sft);
      // element i keeps n_i = q - min(code_i, q) bytes; column k is kept iff code < q - k
      const uint32_t lo = cwd & 0x55555555u, hi = (cwd >> 1) & 0x55555555u;
      const uint32_t lv = live & 0x55555555u;
      const uint32_t z1 = ~(lo | hi) & lv, z2 = ~hi & lv, z3 = ~(lo & hi) & lv;  // code < 1,2,3
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int th = q - c;  // column c kept iff code < th
        m[c] = th <= 0 ? 0u : th == 1 ? z1 : th == 2 ? z2 : th == 3 ? z3 : lv;
        L += __popc(m[c]);
      }
    }
    // lane offsets inside the tile's mid bytes: the group offset from the index + warp scan
    uint32_t incl = L;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += t;
    }
    const uint16_t* woff = reinterpret_cast<const uint16_t*>(S.idx + 16);
    // stream position (tile-relative) of the lane's first byte: blocks before this lane's
    // block in the warp are covered by the warp scan (stream order = lane order)
    const uint32_t start = woff[cw] + incl - L;
    const uint8_t* mid = S.mid + S.mid_sh;
    // (K, V): the lane's effect on the kept-byte word -- columns it never writes pass the
    // previous word through (K), the others end as its last writer left them (V)
    uint32_t K = 0, V = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (m[c]) {
        const int i = (31 - __clz(m[c])) >> 1;  // last element keeping column c
        const uint32_t upto = 0xFFFFFFFFu >> (30 - 2 * i);
        const uint32_t e = start + __popc(m[0] & upto) + __popc(m[1] & upto) +
                           __popc(m[2] & upto) + __popc(m[3] & upto);
        V |= (uint32_t)mid[e - 1 - c] << (8 * c);
      } else {
        K |= 0xFFu << (8 * c);
      }
    }
    // inclusive scan of (K, V) over the 8 lanes of the block (index propagation,
    // parallel.py:79-101): (K_a, V_a) then (K_b, V_b) = (K_a & K_b, (V_a & K_b) | V_b)
#pragma unroll
    for (int d = 1; d < 8; d <<= 1) {
      const uint32_t kp = __shfl_up_sync(kFull, K, d), vp = __shfl_up_sync(kFull, V, d);
      if (g >= d) {
        V = (vp & K) | V;
        K = kp & K;
      }
    }
    uint32_t tin = __shfl_up_sync(kFull, V, 1);
    if (g == 0) tin = 0;  // the zero word before the block start

    float r[16];
    float amax = 0.f;
    const uint32_t qm = __reduce_max_sync(kFull, nc ? (uint32_t)q : 0u);
    if (nc) {
      const uint32_t e = smem_u32(mid) + start;
      const uint32_t sh = (uint32_t)(32 - 8 * q + sft);
      switch (qm) {  // warp-uniform: largest q among the warp's NC blocks
        case 1: decode16<1>(r, m, tin, e, sh, mu, amax); break;
        case 2: decode16<2>(r, m, tin, e, sh, mu, amax); break;
        case 3: decode16<3>(r, m, tin, e, sh, mu, amax); break;
        default: decode16<4>(r, m, tin, e, sh, mu, amax); break;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = mu;  // constant block (pipeline.py:219-220)
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[st]);  // all reads of this stage done
    if (nc && !(amax <= 3.402823466e+38f)) {
      // only live values count (dead ones of a short last block are never stored)
      for (int i = 0; i < nlive; ++i) bad |= !(fabsf(r[i]) <= 3.402823466e+38f);
    }
    if (exists) badmu |= nonfinite(mu);
    float* dst = a.out + (b << 7) + 16 * g;
    if (nlive == 16 && out32) {  // two whole 32-byte sectors per lane
      st_stream_v8(dst, r);
      st_stream_v8(dst + 8, r + 8);
    } else if (nlive == 16) {
#pragma unroll
      for (int v = 0; v < 4; ++v)
        st_stream_f4(dst + 4 * v, make_float4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]));
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < nlive) dst[i] = r[i];
    }
  }
  if (__any_sync(kFull, bad) && lane == 0) atomicOr(a.err, kErrNonFinite);
  if (__any_sync(kFull, badmu) && lane == 0) atomicOr(a.err, kErrMuNonFinite);
}

void launch_decode128(const Decode128Args& a, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(decode128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(DecSmem));
    configured = true;
  }
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  static int per_sm = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode128_kernel, kDecThreads,
                                                  sizeof(DecSmem));
    if (per_sm < 1) per_sm = 1;
  }
  const uint64_t want = (uint64_t)nsm * per_sm;
  const uint32_t grid = (uint32_t)(a.ntiles < want ? a.ntiles : want);
  decode128_kernel<<<grid, kDecThreads, sizeof(DecSmem), s>>>(a);
}

}  // namespace szx
