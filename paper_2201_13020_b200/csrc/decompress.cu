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
// Per-launch phase counters of K3 (cycles summed over CTAs), profiling builds only
// (-DSZX_STATS): [0] phase 1 (map + look-back), [1] row loads + counts, [2] groups + entries,
// [3] phase 3 (look-back + rebase), [4] chunks, [5] phase-1 look-back alone, [6] phase-3
// look-back alone.
__device__ unsigned long long g_index_stats[8];
#ifdef SZX_STATS
#define IDX_T0(v) const long long v = clock64()
#define IDX_ADD(i, v) if (threadIdx.x == 0) atomicAdd(&g_index_stats[i], (unsigned long long)(clock64() - (v)))
#else
#define IDX_T0(v)
#define IDX_ADD(i, v)
#endif

__device__ unsigned long long g_decode_stats[8];

cudaError_t index_stats(unsigned long long* out8, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out8, g_index_stats, 8 * sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    e = cudaMemcpyToSymbol(g_index_stats, z, sizeof z);
  }
  return e;
}
cudaError_t decode_stats(unsigned long long* out8, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out8, g_decode_stats, 8 * sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    e = cudaMemcpyToSymbol(g_decode_stats, z, sizeof z);
  }
  return e;
}

namespace {
constexpr int kIdxTiles = 32 / kIndexCtasPerSm;          // decode tiles per chunk
constexpr int kIdxBlocks = kIdxTiles * kDecTileBlocks;   // 2048 blocks per chunk
constexpr int kIdxBufs = 2;                              // chunks in flight
constexpr int kIdxThreads = 512 / kIndexCtasPerSm;
constexpr int kIdxGroups = kIdxBlocks / kFastBPW;        // 4-block groups per chunk (512)
constexpr int kIdxMaxRanges = kIndexMaxRanges;          // grid size cap (abi.cu index_layout)
constexpr int kIdxMaxChunks = 1024;                      // per CTA: up to 2M blocks

// sum over the 16 codes of a 32-bit code word of min(code, q)   (pipeline.py:208)
// = #(code >= 1) + [q >= 2] #(code >= 2) + [q >= 3] #(code >= 3): the even bits of
// (w | w >> 1) are (code >= 1), the odd bits of w (code >= 2), the even bits of (w & w >> 1)
// (code >= 3).  Branch-free (rows of one warp have different q), popcounts on the XU pipe.
__device__ __forceinline__ uint32_t sum_min_codes(uint32_t w, uint32_t m2, uint32_t m3) {
  return __popc(((w | (w >> 1)) & 0x55555555u) | (w & m2)) + __popc(w & (w >> 1) & m3);
}
__device__ __forceinline__ void min_code_masks(int q, uint32_t& m2, uint32_t& m3) {
  m2 = q >= 2 ? 0xAAAAAAAAu : 0u;
  m3 = q >= 3 ? 0x55555555u : 0u;
}

// constant-map word of decode tile t (64 blocks, LSB-first), masked to the tile's blocks
__device__ __forceinline__ unsigned long long map_word(const uint8_t* map, uint64_t t, uint64_t nb,
                                                       int& nv) {
  const uint64_t tb = t * kDecTileBlocks;
  nv = (int)umin64(kDecTileBlocks, nb - tb);
  const uint8_t* mp = map + 8 * t;
  const int nbytes = (nv + 7) >> 3;
  unsigned long long cb = 0;
  if (nbytes == 8 && ((uintptr_t)mp & 3) == 0) {
    cb = (unsigned long long)reinterpret_cast<const uint32_t*>(mp)[0] |
         ((unsigned long long)reinterpret_cast<const uint32_t*>(mp)[1] << 32);
  } else {
    for (int i = 0; i < nbytes; ++i) cb |= (unsigned long long)mp[i] << (8 * i);
  }
  return cb & (nv >= 64 ? ~0ull : ((1ull << nv) - 1));
}

// Block sizes 64 / 128 / 256 / 512 index 8192-value tiles (8192 / bs blocks); the buffers
// are sized for the most blocks per tile (bs 64: 128).
constexpr int kIdxMaxTB = 128;
constexpr int kIdxMaxBlocks = kIdxTiles * kIdxMaxTB;

// constant-map bits of tile t (kTB blocks, LSB-first) as kMapW words, masked to its blocks
template <int BS>
__device__ __forceinline__ void map_words(const uint8_t* map, uint64_t t, uint64_t nb, int& nv,
                                          uint32_t (&w)[4]) {
  constexpr int kTB = 8192 / BS, kBytes = kTB / 8;
  const uint64_t tb = t * kTB;
  nv = (int)umin64(kTB, nb - tb);
  const uint8_t* mp = map + (uint64_t)kBytes * t;
  const int nbytes = (nv + 7) >> 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) w[i] = 0;
  if (nbytes == kBytes && kBytes >= 4 && ((uintptr_t)mp & 3) == 0) {
#pragma unroll
    for (int i = 0; i < (kBytes >= 4 ? kBytes / 4 : 1); ++i) w[i] = reinterpret_cast<const uint32_t*>(mp)[i];
  } else {
    for (int i = 0; i < nbytes; ++i) w[i >> 2] |= (uint32_t)mp[i] << (8 * (i & 3));
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int vb = nv - 32 * i;
    w[i] &= vb >= 32 ? kFull : vb <= 0 ? 0u : ((1u << vb) - 1);
  }
}

struct IdxBuf {
  uint8_t codes[kIdxBlocks * 32 + 32];      // 2048 code bytes per tile for every block size
  uint8_t req[kIdxMaxBlocks + 32];
  uint8_t mu[kIdxMaxBlocks * 4 + 32];
  uint8_t map[kIdxTiles * kIdxMaxTB / 8 + 32];
  uint32_t codes_sh, req_sh, mu_sh, map_sh;
};
struct IdxSmem {
  IdxBuf buf[kIdxBufs];
  uint32_t cmap[kIdxTiles][4];               // each tile's constant-map words
  uint32_t ncpre[kIdxTiles + 1];
  uint32_t blkmid[kIdxMaxBlocks];
  uint32_t goff[kIdxGroups];
  uint32_t tmid[kIdxTiles];
  uint32_t cnc[kIdxMaxChunks + 1];           // NC blocks per chunk -> exclusive prefix
  uint32_t red[kIdxThreads / 32];
  uint64_t full[kIdxBufs];
  unsigned long long base;
};

struct Plan16 {
  const uint8_t* src;
  uint32_t bytes, shift;
};
__device__ __forceinline__ Plan16 plan16(const uint8_t* base, uint64_t off, uint64_t len) {
  Plan16 p;
  const uintptr_t s = (uintptr_t)(base + off);
  const uintptr_t a0 = s & ~(uintptr_t)15;
  p.src = reinterpret_cast<const uint8_t*>(a0);
  p.shift = (uint32_t)(s - a0);
  p.bytes = len ? (uint32_t)(((s + len + 15) & ~(uintptr_t)15) - a0) : 0;
  return p;
}

// 4 bytes at shared byte address `p` (any alignment), little-endian
__device__ __forceinline__ uint32_t lds32_any(const uint8_t* p) {
  const uintptr_t a = (uintptr_t)p;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
  return __funnelshift_r(w[0], w[1], 8 * (uint32_t)(a & 3));
}
}  // namespace

// One CTA per SM, each owning a contiguous range of decode tiles:
//   1. NC blocks per 2048-block chunk of the range (map popcounts) -> decoupled look-back
//      over the CTAs for the range's first NC block;
//   2. each chunk's code rows and req bytes arrive by ONE bulk copy each (TMA engine, double
//      buffered: chunk j+2 is in flight while chunk j is counted), per-block mid counts,
//      per-group offsets, index entries (mid bytes relative to the range start);
//   3. the range's mid total -> second look-back over the CTAs; every entry gets the base.
// Batched (kBatch): blockIdx.y is the field, `fields[blockIdx.y]` its arguments, and the
// field's own a.ngroups CTAs (of the grid's gridDim.x) index it.
template <bool kBatch, int BS = 128>
__global__ void __launch_bounds__(kIdxThreads, kIndexCtasPerSm)
    index128_kernel(IndexArgs a0, const IndexArgs* __restrict__ fields) {
  constexpr int kLPB = BS / 16, kBPW = 32 / kLPB, kTB = 16 * kBPW;  // decode tile = kTB blocks
  constexpr int kMapW = (kTB + 31) / 32, kRowW = BS / 16;           // map words, code row words
  extern __shared__ __align__(128) uint8_t idx_smem_raw[];
  IdxSmem& sm = *reinterpret_cast<IdxSmem*>(idx_smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const IndexArgs a = kBatch ? fields[blockIdx.y] : a0;
  const uint32_t c = blockIdx.x, G = kBatch ? a.ngroups : gridDim.x;
  if (kBatch && c >= G) return;
  const uint64_t n = a.n, nb = (n + BS - 1) / BS;
  const uint64_t ntiles = (nb + kTB - 1) / kTB;
  const uint64_t r0 = ntiles * c / G, r1 = ntiles * (c + 1) / G;  // this CTA's tiles
  const uint32_t nch = (uint32_t)((r1 - r0 + kIdxTiles - 1) / kIdxTiles);
  const uint32_t ew = kIndexEntryBytes / 8;
  uint32_t flags = 0;

  if (tid == 0) {
    for (int b = 0; b < kIdxBufs; ++b) mbar_init(&sm.full[b], 1);
    fence_barrier_init();
  }
  for (uint32_t j = tid; j <= nch; j += kIdxThreads) sm.cnc[j] = 0;
  __syncthreads();

  // ---- 1. NC blocks per chunk of the range; NC blocks before the range --------------------
  IDX_T0(t_p1);
  for (uint64_t t = r0 + tid; t < r1; t += kIdxThreads) {
    int nv;
    uint32_t w[4];
    map_words<BS>(a.map, t, nb, nv, w);
    uint32_t nc = nv;
#pragma unroll
    for (int i = 0; i < kMapW; ++i) nc -= __popc(w[i]);
    atomicAdd(&sm.cnc[(t - r0) / kIdxTiles], nc);
  }
  // small maps (<= 2 MiB, 16 M blocks): every CTA sums the map words before its range
  // directly (L2-resident, no cross-CTA wait); larger ones use a decoupled look-back
  const bool direct = nb <= a.direct_limit;
  uint32_t before = 0;
  if (direct) {
    // tiles before the range are full: NC = blocks - popcount of their map bytes
    // [0, r0 kTB / 8); 16 independent 4-byte loads in flight per thread
    const uint64_t nbytes = r0 * (kTB / 8);
    uint32_t pop = 0;
    uint64_t done = 0;
    if (((uintptr_t)a.map & 3) == 0) {
      const uint32_t* m32 = reinterpret_cast<const uint32_t*>(a.map);
      const uint64_t nw = nbytes >> 2;
      for (; done + 16 * kIdxThreads <= nw; done += 16 * kIdxThreads) {
        uint32_t w[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) w[u] = __ldg(m32 + done + (uint64_t)u * kIdxThreads + tid);
#pragma unroll
        for (int u = 0; u < 16; ++u) pop += __popc(w[u]);
      }
      for (uint64_t i = done + tid; i < nw; i += kIdxThreads) pop += __popc(__ldg(m32 + i));
      done = nw << 2;  // bytes
    }
    for (uint64_t i = done + tid; i < nbytes; i += kIdxThreads) pop += __popc((uint32_t)a.map[i]);
    // before = r0 kTB - pop: each thread's share (the warp and CTA sums follow)
    before = (tid == 0 ? (uint32_t)(r0 * kTB) : 0u) - pop;
    before = __reduce_add_sync(kFull, before);
    if (lane == 0) sm.red[warp] = before;
  }
  __syncthreads();
  if (warp == 0) {  // exclusive prefix over the chunks (range-relative)
    uint32_t carry = 0;
    for (uint32_t j0 = 0; j0 <= nch; j0 += 32) {
      const uint32_t j = j0 + lane;
      const uint32_t v = j < nch ? sm.cnc[j] : 0u;
      const uint32_t incl = warp_incl_scan(v) + carry;
      if (j <= nch) sm.cnc[j] = incl - v;
      carry = __shfl_sync(kFull, incl, 31);
    }
    uint64_t ex;
    if (direct) {
      const uint32_t v = lane < kIdxThreads / 32 ? sm.red[lane] : 0u;
      ex = __reduce_add_sync(kFull, v);
    } else {
      IDX_T0(t_lb1);
      ex = lookback_wide<4>(a.status_nc, c, carry);  // carry = range NC total
      IDX_ADD(5, t_lb1);
    }
    if (lane == 0) sm.base = ex;
  }
  __syncthreads();
  IDX_ADD(0, t_p1);
  const uint64_t pre_nc_range = sm.base;

  // producer: chunk j's code rows, req bytes, mu and map words (contiguous pool ranges)
  auto issue = [&](uint32_t j) {
    IdxBuf& B = sm.buf[j % kIdxBufs];
    uint64_t* bar = &sm.full[j % kIdxBufs];
    const uint64_t nc0 = pre_nc_range + sm.cnc[j], nc1 = pre_nc_range + sm.cnc[j + 1];
    const uint64_t t0 = r0 + (uint64_t)j * kIdxTiles;
    const uint64_t ntc = umin64(kIdxTiles, r1 - t0);
    const uint64_t b0 = t0 * kTB, nbc = umin64(nb, b0 + ntc * kTB) - b0;
    const Plan16 pc = plan16(a.codes, (BS / 4) * nc0, (BS / 4) * (nc1 - nc0));
    const Plan16 pr = plan16(a.req, nc0, nc1 - nc0);
    const Plan16 pu = plan16(reinterpret_cast<const uint8_t*>(a.mu), 4 * b0, 4 * nbc);
    const Plan16 pp = plan16(a.map, (kTB / 8) * t0, (nbc + 7) >> 3);
    B.codes_sh = pc.shift;
    B.req_sh = pr.shift;
    B.mu_sh = pu.shift;
    B.map_sh = pp.shift;
    mbar_arrive_expect_tx(bar, pc.bytes + pr.bytes + pu.bytes + pp.bytes);
    if (pc.bytes) bulk_g2s(B.codes, pc.src, pc.bytes, bar);
    if (pr.bytes) bulk_g2s(B.req, pr.src, pr.bytes, bar);
    bulk_g2s(B.mu, pu.src, pu.bytes, bar);
    bulk_g2s(B.map, pp.src, pp.bytes, bar);
  };
  if (tid == 0)
    for (uint32_t j = 0; j < nch && j < kIdxBufs; ++j) issue(j);
  uint64_t run_mid = 0;  // mid bytes before the current chunk (range-relative)

  // ---- 2. chunks of 32 tiles ----------------------------------------------------------------
  for (uint32_t j = 0; j < nch; ++j) {
    IDX_T0(t_rows);
#ifdef SZX_STATS
    if (tid == 0) atomicAdd(&g_index_stats[4], 1ull);
#endif
    const uint64_t ct0 = r0 + (uint64_t)j * kIdxTiles;
    const int nt = (int)umin64(kIdxTiles, r1 - ct0);
    const uint64_t run_nc = pre_nc_range + sm.cnc[j];
    IDX_T0(t_w);
    mbar_wait(&sm.full[j % kIdxBufs], (j / kIdxBufs) & 1);
    IDX_ADD(5, t_w);
    const IdxBuf& B = sm.buf[j % kIdxBufs];
    // mu of every block in the chunk must be finite (container.py:198-199)
    {
      const uint32_t nbc = (uint32_t)(umin64(nb, (ct0 + nt) * kTB) - ct0 * kTB);
      for (uint32_t b = tid; b < nbc; b += kIdxThreads)
        if (nonfinite(__uint_as_float(lds32_any(B.mu + B.mu_sh + 4 * b)))) flags |= kErrMuNonFinite;
    }
    // per-tile NC counts (warp 0: one tile per lane), from the staged map words
    if (warp == 0) {
      uint32_t nc = 0;
      if (lane < nt) {
        const uint64_t tb = (ct0 + lane) * kTB;
        const int nv = (int)umin64(kTB, nb - tb);
        const uint8_t* mp = B.map + B.map_sh + (kTB / 8) * lane;
        nc = nv;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int vb = nv - 32 * w;
          const uint32_t vm = vb >= 32 ? kFull : vb <= 0 ? 0u : ((1u << vb) - 1);
          const uint32_t cw = w < kMapW ? lds32_any(mp + 4 * w) & vm : 0u;
          sm.cmap[lane][w] = cw;
          nc -= __popc(cw);
        }
      }
      const uint32_t incl = warp_incl_scan(nc);
      if (lane < kIdxTiles) sm.ncpre[lane] = incl - nc;
      if (lane == kIdxTiles - 1) sm.ncpre[kIdxTiles] = incl;
    }
    __syncthreads();
    const uint32_t nc_c = sm.ncpre[kIdxTiles];
    // the field's last block may be short; it is the chunk's last NC block when it is NC
    uint32_t tail_rank = ~0u, tail_cnt = 128;
    if (ct0 + nt == ntiles) {
      const uint64_t lastb = nb - 1;
      const uint32_t lb = (uint32_t)(lastb - ct0 * kTB);
      if (!((sm.cmap[lb / kTB][(lb % kTB) >> 5] >> (lb & 31)) & 1)) {
        tail_rank = nc_c - 1;
        tail_cnt = (uint32_t)(n - lastb * BS);
      }
    }
    const bool al16 = (B.codes_sh & 15) == 0;
    // mid bytes per NC block from the staged code rows: 4 independent rows per thread in
    // flight (the chain LDS -> popcounts -> sum is latency-bound one row at a time)
    // code word i (16 codes) of NC row r: a row is BS / 4 bytes = kRowW words
    auto row_word4 = [&](uint32_t r, int i, uint32_t (&w)[4]) {  // words i .. i + 3
      const uint8_t* p = B.codes + B.codes_sh + (BS / 4) * r + 4 * i;
      if (al16) {
        const uint4 x = *reinterpret_cast<const uint4*>(p);
        w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = lds32_any(p + 4 * k);
      }
    };
    auto row_q = [&](uint32_t r) {
      const int rq = B.req[B.req_sh + r];
      if (rq < 1 || rq > 32) flags |= kErrBadReq;  // container.py:206-207
      int q, s;
      q_s_of(rq > 32 ? 32 : (rq < 1 ? 1 : rq), q, s);
      return q;
    };
    for (uint32_t r0 = tid; r0 < nc_c; r0 += 4 * kIdxThreads) {
      uint32_t cnt[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t r = r0 + u * kIdxThreads;
        cnt[u] = 0;
        if (r < nc_c) {
          const int q = row_q(r);
          uint32_t m2, m3;
          min_code_masks(q, m2, m3);
          cnt[u] = BS * q;
#pragma unroll
          for (int i = 0; i < kRowW; i += 4) {
            uint32_t w[4];
            row_word4(r, i, w);
#pragma unroll
            for (int k = 0; k < 4; ++k) cnt[u] -= sum_min_codes(w[k], m2, m3);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (r0 + u * kIdxThreads < nc_c) sm.blkmid[r0 + u * kIdxThreads] = cnt[u];
    }
    // the field's short last block: codes past the field's end are absent from the pool
    // (zero padding bits); recounted by the thread that counted it as a full row above
    if (tail_rank != ~0u && tid == (int)(tail_rank % kIdxThreads)) {
      const uint32_t r = tail_rank;
      const int q = row_q(r);
      uint32_t m2, m3;
      min_code_masks(q, m2, m3);
      const uint32_t ncodes = tail_cnt;
      const uint32_t nbytes = (ncodes + 3) >> 2;
      uint32_t cnt = 0;
#pragma unroll
      for (int i = 0; i < kRowW; ++i) {
        uint32_t w4[4];
        row_word4(r, i & ~3, w4);
        const uint32_t base = 16 * i;
        // bytes past the pool's code bytes were not part of the stream: ignore them
        const uint32_t bytes_here = nbytes <= 4 * (uint32_t)i ? 0 : umin64(4, nbytes - 4 * i);
        const uint32_t wmask = bytes_here >= 4 ? kFull : ((1u << (8 * bytes_here)) - 1);
        const uint32_t wi = w4[i & 3] & wmask;
        const uint32_t valid = ncodes <= base ? 0 : (ncodes - base >= 16 ? 16 : ncodes - base);
        const uint32_t live = valid >= 16 ? kFull : ((1u << (2 * valid)) - 1);
        if (wi & ~live) flags |= kErrCodePadding;  // container.py:304-305
        cnt += valid * q - sum_min_codes(wi & live, m2, m3);
      }
      sm.blkmid[r] = cnt;
    }
    __syncthreads();
    if (tid == 0 && j + kIdxBufs < nch) issue(j + kIdxBufs);  // buffer is free again
    IDX_ADD(1, t_rows);
    IDX_T0(t_grp);
    // per 4-block group (one per thread): mid bytes, tile-relative offsets, tile totals
    if (tid < kIdxGroups) {
      const int gi = tid;
      const int t = gi / 16;  // tile of this group (16 groups of kBPW blocks per tile)
      uint32_t gs = 0;
      if (t < nt) {
        const uint64_t tb = (ct0 + t) * kTB;
        const int nv = (int)umin64(kTB, nb - tb);
        uint32_t ncw[kMapW];  // NC bits of the tile
#pragma unroll
        for (int w = 0; w < kMapW; ++w) {
          const int vb = nv - 32 * w;
          ncw[w] = ~sm.cmap[t][w] & (vb >= 32 ? kFull : vb <= 0 ? 0u : ((1u << vb) - 1));
        }
        uint32_t rank = sm.ncpre[t];  // NC blocks of the tile before the group
        const int lb0 = (gi % 16) * kBPW;
#pragma unroll
        for (int w = 0; w < kMapW; ++w) {
          const int below = lb0 - 32 * w;
          rank += __popc(ncw[w] & (below >= 32 ? kFull : below <= 0 ? 0u : ((1u << below) - 1)));
        }
#pragma unroll
        for (int jj = 0; jj < kBPW; ++jj) {
          const int lb = lb0 + jj;  // block in tile (a group never straddles a map word)
          uint32_t wv = ncw[0];
#pragma unroll
          for (int w = 1; w < kMapW; ++w)
            if ((lb >> 5) == w) wv = ncw[w];
          if ((wv >> (lb & 31)) & 1) gs += sm.blkmid[rank++];
        }
      }
      // segmented (16-lane) inclusive scan: lanes 0-15 and 16-31 of a warp are two tiles
      uint32_t incl = gs;
#pragma unroll
      for (int d = 1; d < 16; d <<= 1) {
        const uint32_t v = __shfl_up_sync(kFull, incl, d);
        if ((lane & 15) >= d) incl += v;
      }
      sm.goff[gi] = incl - gs;
      if ((lane & 15) == 15) sm.tmid[t] = incl;
    }
    __syncthreads();
    // index entries of the chunk (mid bytes relative to the range start)
    if (warp == 0) {
      const uint32_t v = lane < nt ? sm.tmid[lane] : 0u;
      const uint32_t incl = warp_incl_scan(v);
      if (lane < nt) {
        uint64_t* e = a.index + ew * (ct0 + lane);
        uint64_t wo[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t* o = &sm.goff[16 * lane + 4 * i];
          wo[i] = (uint64_t)o[0] | ((uint64_t)o[1] << 16) | ((uint64_t)o[2] << 32) |
                  ((uint64_t)o[3] << 48);
        }
        reinterpret_cast<ulonglong2*>(e)[0] = make_ulonglong2(run_nc + sm.ncpre[lane], run_mid + incl - v);
        reinterpret_cast<ulonglong2*>(e)[1] = make_ulonglong2(wo[0], wo[1]);
        reinterpret_cast<ulonglong2*>(e)[2] = make_ulonglong2(wo[2], wo[3]);
        reinterpret_cast<ulonglong2*>(e)[3] = make_ulonglong2(c, 0);  // range -> base table
      }
      if (lane == 31) sm.red[0] = incl;  // chunk mid total
    }
    __syncthreads();
    run_mid += sm.red[0];
    __syncthreads();
    IDX_ADD(2, t_grp);
  }
  const uint64_t nc_end = pre_nc_range + sm.cnc[nch];

  // ---- 3. range bases: the last CTA to finish scans the range totals (no waiting) -------
  // The entries keep range-relative mid offsets; base[c] (after the closing entry) turns them
  // into stream offsets -- the decoder adds it.
  IDX_T0(t_p3);
  flags = __reduce_or_sync(kFull, flags);
  if (lane == 0 && flags) atomicOr(a.err, flags);
  uint64_t* base = a.index + ew * (ntiles + 1);
  if (tid == 0) {
    a.status_mid[c] = run_mid;  // range mid total
    __threadfence();
    const uint32_t done = atomicAdd(a.counter, 1u);
    sm.red[0] = done == G - 1;
  }
  __syncthreads();
  if (sm.red[0]) {  // last CTA: exclusive scan of the G range totals -> base table
    __threadfence();
    if (warp == 0) {
      // every range total in flight at once (G <= 256): one L2 round trip, then the scan
      constexpr int kPer = kIdxMaxRanges / 32;
      uint64_t tot[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const uint32_t j = 32 * u + lane;
        tot[u] = j < G ? ld_relaxed(a.status_mid + j) : 0ull;
      }
      uint64_t carry = 0;
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const uint32_t j0 = 32 * u;
        if (j0 >= G) break;
        const uint32_t j = j0 + lane;
        const uint64_t v = tot[u];
        uint64_t incl = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint64_t t = __shfl_up_sync(kFull, incl, d);
          if (lane >= d) incl += t;
        }
        incl += carry;
        if (j < G) base[j] = incl - v;
        carry = __shfl_sync(kFull, incl, 31);
      }
      if (lane == 0) *a.mid_total = carry;  // mid-pool length the codes imply
    }
  }
  if (c == G - 1 && tid == 0) {  // closing entry (range-relative like the others) + NC total
    uint64_t* e = a.index + ew * ntiles;
    reinterpret_cast<ulonglong2*>(e)[0] = make_ulonglong2(nc_end, run_mid);
    reinterpret_cast<ulonglong2*>(e)[3] = make_ulonglong2(G - 1, 0);
    *a.nc_total = nc_end;
  }
  IDX_ADD(3, t_p3);
}

namespace {
template <int BS>
void launch_index_bs(const IndexArgs& a, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(index128_kernel<false, BS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(IdxSmem));
    configured = true;
  }
  index128_kernel<false, BS><<<a.ngroups, kIdxThreads, sizeof(IdxSmem), s>>>(a, nullptr);
}
}  // namespace

void launch_index128(const IndexArgs& a, cudaStream_t s) {
  switch (a.bs) {
    case 64: launch_index_bs<64>(a, s); break;
    case 256: launch_index_bs<256>(a, s); break;
    case 512: launch_index_bs<512>(a, s); break;
    default: launch_index_bs<128>(a, s); break;
  }
}

uint32_t index_batch_groups(uint64_t n) {  // one full chunk per CTA, <= the single-field cap
  const uint64_t nb = (n + 127) >> 7, nt = (nb + kDecTileBlocks - 1) / kDecTileBlocks;
  const uint64_t g = (nt + kIdxTiles - 1) / kIdxTiles;
  return (uint32_t)(g < 1 ? 1 : (g > (uint64_t)kIdxMaxRanges ? kIdxMaxRanges : g));
}

void launch_index128_batch(const IndexArgs* d_fields, uint32_t nfields, uint32_t max_groups,
                           cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(index128_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(IdxSmem));
    configured = true;
  }
  IndexArgs dummy{};
  index128_kernel<true><<<dim3(max_groups, nfields), kIdxThreads, sizeof(IdxSmem), s>>>(dummy,
                                                                                       d_fields);
}

// =========================================================================================
// K3 v2: one chunk of 16 decode tiles per CTA, many CTAs resident
// =========================================================================================
// The range-per-SM K3 above processes its chunks one after another, each a chain of
// dependent phases (loads, row counts, group scan, entries) with one CTA per SM to hide the
// latency, so it runs at ~0.2 of HBM.  Here every chunk is its own CTA (256 threads, ~43 KB
// of shared memory, four CTAs per SM): chunk ids come from an atomic counter in CTA start
// order, the chunk's NC blocks before it from a decoupled look-back over the chunks' map
// popcounts, and its mid bytes before it from a second look-back over the chunks' mid
// totals; the entries hold absolute offsets (one range, base 0) -- the same index format
// (IndexArgs) the decoder reads.  Same checks as K3: req in 1..32, zero padding bits of the
// last row, finite mu.
namespace {
constexpr int kV2Tiles = 16;                                 // decode tiles per chunk
constexpr int kV2Blocks = kV2Tiles * kDecTileBlocks;         // 1024
constexpr int kV2Threads = 256;
constexpr int kV2Groups = kV2Blocks / kFastBPW;              // 256: one per thread
static_assert(kV2Groups == kV2Threads, "one 4-block group per thread");

struct IdxV2Smem {
  uint8_t codes[kV2Blocks * 32 + 32];
  uint8_t req[kV2Blocks + 32];
  uint32_t blkmid[kV2Blocks];
  uint32_t goff[kV2Groups];
  unsigned long long cbits[kV2Tiles];
  uint32_t ncpre[kV2Tiles + 1];
  uint32_t tmid[kV2Tiles];
  uint32_t codes_sh, req_sh, chunk, flags;
  unsigned long long pre_nc, pre_mid;
  uint64_t full;
};
}  // namespace

__global__ void __launch_bounds__(kV2Threads, 4) index128v2_kernel(IndexArgs a) {
  __shared__ __align__(128) IdxV2Smem sm;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t n = a.n, nb = (n + 127) >> 7;
  const uint64_t ntiles = (nb + kDecTileBlocks - 1) / kDecTileBlocks;
  const uint32_t nchunks = (uint32_t)((ntiles + kV2Tiles - 1) / kV2Tiles);
  if (tid == 0) {
    sm.chunk = atomicAdd(a.counter, 1u);  // start order: lower chunks are already running
    sm.flags = 0;
    mbar_init(&sm.full, 1);
    fence_barrier_init();
  }
  __syncthreads();
  const uint32_t c = sm.chunk;
  if (c >= nchunks) return;
  const uint64_t t0 = (uint64_t)c * kV2Tiles;
  const int nt = (int)umin64(kV2Tiles, ntiles - t0);
  const uint64_t b0 = t0 * kDecTileBlocks;
  const uint32_t nbc = (uint32_t)(umin64(nb, b0 + (uint64_t)nt * kDecTileBlocks) - b0);
  uint32_t flags = 0;

  // ---- NC blocks per tile (map popcounts) and before the chunk (look-back 1) ---------------
  if (warp == 0) {
    uint32_t nc = 0;
    if (lane < nt) {
      int nv;
      const unsigned long long cb = map_word(a.map, t0 + lane, nb, nv);
      sm.cbits[lane] = cb;
      nc = (uint32_t)__popcll(~cb & (nv >= 64 ? ~0ull : ((1ull << nv) - 1)));
    }
    const uint32_t incl = warp_incl_scan(nc);
    if (lane < kV2Tiles) sm.ncpre[lane] = incl - nc;
    const uint32_t tot = __shfl_sync(kFull, incl, 31);
    if (lane == 0) sm.ncpre[kV2Tiles] = tot;
    const uint64_t ex = lookback_wide<4>(a.status_nc, c, tot);
    if (lane == 0) {
      sm.pre_nc = ex;
      // the chunk's code rows, req bytes (one bulk copy each)
      const Plan16 pc = plan16(a.codes, 32 * ex, 32 * (uint64_t)tot);
      const Plan16 pr = plan16(a.req, ex, tot);
      sm.codes_sh = pc.shift;
      sm.req_sh = pr.shift;
      mbar_arrive_expect_tx(&sm.full, pc.bytes + pr.bytes);
      if (pc.bytes) bulk_g2s(sm.codes, pc.src, pc.bytes, &sm.full);
      if (pr.bytes) bulk_g2s(sm.req, pr.src, pr.bytes, &sm.full);
    }
  }
  // mu of every block of the chunk must be finite (container.py:198-199), while the rows load
  for (uint32_t b = tid; b < nbc; b += kV2Threads)
    if (nonfinite(a.mu[b0 + b])) flags |= kErrMuNonFinite;
  __syncthreads();
  const uint32_t nc_c = sm.ncpre[kV2Tiles];
  mbar_wait(&sm.full, 0);
  // the field's last block may be short; it is the chunk's last NC block when it is NC
  uint32_t tail_rank = ~0u, tail_cnt = 128;
  if (t0 + nt == ntiles) {
    const uint64_t lastb = nb - 1;
    const uint32_t lb = (uint32_t)(lastb - b0);
    if (!((sm.cbits[lb >> 6] >> (lb & 63)) & 1)) {
      tail_rank = nc_c - 1;
      tail_cnt = (uint32_t)(n - lastb * 128);
    }
  }
  const uint8_t* rows = sm.codes + sm.codes_sh;
  const uint8_t* reqs = sm.req + sm.req_sh;
  const bool al16 = (sm.codes_sh & 15) == 0;
  auto row_words = [&](uint32_t r, uint32_t (&w)[8]) {
    const uint8_t* p = rows + 32 * r;
    if (al16) {
      const uint4 x0 = reinterpret_cast<const uint4*>(p)[0], x1 = reinterpret_cast<const uint4*>(p)[1];
      w[0] = x0.x; w[1] = x0.y; w[2] = x0.z; w[3] = x0.w; w[4] = x1.x; w[5] = x1.y; w[6] = x1.z; w[7] = x1.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = lds32_any(p + 4 * i);
    }
  };
  auto row_q = [&](uint32_t r) {
    const int rq = reqs[r];
    if (rq < 1 || rq > 32) flags |= kErrBadReq;  // container.py:206-207
    int q, s;
    q_s_of(rq > 32 ? 32 : (rq < 1 ? 1 : rq), q, s);
    return q;
  };
  // mid bytes per NC block: sum over its codes of q - min(code, q) (pipeline.py:208)
  {
    uint32_t cnt[kV2Blocks / kV2Threads];
#pragma unroll
    for (int u = 0; u < kV2Blocks / kV2Threads; ++u) {
      const uint32_t r = tid + u * kV2Threads;
      cnt[u] = 0;
      if (r < nc_c) {
        const int q = row_q(r);
        uint32_t m2, m3;
        min_code_masks(q, m2, m3);
        uint32_t w[8];
        row_words(r, w);
        cnt[u] = 128 * q;
#pragma unroll
        for (int i = 0; i < 8; ++i) cnt[u] -= sum_min_codes(w[i], m2, m3);
      }
    }
#pragma unroll
    for (int u = 0; u < kV2Blocks / kV2Threads; ++u)
      if (tid + u * kV2Threads < nc_c) sm.blkmid[tid + u * kV2Threads] = cnt[u];
  }
  // the short last block: codes past the field's end are absent (zero padding bits)
  if (tail_rank != ~0u && tid == (int)(tail_rank % kV2Threads)) {
    const uint32_t r = tail_rank;
    const int q = row_q(r);
    uint32_t m2, m3;
    min_code_masks(q, m2, m3);
    uint32_t w[8];
    row_words(r, w);
    const uint32_t nbytes = (tail_cnt + 3) >> 2;
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t base = 16 * i;
      const uint32_t bytes_here = nbytes <= 4 * (uint32_t)i ? 0 : (uint32_t)umin64(4, nbytes - 4 * i);
      const uint32_t wmask = bytes_here >= 4 ? kFull : ((1u << (8 * bytes_here)) - 1);
      const uint32_t wi = w[i] & wmask;
      const uint32_t valid = tail_cnt <= base ? 0 : (tail_cnt - base >= 16 ? 16 : tail_cnt - base);
      const uint32_t live = valid >= 16 ? kFull : ((1u << (2 * valid)) - 1);
      if (wi & ~live) flags |= kErrCodePadding;  // container.py:304-305
      cnt += valid * q - sum_min_codes(wi & live, m2, m3);
    }
    sm.blkmid[r] = cnt;
  }
  __syncthreads();
  // per 4-block group (one per thread): mid bytes, tile-relative offsets, tile totals
  {
    const int gi = tid;
    const int t = gi / (kDecTileBlocks / kFastBPW);  // 16 groups per tile
    uint32_t gs = 0;
    if (t < nt) {
      const unsigned long long cb = sm.cbits[t];
      const uint64_t tb = (t0 + t) * kDecTileBlocks;
      const int nv = (int)umin64(kDecTileBlocks, nb - tb);
      const unsigned long long ncm = ~cb & (nv >= 64 ? ~0ull : ((1ull << nv) - 1));
#pragma unroll
      for (int jj = 0; jj < kFastBPW; ++jj) {
        const int lb = (gi % (kDecTileBlocks / kFastBPW)) * kFastBPW + jj;
        if ((ncm >> lb) & 1) gs += sm.blkmid[sm.ncpre[t] + __popcll(ncm & ((1ull << lb) - 1))];
      }
    }
    uint32_t incl = gs;
#pragma unroll
    for (int d = 1; d < 16; d <<= 1) {
      const uint32_t v = __shfl_up_sync(kFull, incl, d);
      if ((lane & 15) >= d) incl += v;
    }
    sm.goff[gi] = incl - gs;
    if ((lane & 15) == 15 && t < kV2Tiles) sm.tmid[t] = incl;
  }
  flags = __reduce_or_sync(kFull, flags);
  if (lane == 0 && flags) atomicOr(&sm.flags, flags);
  __syncthreads();
  // ---- mid bytes before the chunk (look-back 2), entries ------------------------------------
  if (warp == 0) {
    const uint32_t v = lane < nt ? sm.tmid[lane] : 0u;
    const uint32_t incl = warp_incl_scan(v);
    const uint32_t tot = __shfl_sync(kFull, incl, 31);
    const uint64_t ex = lookback_wide<4>(a.status_mid, c, tot);
    const uint32_t ew = kIndexEntryBytes / 8;
    if (lane < nt) {
      uint64_t* e = a.index + ew * (t0 + lane);
      uint64_t wo[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t* o = &sm.goff[16 * lane + 4 * i];
        wo[i] = (uint64_t)o[0] | ((uint64_t)o[1] << 16) | ((uint64_t)o[2] << 32) |
                ((uint64_t)o[3] << 48);
      }
      reinterpret_cast<ulonglong2*>(e)[0] = make_ulonglong2(sm.pre_nc + sm.ncpre[lane], ex + incl - v);
      reinterpret_cast<ulonglong2*>(e)[1] = make_ulonglong2(wo[0], wo[1]);
      reinterpret_cast<ulonglong2*>(e)[2] = make_ulonglong2(wo[2], wo[3]);
      reinterpret_cast<ulonglong2*>(e)[3] = make_ulonglong2(0, 0);  // range 0 (base 0)
    }
    if (c == nchunks - 1 && lane == 0) {  // closing entry, the one range base, totals
      uint64_t* e = a.index + ew * ntiles;
      const uint64_t nc_end = sm.pre_nc + sm.ncpre[kV2Tiles], mid_end = ex + tot;
      reinterpret_cast<ulonglong2*>(e)[0] = make_ulonglong2(nc_end, mid_end);
      reinterpret_cast<ulonglong2*>(e)[1] = make_ulonglong2(0, 0);
      reinterpret_cast<ulonglong2*>(e)[2] = make_ulonglong2(0, 0);
      reinterpret_cast<ulonglong2*>(e)[3] = make_ulonglong2(0, 0);
      e[ew] = 0;  // base[0]
      *a.nc_total = nc_end;
      *a.mid_total = mid_end;
    }
    if (lane == 0 && sm.flags) atomicOr(a.err, sm.flags);
  }
}

void launch_index128v2(const IndexArgs& a, cudaStream_t s) {
  const uint64_t nb = (a.n + 127) >> 7, nt = (nb + kDecTileBlocks - 1) / kDecTileBlocks;
  const uint64_t nchunks = (nt + kV2Tiles - 1) / kV2Tiles;
  index128v2_kernel<<<(uint32_t)nchunks, kV2Threads, 0, s>>>(a);
}

uint64_t index128v2_chunks(uint64_t n) {
  const uint64_t nb = (n + 127) >> 7, nt = (nb + kDecTileBlocks - 1) / kDecTileBlocks;
  return (nt + kV2Tiles - 1) / kV2Tiles;
}

// =========================================================================================
// K2: persistent decoder
// =========================================================================================
namespace {
#ifndef SZX_K2_WAIT
#define SZX_K2_WAIT 1   // compute warps: hardware-suspending try_wait (no poll loop)
#endif
constexpr int kDecWarps = 16;                        // compute warps 0..15, producer warp 16
constexpr int kDecThreads = (kDecWarps + 1) * 32;
#ifndef SZX_K2_STAGES
#define SZX_K2_STAGES 3
#endif
constexpr int kDecStages = SZX_K2_STAGES;
#ifndef SZX_K2_CTAS
#define SZX_K2_CTAS 2  // resident CTAs per SM (3 needs SZX_K2_STAGES=2 and <= 40 registers)
#endif

constexpr int kDecMaxTB = 128;                       // blocks per tile, smallest fast bs
struct __align__(16) DecStage {
  uint8_t slack[16];                                  // column loads may look 4 bytes back
  uint8_t mid[kDecTileBlocks * 512 + 32];
  uint8_t codes[kDecTileBlocks * 32 + 32];
  uint8_t mu[kDecMaxTB * 4 + 32];                   // bs 64: 128 blocks per tile
  uint8_t req[kDecMaxTB + 32];
  uint8_t map[32];
  uint8_t idx[kIndexEntryBytes];                      // this tile's index entry (group offsets)
  uint32_t tile, mid_sh, codes_sh, mu_sh, req_sh, map_sh, pad0, pad1;
};

constexpr int kDecMaxRanges = kIdxMaxRanges;         // K3 ranges (one per SM) <= 256

struct DecSmem {
  DecStage st[kDecStages];
  uint64_t full[kDecStages];
  uint64_t empty[kDecStages];
  unsigned long long base[kDecMaxRanges];            // K3 range bases (producer only)
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
// e: shared address of the lane's first mid byte; mul[k] = 2^(32 - 8q + s + 8k), so that
// sum_k T_k * mul[k] = (kept-byte word << (32 - 8q)) << s on the FMA pipe (the ALU pipe is
// the busy one); nan accumulates r * 0, which stays 0 unless some r is inf/NaN.
// Element i's kept bytes are [e_i - n_i, e_i) in big-endian order, so column k (0 = last
// kept byte) sits at e_i - 1 - k (pipeline.py:193-214, blockcodec.py:150-158); a column
// register keeps the reused byte when the element does not load it.
// One element's column loads: predicate k = bit 2i of m[k] (element keeps > k bytes), the
// stream position advances by the number of kept bytes, then kept column k is read at
// e_i - 1 - k into its column register (which otherwise keeps the reused byte).  Written in
// PTX so each predicate is a single LOP3 bit test against an immediate.
template <int QM, int I>
__device__ __forceinline__ void elem_cols(uint32_t& e, uint32_t& T0, uint32_t& T1, uint32_t& T2,
                                          uint32_t& T3, const uint32_t (&m)[4]) {
  constexpr uint32_t kBit = 1u << (2 * I);
  if constexpr (QM == 1) {
    asm volatile(
        "{\n .reg .pred p0;\n .reg .b32 t;\n and.b32 t, %2, %3;\n setp.ne.b32 p0, t, 0;\n"
        " @p0 add.u32 %1, %1, 1;\n @p0 ld.shared.u8 %0, [%1+-1];\n}\n"
        : "+r"(T0), "+r"(e) : "r"(m[0]), "n"(kBit));
  } else if constexpr (QM == 2) {
    asm volatile(
        "{\n .reg .pred p0, p1;\n .reg .b32 t;\n and.b32 t, %3, %5;\n setp.ne.b32 p0, t, 0;\n"
        " and.b32 t, %4, %5;\n setp.ne.b32 p1, t, 0;\n"
        " @p0 add.u32 %2, %2, 1;\n @p1 add.u32 %2, %2, 1;\n"
        " @p0 ld.shared.u8 %0, [%2+-1];\n @p1 ld.shared.u8 %1, [%2+-2];\n}\n"
        : "+r"(T0), "+r"(T1), "+r"(e) : "r"(m[0]), "r"(m[1]), "n"(kBit));
  } else if constexpr (QM == 3) {
    asm volatile(
        "{\n .reg .pred p0, p1, p2;\n .reg .b32 t;\n and.b32 t, %4, %7;\n setp.ne.b32 p0, t, 0;\n"
        " and.b32 t, %5, %7;\n setp.ne.b32 p1, t, 0;\n and.b32 t, %6, %7;\n setp.ne.b32 p2, t, 0;\n"
        " @p0 add.u32 %3, %3, 1;\n @p1 add.u32 %3, %3, 1;\n @p2 add.u32 %3, %3, 1;\n"
        " @p0 ld.shared.u8 %0, [%3+-1];\n @p1 ld.shared.u8 %1, [%3+-2];\n"
        " @p2 ld.shared.u8 %2, [%3+-3];\n}\n"
        : "+r"(T0), "+r"(T1), "+r"(T2), "+r"(e) : "r"(m[0]), "r"(m[1]), "r"(m[2]), "n"(kBit));
  } else {
    asm volatile(
        "{\n .reg .pred p0, p1, p2, p3;\n .reg .b32 t;\n and.b32 t, %5, %9;\n setp.ne.b32 p0, t, 0;\n"
        " and.b32 t, %6, %9;\n setp.ne.b32 p1, t, 0;\n and.b32 t, %7, %9;\n setp.ne.b32 p2, t, 0;\n"
        " and.b32 t, %8, %9;\n setp.ne.b32 p3, t, 0;\n"
        " @p0 add.u32 %4, %4, 1;\n @p1 add.u32 %4, %4, 1;\n @p2 add.u32 %4, %4, 1;\n"
        " @p3 add.u32 %4, %4, 1;\n"
        " @p0 ld.shared.u8 %0, [%4+-1];\n @p1 ld.shared.u8 %1, [%4+-2];\n"
        " @p2 ld.shared.u8 %2, [%4+-3];\n @p3 ld.shared.u8 %3, [%4+-4];\n}\n"
        : "+r"(T0), "+r"(T1), "+r"(T2), "+r"(T3), "+r"(e)
        : "r"(m[0]), "r"(m[1]), "r"(m[2]), "r"(m[3]), "n"(kBit));
  }
}

#ifndef SZX_K2_ABL
#define SZX_K2_ABL 0
#endif
#ifndef SZX_K2_F2
#define SZX_K2_F2 1  // packed f32x2 adds / non-finite FMAs (FADD2 / FFMA2), two elements each
#endif

template <int QM, int I>
__device__ __forceinline__ uint32_t elem_word(uint32_t& e, uint32_t& T0, uint32_t& T1,
                                              uint32_t& T2, uint32_t& T3, const uint32_t (&m)[4],
                                              const uint32_t (&mul)[4]) {
  elem_cols<QM, I>(e, T0, T1, T2, T3, m);
  uint32_t bits = T0 * mul[0];
  if (QM >= 2) bits += T1 * mul[1];
  if (QM >= 3) bits += T2 * mul[2];
  if (QM >= 4) bits += T3 * mul[3];
  return bits;  // (w << s) as float32 bits (pipeline.py:222)
}

template <int QM, int I>
__device__ __forceinline__ void decode_elems(float (&r)[16], const uint32_t (&m)[4], uint32_t& e,
                                             uint32_t& T0, uint32_t& T1, uint32_t& T2,
                                             uint32_t& T3, const uint32_t (&mul)[4], float mu,
                                             float& nan, uint64_t& nan2, uint64_t mu2) {
  if constexpr (I < 16) {
#if SZX_K2_F2
    // two elements per packed add: each lane of add.rn.f32x2 is the IEEE RN float32 add of
    // pipeline.py:223 (+ mu in float32); r * 0 stays 0 unless r is inf / NaN
    const uint32_t b0 = elem_word<QM, I>(e, T0, T1, T2, T3, m, mul);
    const uint32_t b1 = elem_word<QM, I + 1>(e, T0, T1, T2, T3, m, mul);
    uint64_t w, y;
    asm("mov.b64 %0, {%1, %2};" : "=l"(w) : "r"(b0), "r"(b1));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(y) : "l"(w), "l"(mu2));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(nan2) : "l"(y), "l"(0ull));
    uint32_t y0, y1;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(y0), "=r"(y1) : "l"(y));
    r[I] = __uint_as_float(y0);
    r[I + 1] = __uint_as_float(y1);
    decode_elems<QM, I + 2>(r, m, e, T0, T1, T2, T3, mul, mu, nan, nan2, mu2);
#else
    const uint32_t bits = elem_word<QM, I>(e, T0, T1, T2, T3, m, mul);
    // pipeline.py:222-223 -- (w << s) as float32, + mu in float32
    r[I] = __fadd_rn(__uint_as_float(bits), mu);
    nan = __fmaf_rn(r[I], 0.f, nan);
    decode_elems<QM, I + 1>(r, m, e, T0, T1, T2, T3, mul, mu, nan, nan2, mu2);
#endif
  }
}

template <int QM>
__device__ __forceinline__ void decode16(float (&r)[16], const uint32_t (&m)[4], uint32_t tin,
                                         uint32_t e, const uint32_t (&mul)[4], float mu,
                                         float& nan) {
  uint32_t T0 = tin & 0xFF, T1 = (tin >> 8) & 0xFF, T2 = (tin >> 16) & 0xFF, T3 = tin >> 24;
  uint64_t nan2 = 0, mu2;
  asm("mov.b64 %0, {%1, %1};" : "=l"(mu2) : "r"(__float_as_uint(mu)));
  decode_elems<QM, 0>(r, m, e, T0, T1, T2, T3, mul, mu, nan, nan2, mu2);
#if SZX_K2_F2
  uint32_t n0, n1;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(n0), "=r"(n1) : "l"(nan2));
  nan = __fadd_rn(nan, __fadd_rn(__uint_as_float(n0), __uint_as_float(n1)));
#endif
}
}  // namespace

// One lane's decode for a warp whose largest q is QM (warp-uniform; lanes with a smaller q
// or a constant block simply leave the higher columns empty):
//   column masks m[c] (bit 2i: element i keeps more than c bytes, i.e. code_i < q - c) and the
//   lane's byte count L; its stream position = the group offset from the index + a warp scan
//   of L (stream order = lane order); the (K, V) effect of the lane on the kept-byte word --
//   columns it never writes pass the previous word through (K), the others end as their last
//   writer left them (V) -- scanned over the block's 8 lanes (index propagation,
//   parallel.py:79-101); then the 16 elements (pipeline.py:193-224).
template <int QM, int LPB = 8>
__device__ __forceinline__ void lane_decode(float (&r)[16], float& nan, bool nc, int q, int sft,
                                            uint32_t cwd, uint32_t live, uint32_t gstart,
                                            const uint8_t* mid, float mu, int lane, int g) {
  if (q > QM) __builtin_unreachable();
  uint32_t m[4] = {0, 0, 0, 0};
  uint32_t L = 0;
  if (nc) {
    const uint32_t lo = cwd & 0x55555555u, hi = (cwd >> 1) & 0x55555555u;
    const uint32_t lv = live & 0x55555555u;
    const uint32_t z1 = ~(lo | hi) & lv, z2 = ~hi & lv, z3 = ~(lo & hi) & lv;  // code < 1,2,3
#pragma unroll
    for (int c = 0; c < QM; ++c) {
      const int th = q - c;  // column c kept iff code < th
      m[c] = th <= 0 ? 0u : th == 1 ? z1 : th == 2 ? z2 : th == 3 ? z3 : lv;
      L += __popc(m[c]);
    }
  }
  uint32_t incl = L;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += t;
  }
  const uint32_t start = gstart + incl - L;
  // The last element keeping column c ends at start + L minus the bytes of the elements
  // after it, which keep at most c bytes each: sum_{k<c} popc(m[k] above it).
  uint32_t K = QM >= 4 ? 0u : (0xFFFFFFFFu << (8 * QM)), V = 0;
#pragma unroll
  for (int c = 0; c < QM; ++c) {
    if (m[c]) {
      const int i = (31 - __clz(m[c])) >> 1;  // last element keeping column c
      const uint32_t above = i >= 15 ? 0u : (0xFFFFFFFFu << (2 * i + 2));
      uint32_t after = 0;
#pragma unroll
      for (int k = 0; k < c; ++k) after += __popc(m[k] & above);
      V |= (uint32_t)mid[start + L - after - 1 - c] << (8 * c);
    } else {
      K |= 0xFFu << (8 * c);
    }
  }
  // (K_a, V_a) then (K_b, V_b) = (K_a & K_b, (V_a & K_b) | V_b), over the block's LPB lanes
#pragma unroll
  for (int d = 1; d < LPB; d <<= 1) {
    const uint32_t kp = __shfl_up_sync(kFull, K, d), vp = __shfl_up_sync(kFull, V, d);
    if (g >= d) {
      V = (vp & K) | V;
      K = kp & K;
    }
  }
  uint32_t tin = __shfl_up_sync(kFull, V, 1);
  if (g == 0) tin = 0;  // the zero word before the block start
  if (nc) {
#if SZX_K2_ABL & 1  // timing ablation (wrong output): lane-adjacent column loads, no conflicts
    const uint32_t e = smem_u32(mid) + 8 + (uint32_t)lane;
#else
    const uint32_t e = smem_u32(mid) + start;
#endif
    const uint32_t sh = (uint32_t)(32 - 8 * q + sft);
    uint32_t mul[4] = {0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < QM; ++c) mul[c] = c < q ? 1u << (sh + 8 * c) : 0u;
    decode16<QM>(r, m, tin, e, mul, mu, nan);
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = mu;  // constant block (pipeline.py:219-220)
  }
}

// Batched (kBatch): the launch's tiles [a.tile_begin, a.tile_end) are the concatenation of
// the fields' decode tiles (field f from tile0s[f]); every tile takes its pools, index and
// output from fields[f] (its K3 range bases from the field's index, not shared memory).
// BS: the block size (64, 128, 256 or 512); a decode tile is 8192 values = 8192 / BS blocks.
template <bool kBatch, int BS = 128>
#if SZX_K2_CTAS >= 3
__global__ void __maxnreg__(40)
#else
__global__ void __launch_bounds__(kDecThreads, SZX_K2_CTAS)
#endif
    decode128_kernel(Decode128Args a, const Decode128Args* __restrict__ fields,
                     const uint64_t* __restrict__ tile0s, uint32_t nfields) {
  constexpr int kLPB = BS / 16;            // lanes per block
  constexpr int kBPW = 32 / kLPB;          // blocks per warp (group)
  constexpr int kTB = 16 * kBPW;           // blocks per decode tile
  constexpr int kMapW = (kTB + 31) / 32;   // constant-map words per tile
  static_assert(kTB * BS == 8192, "8192-value decode tiles");
  extern __shared__ __align__(128) uint8_t smem_raw[];
  DecSmem& sm = *reinterpret_cast<DecSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

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
    if (!kBatch) {  // the K3 range bases (after the closing index entry) into shared memory
      const uint32_t ew = kIndexEntryBytes / 8;
      uint32_t G = (uint32_t)a.index[ew * a.ntiles + 6] + 1;
      G = G < kDecMaxRanges ? G : kDecMaxRanges;
      for (uint32_t i = lane; i < G; i += 32) sm.base[i] = a.index[ew * (a.ntiles + 1) + i];
      __syncwarp();
    }
    if (lane == 0) {
      // the index entries are loaded one tile ahead, so their latency overlaps the wait for
      // a free slot instead of delaying the bulk copies
      const uint32_t ew = kIndexEntryBytes / 8;
      // entries hold range-relative mid offsets; base[range] follows the closing entry
      auto load_idx = [&](const Decode128Args& fa, uint64_t t, ulonglong2& x0, ulonglong2& x1) {
        if (t < fa.ntiles) {
          x0 = *reinterpret_cast<const ulonglong2*>(fa.index + ew * t);
          x1 = *reinterpret_cast<const ulonglong2*>(fa.index + ew * (t + 1));
          const uint32_t c0 = (uint32_t)fa.index[ew * t + 6], c1 = (uint32_t)fa.index[ew * (t + 1) + 6];
          if (kBatch) {
            const uint64_t* base = fa.index + ew * (fa.ntiles + 1);
            x0.y += base[c0];
            x1.y += base[c1];
          } else {
            x0.y += sm.base[c0 < kDecMaxRanges ? c0 : 0];
            x1.y += sm.base[c1 < kDecMaxRanges ? c1 : 0];
          }
        }
      };
      // field of a launch tile (batched: tiles only increase, the search moves forward)
      uint32_t fnext = 0;
      auto field_of = [&](uint64_t t, uint32_t& f) {
        if (kBatch)
          while (f + 1 < nfields && t >= tile0s[f + 1]) ++f;
        return kBatch ? t - tile0s[f] : t;
      };
      ulonglong2 n0 = make_ulonglong2(0, 0), n1 = make_ulonglong2(0, 0);
      {
        const uint64_t t = a.tile_begin + blockIdx.x;
        if (t < a.tile_end) {
          const uint64_t lt = field_of(t, fnext);
          load_idx(kBatch ? fields[fnext] : a, lt, n0, n1);
        }
      }
      for (uint32_t k = 0;; ++k) {
        const int s = k % kDecStages;
        const uint64_t tile = a.tile_begin + (uint64_t)blockIdx.x + (uint64_t)k * gridDim.x;
        const ulonglong2 e0 = n0, e1 = n1;
        const uint32_t f = fnext;
        const uint64_t lt = kBatch ? tile - tile0s[f] : tile;
        if (tile + gridDim.x < a.tile_end) {
          const uint64_t ltn = field_of(tile + gridDim.x, fnext);
          load_idx(kBatch ? fields[fnext] : a, ltn, n0, n1);
        }
        mbar_wait_sleep(&sm.empty[s], ((k / kDecStages) & 1) ^ 1);
        DecStage& S = sm.st[s];
        if (tile >= a.tile_end) {
          S.tile = ~0u;
          mbar_arrive(&sm.full[s]);
          break;
        }
        const Decode128Args& fa = kBatch ? fields[f] : a;
        const uint64_t nb = (fa.n + BS - 1) / BS;
        const uint32_t nv = (uint32_t)umin64(kTB, nb - lt * kTB);
        uint64_t m0 = e0.y, m1 = e1.y;
        if (m1 > fa.mid_len) {  // codes imply more mid bytes than present: never read past
          atomicOr(fa.err, kErrUnderrun);
          m1 = fa.mid_len;
          m0 = m0 < m1 ? m0 : m1;
        }
        if (m1 - m0 > kDecTileBlocks * 512) m1 = m0 + kDecTileBlocks * 512;  // corrupt index
        const BulkPlan pm = plan(fa.mid, m0, m1 - m0);
        const BulkPlan pc = plan(fa.codes, (BS / 4) * e0.x, (BS / 4) * (e1.x - e0.x));
        const BulkPlan pu = plan(reinterpret_cast<const uint8_t*>(fa.mu), 4 * lt * kTB, 4 * nv);
        const BulkPlan pr = plan(fa.req, e0.x, e1.x - e0.x);
        const BulkPlan pp = plan(fa.map, (kTB / 8) * lt, (nv + 7) >> 3);
        S.tile = (uint32_t)lt;
        S.pad0 = f;  // the tile's field (batched)
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
        bulk_g2s(S.idx, fa.index + ew * lt, kIndexEntryBytes, &sm.full[s]);
      }
    }
    return;
  }

  // ---------------------------------------------------------------- compute warps (0..15)
  // warp cw decodes blocks kBPW cw .. of every tile (its group), lane l the 16 values
  // 16 (l % kLPB) .. of block kBPW cw + l / kLPB (the encoder's layout)
  const int cw = warp;
  const int jl = cw * kBPW + lane / kLPB;  // block of the tile this lane decodes
  const int g = lane % kLPB;               // 16-value group within the block
  bool bad = false, badmu = false;
  for (uint32_t k = 0;; ++k) {
    const int st = k % kDecStages;
#ifdef SZX_STATS
    const long long tw0 = clock64();
#endif
#if SZX_K2_WAIT == 1
    while (!mbar_try_wait_hint(&sm.full[st], (k / kDecStages) & 1)) {
    }
#elif SZX_K2_WAIT == 2
    mbar_wait_backoff(&sm.full[st], (k / kDecStages) & 1, 128, 512);
#else
    mbar_wait(&sm.full[st], (k / kDecStages) & 1);
#endif
#ifdef SZX_STATS
    if (lane == 0) {  // per warp: [0] wait for the stage, [1] tiles, [2] busy
      atomicAdd(&g_decode_stats[0], (unsigned long long)(clock64() - tw0));
      atomicAdd(&g_decode_stats[1], 1ull);
    }
    const long long tb0 = clock64();
#endif
    const DecStage& S = sm.st[st];
    if (S.tile == ~0u) break;
    const Decode128Args& fa = kBatch ? fields[S.pad0] : a;
    const uint64_t n = fa.n, nb = (n + BS - 1) / BS;
    const bool out32 = ((uintptr_t)fa.out & 31) == 0;
    const uint64_t tb = (uint64_t)S.tile * kTB;
    const int nvalid = (int)umin64(kTB, nb - tb);
    // the tile's constant-map bits (kTB, LSB-first), masked to its blocks
    // the tile's constant-map bits (kTB, LSB-first), masked to its blocks; the block's NC flag
    // and its NC rank in the tile (non-constant valid blocks before it)
    const bool exists = jl < nvalid;
    bool nc;
    uint32_t rnk = 0;
    if constexpr (kTB == 64) {  // bs 128: one 64-bit word
      const uint8_t* mp = S.map + S.map_sh;
      unsigned long long cbits =
          (S.map_sh & 7) == 0  // 8-byte map words of 64-block tiles are aligned in the pool
              ? *reinterpret_cast<const unsigned long long*>(mp)
              : (unsigned long long)lds_u32_any(mp) | ((unsigned long long)lds_u32_any(mp + 4) << 32);
      const unsigned long long vmask = nvalid >= 64 ? ~0ull : ((1ull << nvalid) - 1);
      cbits &= vmask;
      nc = exists && !((cbits >> jl) & 1);
      if (nc) rnk = __popcll(~cbits & vmask & ((1ull << jl) - 1));
    } else {
      uint32_t mw[kMapW];
      const uint8_t* mp = S.map + S.map_sh;
#pragma unroll
      for (int w = 0; w < kMapW; ++w) {
        const int vb = nvalid - 32 * w;  // valid bits in word w
        mw[w] = lds_u32_any(mp + 4 * w) & (vb >= 32 ? kFull : vb <= 0 ? 0u : ((1u << vb) - 1));
      }
      uint32_t jw = mw[0];  // map word of block jl (selected, not indexed: no local memory)
#pragma unroll
      for (int w = 1; w < kMapW; ++w)
        if ((jl >> 5) == w) jw = mw[w];
      nc = exists && !((jw >> (jl & 31)) & 1);
      if (nc) {
#pragma unroll
        for (int w = 0; w < kMapW; ++w) {
          const int vb = nvalid - 32 * w;
          const uint32_t valid = vb >= 32 ? kFull : vb <= 0 ? 0u : ((1u << vb) - 1);
          const int below = jl - 32 * w;  // bits of word w before block jl
          const uint32_t bm = below >= 32 ? kFull : below <= 0 ? 0u : ((1u << below) - 1);
          rnk += __popc(~mw[w] & valid & bm);
        }
      }
    }
    const uint64_t b = tb + jl;
    const float mu = !exists ? 0.f
                     : ((S.mu_sh & 3) == 0
                            ? *reinterpret_cast<const float*>(S.mu + S.mu_sh + 4 * jl)
                            : __uint_as_float(lds_u32_any(S.mu + S.mu_sh + 4 * jl)));
    // live values of this lane (the field's last block may be short)
    const bool full_tile = ((uint64_t)S.tile + 1) * kTB * BS <= n;
    const uint64_t bvals = exists ? umin64(n - b * BS, BS) : 0;
    const int nlive = full_tile ? 16
                      : (int)umin64(16, bvals > 16u * (uint64_t)g ? bvals - 16u * (uint64_t)g : 0);
    int q = 0, sft = 0;
    uint32_t cwd = 0, live = 0;
    if (nc) {
      const uint32_t r = rnk;
      const uint8_t* cp = S.codes + S.codes_sh + (BS / 4) * r + 4 * g;
      cwd = (S.codes_sh & 3) == 0 ? *reinterpret_cast<const uint32_t*>(cp) : lds_u32_any(cp);
      live = nlive >= 16 ? kFull : ((1u << (2 * nlive)) - 1);
      cwd &= live;
      int rq = S.req[S.req_sh + r];
      rq = rq < 1 ? 1 : (rq > 32 ? 32 : rq);  // K3 flags bad req; keep the decode in bounds
      q_s_of(rq, q, sft);
    }
    float r[16];
    float nan = 0.f;
    const uint32_t qm = __reduce_max_sync(kFull, nc ? (uint32_t)q : 0u);
    const uint16_t* woff = reinterpret_cast<const uint16_t*>(S.idx + 16);
    const uint8_t* mid = S.mid + S.mid_sh;
    const uint32_t gs = woff[cw];
    switch (qm) {  // warp-uniform: largest q among the warp's NC blocks
      case 0:  // every block of the warp is constant (pipeline.py:219-220)
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = mu;
        break;
      case 1: lane_decode<1, kLPB>(r, nan, nc, q, sft, cwd, live, gs, mid, mu, lane, g); break;
      case 2: lane_decode<2, kLPB>(r, nan, nc, q, sft, cwd, live, gs, mid, mu, lane, g); break;
      case 3: lane_decode<3, kLPB>(r, nan, nc, q, sft, cwd, live, gs, mid, mu, lane, g); break;
      default: lane_decode<4, kLPB>(r, nan, nc, q, sft, cwd, live, gs, mid, mu, lane, g); break;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[st]);  // all reads of this stage done
    if (nc && nan != 0.f) {
      // only live values count (dead ones of a short last block are never stored)
#pragma unroll
      for (int i = 0; i < 16; ++i) bad |= i < nlive && !(fabsf(r[i]) <= 3.402823466e+38f);
    }
    if (exists) badmu |= nonfinite(mu);
    if (kBatch) {  // flags belong to the tile's field
      if (__any_sync(kFull, bad) && lane == 0) atomicOr(fa.err, kErrNonFinite);
      if (__any_sync(kFull, badmu) && lane == 0) atomicOr(fa.err, kErrMuNonFinite);
      bad = badmu = false;
    }
    float* dst = fa.out + b * BS + 16 * g;
#ifdef SZX_STATS
    if (lane == 0) atomicAdd(&g_decode_stats[2], (unsigned long long)(clock64() - tb0));
#endif
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

namespace {
int decode_grid_cap() {
  static int cap = 0;
  if (!cap) {
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
    cudaFuncSetAttribute(decode128_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(DecSmem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode128_kernel<true>, kDecThreads,
                                                  sizeof(DecSmem));
    cap = nsm * (per_sm < 1 ? 1 : per_sm);
  }
  return cap;
}
}  // namespace

void launch_decode128_batch(const Decode128Args& a, const Decode128Args* d_fields,
                            const uint64_t* d_tile0s, uint32_t nfields, cudaStream_t s) {
  const uint64_t want = (uint64_t)decode_grid_cap();
  const uint64_t tiles = a.tile_end - a.tile_begin;
  const uint32_t grid = (uint32_t)(tiles < want ? tiles : want);
  if (grid)
    decode128_kernel<true><<<grid, kDecThreads, sizeof(DecSmem), s>>>(a, d_fields, d_tile0s,
                                                                      nfields);
}

namespace {
template <int BS>
void launch_decode_bs(const Decode128Args& a, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(decode128_kernel<false, BS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode128_kernel<false, BS>, kDecThreads,
                                                  sizeof(DecSmem));
    if (per_sm < 1) per_sm = 1;
  }
  const uint64_t want = (uint64_t)nsm * per_sm;
  const uint64_t tiles = a.tile_end - a.tile_begin;
  const uint32_t grid = (uint32_t)(tiles < want ? tiles : want);
  if (grid) decode128_kernel<false, BS><<<grid, kDecThreads, sizeof(DecSmem), s>>>(a, nullptr, nullptr, 1);
}
}  // namespace

void launch_decode128(const Decode128Args& a, cudaStream_t s) {
  switch (a.bs) {
    case 64: launch_decode_bs<64>(a, s); break;
    case 256: launch_decode_bs<256>(a, s); break;
    case 512: launch_decode_bs<512>(a, s); break;
    default: launch_decode_bs<128>(a, s); break;
  }
}

}  // namespace szx
