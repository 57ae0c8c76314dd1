// analysis.cu -- the measurement side of the reference package on the device:
//   A1 accounting_kernel   pipeline.py:119-132 (compress_with_accounting's unshifted shadow
//                          scheme; the shifted side is 8 * mid_len of the K1 stream)
//   A2 quality_kernel      metrics.py:78-103   (max |a-b|, sum (a-b)^2, range of a: one pass)
//   A3 block_range_kernel  metrics.py:128-146  (block_range_cdf counts per threshold)
//   A4 scan_*_kernel       parallel.py:21-44   (prefix_scan, exclusive int64)
//   A5 propagate_kernel    parallel.py:74-101  (propagate_round / propagate_indices)
// All HBM-bound streaming passes; float64 arithmetic follows the reference's NumPy
// promotion exactly (explicit __d*_rn), integer sums are order-independent.
#include <cfloat>

#include "szx_device.cuh"
#include "szx_kernels.h"

namespace szx {

namespace {
constexpr int kAThreads = 256;
constexpr int kAWarps = kAThreads / 32;

// leading zero bytes of a u32, 0..4 (pipeline.py:84-91)
__device__ __forceinline__ uint32_t lzbytes(uint32_t x) { return (uint32_t)__clz(x) >> 3; }

// f32 min / max of one block (one warp, any block size), lanes read consecutive values.
__device__ __forceinline__ void block_minmax(const float* __restrict__ x, uint32_t cnt, int lane,
                                             float& mn, float& mx) {
  mn = FLT_MAX;
  mx = -FLT_MAX;
  uint32_t i = lane;
#pragma unroll 4
  for (; i < cnt; i += 32) {
    const float v = __ldg(x + i);
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(kFull, mn, d));
    mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, d));
  }
}
}  // namespace

// ---- A1: unshifted-scheme bits (pipeline.py:119-129) -------------------------------------
// Per NC element: w = bits(x -f32 mu) (no shift), prev = previous w in the block (0 at the
// block start, pipeline.py:108-111 / 121-123), reuse = min(3, lzb(w ^ prev), req // 8),
// bits = req - 8 * reuse.  One warp per block (grid-stride), the classification is the
// compress kernels' own classify() (pipeline.py:54-81), so NC blocks and req are identical.
__global__ void __launch_bounds__(kAThreads) accounting_kernel(const float* __restrict__ x,
                                                               uint64_t n, uint32_t bs, double e,
                                                               int pe,
                                                               unsigned long long* bits_out) {
  const int lane = threadIdx.x & 31;
  const uint64_t nb = (n + bs - 1) / bs;
  const uint64_t wstride = (uint64_t)gridDim.x * kAWarps;
  unsigned long long acc = 0;
  for (uint64_t b = (uint64_t)blockIdx.x * kAWarps + (threadIdx.x >> 5); b < nb; b += wstride) {
    const uint64_t start = b * bs;
    const uint32_t cnt = (uint32_t)umin64(bs, n - start);
    const float* xb = x + start;
    float mn, mx;
    block_minmax(xb, cnt, lane, mn, mx);
    const BlockClass c = classify(mn, mx, e, pe);
    if (c.cst) continue;  // warp-uniform
    const uint32_t req = (uint32_t)c.req, rb = req >> 3;
    uint32_t carry = 0;   // w of the previous chunk's last element (0 at the block start)
    for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
      const uint32_t i = i0 + lane;
      const bool live = i < cnt;
      const uint32_t w = live ? __float_as_uint(__fsub_rn(__ldg(xb + i), c.mu)) : 0u;
      uint32_t prev = __shfl_up_sync(kFull, w, 1);
      if (lane == 0) prev = carry;
      carry = __shfl_sync(kFull, w, 31);
      uint32_t reuse = lzbytes(w ^ prev);
      reuse = reuse < 3 ? reuse : 3;
      reuse = reuse < rb ? reuse : rb;
      if (live) acc += req - 8 * reuse;
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(kFull, acc, d);
  if (lane == 0 && acc) atomicAdd(bits_out, acc);
}

// ---- A2: quality measures in one pass (metrics.py:78-103) -------------------------------
// d = f64(a) - f64(b) (NumPy promotes both float32 arrays to float64 first), max |d|,
// sum d*d, and the f32 min / max of a (psnr's range: f64(max) - f64(min) on the host).
// A NaN difference (inf - inf, NaN input) is counted so the host can return NaN as NumPy
// would.  Per-CTA partials, reduced in a fixed order by the last CTA (deterministic).
struct QualPart {
  double maxabs, sumsq;
  float mn, mx;
  uint32_t nan, pad;
};

__device__ __forceinline__ void qual_acc(float a, float b, double& m, double& s, float& mn,
                                         float& mx, uint32_t& nan) {
  const double d = __dsub_rn((double)a, (double)b);
  const double ad = fabs(d);
  nan += d != d;
  m = ad > m ? ad : m;
  s = __dadd_rn(s, __dmul_rn(d, d));
  mn = fminf(mn, a);
  mx = fmaxf(mx, a);
}

__global__ void __launch_bounds__(kAThreads) quality_kernel(const float* __restrict__ a,
                                                            const float* __restrict__ b,
                                                            uint64_t n, QualPart* parts,
                                                            uint32_t* counter, double* out) {
  __shared__ QualPart sp[kAWarps];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double m = 0.0, s = 0.0;
  float mn = FLT_MAX, mx = -FLT_MAX;
  uint32_t nan = 0;
  const uint64_t stride = (uint64_t)gridDim.x * kAThreads;
  const uint64_t first = (uint64_t)blockIdx.x * kAThreads + tid;
  const bool vec = (((uintptr_t)a | (uintptr_t)b) & 15) == 0;
  uint64_t tail0 = 0;
  if (vec) {
    const uint64_t nvec = n >> 2;
    for (uint64_t i = first; i < nvec; i += stride) {
      const float4 va = ld_stream_f4(a + 4 * i), vb = ld_stream_f4(b + 4 * i);
      qual_acc(va.x, vb.x, m, s, mn, mx, nan);
      qual_acc(va.y, vb.y, m, s, mn, mx, nan);
      qual_acc(va.z, vb.z, m, s, mn, mx, nan);
      qual_acc(va.w, vb.w, m, s, mn, mx, nan);
    }
    tail0 = 4 * nvec;
  }
  for (uint64_t i = tail0 + first; i < n; i += stride) qual_acc(a[i], b[i], m, s, mn, mx, nan);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const double om = __shfl_xor_sync(kFull, m, d);
    m = om > m ? om : m;
    s = __dadd_rn(s, __shfl_xor_sync(kFull, s, d));
    mn = fminf(mn, __shfl_xor_sync(kFull, mn, d));
    mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, d));
    nan += __shfl_xor_sync(kFull, nan, d);
  }
  if (lane == 0) sp[warp] = QualPart{m, s, mn, mx, nan, 0};
  __syncthreads();
  if (tid == 0) {
    QualPart p = sp[0];
    for (int w = 1; w < kAWarps; ++w) {
      p.maxabs = sp[w].maxabs > p.maxabs ? sp[w].maxabs : p.maxabs;
      p.sumsq = __dadd_rn(p.sumsq, sp[w].sumsq);
      p.mn = fminf(p.mn, sp[w].mn);
      p.mx = fmaxf(p.mx, sp[w].mx);
      p.nan += sp[w].nan;
    }
    parts[blockIdx.x] = p;
    __threadfence();
    s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last || tid != 0) return;
  __threadfence();
  QualPart p{0.0, 0.0, FLT_MAX, -FLT_MAX, 0, 0};
  for (uint32_t k = 0; k < gridDim.x; ++k) {  // fixed order: same bits every run
    const volatile QualPart& q = parts[k];
    p.maxabs = q.maxabs > p.maxabs ? q.maxabs : p.maxabs;
    p.sumsq = __dadd_rn(p.sumsq, q.sumsq);
    p.mn = fminf(p.mn, q.mn);
    p.mx = fmaxf(p.mx, q.mx);
    p.nan += q.nan;
  }
  out[0] = p.maxabs;
  out[1] = p.sumsq;
  out[2] = (double)p.mn;
  out[3] = (double)p.mx;
  out[4] = (double)p.nan;
  *counter = 0;  // re-arm
}

// ---- A3: block_range_cdf counts (metrics.py:128-146) -------------------------------------
// rel = (f64(block max) - f64(block min)) / global_range; count rel <= t per threshold.  The
// reference pads the last block with values[-1], which never changes its min / max.
constexpr int kMaxThresholds = 64;

__global__ void __launch_bounds__(kAThreads) block_range_kernel(
    const float* __restrict__ x, uint64_t n, uint32_t bs, double grange,
    const double* __restrict__ thr, uint32_t nthr, unsigned long long* counts) {
  __shared__ double s_thr[kMaxThresholds];
  __shared__ unsigned long long s_cnt[kMaxThresholds];
  for (uint32_t t = threadIdx.x; t < nthr; t += kAThreads) {
    s_thr[t] = thr[t];
    s_cnt[t] = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t nb = (n + bs - 1) / bs;
  const uint64_t wstride = (uint64_t)gridDim.x * kAWarps;
  for (uint64_t b = (uint64_t)blockIdx.x * kAWarps + (threadIdx.x >> 5); b < nb; b += wstride) {
    const uint64_t start = b * bs;
    float mn, mx;
    block_minmax(x + start, (uint32_t)umin64(bs, n - start), lane, mn, mx);
    const double rel = __ddiv_rn(__dsub_rn((double)mx, (double)mn), grange);
    for (uint32_t t = lane; t < nthr; t += 32)
      if (rel <= s_thr[t]) atomicAdd(&s_cnt[t], 1ull);
  }
  __syncthreads();
  for (uint32_t t = threadIdx.x; t < nthr; t += kAThreads)
    if (s_cnt[t]) atomicAdd(&counts[t], s_cnt[t]);
}

// ---- A4: exclusive int64 prefix scan (parallel.py:21-44) ---------------------------------
// Three passes over 2048-value tiles: tile sums, a single-CTA scan of the tile sums, then
// each tile's local scan plus its offset.  int64 wraps like NumPy's int64 adds.
constexpr int kScanItems = 8;
constexpr int kScanTile = kAThreads * kScanItems;

__device__ __forceinline__ long long block_excl_scan(long long v, long long* s_warp,
                                                     long long& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const long long t = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += t;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  long long wpre = 0;
  total = 0;
  for (int w = 0; w < kAWarps; ++w) {
    const long long sw = s_warp[w];
    if (w < warp) wpre += sw;
    total += sw;
  }
  __syncthreads();
  return wpre + incl - v;
}

__global__ void __launch_bounds__(kAThreads) scan_sums_kernel(const long long* __restrict__ in,
                                                              uint64_t n, long long* sums) {
  __shared__ long long s_warp[kAWarps];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  long long v = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint64_t i = base + (uint64_t)k * kAThreads + threadIdx.x;
    if (i < n) v += in[i];
  }
  long long total;
  block_excl_scan(v, s_warp, total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kAThreads) scan_tiles_kernel(long long* sums, uint64_t ntiles) {
  __shared__ long long s_warp[kAWarps];
  long long carry = 0;
  for (uint64_t b = 0; b < ntiles; b += kAThreads) {
    const uint64_t i = b + threadIdx.x;
    const long long v = i < ntiles ? sums[i] : 0;
    long long total;
    const long long ex = block_excl_scan(v, s_warp, total);
    if (i < ntiles) sums[i] = carry + ex;
    carry += total;
  }
}

__global__ void __launch_bounds__(kAThreads) scan_apply_kernel(const long long* __restrict__ in,
                                                               uint64_t n,
                                                               const long long* __restrict__ offs,
                                                               long long* out) {
  __shared__ long long s_warp[kAWarps];
  // thread t owns the kScanItems consecutive values base + t*kScanItems ..
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  long long v[kScanItems];
  long long sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < n ? in[base + k] : 0;
    sum += v[k];
  }
  long long total;
  long long run = offs[blockIdx.x] + block_excl_scan(sum, s_warp, total);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
}

// ---- A5: index propagation (parallel.py:74-101) ------------------------------------------
// propagate_indices: column j of the (count, q) position matrix is the running maximum of
// (i + 1 if byte j of element i is a mid byte, i.e. j >= min(code_i, q), else 0) -- what
// ceil(log2 count) stride-doubling rounds of propagate_round converge to.  One CTA, the
// columns scanned together, chunk by chunk with a carried maximum.
__global__ void __launch_bounds__(1024) propagate_kernel(const uint8_t* __restrict__ codes,
                                                         uint32_t count, uint32_t q,
                                                         long long* pos) {
  __shared__ uint32_t s_warp[32][4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t carry[4] = {0, 0, 0, 0};
  for (uint32_t c0 = 0; c0 < count; c0 += 1024) {
    const uint32_t i = c0 + threadIdx.x;
    const uint32_t code = i < count ? min((uint32_t)codes[i], q) : 4u;
    uint32_t v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[j] = (i < count && (uint32_t)j >= code) ? i + 1 : 0u;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, v[j], d);
        if (lane >= d) v[j] = max(v[j], t);
      }
    }
    if (lane == 31)
#pragma unroll
      for (int j = 0; j < 4; ++j) s_warp[warp][j] = v[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t pre = carry[j], all = carry[j];
      for (int w = 0; w < 32; ++w) {
        const uint32_t sw = s_warp[w][j];
        if (w < warp) pre = max(pre, sw);
        all = max(all, sw);
      }
      v[j] = max(v[j], pre);
      carry[j] = all;
    }
    __syncthreads();
    if (i < count)
      for (uint32_t j = 0; j < q; ++j) pos[(uint64_t)i * q + j] = v[j];
  }
}

// propagate_round: next[r] = max(p[r], p[r - stride]) for r >= stride (rows of `cols`).
__global__ void __launch_bounds__(kAThreads) propagate_round_kernel(const long long* __restrict__ p,
                                                                    uint64_t rows, uint32_t cols,
                                                                    uint64_t stride,
                                                                    long long* out) {
  const uint64_t total = rows * cols;
  for (uint64_t k = (uint64_t)blockIdx.x * kAThreads + threadIdx.x; k < total;
       k += (uint64_t)gridDim.x * kAThreads) {
    const uint64_t r = k / cols;
    long long v = p[k];
    if (r >= stride) {
      const long long u = p[k - stride * cols];
      v = u > v ? u : v;
    }
    out[k] = v;
  }
}

// ---- launchers -----------------------------------------------------------------------------
namespace {
int sms() {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || nsm <= 0)
      nsm = 148;
  }
  return nsm;
}
// one warp per block, up to 8 resident CTAs per SM
int warp_grid(uint64_t nb) {
  const uint64_t want = (nb + kAWarps - 1) / kAWarps;
  const uint64_t cap = (uint64_t)sms() * 8;
  return (int)(want < cap ? (want ? want : 1) : cap);
}
}  // namespace

int quality_grid(uint64_t n) {
  const uint64_t want = (n / 4 + kAThreads - 1) / kAThreads;
  const uint64_t cap = (uint64_t)sms() * 8;
  return (int)(want < cap ? (want ? want : 1) : cap);
}
size_t quality_part_bytes() { return sizeof(QualPart); }
uint64_t scan_tiles(uint64_t n) { return (n + kScanTile - 1) / kScanTile; }
uint32_t max_thresholds() { return kMaxThresholds; }

void launch_accounting(const float* x, uint64_t n, uint32_t bs, double e, int pe,
                       unsigned long long* bits, cudaStream_t s) {
  accounting_kernel<<<warp_grid((n + bs - 1) / bs), kAThreads, 0, s>>>(x, n, bs, e, pe, bits);
}

void launch_quality(const float* a, const float* b, uint64_t n, void* parts, uint32_t* counter,
                    double* out, cudaStream_t s) {
  quality_kernel<<<quality_grid(n), kAThreads, 0, s>>>(a, b, n, static_cast<QualPart*>(parts),
                                                       counter, out);
}

void launch_block_range(const float* x, uint64_t n, uint32_t bs, double grange, const double* thr,
                        uint32_t nthr, unsigned long long* counts, cudaStream_t s) {
  block_range_kernel<<<warp_grid((n + bs - 1) / bs), kAThreads, 0, s>>>(x, n, bs, grange, thr,
                                                                         nthr, counts);
}

void launch_prefix_scan(const long long* in, uint64_t n, long long* out, long long* sums,
                        cudaStream_t s) {
  const uint64_t nt = scan_tiles(n);
  scan_sums_kernel<<<(unsigned)nt, kAThreads, 0, s>>>(in, n, sums);
  scan_tiles_kernel<<<1, kAThreads, 0, s>>>(sums, nt);
  scan_apply_kernel<<<(unsigned)nt, kAThreads, 0, s>>>(in, n, sums, out);
}

void launch_propagate(const uint8_t* codes, uint32_t count, uint32_t q, long long* pos,
                      cudaStream_t s) {
  propagate_kernel<<<1, 1024, 0, s>>>(codes, count, q, pos);
}

void launch_propagate_round(const long long* p, uint64_t rows, uint32_t cols, uint64_t stride,
                            long long* out, cudaStream_t s) {
  const uint64_t total = rows * cols;
  uint64_t g = (total + kAThreads - 1) / kAThreads;
  const uint64_t cap = (uint64_t)sms() * 8;
  g = g < cap ? (g ? g : 1) : cap;
  propagate_round_kernel<<<(unsigned)g, kAThreads, 0, s>>>(p, rows, cols, stride, out);
}

}  // namespace szx
