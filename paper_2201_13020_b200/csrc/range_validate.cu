// range_validate.cu -- K0 (global range + finite check) and K3 (stream pool validation).
#include <cfloat>

#include "szx_device.cuh"
#include "szx_kernels.h"

namespace szx {

// ---- K0: DataField.__post_init__ finite check + global min/max (container.py:84-87) -----
constexpr int kRangeThreads = 512;

// CTAs for a range pass over n values (host and device agree).
__host__ __device__ __forceinline__ int range_grid_dev(uint64_t n) {
  const uint64_t vec = (n + 3) / 4;
  uint64_t g = (vec + kRangeThreads * 4 - 1) / (kRangeThreads * 4);
  if (g < 1) g = 1;
  if (g > 148 * 4) g = 148 * 4;
  return (int)g;
}

// One range pass of `x` by CTA `cta` of `G` (the last of the G CTAs to finish reduces the
// partials into result[0..1]).
__device__ __forceinline__ void range_body(const float* __restrict__ x, uint64_t n,
                                           uint32_t cta, uint32_t G, float* partials,
                                           uint32_t* counter, float* result, uint32_t* err) {
  __shared__ float s_mn[kRangeThreads / 32], s_mx[kRangeThreads / 32];
  __shared__ uint32_t s_bad[kRangeThreads / 32];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float mn = FLT_MAX, mx = -FLT_MAX;
  uint32_t bad = 0;
  // scalar head up to 16-byte alignment, then 16-byte vectors, then scalar tail
  const uint64_t head = umin64(n, ((16 - ((uintptr_t)x & 15)) & 15) >> 2);
  const uint64_t nvec = (n - head) >> 2;
  const float4* xv = reinterpret_cast<const float4*>(x + head);
  const uint64_t stride = (uint64_t)G * blockDim.x;
  uint64_t i = (uint64_t)cta * blockDim.x + tid;
  for (; i + 3 * stride < nvec; i += 4 * stride) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = ld_stream_f4(reinterpret_cast<const float*>(xv + i + u * stride));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      mn = fminf(mn, fminf(fminf(v[u].x, v[u].y), fminf(v[u].z, v[u].w)));
      mx = fmaxf(mx, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
      bad |= nonfinite(v[u].x) | nonfinite(v[u].y) | nonfinite(v[u].z) | nonfinite(v[u].w);
    }
  }
  for (; i < nvec; i += stride) {
    const float4 v = ld_stream_f4(reinterpret_cast<const float*>(xv + i));
    mn = fminf(mn, fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
    mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    bad |= nonfinite(v.x) | nonfinite(v.y) | nonfinite(v.z) | nonfinite(v.w);
  }
  if (cta == 0) {
    const uint64_t tail0 = head + 4 * nvec;
    for (uint64_t k = tid; k < head; k += blockDim.x) {
      const float v = x[k];
      mn = fminf(mn, v); mx = fmaxf(mx, v); bad |= nonfinite(v);
    }
    for (uint64_t k = tail0 + tid; k < n; k += blockDim.x) {
      const float v = x[k];
      mn = fminf(mn, v); mx = fmaxf(mx, v); bad |= nonfinite(v);
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(kFull, mn, d));
    mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, d));
    bad |= __shfl_xor_sync(kFull, bad, d);
  }
  if (lane == 0) { s_mn[warp] = mn; s_mx[warp] = mx; s_bad[warp] = bad; }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kRangeThreads / 32; ++w) {
      mn = fminf(mn, s_mn[w]); mx = fmaxf(mx, s_mx[w]); bad |= s_bad[w];
    }
    partials[2 * cta] = mn;
    partials[2 * cta + 1] = mx;
    if (bad) atomicOr(err, kErrNonFinite);
    __threadfence();
    s_last = atomicAdd(counter, 1u) == G - 1;
  }
  __syncthreads();
  if (!s_last) return;
  // last CTA: reduce the per-CTA partials
  __threadfence();
  mn = FLT_MAX; mx = -FLT_MAX;
  for (uint32_t k = tid; k < G; k += blockDim.x) {
    mn = fminf(mn, __ldcg(partials + 2 * k));
    mx = fmaxf(mx, __ldcg(partials + 2 * k + 1));
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(kFull, mn, d));
    mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, d));
  }
  if (lane == 0) { s_mn[warp] = mn; s_mx[warp] = mx; }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kRangeThreads / 32; ++w) { mn = fminf(mn, s_mn[w]); mx = fmaxf(mx, s_mx[w]); }
    result[0] = mn;
    result[1] = mx;
    *counter = 0;  // re-arm for the next launch
  }
}

__global__ void __launch_bounds__(kRangeThreads) range_kernel(const float* __restrict__ x,
                                                              uint64_t n, float* partials,
                                                              uint32_t* counter, float* result,
                                                              uint32_t* err) {
  range_body(x, n, blockIdx.x, gridDim.x, partials, counter, result, err);
}

// Batched (one launch for many fields, BASELINE configs[2]): CTA (b, f) of a (G, F) grid
// ranges field f; per-field partials (2G floats), counter, result pair and error word.
__global__ void __launch_bounds__(kRangeThreads) range_batch_kernel(const RangeField* __restrict__ fs,
                                                                    float* partials,
                                                                    uint32_t* counters,
                                                                    float* results,
                                                                    uint32_t* errs) {
  const uint32_t f = blockIdx.y, G = gridDim.x;
  const RangeField d = fs[f];
  const uint32_t g = (uint32_t)range_grid_dev(d.n);  // this field's share of the grid
  if (blockIdx.x >= g) return;
  range_body(d.x, d.n, blockIdx.x, g, partials + 2 * (uint64_t)G * f, counters + f,
             results + 2 * f, errs + f);
}

void launch_range_batch(const RangeField* d_fields, uint32_t nfields, int grid, float* partials,
                        uint32_t* counters, float* results, uint32_t* errs, cudaStream_t s) {
  range_batch_kernel<<<dim3(grid, nfields), kRangeThreads, 0, s>>>(d_fields, partials, counters,
                                                                   results, errs);
}

int range_grid(uint64_t n) { return range_grid_dev(n); }

void launch_range(const float* x, uint64_t n, float* partials, uint32_t* counter,
                  float* result, uint32_t* err, int grid, cudaStream_t s) {
  range_kernel<<<grid, kRangeThreads, 0, s>>>(x, n, partials, counter, result, err);
}

// ---- K3: mid-pool length + pool checks for deserialized / user-built streams -----------
// One thread per code byte (4 codes).  NC block r owns codes [r*bs, r*bs + count) because
// every NC block before the last is full (pipeline.py:46-51).
constexpr int kValThreads = 256;

__global__ void __launch_bounds__(kValThreads) validate_kernel(
    const uint8_t* __restrict__ req, uint64_t n_nc, const uint8_t* __restrict__ codes,
    uint64_t m, const float* __restrict__ mu, uint64_t nb, uint32_t bs,
    unsigned long long* mid_total, uint32_t* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t ncb = (m + 3) >> 2;
  unsigned long long total = 0;
  uint32_t flags = 0;
  for (uint64_t t = t0; t < ncb; t += stride) {
    const uint32_t cb = codes[t];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint64_t g = 4 * t + i;
      const int c = (cb >> (2 * i)) & 3;
      if (g < m) {
        const int rq = req[g / bs];
        int q, s;
        q_s_of(rq, q, s);
        total += (unsigned long long)(q - min(c, q));
      } else if (c) {
        flags |= kErrCodePadding;  // container.py:304-305
      }
    }
  }
  for (uint64_t t = t0; t < n_nc; t += stride) {
    const int rq = req[t];
    if (rq < 1 || rq > 32) flags |= kErrBadReq;  // container.py:206-207
  }
  for (uint64_t t = t0; t < nb; t += stride) {
    if (nonfinite(mu[t])) flags |= kErrMuNonFinite;  // container.py:198-199
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) total += __shfl_xor_sync(kFull, total, d);
  flags = __reduce_or_sync(kFull, flags);
  if ((threadIdx.x & 31) == 0) {
    if (total) atomicAdd(mid_total, total);
    if (flags) atomicOr(err, flags);
  }
}

void launch_validate(const uint8_t* req, uint64_t n_nc, const uint8_t* codes, uint64_t m,
                     const float* mu, uint64_t nb, uint32_t bs, unsigned long long* mid_total,
                     uint32_t* err, cudaStream_t s) {
  const uint64_t work = max(max((m + 3) / 4, n_nc), nb);
  uint64_t g = (work + kValThreads - 1) / kValThreads;
  if (g < 1) g = 1;
  if (g > 148 * 8) g = 148 * 8;
  validate_kernel<<<(int)g, kValThreads, 0, s>>>(req, n_nc, codes, m, mu, nb, bs, mid_total, err);
}

}  // namespace szx
