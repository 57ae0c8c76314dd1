// abi.cu -- extern "C" boundary of libszx_b200.so (declared in include/szx_b200.h).
//
// Device-pointer entry points: chunking, scratch layout and kernel selection.
// Host-buffer entry points: the reference's user-level calls
//   serialize(compress(DataField(x), cfg))   container.py:309-326, pipeline.py:177-183
//   decompress(deserialize(blob)).values     container.py:349-416, pipeline.py:227-260
// on a library-owned device arena, with the container header handled here on the host.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/szx_b200.h"
#include "szx_kernels.h"

using namespace szx;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(SZX_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CU(call)                                          \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);   \
  } while (0)

inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

int num_sms() {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || nsm <= 0)
      nsm = 148;
  }
  return nsm;
}
inline bool aligned(const void* p, uintptr_t a) { return ((uintptr_t)p & (a - 1)) == 0; }

// ---- chunk plan -----------------------------------------------------------------------
// The look-back payload packs (non-constant blocks : 26 bits, mid bytes : 36 bits); a
// chunk is bounded so neither field can overflow, and chunks start on 64-block multiples
// so every chunk's map bytes and (for bs == 128) code bytes are whole bytes.
struct Plan {
  uint64_t nb, chunk_blocks, nchunks, tile_blocks, tiles_total;
  bool fast;
};

uint64_t g_chunk_override = 0;  // testing hook: szx_set_max_chunk_blocks
// K3 sums the map words before its range directly up to this many blocks (2 MiB of map),
// beyond it a decoupled look-back over the CTAs; testing hook: szx_set_index_direct_limit
uint64_t g_index_direct_limit = 1ull << 24;
// K3 kernel: 1 = one range per SM (index128_kernel, default), 2 = one 16-tile chunk per CTA
// (index128v2_kernel: 46 vs 31 us on NYX, its two chained look-backs per chunk cost more than
// the serial chunks of v1); testing hook szx_set_index_kernel
int g_index_kernel = 1;

// bs == 128 compress kernel: 1 = the CTA-tile compress128_kernel (64-block tiles, faster on
// smooth fields), 2 = the warp-autonomous encode128_kernel (88-block super-tiles, faster on
// noisy fields); testing / benchmarking hook szx_set_compress_variant
int g_k1_variant = 1;

// compress: the tiled kernels for the fast block sizes; decompress: K3 + K2 exist for bs == 128
// only, every other block size decodes with the generic kernel (kGenTileBlocks tiles)
Plan make_plan(uint64_t n, uint32_t bs, bool compress = true) {
  Plan p{};
  p.nb = ceil_div(n, bs);
  p.fast = fast_bs(bs);
  // bs == 128: the selected compress variant's tiles (szx_compress_scratch_bytes sizes scratch
  // for the smallest, so a variant switch between the size query and the launch stays in
  // bounds); bs 64 / 256 / 512: variant 1's 8192-value tiles
  p.tile_blocks = !p.fast      ? kGenTileBlocks
                  : bs != 128 ? 8192 / bs
                  : (g_k1_variant == 2   ? kEncTileBlocks
                     : g_k1_variant == 3 ? kV3TileBlocks
                     : g_k1_variant == 5 ? kV5TileBlocks
                                         : kCompTileBlocks);
  uint64_t cap = (1ull << 26) - 64;
  const uint64_t by_bytes = (1ull << 33) / bs;
  if (by_bytes < cap) cap = by_bytes;
  if (g_chunk_override && g_chunk_override < cap) cap = g_chunk_override;
  // chunks start on whole tiles (and whole 64-block map words)
  const uint64_t unit = (p.fast && bs != 128 && p.tile_blocks > 64) ? p.tile_blocks : 64;
  cap = cap / unit * unit;
  if (cap < unit) cap = unit;
  p.chunk_blocks = p.nb < cap ? p.nb : cap;
  p.nchunks = p.nb ? ceil_div(p.nb, p.chunk_blocks) : 0;
  p.tiles_total = 0;
  for (uint64_t c = 0; c < p.nchunks; ++c) {
    const uint64_t b0 = c * p.chunk_blocks;
    const uint64_t b1 = b0 + p.chunk_blocks < p.nb ? b0 + p.chunk_blocks : p.nb;
    p.tiles_total += ceil_div(b1 - b0, p.tile_blocks);
  }
  return p;
}

size_t scratch_layout(const Plan& p, int chains, size_t* off_counter, size_t* off_status) {
  size_t off = sizeof(Totals) * (p.nchunks + 1);
  *off_counter = off;
  off += 8 * ((p.nchunks + 1) / 2 + 1);
  off = (off + 255) & ~size_t(255);
  *off_status = off;
  off += 8 * p.tiles_total * chains;
  return off;
}

bool valid_bs(uint32_t bs) { return bs >= 8 && bs <= 65535; }

int compress_impl(const float* d_x, uint64_t n, uint32_t bs, double e, uint8_t* d_map,
                  float* d_mu, uint8_t* d_req, uint8_t* d_codes, uint8_t* d_mid,
                  szx_totals* d_totals, uint32_t* d_err, void* d_scratch, size_t scratch_bytes,
                  uint64_t* d_index, void* stream);

}  // namespace

extern "C" {

const char* szx_version(void) { return "szx-b200 0.1.0 (sm_100a)"; }
const char* szx_last_error(void) { return g_err.c_str(); }
int32_t szx_bound_exponent(double e) {
  int ex = 0;
  std::frexp(e, &ex);
  return ex - 1;
}

int szx_debug_stats(uint64_t* out8, int reset) {
  unsigned long long h[16];
  // reset bit 0: clear after reading; bits 1-2 select the kernel (0 compress, 1 index, 2 decode)
  const int which = (reset >> 1) & 7;
  CU(which == 4   ? szx::v3_stats(h, (reset & 1) != 0)
     : which == 1 ? szx::index_stats(h, (reset & 1) != 0)
     : which == 2 ? szx::decode_stats(h, (reset & 1) != 0)
     : which == 3 ? szx::encode_stats(h, (reset & 1) != 0)
                  : szx::compress_stats(h, (reset & 1) != 0));
  const int nout = which >= 3 ? 16 : 8;  // encode128 / compress128v3 keep 16 counters
  for (int i = 0; i < nout; ++i) out8[i] = h[i];
  return SZX_OK;
}

int szx_debug_trace(void* d_buf) {
  CU(szx::k1_trace_buffer(static_cast<unsigned long long*>(d_buf)));
  return SZX_OK;
}

int szx_set_index_kernel(int kernel) {
  const int old = g_index_kernel;
  if (kernel == 1 || kernel == 2) g_index_kernel = kernel;
  return old;
}

uint64_t szx_set_index_direct_limit(uint64_t blocks) {
  const uint64_t old = g_index_direct_limit;
  g_index_direct_limit = blocks;
  return old;
}

uint64_t szx_set_max_chunk_blocks(uint64_t blocks) {
  const uint64_t old = g_chunk_override;
  g_chunk_override = blocks;
  return old;
}

uint64_t szx_num_blocks(uint64_t n, uint32_t bs) { return bs ? ceil_div(n, bs) : 0; }
uint64_t szx_map_bytes(uint64_t n, uint32_t bs) {
  // rounded up to the 4-byte tile words the bs == 128 kernel stores
  return ceil_div(ceil_div(szx_num_blocks(n, bs), 8), 4) * 4;
}
// worst-case packed code bytes, word-rounded, plus the decoder's 32-byte row + 16-byte
// alignment slack for a short last block
uint64_t szx_codes_capacity(uint64_t n) { return ceil_div(ceil_div(n, 4), 4) * 4 + 64; }

// ---- K0 ---------------------------------------------------------------------------------
size_t szx_range_scratch_bytes(uint64_t n) {
  return 256 + 8 * (size_t)range_grid(n);
}

int szx_range_f32(const float* d_x, uint64_t n, float* d_minmax, uint32_t* d_err,
                  void* d_scratch, size_t scratch_bytes, void* stream) {
  if (n == 0) return fail(SZX_ERR_INVALID_ARG, "empty dataset");
  if (scratch_bytes < szx_range_scratch_bytes(n) || !aligned(d_scratch, 256))
    return fail(SZX_ERR_INVALID_ARG, "range scratch too small or misaligned");
  const int grid = range_grid(n);
  uint32_t* counter = static_cast<uint32_t*>(d_scratch);
  float* partials = reinterpret_cast<float*>(static_cast<char*>(d_scratch) + 256);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CU(cudaMemsetAsync(counter, 0, 4, s));
  launch_range(d_x, n, partials, counter, d_minmax, d_err, grid, s);
  CU(cudaGetLastError());
  return SZX_OK;
}

// ---- K1 ---------------------------------------------------------------------------------
size_t szx_compress_scratch_bytes(uint64_t n, uint32_t bs) {
  if (!valid_bs(bs)) return 0;
  size_t a, b;
  const int v = g_k1_variant;
  // the smallest tiles of the bs == 128 kernels (most look-back words): variant 5's
  // 32-block tiles, else variant 1's 64
  g_k1_variant = kV5TileBlocks < kCompTileBlocks ? 5 : 1;
  const size_t bytes = scratch_layout(make_plan(n, bs), 1, &a, &b);
  g_k1_variant = v;
  return bytes;
}

int szx_set_compress_variant(int variant) {
  const int old = g_k1_variant;
  if (variant >= 1 && variant <= 5) g_k1_variant = variant;
  return old;
}

int szx_compress_emits_index(uint32_t bs) {
  return fast_bs(bs) && (bs != 128 || g_k1_variant == 1);  // bs != 128 always runs variant 1
}

int szx_compress_indexed_f32(const float* d_x, uint64_t n, uint32_t bs, double e, uint8_t* d_map,
                             float* d_mu, uint8_t* d_req, uint8_t* d_codes, uint8_t* d_mid,
                             szx_totals* d_totals, uint32_t* d_err, void* d_scratch,
                             size_t scratch_bytes, uint64_t* d_index, void* stream) {
  if (!szx_compress_emits_index(bs))
    return fail(SZX_ERR_INVALID_ARG,
                "the decode index is emitted for block sizes 64/128/256/512 by the default kernel");
  if (!aligned(d_index, 16)) return fail(SZX_ERR_ALIGN, "index needs 16-byte alignment");
  return compress_impl(d_x, n, bs, e, d_map, d_mu, d_req, d_codes, d_mid, d_totals, d_err,
                       d_scratch, scratch_bytes, d_index, stream);
}

int szx_compress_f32(const float* d_x, uint64_t n, uint32_t bs, double e, uint8_t* d_map,
                     float* d_mu, uint8_t* d_req, uint8_t* d_codes, uint8_t* d_mid,
                     szx_totals* d_totals, uint32_t* d_err, void* d_scratch,
                     size_t scratch_bytes, void* stream) {
  return compress_impl(d_x, n, bs, e, d_map, d_mu, d_req, d_codes, d_mid, d_totals, d_err,
                       d_scratch, scratch_bytes, nullptr, stream);
}

}  // extern "C"

namespace {
int compress_impl(const float* d_x, uint64_t n, uint32_t bs, double e, uint8_t* d_map,
                  float* d_mu, uint8_t* d_req, uint8_t* d_codes, uint8_t* d_mid,
                  szx_totals* d_totals, uint32_t* d_err, void* d_scratch, size_t scratch_bytes,
                  uint64_t* d_index, void* stream) {
  if (n == 0) return fail(SZX_ERR_INVALID_ARG, "empty dataset");
  if (!valid_bs(bs)) return fail(SZX_ERR_INVALID_ARG, "block size outside 8..65535");
  if (!(e > 0) || !std::isfinite(e)) return fail(SZX_ERR_INVALID_ARG, "bound must be positive finite");
  if (!aligned(d_x, 16) || !aligned(d_mid, 16) || !aligned(d_map, 4) || !aligned(d_codes, 4) ||
      !aligned(d_mu, 4))
    return fail(SZX_ERR_ALIGN, "x/mid need 16-byte, map/codes/mu 4-byte alignment");
  const Plan p = make_plan(n, bs);
  size_t off_counter, off_status;
  const size_t need = scratch_layout(p, 1, &off_counter, &off_status);
  if (scratch_bytes < need || !aligned(d_scratch, 256))
    return fail(SZX_ERR_INVALID_ARG, "compress scratch too small or misaligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* sc = static_cast<char*>(d_scratch);
  CU(cudaMemsetAsync(sc, 0, need, s));
  if (!p.fast) CU(cudaMemsetAsync(d_codes, 0, szx_codes_capacity(n), s));
  Totals* slots = reinterpret_cast<Totals*>(sc);
  uint32_t* counters = reinterpret_cast<uint32_t*>(sc + off_counter);
  uint64_t* status = reinterpret_cast<uint64_t*>(sc + off_status);
  uint64_t tile_off = 0;
  for (uint64_t c = 0; c < p.nchunks; ++c) {
    const uint64_t b0 = c * p.chunk_blocks;
    const uint64_t b1 = b0 + p.chunk_blocks < p.nb ? b0 + p.chunk_blocks : p.nb;
    const uint64_t v0 = b0 * bs, v1 = b1 * bs < n ? b1 * bs : n;
    CompressArgs a{};
    a.x = d_x + v0;
    a.n = v1 - v0;
    a.bs = bs;
    a.e = e;
    a.pe = szx_bound_exponent(e);
    a.map = d_map + b0 / 8;
    a.mu = d_mu + b0;
    a.req = d_req;
    a.codes = d_codes;
    a.mid = d_mid;
    a.base = c ? &slots[c] : nullptr;
    a.totals = c + 1 == p.nchunks ? reinterpret_cast<Totals*>(d_totals) : &slots[c + 1];
    a.ntiles = (uint32_t)ceil_div(b1 - b0, p.tile_blocks);
    a.status = status + tile_off;
    a.counter = counters + c;
    a.err = d_err;
    if (d_index) {
      a.index = d_index;
      const uint64_t tb = 8192 / bs;  // blocks per 8192-value tile (compress = decode tiles)
      a.idx_tile0 = b0 / tb;
      a.idx_ntiles = ceil_div(p.nb, tb);
      a.idx_last = c + 1 == p.nchunks;
    }
    tile_off += a.ntiles;
    if (p.fast && bs != 128) CU(launch_compress_fast(a, s));
    else if (p.fast) CU(g_k1_variant == 1   ? launch_compress128(a, s)
                   : g_k1_variant == 3 ? launch_compress128v3(a, s)
                   : g_k1_variant == 4 ? launch_compress128v4(a, s)
                   : g_k1_variant == 5 ? launch_compress128v5(a, s)
                                       : launch_encode128(a, s));
    else launch_compress_generic(a, s);
    CU(cudaGetLastError());
  }
  return SZX_OK;
}

}  // namespace

extern "C" {

// ---- K3 ---------------------------------------------------------------------------------
int szx_validate_f32(const uint8_t* d_req, uint64_t n_nc, const uint8_t* d_codes, uint64_t m,
                     const float* d_mu, uint64_t nb, uint32_t bs, uint64_t* d_mid_total,
                     uint32_t* d_err, void* stream) {
  if (!valid_bs(bs)) return fail(SZX_ERR_INVALID_ARG, "block size outside 8..65535");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CU(cudaMemsetAsync(d_mid_total, 0, 8, s));
  launch_validate(d_req, n_nc, d_codes, m, d_mu, nb, bs,
                  reinterpret_cast<unsigned long long*>(d_mid_total), d_err, s);
  CU(cudaGetLastError());
  return SZX_OK;
}

// ---- K3 index + K2 decode ---------------------------------------------------------------
namespace {
struct IndexLayout {
  uint64_t ntiles, ngroups, nstatus;
  size_t off_index, off_status, off_counter, off_stats, total;
};
IndexLayout index_layout(uint64_t n) {
  IndexLayout L{};
  const uint64_t nb = ceil_div(n, 128);
  L.ntiles = ceil_div(nb, kDecTileBlocks);
  // K3 runs kIndexCtasPerSm CTAs per SM, each owning a contiguous range of decode tiles
  // (<= kIndexMaxRanges ranges: the decoder keeps their bases in shared memory)
  const uint64_t want = (uint64_t)num_sms() * kIndexCtasPerSm;
  const uint64_t ctas = want < (uint64_t)kIndexMaxRanges ? want : (uint64_t)kIndexMaxRanges;
  L.ngroups = L.ntiles < ctas ? L.ntiles : ctas;
  size_t off = 0;
  L.off_index = off;  // entries + closing entry + one mid base per K3 range (szx_index_bytes)
  off += kIndexEntryBytes * (L.ntiles + 1) + 8 * ((L.ngroups + 1) & ~1ull);
  off = (off + 255) & ~size_t(255);
  L.off_status = off;
  // two look-back words per K3 range (v1) or per 16-tile chunk (v2)
  const uint64_t nst = L.ngroups > index128v2_chunks(n) ? L.ngroups : index128v2_chunks(n);
  L.nstatus = nst;
  off += 16 * nst;
  L.off_counter = off;
  off += 16;
  L.off_stats = off;  // nc_total, mid_total
  off += 16;
  L.total = (off + 255) & ~size_t(255);
  return L;
}
}  // namespace

uint64_t szx_index_bytes(uint64_t n, uint32_t bs) {
  // 8192-value tiles for every fast block size: ceil(ceil(n / bs) / (8192 / bs)) = ceil(n / 8192)
  if (!fast_bs(bs) || n == 0) return 0;
  const IndexLayout L = index_layout(n);  // entries + closing entry + one base per K3 range
  return kIndexEntryBytes * (L.ntiles + 1) + 8 * ((L.ngroups + 1) & ~1ull);
}

size_t szx_index_scratch_bytes(uint64_t n, uint32_t bs) {
  return fast_bs(bs) ? index_layout(n).total : 0;
}

int szx_index_f32(const uint8_t* d_map, const float* d_mu, const uint8_t* d_req,
                  const uint8_t* d_codes, uint64_t n, uint32_t bs, uint64_t* d_index,
                  uint64_t* d_stats, uint32_t* d_err, void* d_scratch, size_t scratch_bytes,
                  void* stream) {
  if (n == 0) return fail(SZX_ERR_INVALID_ARG, "empty stream");
  if (!fast_bs(bs))
    return fail(SZX_ERR_INVALID_ARG, "the tile index exists for block sizes 64/128/256/512");
  if (!aligned(d_index, 16) || !aligned(d_mu, 4))
    return fail(SZX_ERR_ALIGN, "index needs 16-byte, mu 4-byte alignment");
  const IndexLayout L = index_layout(n);
  if (scratch_bytes < L.total || !aligned(d_scratch, 256))
    return fail(SZX_ERR_INVALID_ARG, "index scratch too small or misaligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* sc = static_cast<char*>(d_scratch);
  CU(cudaMemsetAsync(sc + L.off_status, 0, L.total - L.off_status, s));
  IndexArgs a{};
  a.map = d_map;
  a.mu = d_mu;
  a.req = d_req;
  a.codes = d_codes;
  a.n = n;
  a.index = d_index;
  a.nc_total = reinterpret_cast<unsigned long long*>(d_stats);
  a.mid_total = reinterpret_cast<unsigned long long*>(d_stats) + 1;
  a.err = d_err;
  a.status_nc = reinterpret_cast<uint64_t*>(sc + L.off_status);
  a.status_mid = a.status_nc + L.nstatus;
  a.counter = reinterpret_cast<uint32_t*>(sc + L.off_counter);
  a.ngroups = (uint32_t)L.ngroups;
  a.direct_limit = g_index_direct_limit;
  a.bs = bs;
  if (g_index_kernel == 2 && bs == 128) launch_index128v2(a, s);
  else launch_index128(a, s);
  CU(cudaGetLastError());
  return SZX_OK;
}

int szx_decompress_indexed_f32(const uint8_t* d_map, const float* d_mu, const uint8_t* d_req,
                               const uint8_t* d_codes, const uint8_t* d_mid, uint64_t mid_len,
                               uint64_t n, uint32_t bs, const uint64_t* d_index, float* d_out,
                               uint32_t* d_err, void* stream) {
  if (n == 0) return fail(SZX_ERR_INVALID_ARG, "empty stream");
  if (!fast_bs(bs))
    return fail(SZX_ERR_INVALID_ARG, "indexed decode exists for block sizes 64/128/256/512");
  if (!aligned(d_out, 16) || !aligned(d_index, 16) || !aligned(d_mu, 4))
    return fail(SZX_ERR_ALIGN, "out/index need 16-byte, mu 4-byte alignment");
  Decode128Args a{};
  a.map = d_map;
  a.mu = d_mu;
  a.req = d_req;
  a.codes = d_codes;
  a.mid = d_mid;
  a.mid_len = mid_len;
  a.index = d_index;
  a.out = d_out;
  a.n = n;
  a.ntiles = ceil_div(n, (uint64_t)8192);  // 8192-value tiles
  a.tile_begin = 0;
  a.tile_end = a.ntiles;
  a.err = d_err;
  a.bs = bs;
  launch_decode128(a, static_cast<cudaStream_t>(stream));
  CU(cudaGetLastError());
  return SZX_OK;
}

size_t szx_decompress_scratch_bytes(uint64_t n, uint32_t bs) {
  if (!valid_bs(bs)) return 0;
  if (fast_bs(bs)) return index_layout(n).total;
  size_t a, b;
  return scratch_layout(make_plan(n, bs, false), 2, &a, &b);
}

int szx_decompress_f32(const uint8_t* d_map, const float* d_mu, const uint8_t* d_req,
                       const uint8_t* d_codes, const uint8_t* d_mid, uint64_t mid_len,
                       uint64_t n, uint32_t bs, float* d_out, szx_totals* d_totals,
                       uint32_t* d_err, void* d_scratch, size_t scratch_bytes, void* stream) {
  if (n == 0) return fail(SZX_ERR_INVALID_ARG, "empty stream");
  if (!valid_bs(bs)) return fail(SZX_ERR_INVALID_ARG, "block size outside 8..65535");
  if (fast_bs(bs)) {  // scan of the stored sizes (K3), then one decode pass (K2)
    const IndexLayout L = index_layout(n);
    if (scratch_bytes < L.total || !aligned(d_scratch, 256))
      return fail(SZX_ERR_INVALID_ARG, "decompress scratch too small or misaligned");
    char* sc = static_cast<char*>(d_scratch);
    uint64_t* index = reinterpret_cast<uint64_t*>(sc + L.off_index);
    uint64_t* stats = reinterpret_cast<uint64_t*>(sc + L.off_stats);
    int rc = szx_index_f32(d_map, d_mu, d_req, d_codes, n, bs, index, stats, d_err, d_scratch,
                           scratch_bytes, stream);
    if (rc) return rc;
    rc = szx_decompress_indexed_f32(d_map, d_mu, d_req, d_codes, d_mid, mid_len, n, bs, index,
                                    d_out, d_err, stream);
    if (rc) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // d_totals = {n_nc, 0, mid_len implied by the codes, 0}
    CU(cudaMemsetAsync(d_totals, 0, sizeof(szx_totals), s));
    CU(cudaMemcpyAsync(&d_totals->n_nc, stats, 8, cudaMemcpyDeviceToDevice, s));
    CU(cudaMemcpyAsync(&d_totals->mid_len, stats + 1, 8, cudaMemcpyDeviceToDevice, s));
    return SZX_OK;
  }
  const Plan p = make_plan(n, bs, false);
  if (!aligned(d_out, 16) || !aligned(d_mid, 16))
    return fail(SZX_ERR_ALIGN, "out/mid need 16-byte alignment");
  size_t off_counter, off_status;
  const size_t need = scratch_layout(p, 2, &off_counter, &off_status);
  if (scratch_bytes < need || !aligned(d_scratch, 256))
    return fail(SZX_ERR_INVALID_ARG, "decompress scratch too small or misaligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* sc = static_cast<char*>(d_scratch);
  CU(cudaMemsetAsync(sc, 0, need, s));
  Totals* slots = reinterpret_cast<Totals*>(sc);
  uint32_t* counters = reinterpret_cast<uint32_t*>(sc + off_counter);
  uint64_t* status = reinterpret_cast<uint64_t*>(sc + off_status);
  uint64_t tile_off = 0;
  for (uint64_t c = 0; c < p.nchunks; ++c) {
    const uint64_t b0 = c * p.chunk_blocks;
    const uint64_t b1 = b0 + p.chunk_blocks < p.nb ? b0 + p.chunk_blocks : p.nb;
    const uint64_t v0 = b0 * bs, v1 = b1 * bs < n ? b1 * bs : n;
    DecompressArgs a{};
    a.map = d_map + b0 / 8;
    a.mu = d_mu + b0;
    a.req = d_req;
    a.codes = d_codes;
    a.mid = d_mid;
    a.mid_len = mid_len;
    a.out = d_out + v0;
    a.n = v1 - v0;
    a.bs = bs;
    a.base = c ? &slots[c] : nullptr;
    a.totals = c + 1 == p.nchunks ? reinterpret_cast<Totals*>(d_totals) : &slots[c + 1];
    a.ntiles = (uint32_t)ceil_div(b1 - b0, p.tile_blocks);
    a.status_nc = status + tile_off;
    a.status_mid = status + p.tiles_total + tile_off;
    a.counter = counters + c;
    a.err = d_err;
    tile_off += a.ntiles;
    launch_decompress_generic(a, s);
    CU(cudaGetLastError());
  }
  return SZX_OK;
}

}  // extern "C"

// =========================================================================================
// Host-buffer API
// =========================================================================================
namespace {

constexpr size_t kHead = 17;  // struct "<4sBBHdB" (container.py:35)

constexpr int kPipeParts = 32;  // host pipelines: at most this many copy parts / decode chunks

struct Ctx {
  std::mutex mu;
  bool ready = false;
  cudaStream_t stream = nullptr;            // kernels
  cudaStream_t s_in = nullptr, s_out = nullptr;  // host->device / device->host copies
  cudaEvent_t ev_head = nullptr, ev_pre = nullptr, ev_mid[kPipeParts] = {}, ev_dec[kPipeParts] = {};
  char* arena = nullptr;
  size_t cap = 0;
  int parts = 8;  // decompress: mid H2D parts = decode chunks (szx_set_host_pipeline)
  // pinned host copy of the decode index + stream checks (a pageable destination would make
  // the index read-back a staged, synchronous copy on the decompress critical path)
  uint64_t* h_idx = nullptr;
  size_t h_idx_cap = 0;
  uint8_t* h_small = nullptr;  // 256 pinned bytes for the compress path's small read-backs
  uint64_t* h_plan = nullptr;  // mapped pinned: plan_bounds_kernel output (kPipeParts + 2)
  // szx_set_host_pipeline(.., trace = 1): timing events at the pipeline stages, printed to
  // stderr after each host call (benchmarking aid)
  bool trace = false;
  int ntr = 0;
  cudaEvent_t tr_ev[192] = {};
  const char* tr_name[192] = {};
  int tr_idx[192] = {};
};
Ctx g_ctx;

// The decode plan's mid offsets, written by the GPU straight into mapped pinned memory:
// out[j] = mid_before(t_j) for the P chunk bounds t_j = ntiles (j + 1) / P, out[P] the stream's
// derived mid total, out[P + 1] the error word.  (A copy-engine read-back would queue behind
// the first chunk's device->host copy.)
__global__ void plan_bounds_kernel(const uint64_t* __restrict__ idx, uint64_t ntiles, int P,
                                   const uint64_t* __restrict__ stats,
                                   const uint32_t* __restrict__ err, volatile uint64_t* out) {
  const int j = threadIdx.x;
  constexpr uint64_t ew = kIndexEntryBytes / 8;
  if (j < P) {
    const uint64_t t = ntiles * (uint64_t)(j + 1) / (uint64_t)P;
    const uint64_t c = idx[ew * t + 6];
    out[j] = idx[ew * t + 1] + idx[ew * (ntiles + 1) + c];
  } else if (j == P) {
    out[P] = stats[1];
  } else if (j == P + 1) {
    out[P + 1] = *err;
  }
}

void trace_mark(const char* name, cudaStream_t st, int idx = -1) {
  if (!g_ctx.trace || g_ctx.ntr >= 192) return;
  cudaEvent_t& e = g_ctx.tr_ev[g_ctx.ntr];
  if (!e) cudaEventCreate(&e);
  cudaEventRecord(e, st);
  g_ctx.tr_name[g_ctx.ntr] = name;
  g_ctx.tr_idx[g_ctx.ntr] = idx;
  ++g_ctx.ntr;
}
void trace_dump(const char* what) {
  if (!g_ctx.trace) return;
  cudaDeviceSynchronize();
  std::fprintf(stderr, "[szx host trace] %s\n", what);
  for (int i = 0; i < g_ctx.ntr; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, g_ctx.tr_ev[0], g_ctx.tr_ev[i]);
    if (g_ctx.tr_idx[i] >= 0)
      std::fprintf(stderr, "  %8.3f ms  %s[%d]\n", ms, g_ctx.tr_name[i], g_ctx.tr_idx[i]);
    else
      std::fprintf(stderr, "  %8.3f ms  %s\n", ms, g_ctx.tr_name[i]);
  }
  g_ctx.ntr = 0;
}

int ctx_ready() {
  if (g_ctx.ready) return SZX_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(SZX_ERR_NO_DEVICE, "no CUDA device visible (the library has no CPU path)");
  CU(cudaStreamCreateWithFlags(&g_ctx.stream, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&g_ctx.s_in, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&g_ctx.s_out, cudaStreamNonBlocking));
  CU(cudaMallocHost(&g_ctx.h_small, 256));
  CU(cudaHostAlloc(&g_ctx.h_plan, 8 * (kPipeParts + 2), cudaHostAllocMapped));
  CU(cudaEventCreateWithFlags(&g_ctx.ev_head, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&g_ctx.ev_pre, cudaEventDisableTiming));
  for (int i = 0; i < kPipeParts; ++i) {
    CU(cudaEventCreateWithFlags(&g_ctx.ev_mid[i], cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&g_ctx.ev_dec[i], cudaEventDisableTiming));
  }
  g_ctx.ready = true;
  return SZX_OK;
}

int ctx_reserve(size_t bytes) {
  if (bytes <= g_ctx.cap) return SZX_OK;
  if (g_ctx.arena) CU(cudaFree(g_ctx.arena));
  g_ctx.arena = nullptr;
  g_ctx.cap = 0;
  const size_t want = bytes + bytes / 8;
  CU(cudaMalloc(&g_ctx.arena, want));
  g_ctx.cap = want;
  return SZX_OK;
}

struct Bump {
  size_t off = 0;
  size_t take(size_t bytes, size_t align = 256) {
    off = (off + align - 1) / align * align;
    const size_t at = off;
    off += bytes;
    return at;
  }
};

void put_le(uint8_t* p, uint64_t v, int nbytes) {
  for (int i = 0; i < nbytes; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
uint64_t get_le(const uint8_t* p, int nbytes) {
  uint64_t v = 0;
  for (int i = 0; i < nbytes; ++i) v |= (uint64_t)p[i] << (8 * i);
  return v;
}

// Header parse with the reference's check order (container.py:351-370).
struct Header {
  uint32_t bs, ndims;
  double e;
  uint64_t n, nb;
  size_t pos;  // first byte after dims
  std::vector<uint64_t> dims;
};

int parse_header(const uint8_t* in, uint64_t len, Header& h) {
  if (len < kHead) return fail(SZX_ERR_TRUNCATED, "stream ends inside header");
  if (std::memcmp(in, "UFZX", 4) != 0) return fail(SZX_ERR_MAGIC, "bad magic");
  if (in[4] != 1) return fail(SZX_ERR_VERSION, "unsupported version");
  if (in[5] == 1) return fail(SZX_ERR_DTYPE, "float64 payloads are reserved and not supported");
  if (in[5] != 0) return fail(SZX_ERR_DTYPE, "unknown dtype code");
  h.bs = (uint32_t)get_le(in + 6, 2);
  uint64_t ebits = get_le(in + 8, 8);
  std::memcpy(&h.e, &ebits, 8);
  h.ndims = in[16];
  if (h.ndims < 1) return fail(SZX_ERR_INCONSISTENT, "ndims must be >= 1");
  if (len < kHead + 8ull * h.ndims) return fail(SZX_ERR_TRUNCATED, "stream ends inside dims");
  h.dims.resize(h.ndims);
  h.n = 1;
  bool overflow = false;
  for (uint32_t i = 0; i < h.ndims; ++i) {
    h.dims[i] = get_le(in + kHead + 8 * i, 8);
    if (h.dims[i] == 0) return fail(SZX_ERR_INCONSISTENT, "zero dimension");
  }
  for (uint32_t i = 0; i < h.ndims; ++i) {
    if (h.dims[i] && h.n > UINT64_MAX / h.dims[i]) overflow = true;
    h.n *= h.dims[i];
  }
  if (!valid_bs(h.bs)) return fail(SZX_ERR_INCONSISTENT, "block size out of range");
  if (!(h.e > 0) || !std::isfinite(h.e)) return fail(SZX_ERR_INCONSISTENT, "error bound not positive finite");
  if (overflow) return fail(SZX_ERR_TRUNCATED, "dims product overflows");
  h.nb = ceil_div(h.n, h.bs);
  h.pos = kHead + 8ull * h.ndims;
  return SZX_OK;
}

}  // namespace

extern "C" {

int szx_set_host_pipeline(int parts, int trace) {
  std::lock_guard<std::mutex> lock(g_ctx.mu);
  const int old = g_ctx.parts;
  if (parts >= 1 && parts <= kPipeParts) g_ctx.parts = parts;
  g_ctx.trace = trace != 0;
  g_ctx.ntr = 0;
  return old;
}

uint64_t szx_compress_bound(uint64_t n, uint32_t ndims, uint32_t bs) {
  if (!valid_bs(bs)) return 0;
  const uint64_t nb = ceil_div(n, bs);
  return kHead + 8ull * ndims + ceil_div(nb, 8) + 4 * nb + nb + ceil_div(2 * n, 8) + 4 * n;
}

int szx_compress_host(const float* h_x, const uint64_t* dims, uint32_t ndims, uint32_t bs,
                      int32_t rel_mode, double magnitude, uint8_t* h_out,
                      uint64_t out_capacity, uint64_t* out_len) {
  std::lock_guard<std::mutex> lock(g_ctx.mu);
  if (ndims < 1 || ndims > 255) return fail(SZX_ERR_INVALID_ARG, "dims must be positive");
  uint64_t n = 1;
  for (uint32_t i = 0; i < ndims; ++i) {
    if (dims[i] == 0) return fail(SZX_ERR_INVALID_ARG, "dims must be positive");
    if (n > UINT64_MAX / dims[i]) return fail(SZX_ERR_INVALID_ARG, "dims product overflows");
    n *= dims[i];
  }
  // every device byte count below (4n input, 4n + 16 mid) must fit a size_t
  if (n > (SIZE_MAX - 4096) / 8) return fail(SZX_ERR_INVALID_ARG, "dataset too large");
  if (!valid_bs(bs)) return fail(SZX_ERR_INVALID_ARG, "block size outside 8..65535");
  if (!(magnitude > 0) || !std::isfinite(magnitude))
    return fail(SZX_ERR_INVALID_ARG, "bound magnitude must be positive and finite");
  if (rel_mode != 0 && rel_mode != 1) return fail(SZX_ERR_INVALID_ARG, "unknown bound mode");
  int rc = ctx_ready();
  if (rc) return rc;

  const uint64_t nb = ceil_div(n, bs);
  Bump b;
  const size_t o_x = b.take(4 * n);
  const size_t o_map = b.take(szx_map_bytes(n, bs));
  const size_t o_mu = b.take(4 * nb);
  const size_t o_req = b.take(nb);
  const size_t o_codes = b.take(szx_codes_capacity(n));
  const size_t o_mid = b.take(4 * n + 16);
  const size_t o_small = b.take(256);
  const size_t rs = szx_range_scratch_bytes(n);
  const size_t o_rs = b.take(rs);
  const size_t cs = szx_compress_scratch_bytes(n, bs);
  const size_t o_cs = b.take(cs);
  rc = ctx_reserve(b.off);
  if (rc) return rc;
  char* A = g_ctx.arena;
  cudaStream_t s = g_ctx.stream;
  float* d_x = reinterpret_cast<float*>(A + o_x);
  float* d_minmax = reinterpret_cast<float*>(A + o_small);
  uint32_t* d_err = reinterpret_cast<uint32_t*>(A + o_small + 16);
  szx_totals* d_tot = reinterpret_cast<szx_totals*>(A + o_small + 64);

  trace_mark("start", s);
  CU(cudaMemcpyAsync(d_x, h_x, 4 * n, cudaMemcpyHostToDevice, s));
  trace_mark("h2d input", s);
  CU(cudaMemsetAsync(d_err, 0, 4, s));
  rc = szx_range_f32(d_x, n, d_minmax, d_err, A + o_rs, rs, s);
  if (rc) return rc;
  trace_mark("K0 range", s);
  struct Small { float mm[2]; uint32_t err; szx_totals t; };
  Small& small = *reinterpret_cast<Small*>(g_ctx.h_small);  // pinned
  static_assert(sizeof(Small) <= 256, "pinned scratch");
  CU(cudaMemcpyAsync(&small.mm, d_minmax, 8, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&small.err, d_err, 4, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (small.err & SZX_FLAG_NONFINITE) return fail(SZX_ERR_NONFINITE, "non-finite value in dataset");
  // pipeline.py:34-43
  double e = magnitude;
  if (rel_mode) {
    e = magnitude * ((double)small.mm[1] - (double)small.mm[0]);
    if (e == 0) return fail(SZX_ERR_ZERO_RANGE, "relative bound on a zero-range dataset resolves to 0");
  }
  uint8_t* d_map = reinterpret_cast<uint8_t*>(A + o_map);
  float* d_mu = reinterpret_cast<float*>(A + o_mu);
  uint8_t* d_req = reinterpret_cast<uint8_t*>(A + o_req);
  uint8_t* d_codes = reinterpret_cast<uint8_t*>(A + o_codes);
  uint8_t* d_mid = reinterpret_cast<uint8_t*>(A + o_mid);
  rc = szx_compress_f32(d_x, n, bs, e, d_map, d_mu, d_req, d_codes, d_mid, d_tot, d_err,
                        A + o_cs, cs, s);
  if (rc) return rc;
  trace_mark("K1 compress", s);
  // the map and mu pools sit at fixed stream offsets: their read-back starts before the
  // totals come back
  const uint64_t map_b = ceil_div(nb, 8);
  const uint64_t pos0 = kHead + 8ull * ndims;
  // (when they do not fit, the total does not either and the call fails below)
  if (pos0 + map_b + 4 * nb <= out_capacity) {
    CU(cudaMemcpyAsync(h_out + pos0, d_map, map_b, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(h_out + pos0 + map_b, d_mu, 4 * nb, cudaMemcpyDeviceToHost, s));
  }
  CU(cudaMemcpyAsync(&small.t, d_tot, sizeof(szx_totals), cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&small.err, d_err, 4, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  const szx_totals t = small.t;
  if (small.err & SZX_FLAG_BAD_REQ) return fail(SZX_ERR_BAD_REQ, "required bit length outside 1..32");
  // container.py:255-266
  const uint64_t code_b = ceil_div(2 * t.m, 8);
  const uint64_t total = kHead + 8ull * ndims + map_b + 4 * nb + t.n_nc + code_b + t.mid_len;
  if (out_len) *out_len = total;
  if (total > out_capacity) return fail(SZX_ERR_CAPACITY, "output buffer too small");
  // container.py:312-320 header
  std::memcpy(h_out, "UFZX", 4);
  h_out[4] = 1;
  h_out[5] = 0;
  put_le(h_out + 6, bs, 2);
  uint64_t ebits;
  std::memcpy(&ebits, &e, 8);
  put_le(h_out + 8, ebits, 8);
  h_out[16] = (uint8_t)ndims;
  for (uint32_t i = 0; i < ndims; ++i) put_le(h_out + kHead + 8 * i, dims[i], 8);
  uint64_t pos = pos0 + map_b + 4 * nb;  // map and mu are already on their way (fits_fixed)
  if (t.n_nc) CU(cudaMemcpyAsync(h_out + pos, d_req, t.n_nc, cudaMemcpyDeviceToHost, s));
  pos += t.n_nc;
  if (code_b) CU(cudaMemcpyAsync(h_out + pos, d_codes, code_b, cudaMemcpyDeviceToHost, s));
  pos += code_b;
  trace_mark("d2h map..codes", s);
  if (t.mid_len) CU(cudaMemcpyAsync(h_out + pos, d_mid, t.mid_len, cudaMemcpyDeviceToHost, s));
  trace_mark("d2h mid", s);
  CU(cudaStreamSynchronize(s));
  trace_dump("szx_compress_host");
  return SZX_OK;
}

int szx_stream_info(const uint8_t* h_in, uint64_t len, uint64_t* n_values, uint32_t* ndims,
                    uint64_t* dims_out, uint32_t dims_capacity, uint32_t* block_size,
                    double* error_bound) {
  Header h;
  int rc = parse_header(h_in, len, h);
  if (rc) return rc;
  if (n_values) *n_values = h.n;
  if (ndims) *ndims = h.ndims;
  if (block_size) *block_size = h.bs;
  if (error_bound) *error_bound = h.e;
  if (dims_out)
    for (uint32_t i = 0; i < h.ndims && i < dims_capacity; ++i) dims_out[i] = h.dims[i];
  return SZX_OK;
}

int szx_decompress_host(const uint8_t* h_in, uint64_t len, float* h_out, uint64_t n_capacity) {
  std::lock_guard<std::mutex> lock(g_ctx.mu);
  Header h;
  int rc = parse_header(h_in, len, h);
  if (rc) return rc;
  const uint64_t n = h.n, nb = h.nb, bs = h.bs;
  if (n > n_capacity) return fail(SZX_ERR_CAPACITY, "output buffer too small");
  // container.py:377-381 constant map + padding bits
  uint64_t pos = h.pos;
  const uint64_t map_b = ceil_div(nb, 8);
  if (len - pos < map_b) return fail(SZX_ERR_TRUNCATED, "stream ends inside constant map");
  const uint8_t* map = h_in + pos;
  uint64_t n_const = 0;
  {  // SWAR popcount, 8 map bytes per step (no popcnt instruction assumed on the host)
    uint64_t i = 0;
    for (; i + 8 <= map_b; i += 8) {
      uint64_t w;
      std::memcpy(&w, map + i, 8);
      w = w - ((w >> 1) & 0x5555555555555555ull);
      w = (w & 0x3333333333333333ull) + ((w >> 2) & 0x3333333333333333ull);
      w = (w + (w >> 4)) & 0x0F0F0F0F0F0F0F0Full;
      n_const += (w * 0x0101010101010101ull) >> 56;
    }
    for (; i < map_b; ++i)
      for (uint8_t v = map[i]; v; v &= (uint8_t)(v - 1)) ++n_const;
  }
  if (nb % 8) {
    const uint8_t padmask = (uint8_t)(0xFFu << (nb % 8));
    if (map[map_b - 1] & padmask) return fail(SZX_ERR_INCONSISTENT, "nonzero padding bits in constant map");
  }
  pos += map_b;
  if (len - pos < 4 * nb) return fail(SZX_ERR_TRUNCATED, "stream ends inside mu array");
  const uint64_t o_mu = pos;
  pos += 4 * nb;
  const uint64_t n_nc = nb - n_const;
  if (len - pos < n_nc) return fail(SZX_ERR_TRUNCATED, "stream ends inside req_len array");
  const uint64_t o_req = pos;
  {  // branch-free so the compiler vectorises it (~1 M req bytes at NYX size)
    const uint8_t* rq = h_in + o_req;
    uint32_t bad = 0;
    for (uint64_t i = 0; i < n_nc; ++i) bad |= (uint8_t)(rq[i] - 1) > 31;
    if (bad) return fail(SZX_ERR_INCONSISTENT, "required bit length outside 1..32");
  }
  pos += n_nc;
  // NC element count: every NC block is full except possibly the last block
  const bool last_nc = !((map[(nb - 1) >> 3] >> ((nb - 1) & 7)) & 1);
  const uint64_t tail = n - (nb - 1) * bs;
  const uint64_t m = n_nc * bs - (last_nc ? bs - tail : 0);
  const uint64_t code_b = ceil_div(2 * m, 8);
  if (len - pos < code_b) return fail(SZX_ERR_TRUNCATED, "stream ends inside leading code pool");
  const uint64_t o_codes = pos;
  if (m % 4) {
    const uint8_t padmask = (uint8_t)(0xFFu << (2 * (m % 4)));
    if (h_in[o_codes + code_b - 1] & padmask)
      return fail(SZX_ERR_INCONSISTENT, "nonzero padding bits in leading code pool");
  }
  pos += code_b;
  const uint64_t o_mid = pos, remaining = len - pos;

  rc = ctx_ready();
  if (rc) return rc;
  // place the blob so the mid pool lands 16-byte aligned, padded past the end; map and mu
  // get aligned copies when their offsets in the blob are not word-aligned
  Bump b;
  const size_t o_blob = b.take(len + 64);
  const size_t lead = (16 - (o_mid & 15)) & 15;
  const size_t o_out = b.take(4 * n);
  const size_t o_small = b.take(256);
  const size_t ds = szx_decompress_scratch_bytes(n, h.bs);
  const size_t o_ds = b.take(ds);
  const size_t o_mapc = b.take(map_b + 8);
  const size_t o_mua = b.take(4 * nb + 16);
  // the first decode chunk's own index pass (szx_decompress_host pipeline, fast block sizes)
  const uint64_t ntl = fast_bs(h.bs) ? index_layout(n).ntiles : 0;
  const size_t pds = g_ctx.parts >= 2 && ntl / g_ctx.parts >= 1
                         ? szx_decompress_scratch_bytes((ntl / g_ctx.parts) * 8192, h.bs)
                         : 0;
  const size_t o_pds = pds ? b.take(pds) : 0;
  rc = ctx_reserve(b.off);
  if (rc) return rc;
  char* A = g_ctx.arena;
  cudaStream_t s = g_ctx.stream;
  uint8_t* d_blob = reinterpret_cast<uint8_t*>(A + o_blob) + lead;
  float* d_out = reinterpret_cast<float*>(A + o_out);
  uint32_t* d_err = reinterpret_cast<uint32_t*>(A + o_small);
  szx_totals* d_tot = reinterpret_cast<szx_totals*>(A + o_small + 64);
  if (fast_bs(h.bs)) {
    // Pipelined: the pools before the mid bytes go up first, K3 indexes them while the mid
    // bytes follow in kPipeParts pieces; each decode chunk waits only for the piece holding
    // its last mid byte, and its values go back on a second copy stream while later chunks
    // decode -- so the host->device and device->host copies overlap.
    const IndexLayout L = index_layout(n);
    uint64_t* d_index = reinterpret_cast<uint64_t*>(A + o_ds + L.off_index);
    uint64_t* d_stats = reinterpret_cast<uint64_t*>(A + o_ds + L.off_stats);
    cudaStream_t si = g_ctx.s_in, so = g_ctx.s_out;
    CU(cudaMemsetAsync(d_err, 0, 4, s));
    const int P = g_ctx.parts;
    const uint64_t ntiles = L.ntiles, ew = kIndexEntryBytes / 8;
    // Prefix: the first decode chunk's tiles [0, t1) are indexed by a K3 launch over just
    // their pool prefixes (map, mu, req, codes of the first t1 tiles -- every one of them
    // full), so the first chunk decodes and its values start back while the rest of the
    // pools is still uploading.  Its index entries equal the full index's (both are prefix
    // sums from the stream start).
    const uint64_t t1p = ntiles / P;
    const bool prefix = P >= 2 && t1p >= 1 && o_pds != 0;
    const uint64_t bpt = 8192 / bs;  // blocks per decode tile
    const uint64_t nb1 = t1p * bpt, n1 = t1p * 8192;
    uint64_t nc1 = 0;
    if (prefix) {
      uint64_t cst = 0;
      for (uint64_t i = 0; i < nb1 / 8; ++i) cst += (uint64_t)__builtin_popcount(map[i]);
      nc1 = nb1 - cst;
    }
    // pool (offset in the blob, bytes, bytes of the prefix)
    const uint64_t po[4] = {h.pos, o_mu, o_req, o_codes};
    const uint64_t pz[4] = {map_b, 4 * nb, n_nc, code_b};
    const uint64_t pp[4] = {nb1 / 8, 4 * nb1, nc1, nc1 * (bs / 4)};
    uint64_t part_end[kPipeParts];
    for (int j = 0; j < P; ++j) part_end[j] = remaining * (j + 1) / P;
    auto mid_part = [&](int j) -> int {
      const uint64_t b0 = remaining * j / P, b1 = part_end[j];
      if (b1 > b0)
        CU(cudaMemcpyAsync(d_blob + o_mid + b0, h_in + o_mid + b0, b1 - b0,
                           cudaMemcpyHostToDevice, si));
      if (j == P - 1) CU(cudaMemsetAsync(d_blob + len, 0, 32, si));
      CU(cudaEventRecord(g_ctx.ev_mid[j], si));
      trace_mark("h2d mid part", si, j);
      return SZX_OK;
    };
    trace_mark("start", si);
    if (prefix) {
      for (int q = 0; q < 4; ++q)
        if (pp[q]) CU(cudaMemcpyAsync(d_blob + po[q], h_in + po[q], pp[q], cudaMemcpyHostToDevice, si));
      CU(cudaEventRecord(g_ctx.ev_pre, si));
      trace_mark("h2d prefix pools", si);
      if ((rc = mid_part(0))) return rc;
      for (int q = 0; q < 4; ++q)
        if (pz[q] > pp[q])
          CU(cudaMemcpyAsync(d_blob + po[q] + pp[q], h_in + po[q] + pp[q], pz[q] - pp[q],
                             cudaMemcpyHostToDevice, si));
    } else {
      CU(cudaMemcpyAsync(d_blob, h_in, o_mid, cudaMemcpyHostToDevice, si));
    }
    CU(cudaEventRecord(g_ctx.ev_head, si));
    trace_mark("h2d head pools", si);
    for (int j = prefix ? 1 : 0; j < P; ++j)
      if ((rc = mid_part(j))) return rc;
    // map / mu views K3 and K2 can load as words (aligned copies when the blob offsets are not)
    const uint8_t* d_map = d_blob + h.pos;
    const float* d_mu = reinterpret_cast<const float*>(d_blob + o_mu);
    uint8_t* d_mapc = reinterpret_cast<uint8_t*>(A + o_mapc);
    float* d_mua = reinterpret_cast<float*>(A + o_mua);
    const bool map_copy = ((uintptr_t)d_map & 3) != 0, mu_copy = ((uintptr_t)d_mu & 3) != 0;
    auto align_views = [&](uint64_t map_from, uint64_t map_to, uint64_t mu_from,
                           uint64_t mu_to) -> int {
      if (map_copy && map_to > map_from)
        CU(cudaMemcpyAsync(d_mapc + map_from, d_map + map_from, map_to - map_from,
                           cudaMemcpyDeviceToDevice, s));
      if (mu_copy && mu_to > mu_from)
        CU(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(d_mua) + mu_from,
                           reinterpret_cast<const uint8_t*>(d_mu) + mu_from, mu_to - mu_from,
                           cudaMemcpyDeviceToDevice, s));
      return SZX_OK;
    };
    const uint8_t* v_map = map_copy ? d_mapc : d_map;
    const float* v_mu = mu_copy ? d_mua : d_mu;
    // pinned read-back area: the prefix index (then the error word)
    const uint64_t pre_bytes = prefix ? szx_index_bytes(n1, h.bs) : 0;
    const size_t need_h = pre_bytes + 32;
    if (g_ctx.h_idx_cap < need_h) {
      if (g_ctx.h_idx) CU(cudaFreeHost(g_ctx.h_idx));
      g_ctx.h_idx = nullptr;
      g_ctx.h_idx_cap = 0;
      CU(cudaMallocHost(&g_ctx.h_idx, need_h));
      g_ctx.h_idx_cap = need_h;
    }
    uint64_t* hpre = g_ctx.h_idx;
    uint32_t herr = 0;
    uint32_t* herr_p = reinterpret_cast<uint32_t*>(g_ctx.h_idx + pre_bytes / 8);
    auto decode_chunk = [&](int j, uint64_t t0, uint64_t t1, const uint64_t* d_idx, uint64_t nt,
                            uint64_t nv, uint64_t need) -> int {
      int part = 0;
      while (part < P - 1 && part_end[part] < need) ++part;
      CU(cudaStreamWaitEvent(s, g_ctx.ev_mid[part], 0));
      Decode128Args da{};
      da.map = v_map;
      da.mu = v_mu;
      da.req = d_blob + o_req;
      da.codes = d_blob + o_codes;
      da.mid = d_blob + o_mid;
      da.mid_len = remaining;
      da.index = d_idx;
      da.out = d_out;
      da.n = nv;
      da.ntiles = nt;
      da.tile_begin = t0;
      da.tile_end = t1;
      da.err = d_err;
      da.bs = h.bs;
      launch_decode128(da, s);
      CU(cudaGetLastError());
      CU(cudaEventRecord(g_ctx.ev_dec[j], s));
      CU(cudaStreamWaitEvent(so, g_ctx.ev_dec[j], 0));
      const uint64_t v0 = t0 * 8192;  // 8192-value tiles for every fast block size
      const uint64_t v1 = std::min<uint64_t>(n, t1 * 8192);
      trace_mark("K2 chunk", s, j);
      // in pieces of <= 16 MiB, so a small read-back queued behind them (the index) waits
      // for one piece, not the whole chunk
      for (uint64_t w0 = v0; w0 < v1; w0 += (4u << 20)) {
        const uint64_t w1 = std::min<uint64_t>(v1, w0 + (4u << 20));
        CU(cudaMemcpyAsync(h_out + w0, d_out + w0, 4 * (w1 - w0), cudaMemcpyDeviceToHost, so));
      }
      trace_mark("d2h chunk", so, j);
      return SZX_OK;
    };
    auto drain = [&]() -> int {  // no copy may still target the caller's buffers
      CU(cudaStreamSynchronize(s));
      CU(cudaStreamSynchronize(so));
      CU(cudaStreamSynchronize(si));
      return SZX_OK;
    };
    auto stop = [&](int code, const char* msg) -> int {
      const int d = drain();
      return d ? d : fail(code, msg);
    };
    if (prefix) {
      CU(cudaStreamWaitEvent(s, g_ctx.ev_pre, 0));
      if ((rc = align_views(0, nb1 / 8, 0, 4 * nb1))) return rc;
      const IndexLayout Lp = index_layout(n1);
      uint64_t* d_ipre = reinterpret_cast<uint64_t*>(A + o_pds + Lp.off_index);
      uint64_t* d_spre = reinterpret_cast<uint64_t*>(A + o_pds + Lp.off_stats);
      rc = szx_index_f32(v_map, v_mu, d_blob + o_req, d_blob + o_codes, n1, h.bs, d_ipre, d_spre,
                         d_err, A + o_pds, pds, s);
      if (rc) {
        drain();
        return rc;
      }
      trace_mark("K3 prefix index", s);
      CU(cudaMemcpyAsync(hpre, d_ipre, pre_bytes, cudaMemcpyDeviceToHost, s));
      CU(cudaStreamSynchronize(s));
      const uint64_t c = hpre[ew * t1p + 6];
      const uint64_t need = hpre[ew * t1p + 1] + hpre[ew * (t1p + 1) + c];
      if (need > remaining) return stop(SZX_ERR_TRUNCATED, "stream ends inside mid byte pool");
      if ((rc = decode_chunk(0, 0, t1p, d_ipre, t1p, n1, need))) return rc;
    }
    CU(cudaStreamWaitEvent(s, g_ctx.ev_head, 0));
    if ((rc = align_views(prefix ? nb1 / 8 : 0, map_b, prefix ? 4 * nb1 : 0, 4 * nb))) return rc;
    rc = szx_index_f32(v_map, v_mu, d_blob + o_req, d_blob + o_codes, n, h.bs, d_index, d_stats,
                       d_err, A + o_ds, ds, s);
    if (rc) {
      drain();
      return rc;
    }
    trace_mark("K3 index", s);
    // the chunk bounds' mid offsets and the stream checks come back to plan the chunks
    volatile uint64_t* plan = g_ctx.h_plan;
    plan_bounds_kernel<<<1, 64, 0, s>>>(d_index, ntiles, P, d_stats, d_err, plan);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(s));
    herr = (uint32_t)plan[P + 1];
    // container.py:403-405 then CompressedStream._validate (198-214)
    if (plan[P] > remaining) return stop(SZX_ERR_TRUNCATED, "stream ends inside mid byte pool");
    if (plan[P] < remaining) return stop(SZX_ERR_INCONSISTENT, "trailing bytes after mid pool");
    trace_mark("index on host", s);
    for (int j = prefix ? 1 : 0; j < P; ++j) {
      const uint64_t t0 = ntiles * j / P, t1 = ntiles * (j + 1) / P;
      if (t1 == t0) continue;
      // the chunk's last mid byte is below mid_before(t1)
      if ((rc = decode_chunk(j, t0, t1, d_index, ntiles, n, plan[j]))) return rc;
    }
    CU(cudaMemcpyAsync(herr_p, d_err, 4, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    CU(cudaStreamSynchronize(so));
    CU(cudaStreamSynchronize(si));
    herr = *herr_p;
    trace_dump("szx_decompress_host");
    if (herr & SZX_FLAG_MU_NONFINITE) return fail(SZX_ERR_INCONSISTENT, "non-finite mu");
    if (herr & SZX_FLAG_BAD_REQ)
      return fail(SZX_ERR_INCONSISTENT, "required bit length outside 1..32");
    if (herr & SZX_FLAG_CODE_PADDING)
      return fail(SZX_ERR_INCONSISTENT, "nonzero padding bits in leading code pool");
    if (herr & SZX_FLAG_UNDERRUN) return fail(SZX_ERR_UNDERRUN, "mid pool exhausted");
    if (herr & SZX_FLAG_NONFINITE) return fail(SZX_ERR_NONFINITE, "non-finite value in dataset");
    return SZX_OK;
  }
  CU(cudaMemcpyAsync(d_blob, h_in, len, cudaMemcpyHostToDevice, s));
  CU(cudaMemsetAsync(d_blob + len, 0, 32, s));
  CU(cudaMemsetAsync(d_err, 0, 4, s));
  const uint8_t* d_map = d_blob + h.pos;
  if (((uintptr_t)d_map & 3) != 0) {
    uint8_t* d_mapc = reinterpret_cast<uint8_t*>(A + o_mapc);
    CU(cudaMemcpyAsync(d_mapc, d_map, map_b, cudaMemcpyDeviceToDevice, s));
    d_map = d_mapc;
  }
  const float* d_mu = reinterpret_cast<const float*>(d_blob + o_mu);
  if (((uintptr_t)d_mu & 3) != 0) {
    float* d_mua = reinterpret_cast<float*>(A + o_mua);
    CU(cudaMemcpyAsync(d_mua, d_blob + o_mu, 4 * nb, cudaMemcpyDeviceToDevice, s));
    d_mu = d_mua;
  }
  rc = szx_decompress_f32(d_map, d_mu, d_blob + o_req, d_blob + o_codes, d_blob + o_mid,
                          remaining, n, h.bs, d_out, d_tot, d_err, A + o_ds, ds, s);
  if (rc) return rc;
  szx_totals t;
  uint32_t err = 0;
  CU(cudaMemcpyAsync(&t, d_tot, sizeof t, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&err, d_err, 4, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(h_out, d_out, 4 * n, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  // container.py:403-405 then CompressedStream._validate (198-199)
  if (t.mid_len > remaining) return fail(SZX_ERR_TRUNCATED, "stream ends inside mid byte pool");
  if (t.mid_len < remaining) return fail(SZX_ERR_INCONSISTENT, "trailing bytes after mid pool");
  if (err & SZX_FLAG_MU_NONFINITE) return fail(SZX_ERR_INCONSISTENT, "non-finite mu");
  if (err & SZX_FLAG_UNDERRUN) return fail(SZX_ERR_UNDERRUN, "mid pool exhausted");
  // _assemble builds a DataField of the reconstruction (pipeline.py:224 -> container.py:84)
  if (err & SZX_FLAG_NONFINITE) return fail(SZX_ERR_NONFINITE, "non-finite value in dataset");
  return SZX_OK;
}

}  // extern "C"

// ---- measurement passes (analysis.cu) -------------------------------------------------------
extern "C" {

int szx_accounting_f32(const float* d_x, uint64_t n, uint32_t bs, double e, uint64_t* d_bits,
                       void* stream) {
  if (n == 0) return fail(SZX_ERR_INVALID_ARG, "empty dataset");
  if (!valid_bs(bs)) return fail(SZX_ERR_INVALID_ARG, "block size outside 8..65535");
  if (!(e > 0) || !std::isfinite(e)) return fail(SZX_ERR_INVALID_ARG, "bound must be positive finite");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CU(cudaMemsetAsync(d_bits, 0, 8, s));
  launch_accounting(d_x, n, bs, e, szx_bound_exponent(e),
                    reinterpret_cast<unsigned long long*>(d_bits), s);
  CU(cudaGetLastError());
  return SZX_OK;
}

size_t szx_quality_scratch_bytes(uint64_t n) {
  return 256 + quality_part_bytes() * (size_t)quality_grid(n);
}

int szx_quality_f32(const float* d_a, const float* d_b, uint64_t n, double* d_out5,
                    void* d_scratch, size_t scratch_bytes, void* stream) {
  if (n == 0) return fail(SZX_ERR_INVALID_ARG, "empty dataset");
  if (scratch_bytes < szx_quality_scratch_bytes(n) || !aligned(d_scratch, 256))
    return fail(SZX_ERR_INVALID_ARG, "quality scratch too small or misaligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* counter = static_cast<uint32_t*>(d_scratch);
  CU(cudaMemsetAsync(counter, 0, 4, s));
  launch_quality(d_a, d_b, n, static_cast<char*>(d_scratch) + 256, counter, d_out5, s);
  CU(cudaGetLastError());
  return SZX_OK;
}

int szx_block_range_counts_f32(const float* d_x, uint64_t n, uint32_t bs, double global_range,
                               const double* d_thresholds, uint32_t nthr, uint64_t* d_counts,
                               void* stream) {
  if (n == 0) return fail(SZX_ERR_INVALID_ARG, "empty dataset");
  if (bs == 0) return fail(SZX_ERR_INVALID_ARG, "block size must be positive");
  if (nthr > max_thresholds()) return fail(SZX_ERR_INVALID_ARG, "too many thresholds (max 64)");
  if (!(global_range > 0)) return fail(SZX_ERR_ZERO_RANGE, "zero global value range");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nthr == 0) return SZX_OK;
  CU(cudaMemsetAsync(d_counts, 0, 8 * (size_t)nthr, s));
  launch_block_range(d_x, n, bs, global_range, d_thresholds, nthr,
                     reinterpret_cast<unsigned long long*>(d_counts), s);
  CU(cudaGetLastError());
  return SZX_OK;
}

size_t szx_prefix_scan_scratch_bytes(uint64_t n) { return 256 + 8 * (size_t)scan_tiles(n); }

int szx_prefix_scan_i64(const int64_t* d_in, uint64_t n, int64_t* d_out, void* d_scratch,
                        size_t scratch_bytes, void* stream) {
  if (n == 0) return SZX_OK;
  if (scratch_bytes < szx_prefix_scan_scratch_bytes(n) || !aligned(d_scratch, 8))
    return fail(SZX_ERR_INVALID_ARG, "scan scratch too small or misaligned");
  if (scan_tiles(n) > 0x7FFFFFFFull) return fail(SZX_ERR_INVALID_ARG, "scan too long");
  launch_prefix_scan(reinterpret_cast<const long long*>(d_in), n,
                     reinterpret_cast<long long*>(d_out), static_cast<long long*>(d_scratch),
                     static_cast<cudaStream_t>(stream));
  CU(cudaGetLastError());
  return SZX_OK;
}

int szx_propagate_indices(const uint8_t* d_codes, uint32_t count, uint32_t q,
                          int64_t* d_positions, void* stream) {
  if (q < 1 || q > 4) return fail(SZX_ERR_INVALID_ARG, "bad byte count");
  if (count == 0) return SZX_OK;
  launch_propagate(d_codes, count, q, reinterpret_cast<long long*>(d_positions),
                   static_cast<cudaStream_t>(stream));
  CU(cudaGetLastError());
  return SZX_OK;
}

int szx_propagate_round(const int64_t* d_in, uint64_t rows, uint32_t cols, uint64_t stride,
                        int64_t* d_out, void* stream) {
  if (rows == 0 || cols == 0) return SZX_OK;
  launch_propagate_round(reinterpret_cast<const long long*>(d_in), rows, cols, stride,
                         reinterpret_cast<long long*>(d_out), static_cast<cudaStream_t>(stream));
  CU(cudaGetLastError());
  return SZX_OK;
}

}  // extern "C"

// ---- batched small-field path (BASELINE configs[2]) -------------------------------------------
namespace {
int range_batch_grid(uint32_t nf, const uint64_t* n) {
  int g = 1;
  for (uint32_t f = 0; f < nf; ++f) g = std::max(g, range_grid(n[f]));
  return g;
}
struct BatchLayout {
  size_t off_tmaps, off_counter, off_status, off_groups, total;
  uint64_t tiles;
  std::vector<size_t> groups;  // per field: its group table (decode-index path)
};
BatchLayout batch_layout(uint32_t nf, const uint64_t* n) {
  BatchLayout L{};
  size_t off = ((sizeof(FieldDesc) * nf + 127) / 128) * 128;
  L.off_tmaps = off;
  off += 128 * (size_t)nf;
  L.off_counter = off;
  off += 128;
  L.off_status = off;
  for (uint32_t f = 0; f < nf; ++f) L.tiles += ceil_div(ceil_div(n[f], 128), kV3TileBlocks);
  off += 8 * L.tiles;
  off = (off + 255) & ~size_t(255);
  L.off_groups = off;
  L.groups.resize(nf);
  for (uint32_t f = 0; f < nf; ++f) {  // 2 u64 per 4-block group of every compress tile
    L.groups[f] = off;
    off += 16 * (size_t)kV3Warps * ceil_div(ceil_div(n[f], 128), kV3TileBlocks);
  }
  L.total = (off + 255) & ~size_t(255);
  return L;
}

int compress_batch_impl(uint32_t nfields, const float* const* d_x, const uint64_t* n,
                        const double* e, uint8_t* const* d_map, float* const* d_mu,
                        uint8_t* const* d_req, uint8_t* const* d_codes, uint8_t* const* d_mid,
                        uint64_t* const* d_index, szx_totals* d_totals, uint32_t* d_err,
                        void* d_scratch, size_t scratch_bytes, void* stream) {
  if (nfields == 0) return SZX_OK;
  const uint64_t chunk_cap = (1ull << 26) - 64;  // one look-back chunk per field (make_plan)
  for (uint32_t f = 0; f < nfields; ++f) {
    if (n[f] == 0) return fail(SZX_ERR_INVALID_ARG, "empty dataset");
    if (ceil_div(n[f], 128) > chunk_cap) return fail(SZX_ERR_INVALID_ARG, "batched field too large");
    if (!(e[f] > 0) || !std::isfinite(e[f])) return fail(SZX_ERR_INVALID_ARG, "bound must be positive finite");
    if (!aligned(d_x[f], 16) || !aligned(d_mid[f], 16) || !aligned(d_map[f], 4) ||
        !aligned(d_codes[f], 4) || !aligned(d_mu[f], 4))
      return fail(SZX_ERR_ALIGN, "x/mid need 16-byte, map/codes/mu 4-byte alignment");
    if (d_index && d_index[f] && !aligned(d_index[f], 8))
      return fail(SZX_ERR_ALIGN, "index needs 8-byte alignment");
  }
  const BatchLayout L = batch_layout(nfields, n);
  if (L.tiles >= (1ull << 32)) return fail(SZX_ERR_INVALID_ARG, "batch too large");
  if (scratch_bytes < L.total || !aligned(d_scratch, 256))
    return fail(SZX_ERR_INVALID_ARG, "batch scratch too small or misaligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* sc = static_cast<char*>(d_scratch);
  CU(cudaMemsetAsync(sc + L.off_counter, 0, L.off_groups - L.off_counter, s));
  std::vector<FieldDesc> h(nfields);
  uint64_t t0 = 0;
  bool any_index = false;
  for (uint32_t f = 0; f < nfields; ++f) {
    FieldDesc& d = h[f];
    d.x = d_x[f];
    d.n = n[f];
    d.e = e[f];
    d.pe = szx_bound_exponent(e[f]);
    d.ntiles = (uint32_t)ceil_div(ceil_div(n[f], 128), kV3TileBlocks);
    d.tile0 = t0;
    d.map = d_map[f];
    d.mu = d_mu[f];
    d.req = d_req[f];
    d.codes = d_codes[f];
    d.mid = d_mid[f];
    d.totals = reinterpret_cast<Totals*>(d_totals + f);
    d.index = d_index ? d_index[f] : nullptr;
    d.groups = d.index ? reinterpret_cast<uint64_t*>(sc + L.groups[f]) : nullptr;
    any_index = any_index || d.index;
    t0 += d.ntiles;
  }
  std::vector<uint8_t> hmaps(128 * (size_t)nfields + 64);
  void* hm = hmaps.data() + ((64 - ((uintptr_t)hmaps.data() & 63)) & 63);
  CompressArgs a{};
  a.bs = 128;
  a.status = reinterpret_cast<uint64_t*>(sc + L.off_status);
  a.counter = reinterpret_cast<uint32_t*>(sc + L.off_counter);
  a.err = d_err;
  a.ntiles = (uint32_t)L.tiles;
  a.x = h[0].x;
  a.n = h[0].n;
  FieldDesc* d_fields = reinterpret_cast<FieldDesc*>(sc);
  CU(launch_compress128v3_batch(a, d_fields, h.data(), nfields, sc + L.off_tmaps, hm, s));
  if (any_index) CU(launch_groups_to_index(d_fields, h.data(), nfields, s));
  // the host staging above is pageable: its copies are complete when cudaMemcpyAsync returns
  return SZX_OK;
}
}  // namespace

extern "C" {

size_t szx_range_batch_scratch_bytes(uint32_t nfields, const uint64_t* n) {
  return 256 + ((sizeof(RangeField) * nfields + 255) & ~size_t(255)) + 4 * (size_t)nfields +
         8 * (size_t)range_batch_grid(nfields, n) * nfields + 256;
}

int szx_range_batch_f32(uint32_t nfields, const float* const* d_x, const uint64_t* n,
                        float* d_minmax, uint32_t* d_err, void* d_scratch, size_t scratch_bytes,
                        void* stream) {
  if (nfields == 0) return SZX_OK;
  for (uint32_t f = 0; f < nfields; ++f)
    if (n[f] == 0) return fail(SZX_ERR_INVALID_ARG, "empty dataset");
  if (scratch_bytes < szx_range_batch_scratch_bytes(nfields, n) || !aligned(d_scratch, 256))
    return fail(SZX_ERR_INVALID_ARG, "range scratch too small or misaligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* sc = static_cast<char*>(d_scratch);
  RangeField* d_fields = reinterpret_cast<RangeField*>(sc);
  size_t off = (sizeof(RangeField) * nfields + 255) & ~size_t(255);
  uint32_t* counters = reinterpret_cast<uint32_t*>(sc + off);
  off += ((4 * (size_t)nfields + 255) & ~size_t(255));
  float* partials = reinterpret_cast<float*>(sc + off);
  std::vector<RangeField> h(nfields);
  for (uint32_t f = 0; f < nfields; ++f) h[f] = RangeField{d_x[f], n[f]};
  CU(cudaMemcpyAsync(d_fields, h.data(), sizeof(RangeField) * nfields, cudaMemcpyHostToDevice, s));
  CU(cudaMemsetAsync(counters, 0, 4 * (size_t)nfields, s));
  launch_range_batch(d_fields, nfields, range_batch_grid(nfields, n), partials, counters,
                     d_minmax, d_err, s);
  CU(cudaGetLastError());
  return SZX_OK;
}

size_t szx_compress_batch_scratch_bytes(uint32_t nfields, const uint64_t* n) {
  return batch_layout(nfields, n).total;
}

int szx_compress_batch_f32(uint32_t nfields, const float* const* d_x, const uint64_t* n,
                           const double* e, uint8_t* const* d_map, float* const* d_mu,
                           uint8_t* const* d_req, uint8_t* const* d_codes, uint8_t* const* d_mid,
                           szx_totals* d_totals, uint32_t* d_err, void* d_scratch,
                           size_t scratch_bytes, void* stream) {
  return compress_batch_impl(nfields, d_x, n, e, d_map, d_mu, d_req, d_codes, d_mid, nullptr,
                             d_totals, d_err, d_scratch, scratch_bytes, stream);
}

int szx_compress_batch_indexed_f32(uint32_t nfields, const float* const* d_x, const uint64_t* n,
                                   const double* e, uint8_t* const* d_map, float* const* d_mu,
                                   uint8_t* const* d_req, uint8_t* const* d_codes,
                                   uint8_t* const* d_mid, uint64_t* const* d_index,
                                   szx_totals* d_totals, uint32_t* d_err, void* d_scratch,
                                   size_t scratch_bytes, void* stream) {
  return compress_batch_impl(nfields, d_x, n, e, d_map, d_mu, d_req, d_codes, d_mid, d_index,
                             d_totals, d_err, d_scratch, scratch_bytes, stream);
}

}  // extern "C"

namespace {
struct DecBatchLayout {
  size_t off_dargs, off_tile0, off_zero, off_index, total;
  std::vector<size_t> zero, index;  // per field: status/counter/stats block, index
  std::vector<uint32_t> groups;
  uint32_t max_groups;
  uint64_t tiles;
};
DecBatchLayout dec_batch_layout(uint32_t nf, const uint64_t* n) {
  DecBatchLayout L{};
  auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
  size_t off = al(sizeof(IndexArgs) * nf);
  L.off_dargs = off;
  off += al(sizeof(Decode128Args) * nf);
  L.off_tile0 = off;
  off += al(8 * ((size_t)nf + 1));
  L.off_zero = off;
  L.zero.resize(nf);
  L.groups.resize(nf);
  L.max_groups = 1;
  for (uint32_t f = 0; f < nf; ++f) {
    L.groups[f] = index_batch_groups(n[f]);
    L.max_groups = std::max(L.max_groups, L.groups[f]);
    L.zero[f] = off;  // status_nc, status_mid (G each), counter, stats (nc, mid)
    off += 16 * (size_t)L.groups[f] + 32;
  }
  off = al(off);
  L.off_index = off;
  L.index.resize(nf);
  for (uint32_t f = 0; f < nf; ++f) {
    L.index[f] = off;
    const uint64_t nt = ceil_div(ceil_div(n[f], 128), kDecTileBlocks);
    L.tiles += nt;
    off += al(kIndexEntryBytes * (nt + 1) + 8 * ((size_t)L.groups[f] + 1));
  }
  L.total = al(off);
  return L;
}
}  // namespace

extern "C" {

size_t szx_decompress_batch_scratch_bytes(uint32_t nfields, const uint64_t* n) {
  return dec_batch_layout(nfields, n).total;
}

// d_index null: K3 indexes every field (into the scratch) before K2; else the fields'
// decode indexes are given (szx_compress_batch_indexed_f32) and only K2 runs.
static int decompress_batch_impl(uint32_t nfields, const uint8_t* const* d_map,
                          const float* const* d_mu, const uint8_t* const* d_req,
                          const uint8_t* const* d_codes, const uint8_t* const* d_mid,
                          const uint64_t* mid_len, const uint64_t* n,
                          const uint64_t* const* d_index, float* const* d_out,
                          uint64_t* d_stats, uint32_t* d_err, void* d_scratch,
                          size_t scratch_bytes, void* stream) {
  if (nfields == 0) return SZX_OK;
  for (uint32_t f = 0; f < nfields; ++f) {
    if (n[f] == 0) return fail(SZX_ERR_INVALID_ARG, "empty stream");
    if (!aligned(d_out[f], 16) || !aligned(d_mu[f], 4))
      return fail(SZX_ERR_ALIGN, "out needs 16-byte, mu 4-byte alignment");
    if (d_index && (!d_index[f] || !aligned(d_index[f], 16)))
      return fail(SZX_ERR_ALIGN, "every field needs a 16-byte aligned index");
  }
  const DecBatchLayout L = dec_batch_layout(nfields, n);
  if (scratch_bytes < L.total || !aligned(d_scratch, 256))
    return fail(SZX_ERR_INVALID_ARG, "batch scratch too small or misaligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* sc = static_cast<char*>(d_scratch);
  if (!d_index) CU(cudaMemsetAsync(sc + L.off_zero, 0, L.off_index - L.off_zero, s));
  std::vector<IndexArgs> ia(nfields);
  std::vector<Decode128Args> da(nfields);
  std::vector<uint64_t> t0(nfields + 1);
  uint64_t tiles = 0;
  for (uint32_t f = 0; f < nfields; ++f) {
    uint64_t* zs = reinterpret_cast<uint64_t*>(sc + L.zero[f]);
    uint64_t* index = d_index ? const_cast<uint64_t*>(d_index[f])
                              : reinterpret_cast<uint64_t*>(sc + L.index[f]);
    const uint64_t nt = ceil_div(ceil_div(n[f], 128), kDecTileBlocks);
    IndexArgs& a = ia[f];
    a.map = d_map[f];
    a.mu = d_mu[f];
    a.req = d_req[f];
    a.codes = d_codes[f];
    a.n = n[f];
    a.index = index;
    a.status_nc = zs;
    a.status_mid = zs + L.groups[f];
    a.counter = reinterpret_cast<uint32_t*>(zs + 2 * (size_t)L.groups[f]);
    a.nc_total = reinterpret_cast<unsigned long long*>(d_stats + 2 * (size_t)f);
    a.mid_total = a.nc_total + 1;
    a.err = d_err + f;
    a.ngroups = L.groups[f];
    a.direct_limit = ~0ull;  // batched fields are summed directly
    Decode128Args& d = da[f];
    d.map = d_map[f];
    d.mu = d_mu[f];
    d.req = d_req[f];
    d.codes = d_codes[f];
    d.mid = d_mid[f];
    d.mid_len = mid_len[f];
    d.index = index;
    d.out = d_out[f];
    d.n = n[f];
    d.ntiles = nt;
    d.tile_begin = 0;
    d.tile_end = nt;
    d.err = d_err + f;
    t0[f] = tiles;
    tiles += nt;
  }
  t0[nfields] = tiles;
  IndexArgs* d_ia = reinterpret_cast<IndexArgs*>(sc);
  Decode128Args* d_da = reinterpret_cast<Decode128Args*>(sc + L.off_dargs);
  uint64_t* d_t0 = reinterpret_cast<uint64_t*>(sc + L.off_tile0);
  // d_stats (2 per field) are overwritten by K3; pageable staging: copies complete on return
  if (!d_index) {
    CU(cudaMemsetAsync(d_stats, 0, 16 * (size_t)nfields, s));
    CU(cudaMemcpyAsync(d_ia, ia.data(), sizeof(IndexArgs) * nfields, cudaMemcpyHostToDevice, s));
  }
  CU(cudaMemcpyAsync(d_da, da.data(), sizeof(Decode128Args) * nfields, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(d_t0, t0.data(), 8 * ((size_t)nfields + 1), cudaMemcpyHostToDevice, s));
  if (!d_index) {
    launch_index128_batch(d_ia, nfields, L.max_groups, s);
    CU(cudaGetLastError());
  }
  Decode128Args a{};
  a.tile_begin = 0;
  a.tile_end = tiles;
  a.err = d_err;
  launch_decode128_batch(a, d_da, d_t0, nfields, s);
  CU(cudaGetLastError());
  return SZX_OK;
}


int szx_decompress_batch_f32(uint32_t nfields, const uint8_t* const* d_map,
                             const float* const* d_mu, const uint8_t* const* d_req,
                             const uint8_t* const* d_codes, const uint8_t* const* d_mid,
                             const uint64_t* mid_len, const uint64_t* n, float* const* d_out,
                             uint64_t* d_stats, uint32_t* d_err, void* d_scratch,
                             size_t scratch_bytes, void* stream) {
  return decompress_batch_impl(nfields, d_map, d_mu, d_req, d_codes, d_mid, mid_len, n, nullptr,
                               d_out, d_stats, d_err, d_scratch, scratch_bytes, stream);
}

int szx_decompress_batch_indexed_f32(uint32_t nfields, const uint8_t* const* d_map,
                                     const float* const* d_mu, const uint8_t* const* d_req,
                                     const uint8_t* const* d_codes, const uint8_t* const* d_mid,
                                     const uint64_t* mid_len, const uint64_t* n,
                                     const uint64_t* const* d_index, float* const* d_out,
                                     uint32_t* d_err, void* d_scratch, size_t scratch_bytes,
                                     void* stream) {
  return decompress_batch_impl(nfields, d_map, d_mu, d_req, d_codes, d_mid, mid_len, n, d_index,
                               d_out, nullptr, d_err, d_scratch, scratch_bytes, stream);
}

}  // extern "C"
