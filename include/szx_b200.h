/*
 * szx_b200.h -- C ABI of the B200-native SZx codec (libszx_b200.so).
 *
 * Drop-in boundary for the reference package `ufzx` (pure Python/NumPy; it has no FFI of
 * its own).  Each entry point below names the reference interface it replaces.  Plain
 * pointers and sizes only; `stream` is a cudaStream_t passed as void* (NULL = legacy
 * default stream).  Device-pointer entry points are stream-ordered and never allocate;
 * host-buffer entry points run synchronously on a library-owned context.
 *
 * Byte format: the reference's UFZX container (ufzx/container.py:3-21), bit-exact.
 */
#ifndef SZX_B200_H
#define SZX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The Python facade maps them 1:1 onto the reference exception classes. */
enum {
  SZX_OK = 0,
  SZX_ERR_INVALID_ARG = 1,     /* ValueError (bad block size, bound, dims, empty field)   */
  SZX_ERR_CUDA = 2,            /* CUDA runtime failure (see szx_last_error)                */
  SZX_ERR_ALIGN = 3,           /* device buffer misaligned (x/out/mid 16 B, map/codes 4 B) */
  SZX_ERR_NONFINITE = 4,       /* ValueError("non-finite value in dataset")  container.py:84 */
  SZX_ERR_ZERO_RANGE = 5,      /* ZeroRangeError                             pipeline.py:17 */
  SZX_ERR_BAD_REQ = 6,         /* InconsistentLengthError (req outside 1..32) container.py:206 */
  SZX_ERR_UNDERRUN = 7,        /* PoolUnderrunError                          blockcodec.py:25 */
  SZX_ERR_TRUNCATED = 8,       /* TruncatedStreamError                       container.py:54 */
  SZX_ERR_MAGIC = 9,           /* MalformedMagicError                        container.py:42 */
  SZX_ERR_VERSION = 10,        /* VersionMismatchError                       container.py:46 */
  SZX_ERR_DTYPE = 11,          /* UnsupportedDtypeError                      container.py:50 */
  SZX_ERR_INCONSISTENT = 12,   /* InconsistentLengthError                    container.py:58 */
  SZX_ERR_CAPACITY = 13,       /* caller's output buffer too small                         */
  SZX_ERR_NO_DEVICE = 14       /* no CUDA device: the library has no CPU path              */
};

/* Device-side stream totals (written by the compress / decompress kernels). */
typedef struct szx_totals {
  uint64_t n_nc;    /* non-constant blocks  == bytes in the req pool          */
  uint64_t m;       /* non-constant elements == number of 2-bit codes (compress only) */
  uint64_t mid_len; /* bytes in the mid pool                                  */
  uint64_t pad;
} szx_totals;

/* Device error-flag bits (OR-accumulated into a caller u32). */
enum {
  SZX_FLAG_BAD_REQ = 1,
  SZX_FLAG_NONFINITE = 2,
  SZX_FLAG_UNDERRUN = 4,
  SZX_FLAG_MU_NONFINITE = 8,
  SZX_FLAG_CODE_PADDING = 16
};

const char* szx_version(void);
/* Message of the last failing call on this thread. */
const char* szx_last_error(void);
/* frexp(e).exp - 1 (ufzx/blockcodec.py:62-66). */
int32_t szx_bound_exponent(double e);
/* Testing hook: cap the blocks per kernel launch (0 = default) so the cross-launch carry
 * of pool offsets is exercised at small sizes.  Returns the previous cap. */
uint64_t szx_set_max_chunk_blocks(uint64_t blocks);
/* Testing / benchmarking hook: the bs == 128 compress kernel -- 1 (default) the CTA-tile
 * compress128_kernel, 2 the warp-autonomous encode128_kernel.  Same bytes.  Returns the
 * previous variant. */
int szx_set_compress_variant(int variant);
/* Testing hook: K3 sums the constant map before its tile range directly for streams of up to
 * `blocks` blocks (default 2^24), with a decoupled look-back beyond; returns the old value. */
uint64_t szx_set_index_direct_limit(uint64_t blocks);
/* Testing hook: the index pass (K3) kernel, 1 = one range of tiles per SM (default), 2 = one
 * 16-tile chunk per CTA with two look-backs (slower: 46 vs 31 us on NYX); returns the old value. */
int szx_set_index_kernel(int kernel);
/* Benchmarking hook for the host-buffer entry points: `parts` (1..32) host->device copy parts
 * = decode chunks of szx_decompress_host (default 8; any other value leaves it unchanged, so 0
 * queries it); `trace` != 0 prints the CUDA-event time of each pipeline stage to stderr after
 * every host call.  Returns the previous part count. */
int szx_set_host_pipeline(int parts, int trace);
/* Profiling builds (-DSZX_STATS) only: per-phase cycle counters.  `reset` bit 0 clears
 * after reading, bits 1-2 select the kernel (0 compress128, 1 index, 2 decode,
 * 3 encode128, which fills 16 counters). */
int szx_debug_stats(uint64_t* out8, int reset);
/* Profiling builds (-DSZX_TRACE) only: install a device buffer of 8 u64 per compress tile
 * (NULL: off); the bs == 128 compress kernel stores %globaltimer at each tile's pipeline
 * events (claim, TMA issue, input seen, aggregate, look-back scan, inclusive prefix,
 * write-out start / end). */
int szx_debug_trace(void* d_buf);

/* ---- device-pointer API ------------------------------------------------------------- */

/* Replaces DataField.__post_init__ finite check + global min/max (container.py:84-87).
 * d_minmax[0]=min, d_minmax[1]=max; SZX_FLAG_NONFINITE is OR-ed into *d_err. */
size_t szx_range_scratch_bytes(uint64_t n);
int szx_range_f32(const float* d_x, uint64_t n, float* d_minmax, uint32_t* d_err,
                  void* d_scratch, size_t scratch_bytes, void* stream);

/* Replaces pipeline.compress / parallel.parallel_compress pool construction
 * (pipeline.py:136-183, parallel.py:104-140).  Worst-case pool sizes (caller allocates):
 *   map   szx_map_bytes(n,bs)      (4-byte aligned)
 *   mu    4*nb                     (4-byte aligned)
 *   req   nb
 *   codes szx_codes_capacity(n)    (4-byte aligned)
 *   mid   4*n + 16                 (16-byte aligned)
 * d_x must be 16-byte aligned.  d_totals receives the exact pool lengths; d_err receives
 * SZX_FLAG_BAD_REQ if the reference would reject the stream (container.py:206-207). */
uint64_t szx_num_blocks(uint64_t n, uint32_t block_size);
uint64_t szx_map_bytes(uint64_t n, uint32_t block_size);
uint64_t szx_codes_capacity(uint64_t n);
size_t szx_compress_scratch_bytes(uint64_t n, uint32_t block_size);
int szx_compress_f32(const float* d_x, uint64_t n, uint32_t block_size, double e,
                     uint8_t* d_map, float* d_mu, uint8_t* d_req, uint8_t* d_codes,
                     uint8_t* d_mid, szx_totals* d_totals, uint32_t* d_err, void* d_scratch,
                     size_t scratch_bytes, void* stream);

/* szx_compress_f32 that also writes the decode index szx_index_f32 would compute from the
 * produced pools (d_index: szx_index_bytes, 16-byte aligned) as a by-product of the tile
 * look-back, so decompress of a device-produced stream needs no index pass (K3).  For block
 * sizes 64/128/256/512 (128: with the default kernel; szx_compress_emits_index); otherwise
 * SZX_ERR_INVALID_ARG.  The index has one entry per 8192-value tile for every one of these
 * block sizes (8192 / bs blocks, groups of 512 / bs blocks). */
int szx_compress_emits_index(uint32_t bs);
int szx_compress_indexed_f32(const float* d_x, uint64_t n, uint32_t bs, double e, uint8_t* d_map,
                             float* d_mu, uint8_t* d_req, uint8_t* d_codes, uint8_t* d_mid,
                             szx_totals* d_totals, uint32_t* d_err, void* d_scratch,
                             size_t scratch_bytes, uint64_t* d_index, void* stream);

/* Replaces the mid-pool length derivation and pool checks of deserialize /
 * CompressedStream._validate (container.py:198-214,246-253,304-305,392-402).
 * *d_mid_total is overwritten with the mid length the codes imply. */
int szx_validate_f32(const uint8_t* d_req, uint64_t n_nc, const uint8_t* d_codes, uint64_t m,
                     const float* d_mu, uint64_t nb, uint32_t block_size,
                     uint64_t* d_mid_total, uint32_t* d_err, void* stream);

/* Block size 128: the "scan of the stored sizes" on its own (pipeline.decode_layout,
 * pipeline.py:193-214; container.py:198-214,246-253,304-305 checks).  Writes the tile index
 * to d_index (16-byte aligned, szx_index_bytes): one 64-byte entry per 64-block decode tile
 * {u64 NC blocks before, u64 mid bytes before (relative to the tile's K3 range), u16
 * tile-relative mid offset of each 4-block group x 16, u64 range id, u64 0}, a closing entry,
 * then one u64 mid-byte base per K3 range.  The index is consumed by
 * szx_decompress_indexed_f32 (treat it as opaque).  d_stats[0] = NC blocks, d_stats[1] =
 * mid-pool length implied by the codes; flags BAD_REQ / CODE_PADDING / MU_NONFINITE into
 * *d_err. */
uint64_t szx_index_bytes(uint64_t n, uint32_t block_size);
size_t szx_index_scratch_bytes(uint64_t n, uint32_t block_size);
int szx_index_f32(const uint8_t* d_map, const float* d_mu, const uint8_t* d_req,
                  const uint8_t* d_codes, uint64_t n, uint32_t block_size, uint64_t* d_index,
                  uint64_t* d_stats, uint32_t* d_err, void* d_scratch, size_t scratch_bytes,
                  void* stream);
/* Block size 128: one decode pass given a tile index (pipeline.py:216-260). */
int szx_decompress_indexed_f32(const uint8_t* d_map, const float* d_mu, const uint8_t* d_req,
                               const uint8_t* d_codes, const uint8_t* d_mid, uint64_t mid_len,
                               uint64_t n, uint32_t block_size, const uint64_t* d_index,
                               float* d_out, uint32_t* d_err, void* stream);

/* Replaces pipeline.decompress / parallel.parallel_decompress (pipeline.py:193-260,
 * parallel.py:143-180): for block size 128 the index pass then the decode pass, otherwise
 * one look-back decode pass.  d_mu 4-byte aligned, d_out 16-byte aligned, d_mid 16-byte
 * aligned and readable up to round_up(mid_len,16)+16 bytes.  SZX_FLAG_UNDERRUN is OR-ed into
 * *d_err if the codes need more mid bytes than mid_len (reads are clamped). */
size_t szx_decompress_scratch_bytes(uint64_t n, uint32_t block_size);
int szx_decompress_f32(const uint8_t* d_map, const float* d_mu, const uint8_t* d_req,
                       const uint8_t* d_codes, const uint8_t* d_mid, uint64_t mid_len,
                       uint64_t n, uint32_t block_size, float* d_out, szx_totals* d_totals,
                       uint32_t* d_err, void* d_scratch, size_t scratch_bytes, void* stream);

/* ---- measurement and simulation passes (device pointers, stream-ordered) ------------- */

/* pipeline.compress_with_accounting (pipeline.py:119-132,186-190): *d_bits = sum over NC
 * elements of req - 8*min(3, lzb(w ^ prev_w), req // 8), w the UNSHIFTED bits of x - mu
 * (the shadow scheme of metrics.ShiftAccounting.bits_unshifted_scheme).  The shifted side is
 * 8 * mid_len of the same stream.  Same classification as szx_compress_f32. */
int szx_accounting_f32(const float* d_x, uint64_t n, uint32_t block_size, double e,
                       uint64_t* d_bits, void* stream);

/* metrics.max_abs_error / mse / psnr (metrics.py:78-103) in one pass over both arrays:
 * d_out5 = {max |f64(a)-f64(b)|, sum (f64(a)-f64(b))^2, f64(min a), f64(max a), NaN count}.
 * Deterministic for a given device (fixed-order reduction of per-CTA partials). */
size_t szx_quality_scratch_bytes(uint64_t n);
int szx_quality_f32(const float* d_a, const float* d_b, uint64_t n, double* d_out5,
                    void* d_scratch, size_t scratch_bytes, void* stream);

/* metrics.block_range_cdf (metrics.py:128-146): d_counts[t] = number of blocks whose
 * (f64 max - f64 min) / global_range <= d_thresholds[t] (nthr <= 64). */
int szx_block_range_counts_f32(const float* d_x, uint64_t n, uint32_t block_size,
                               double global_range, const double* d_thresholds, uint32_t nthr,
                               uint64_t* d_counts, void* stream);

/* parallel.prefix_scan (parallel.py:21-44): exclusive int64 scan (wrapping adds). */
size_t szx_prefix_scan_scratch_bytes(uint64_t n);
int szx_prefix_scan_i64(const int64_t* d_in, uint64_t n, int64_t* d_out, void* d_scratch,
                        size_t scratch_bytes, void* stream);

/* parallel.propagate_indices (parallel.py:83-101): d_positions (count x q, row-major int64)
 * = for every byte column the 1-based index of the latest element at or before it whose
 * byte there is a mid byte (0 = the zero word).  d_codes: one leading code per element. */
int szx_propagate_indices(const uint8_t* d_codes, uint32_t count, uint32_t q,
                          int64_t* d_positions, void* stream);
/* parallel.propagate_round (parallel.py:74-80) on a (rows x cols) int64 matrix. */
int szx_propagate_round(const int64_t* d_in, uint64_t rows, uint32_t cols, uint64_t stride,
                        int64_t* d_out, void* stream);

/* ---- batched small fields (BASELINE configs[2]: many fields, one launch per step) ----- */

/* DataField range of every field in ONE launch: d_minmax[2f], d_minmax[2f+1] = min, max of
 * field f; SZX_FLAG_NONFINITE OR-ed into d_err[f] (caller zeroes).  d_x / n: host arrays. */
size_t szx_range_batch_scratch_bytes(uint32_t nfields, const uint64_t* n);
int szx_range_batch_f32(uint32_t nfields, const float* const* d_x, const uint64_t* n,
                        float* d_minmax, uint32_t* d_err, void* d_scratch, size_t scratch_bytes,
                        void* stream);

/* [compress(DataField(x_f), cfg) for f] for block size 128 in ONE launch over all fields'
 * tiles (a decoupled look-back segmented per field).  Host arrays of per-field device
 * pointers / sizes / bounds; pools sized as for szx_compress_f32; d_totals[f] receives field
 * f's pool lengths, d_err the OR of all fields' flags.  Fields of up to 2^26-64 blocks. */
size_t szx_compress_batch_scratch_bytes(uint32_t nfields, const uint64_t* n);
int szx_compress_batch_f32(uint32_t nfields, const float* const* d_x, const uint64_t* n,
                           const double* e, uint8_t* const* d_map, float* const* d_mu,
                           uint8_t* const* d_req, uint8_t* const* d_codes, uint8_t* const* d_mid,
                           szx_totals* d_totals, uint32_t* d_err, void* d_scratch,
                           size_t scratch_bytes, void* stream);
/* The same, also writing each field's decode index (d_index[f]: szx_index_bytes(n[f], 128)
 * bytes, 16-byte aligned, or NULL for none) -- what szx_index_f32 computes from the pools --
 * from per-group offsets the compress launch records, so szx_decompress_batch_indexed_f32
 * decodes the batch without the index pass. */
int szx_compress_batch_indexed_f32(uint32_t nfields, const float* const* d_x, const uint64_t* n,
                                   const double* e, uint8_t* const* d_map, float* const* d_mu,
                                   uint8_t* const* d_req, uint8_t* const* d_codes,
                                   uint8_t* const* d_mid, uint64_t* const* d_index,
                                   szx_totals* d_totals, uint32_t* d_err, void* d_scratch,
                                   size_t scratch_bytes, void* stream);

/* [decompress(stream_f) for f] for block size 128: ONE K3 launch indexing every stream (each
 * field its own CTA ranges) and ONE K2 launch over the decode tiles of all fields.  Host
 * arrays of per-field device pool pointers and sizes; d_out[f] 16-byte aligned; d_stats
 * (device, 2 per field) receives {NC blocks, mid length the codes imply}; flags per field
 * OR-ed into d_err[f] (caller zeroes) as for szx_decompress_f32. */
size_t szx_decompress_batch_scratch_bytes(uint32_t nfields, const uint64_t* n);
int szx_decompress_batch_f32(uint32_t nfields, const uint8_t* const* d_map,
                             const float* const* d_mu, const uint8_t* const* d_req,
                             const uint8_t* const* d_codes, const uint8_t* const* d_mid,
                             const uint64_t* mid_len, const uint64_t* n, float* const* d_out,
                             uint64_t* d_stats, uint32_t* d_err, void* d_scratch,
                             size_t scratch_bytes, void* stream);
/* The same through given decode indexes (d_index[f], from szx_compress_batch_indexed_f32 or
 * szx_index_f32): ONE K2 launch, no index pass (and no d_stats). */
int szx_decompress_batch_indexed_f32(uint32_t nfields, const uint8_t* const* d_map,
                                     const float* const* d_mu, const uint8_t* const* d_req,
                                     const uint8_t* const* d_codes, const uint8_t* const* d_mid,
                                     const uint64_t* mid_len, const uint64_t* n,
                                     const uint64_t* const* d_index, float* const* d_out,
                                     uint32_t* d_err, void* d_scratch, size_t scratch_bytes,
                                     void* stream);

/* ---- host-buffer API (the reference's user-level calls) ------------------------------ */

/* Upper bound of a UFZX stream for n values (container.py:255-266 at worst case). */
uint64_t szx_compress_bound(uint64_t n, uint32_t ndims, uint32_t block_size);

/* ufzx.serialize(ufzx.compress(DataField(x, dims), CompressorConfig(ErrorBound(mode, mag),
 * block_size))) -- mode 0 = "abs", 1 = "rel".  Writes the UFZX bytes to h_out. */
int szx_compress_host(const float* h_x, const uint64_t* dims, uint32_t ndims,
                      uint32_t block_size, int32_t rel_mode, double magnitude, uint8_t* h_out,
                      uint64_t out_capacity, uint64_t* out_len);

/* Header peek: value count and dims of a UFZX stream (container.py:349-370 checks). */
int szx_stream_info(const uint8_t* h_in, uint64_t len, uint64_t* n_values, uint32_t* ndims,
                    uint64_t* dims_out, uint32_t dims_capacity, uint32_t* block_size,
                    double* error_bound);

/* ufzx.decompress(ufzx.deserialize(blob)).values -- writes n float32 values to h_out. */
int szx_decompress_host(const uint8_t* h_in, uint64_t len, float* h_out, uint64_t n_capacity);

#ifdef __cplusplus
}
#endif
#endif /* SZX_B200_H */
