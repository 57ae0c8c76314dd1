// szx_kernels.h -- launch descriptors shared by the C-ABI layer (abi.cu) and the kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace szx {

// Device-resident running totals of one stream (carried from chunk to chunk).
struct Totals {
  uint64_t n_nc;     // non-constant blocks so far (== req pool bytes)
  uint64_t m;        // non-constant elements so far (== number of 2-bit codes)
  uint64_t mid_len;  // mid-pool bytes so far
  uint64_t pad;
};

// Error flag bits (device u32, OR-accumulated).
enum : uint32_t {
  kErrBadReq = 1u,        // an NC block got req outside 1..32      (container.py:206-207)
  kErrNonFinite = 2u,     // non-finite input value                 (container.py:84-85)
  kErrUnderrun = 4u,      // mid pool shorter than the codes imply  (blockcodec.py:155-158)
  kErrMuNonFinite = 8u,   // non-finite mu in a stream              (container.py:198-199)
  kErrCodePadding = 16u,  // nonzero padding bits in the code pool  (container.py:304-305)
};

struct CompressArgs {
  const float* x;        // first value of this chunk
  uint64_t n;            // values in this chunk
  uint32_t bs;           // block size
  double e;              // resolved absolute bound
  int pe;                // frexp(e).exp - 1
  uint8_t* map;          // first map byte of this chunk (chunks start at 32-block multiples)
  float* mu;             // first mu of this chunk
  uint8_t* req;          // req pool base (absolute; chunk offset comes from `base`)
  uint8_t* codes;        // code pool base (absolute)
  uint8_t* mid;          // mid pool base (absolute, 16-byte aligned)
  const Totals* base;    // totals before this chunk
  Totals* totals;        // totals after this chunk (written by the last tile)
  uint64_t* status;      // one look-back word per tile, zeroed
  uint32_t* counter;     // dynamic tile counter, zeroed
  uint32_t* err;         // error flags
  uint32_t ntiles;
  // optional (bs == 128, K1 v1): the decode index K3 would compute (64-byte entry per
  // 64-block tile; see IndexArgs), written as a by-product of the look-back
  uint64_t* index;       // null: not produced
  uint64_t idx_tile0;    // stream-level tile of this chunk's first tile
  uint64_t idx_ntiles;   // stream-level tile count (closing entry)
  int idx_last;          // this chunk writes the closing entry and the base table
};

// One field of a batched bs == 128 compress launch (BASELINE configs[2]): the field's
// values, bound and pools; its tiles are global tiles [tile0, tile0 + ntiles) of the launch.
struct FieldDesc {
  const float* x;
  uint64_t n;
  double e;
  int32_t pe;
  uint32_t ntiles;
  uint64_t tile0;
  uint8_t* map;
  float* mu;
  uint8_t* req;
  uint8_t* codes;
  uint8_t* mid;
  Totals* totals;
  // optional decode index of the field (null: none): the compress kernel records every
  // 4-block group's (NC blocks, mid bytes) before it in `groups` (2 u64 per group), then
  // groups_to_index_kernel turns them into the 64-byte entries K3 would write into `index`
  uint64_t* groups;
  uint64_t* index;
};

struct DecompressArgs {
  const uint8_t* map;    // chunk-relative
  const float* mu;       // chunk-relative
  const uint8_t* req;    // absolute pool bases
  const uint8_t* codes;
  const uint8_t* mid;    // 16-byte aligned, readable up to round_up(mid_len,16)+16
  uint64_t mid_len;      // bytes actually present in the mid pool
  float* out;            // chunk-relative
  uint64_t n;            // values in this chunk
  uint32_t bs;
  const Totals* base;
  Totals* totals;
  uint64_t* status_nc;   // look-back chain over non-constant block counts
  uint64_t* status_mid;  // look-back chain over mid-byte counts
  uint32_t* counter;
  uint32_t* err;
  uint32_t ntiles;
};

// K3 (bs == 128): per-decode-tile (NC blocks before, mid bytes before) + stream checks.
struct IndexArgs {
  const uint8_t* map;
  const float* mu;
  const uint8_t* req;
  const uint8_t* codes;
  uint64_t n;                      // values
  uint64_t* index;                 // 2 * (ntiles + 1) u64: {nc_before, mid_before}
  unsigned long long* mid_total;   // mid-pool length the codes imply
  unsigned long long* nc_total;    // NC block count
  uint32_t* err;
  uint64_t* status_nc;             // one look-back word per group, zeroed
  uint64_t* status_mid;
  uint32_t* counter;               // zeroed
  uint32_t ngroups;
  uint64_t direct_limit;           // maps of up to this many blocks are summed directly
  uint32_t bs;                     // block size: 64, 128 (also 0), 256 or 512; tiles of 8192 values
};

// K2 (bs == 128): decode with a precomputed tile index (no look-back).
struct Decode128Args {
  const uint8_t* map;
  const float* mu;                 // 4-byte aligned
  const uint8_t* req;
  const uint8_t* codes;
  const uint8_t* mid;              // readable to round_up(end,16)
  uint64_t mid_len;                // bytes present in the mid pool (reads are clamped)
  const uint64_t* index;           // 16-byte aligned
  float* out;                      // 16-byte aligned
  uint64_t n;
  uint64_t ntiles;                 // decode tiles of the whole stream (index layout)
  uint64_t tile_begin, tile_end;   // tiles this launch decodes
  uint32_t* err;
  uint32_t bs;                     // block size: 64, 128 (also 0), 256 or 512; tiles of 8192 values
};

// Tile geometry.
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kFastBPW = 4;                         // blocks per warp, bs == 128 path
constexpr int kFastTileBlocks = kWarps * kFastBPW;  // 32 blocks = 4096 values per CTA
constexpr int kGenTileBlocks = kWarps;              // generic path: one warp per block
constexpr int kCompTileBlocks = 64;                 // K1 (bs == 128) tile: 64 blocks = 32 KiB
#ifndef SZX_V3_WARPS
#define SZX_V3_WARPS 18
#endif
constexpr int kV3Warps = SZX_V3_WARPS;              // K1 v3: compute warps = 4-block groups
constexpr int kV3TileBlocks = 4 * kV3Warps;         // K1 v3 tile

cudaError_t compress_stats(unsigned long long* out8, bool reset);
cudaError_t k1_trace_buffer(unsigned long long* d_buf);  // profiling builds (-DSZX_TRACE)
cudaError_t index_stats(unsigned long long* out8, bool reset);
cudaError_t decode_stats(unsigned long long* out8, bool reset);
cudaError_t encode_stats(unsigned long long* out8, bool reset);
cudaError_t v3_stats(unsigned long long* out16, bool reset);
cudaError_t launch_compress128(const CompressArgs& a, cudaStream_t s);
// K1 (variant 1) for the fast-path block sizes 64, 128, 256, 512 (tiles of 8192 values,
// 8192 / bs blocks per tile); a.bs selects the instantiation
constexpr bool fast_bs(uint32_t bs) { return bs == 64 || bs == 128 || bs == 256 || bs == 512; }
cudaError_t launch_compress_fast(const CompressArgs& a, cudaStream_t s);
cudaError_t launch_encode128(const CompressArgs& a, cudaStream_t s);
cudaError_t launch_compress128v3(const CompressArgs& a, cudaStream_t s);
cudaError_t launch_compress128v4(const CompressArgs& a, cudaStream_t s);
// K1 variant 5: the 16 compute warps in SZX_V5_TEAMS teams taking alternate tiles
#ifndef SZX_V5_TEAMS
#define SZX_V5_TEAMS 2
#endif
constexpr int kV5TileBlocks = 4 * 16 / SZX_V5_TEAMS;
cudaError_t launch_compress128v5(const CompressArgs& a, cudaStream_t s);
// batched: `a` carries the launch-wide status / counter / err / ntiles (sum over fields);
// d_fields / d_tmaps (device, 64-byte aligned) the per-field descriptors and tensor maps,
// h_fields / h_tmaps their host copies (the tensor maps are encoded into h_tmaps here)
// the decode index of every field of a batched launch that asked for one (FieldDesc.index)
cudaError_t launch_groups_to_index(const FieldDesc* d_fields, const FieldDesc* h_fields,
                                   uint32_t nfields, cudaStream_t s);
cudaError_t launch_compress128v3_batch(const CompressArgs& a, FieldDesc* d_fields,
                                       const FieldDesc* h_fields, uint32_t nfields,
                                       void* d_tmaps, void* h_tmaps, cudaStream_t s);
// K1 (bs == 128): a CTA's compute warps encode one super-tile of kEncWarps warp tiles of
// kEncWarpBlocks blocks each per step; the look-back runs over super-tiles
#ifndef SZX_K1V2_WARPS
#define SZX_K1V2_WARPS 22
#endif
constexpr int kEncWarps = SZX_K1V2_WARPS;
constexpr int kEncWarpBlocks = 4;
constexpr int kEncTileBlocks = kEncWarps * kEncWarpBlocks;  // 96 blocks
void launch_compress_generic(const CompressArgs& a, cudaStream_t s);
void launch_index128(const IndexArgs& a, cudaStream_t s);
// K3 v2: one 16-tile chunk per CTA (chunk ids from a.counter, look-backs over a.status_nc /
// a.status_mid, one word per chunk each, zeroed)
void launch_index128v2(const IndexArgs& a, cudaStream_t s);
uint64_t index128v2_chunks(uint64_t n);
void launch_decode128(const Decode128Args& a, cudaStream_t s);
// batched (BASELINE configs[2]): K3 over all fields in one (max_groups, nfields) launch, each
// field's own ngroups CTAs; K2 over the concatenated decode tiles of all fields
uint32_t index_batch_groups(uint64_t n);
void launch_index128_batch(const IndexArgs* d_fields, uint32_t nfields, uint32_t max_groups,
                           cudaStream_t s);
void launch_decode128_batch(const Decode128Args& a, const Decode128Args* d_fields,
                            const uint64_t* d_tile0s, uint32_t nfields, cudaStream_t s);
constexpr int kDecTileBlocks = 64;     // K2 (bs == 128) decode tile: 64 blocks
constexpr int kIndexGroupTiles = 16;   // decode tiles per K3 CTA (1024 blocks)
// K3 index entry per decode tile (64 bytes): {NC blocks before, mid bytes before} as u64,
// then the mid-byte offset (u16, tile-relative) of each 4-block group, then zero padding.
constexpr int kIndexEntryBytes = 64;
#ifndef SZX_K3_PER_SM
#define SZX_K3_PER_SM 1
#endif
constexpr int kIndexCtasPerSm = SZX_K3_PER_SM;      // K3 CTAs resident per SM
constexpr int kIndexMaxRanges = 256 * kIndexCtasPerSm;  // K3 ranges (grid size cap)
void launch_decompress_generic(const DecompressArgs& a, cudaStream_t s);

// Global min / max / non-finite flag (container.py:84-87).  `partials` holds
// 2*gridDim floats + a counter; result[0]=min, result[1]=max, *err |= kErrNonFinite.
void launch_range(const float* x, uint64_t n, float* partials, uint32_t* counter,
                  float* result, uint32_t* err, int grid, cudaStream_t s);
int range_grid(uint64_t n);
struct RangeField {
  const float* x;
  uint64_t n;
};
// batched: a (grid, nfields) launch; partials 2*grid floats per field, one counter / result
// pair / error word per field (counters zeroed)
void launch_range_batch(const RangeField* d_fields, uint32_t nfields, int grid, float* partials,
                        uint32_t* counters, float* results, uint32_t* errs, cudaStream_t s);

// Mid-pool length implied by req + codes (container.py:246-253, 392-402) plus the
// stream checks container.py:198-214,304-305 that need a pass over device pools.
void launch_validate(const uint8_t* req, uint64_t n_nc, const uint8_t* codes, uint64_t m,
                     const float* mu, uint64_t nb, uint32_t bs, unsigned long long* mid_total,
                     uint32_t* err, cudaStream_t s);

// analysis.cu: accounting / quality / block-range / scan / propagation passes
void launch_accounting(const float* x, uint64_t n, uint32_t bs, double e, int pe,
                       unsigned long long* bits, cudaStream_t s);
int quality_grid(uint64_t n);
size_t quality_part_bytes();
void launch_quality(const float* a, const float* b, uint64_t n, void* parts, uint32_t* counter,
                    double* out, cudaStream_t s);
uint32_t max_thresholds();
void launch_block_range(const float* x, uint64_t n, uint32_t bs, double grange, const double* thr,
                        uint32_t nthr, unsigned long long* counts, cudaStream_t s);
uint64_t scan_tiles(uint64_t n);
void launch_prefix_scan(const long long* in, uint64_t n, long long* out, long long* sums,
                        cudaStream_t s);
void launch_propagate(const uint8_t* codes, uint32_t count, uint32_t q, long long* pos,
                      cudaStream_t s);
void launch_propagate_round(const long long* p, uint64_t rows, uint32_t cols, uint64_t stride,
                            long long* out, cudaStream_t s);

}  // namespace szx
