// Argument records + launchers of k_dominance.cu, shared with mo_capi.cu.
#pragma once
#include "mo_grid.cuh"

namespace mo {

constexpr int PRESORT_BUCKETS = 65536;   // maximum (workspace sizing)

// Buckets used for R rows: ~one per row, 1024 .. 65536 (the bucket scan is a fixed cost per step).
__host__ __device__ inline int presort_buckets(int R) {
  int nb = 1024;
  while (nb < R && nb < PRESORT_BUCKETS) nb <<= 1;
  return nb;
}

struct PresortArgs {
  const float* F;
  int R, m;
  uint32_t* keyA;   // R: per-row bucket
  int* valA;        // unused (kept for the workspace layout)
  uint32_t* keyB;   // R: per-row S key
  int* valB;        // PRESORT_BUCKETS + 1: bucket counts -> starts
  int* perm;        // sorted position -> row
  float* FS;        // R x m, sorted
  float* SS;        // R, sorted sums
  int* wend;        // R
  float* blkmin;    // ceil(R/256)
  float* blkmax;
  unsigned* ctl;    // [0] min key, [1] max key (reset by the launcher), [2..] fill cursors base
  int* fill;        // PRESORT_BUCKETS
  GridCtx g;
  unsigned long long* trace;
  // stable = 1: rows inside a bucket keep ascending row order (two stable
  // 8-bit radix passes of the bucket key instead of the atomic scatter), so
  // every shard of a sharded sort derives the same position space
  int stable;
  uint32_t* tkey;   // R (stable only)
  int* tval;        // R (stable only)
  // in_step = 1 (mo_step): no memset nodes -- the grid barrier is self-resetting, the key range is
  // reset by the kernel after its last use, and hasdom (nullable) is cleared here for the tile kernel
  int in_step;
  uint8_t* hasdom;
};

int64_t words_per_row(int64_t R);
int launch_presort(const PresortArgs& args, cudaStream_t s);
int launch_dom_tile(const float* F, int64_t R, int m, const uint8_t* valid, uint32_t* bits, cudaStream_t s);
int launch_dom_tile_sorted(const float* FS, const float* blkmin, const float* blkmax, const int* wend, int64_t R,
                           int m, uint32_t* bits, uint8_t* hasdom, cudaStream_t s, bool clear_hasdom = true);
size_t dom_rank_tables_bytes(int64_t R, int m);
// Tile summary (engine path): bit t of row p's tsum words = "word block t (256 dominators) of row p was
// written and is nonzero".  With a summary the rank kernels store only nonzero word blocks and the peel
// reads only flagged blocks (a C3 row has ~15 nonzero blocks of the ~390 below its S bound).
__host__ __device__ inline int64_t tsum_words(int64_t R) { return (((R + 255) / 256) + 31) / 32; }
int launch_dom_rank(const float* FS, const float* blkmin, const float* blkmax, const int* wend, int64_t R, int m,
                    uint32_t* bits, uint8_t* hasdom, uint32_t* tables, cudaStream_t s, uint32_t* tsum = nullptr);
int launch_front_peel(const uint32_t* bits, int64_t R, const uint8_t* valid, int64_t stop_at, int* ranks,
                      int* info, int* resume, uint32_t* ranked, int* front_sizes, unsigned* bar,
                      const int* perm, const uint8_t* hasdom, const int* wend, int* rank_pos,
                      unsigned long long* trace, cudaStream_t s, bool in_step = false,
                      const uint32_t* tsum = nullptr);

}  // namespace mo
