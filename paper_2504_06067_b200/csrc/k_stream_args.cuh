// Argument record + launchers of k_stream.cu (streamed / row-sharded
// non-dominated sort), shared with mo_capi.cu.
#pragma once
#include "mo_grid.cuh"

namespace mo {

constexpr int STREAM_BLK = 256;      // rows per position block (= bit-matrix tile edge)
constexpr int STREAM_CHUNK = 16;     // i-blocks of 256 rows per work item

// ctl[] slots
enum {
  SC_WORK = 0,    // work-queue cursor of k_stream_tiles
  SC_ITEMS = 1,   // items planned for the current launch
  SC_FLN = 2,     // |front list|
  SC_CUM = 3,     // rows ranked so far
  SC_DONE = 4,    // 0 while peeling; k + 1 once front k closed the split
  SC_COUNT = 16
};

struct StreamArgs {
  // presorted rows (k_presort): position space
  const float* FS;       // R x m
  const float* SS;       // R   FP32 row sums (S order)
  const int* wend;       // R   one past the last word that can hold a dominator
  const float* blkmin;   // ceil(R/256)
  const float* blkmax;
  const int* perm;       // position -> row
  int R, m;
  int G, g;              // shards, this shard
  int T;                 // position blocks owned per shard = ceil(nb / G)
  int64_t stop_at;       // n
  int* cnt;              // R   dominator counts (owned rows)
  int* rank_pos;         // R   ranks in position space (replicated)
  uint32_t* mask_local;  // T * 8 words: this shard's slice of the front mask
  const uint32_t* mask_full;  // G * T * 8 words: all slices (after the all-gather)
  int* fl;               // R   front list (positions, ascending)
  float* flmax;          // ceil(R/256) max S per 256-entry block of fl
  int* plan;             // T + 1 work-item prefix
  int* ucnt;             // T   unranked rows per owned block
  int* ctl;              // SC_COUNT
  int* info;             // MO_INFO_COUNT
  int* ranks;            // R   output ranks (row order)
  GridCtx gc;
  // boxed mode (m <= 10): Morton-ordered positions, per-block bounding boxes,
  // all ordered block pairs classified none / all / mixed (k_presort_morton)
  int boxed;
  float* blkbox;         // nb x 2 x m: per 256-row block min[m], max[m]
  float* flbox;          // nb x 2 x m: per 256-entry front-list chunk
  float* blkbox32;       // ceil(R/32) x 2 x m: per 32-row group
  float* flbox32;        // ceil(R/32) x 2 x m: per 32-entry front-list group
  unsigned long long* stats;  // nullable, 4: (i, j) pairs evaluated -- COUNT fast/full, DEC fast/full
  float* blkS32;         // ceil(R/32) x 2: S min / max per 32-row group (boxed)
  float* flS32;          // ceil(R/32) x 2: S min / max per 32-entry front-list group (boxed)
};

// Morton presort of the boxed mode (F -> perm, FS, SS, S block range, boxes)
struct MortonArgs {
  const float* F;
  int R, m;
  uint32_t* keyA;
  int* valA;
  uint32_t* tkey;
  int* tval;
  unsigned* cbox;        // 2 x 16 ordered-uint per-coordinate min / max
  int* perm;
  float* FS;
  float* SS;
  float* blkmin;
  float* blkmax;
  float* blkbox;
  float* blkbox32;
  float* blkS32;
  GridCtx g;
};

int launch_presort_morton(const MortonArgs& a, cudaStream_t s);
int launch_stream_begin(StreamArgs a, cudaStream_t s);
int launch_stream_front(StreamArgs a, int k, cudaStream_t s);
int launch_stream_end(StreamArgs a, cudaStream_t s);
int launch_stream_fused(StreamArgs a, cudaStream_t s);

}  // namespace mo
