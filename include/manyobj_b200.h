/*
 * manyobj_b200.h -- C-ABI of the B200-native NSGA-III survivor-selection +
 * variation engine (libmanyobj_b200.so, sm_100a).
 *
 * The reference ("manyobj", /root/reference/SPEC.md) is a Python package; its
 * hot path is engine.step and the per-op functions it calls.
 * Each entry point below replaces one of those operations; the comment on each
 * cites the reference interface (file:line) it stands in for.  The Python
 * host package paper_2504_06067_b200 binds these with ctypes.
 *
 * Conventions:
 *   - plain device pointers + sizes; no torch/C++ types in signatures;
 *   - the caller allocates every buffer, including the workspace sized by
 *     mo_workspace_bytes(); the library never allocates or frees;
 *   - all work is stream-ordered and asynchronous on `stream`
 *     (a cudaStream_t passed as void*); the caller sets the device;
 *   - status codes map 1:1 onto pkg/src/manyobj/errors.py classes;
 *   - device-side outcomes (split front, domain violations) are written to
 *     caller-provided device int arrays and read lazily by the host.
 */
#ifndef MANYOBJ_B200_H
#define MANYOBJ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes -> pkg/src/manyobj/errors.py:4-41 */
enum {
  MO_OK = 0,
  MO_ERR_SHAPE = 1,      /* ShapeError           errors.py:4  */
  MO_ERR_PARAM = 2,      /* ParameterError       errors.py:8  */
  MO_ERR_BOUNDS = 3,     /* BoundsError          errors.py:12 */
  MO_ERR_EMPTY = 4,      /* EmptySelectionError  errors.py:16 */
  MO_ERR_DOMAIN = 5,     /* DomainError          errors.py:20 */
  MO_ERR_INFEASIBLE = 6, /* InfeasibleSplitError errors.py:32 */
  MO_ERR_CUDA = 7        /* CUDA runtime failure (no reference analogue) */
};

/* Objective-count limits: the engine (mo_step) runs 2 <= m <= MO_MAX_M
 * (Appendix D studies m = 4 ... 512); m <= 16 runs register-array
 * kernels, 16 < m <= MO_MAX_M the runtime-m ("wide") kernels. */
enum { MO_MAX_M = 512 };

/* Problems (DTLZ1/4/6 per the standard suite). */
enum { MO_DTLZ1 = 1, MO_DTLZ2, MO_DTLZ3, MO_DTLZ4, MO_DTLZ5, MO_DTLZ6, MO_DTLZ7 };

/* Split/outcome record written by the selection kernels (device int32[16]). */
enum {
  MO_INFO_L = 0,          /* splitting front index l                       */
  MO_INFO_SELECTED = 1,   /* |F_s| = cumulative size of fronts < l         */
  MO_INFO_K = 2,          /* k = n - |F_s|                                 */
  MO_INFO_NFRONTS = 3,    /* fronts peeled (= l + 1)                       */
  MO_INFO_FL_SIZE = 4,    /* |F_l|                                         */
  MO_INFO_SKIPPED = 5,    /* 1 if cum(<=l) == n and niching was skipped    */
  MO_INFO_NEAREST = 6,    /* individuals promoted by nearest selection     */
  MO_INFO_LEVEL = 7,      /* water-fill level L*                           */
  MO_INFO_SINGULAR = 8,   /* 1 if the intercept solve fell back entirely   */
  MO_INFO_SURVIVORS = 9,  /* survivors written (must equal n)              */
  MO_INFO_ERROR = 10,     /* non-zero status raised on the device          */
  MO_INFO_ASSOC_FALLBACK = 11, /* candidates the lattice-pruned association
                                  could not certify (full scan instead)     */
  MO_INFO_ERROR_FIRST = 12, /* first non-zero device status since the host
                               last zeroed it (sticky: later generations
                               never clear it; the engine raises it)     */
  MO_INFO_COUNT = 16
};

/* VariationConfig; p_m < 0 means 1/d. */
typedef struct mo_var_cfg {
  float eta_c;
  float eta_m;
  float p_c;
  float p_m;
} mo_var_cfg;

/* ---------------------------------------------------------------- sizing */

/* Bytes of workspace mo_step / mo_select need for (n, m, d, w).  The
 * bit-matrix dominates: 2n x round_up(2n, 256)/8 bytes. */
int mo_workspace_bytes(int64_t n, int32_t m, int32_t d, int64_t w, size_t* bytes);

/* Workspace bytes of the per-op entry points (mo_front_peel, mo_normalize,
 * mo_associate, mo_niche_select) for R rows, m objectives, w reference points. */
int mo_workspace_bytes_rows(int64_t R, int32_t m, int64_t w, size_t* bytes);

/* Words per row of the dominance bit-matrix for R rows. */
int64_t mo_bits_words_per_row(int64_t R);

/* Byte offset, inside an mo_step workspace for (n, m, w), of the 64-slot
 * uint64 phase trace (globaltimer ns stamped at phase boundaries of the
 * persistent kernels; diagnostic only). */
int64_t mo_trace_offset(int64_t n, int32_t m, int64_t w);

/* Library build/version string. */
const char* mo_version(void);
/* sizeof(mo_step_args) as compiled into the library (bindings check their mirror against it). */
size_t mo_step_args_bytes(void);

/* --------------------------------------------------- RNG / shuffles (L1) */

/* batchcore.shuffle_rows permutation.  perm[p] = item at
 * position p (new -> old), pos[i] = position of item i; either may be NULL. */
int mo_permutation(int64_t n, uint64_t seed, uint32_t generation, uint32_t stream,
                   int32_t* perm, int32_t* pos, void* stream_);

/* engine.initialize's uniform population, SPEC.md:450-458 (X is n x d). */
int mo_init_population(float* X, int64_t n, int32_t d, uint64_t seed, void* stream_);

/* ----------------------------------------------- problems / variation (L2/L3) */

/* problems.dtlz_eval.  F is n x m.  *domain_flag (device
 * int32, may be NULL) is OR-ed with 1 when any x lies outside [0,1]. */
int mo_dtlz_eval(int32_t problem, const float* X, int64_t n, int32_t d, int32_t m, float* F,
                 int32_t* domain_flag, void* stream_);

/* variation.mating_pool + sbx_pair + polynomial_mutation + clamp, then
 * dtlz_eval of the children, fused.
 * Parents X (n x d) -> offspring Xo (n x d), Fo (n x m).  If ideal != NULL
 * it is lowered to the column minima of Fo (running ideal). */
int mo_vary_eval(int32_t problem, const float* X, int64_t n, int32_t d, int32_t m, uint64_t seed,
                 uint32_t generation, const mo_var_cfg* cfg, float* Xo, float* Fo, float* ideal,
                 void* stream_);

/* --------------------------------------------------------- dominance (L3) */

/* dominance.dominance_matrix, as a bit-matrix:
 * bit i of row j (word i/32 of bits + j*W) is set iff F[i] dominates F[j].
 * valid (uint8 per row, NULL = all valid): invalid rows neither dominate nor
 * are dominated.  W = mo_bits_words_per_row(R). */
int mo_dominance_bits(const float* F, int64_t R, int32_t m, const uint8_t* valid, uint32_t* bits,
                      void* stream_);

/* The engine's sort path (used inside mo_step), exposed for testing and
 * measurement: mo_presort buckets the R rows by a 16-bit quantisation of
 * S = FP32 left-to-right sum of their objectives (S-ordered buckets, arbitrary
 * order inside a bucket) and writes perm[p] (row at position p), FS (R x m
 * rows in that order), SS (their sums), wend[p] (one past the last bit-matrix
 * word that can hold a dominator of p) and blkmin/blkmax (min/max S of every
 * 256-position block, ceil(R/256) floats each).  mo_dominance_bits_sorted then
 * fills `bits` in position space (rows p, words < wend[p] only) and
 * hasdom[p] = 1 iff p has a dominator.  Same reference op as
 * mo_dominance_bits. */
int mo_presort(const float* F, int64_t R, int32_t m, int32_t* perm, float* FS, float* SS, int32_t* wend,
               float* blkmin, float* blkmax, void* workspace, size_t workspace_bytes, void* stream_);
int mo_dominance_bits_sorted(const float* FS, const float* blkmin, const float* blkmax, const int32_t* wend,
                             int64_t R, int32_t m,
                             uint32_t* bits, uint8_t* hasdom, void* stream_);

/* Same bit-matrix and hasdom as mo_dominance_bits_sorted, by per-objective
 * rank masks (k_dom_rank.cu, the engine's kernel for 2 <= m <= MO_MAX_M; m > 16
 * streams the tables in chunks of 8 objectives): for every
 * 256-row block and objective, the sorted values (Eytzinger order) and the 257
 * prefix masks; a row's dominators in a block are the AND over objectives of
 * the prefix masks selected by m binary searches.  tables: device scratch of
 * mo_dominance_tables_bytes(R, m) bytes (0 = unsupported m). */
size_t mo_dominance_tables_bytes(int64_t R, int32_t m);
/* tsum: NULL = store every word block below the S bound (the op-level
 * contract); else the engine's tile summary (R x mo_tile_summary_words(R)
 * uint32, bit t of row p = word block t of row p is nonzero and stored): only
 * nonzero blocks are stored. */
int64_t mo_tile_summary_words(int64_t R);
int mo_dominance_bits_ranked(const float* FS, const float* blkmin, const float* blkmax, const int32_t* wend,
                             int64_t R, int32_t m, uint32_t* bits, uint8_t* hasdom, void* tables,
                             size_t tables_bytes, uint32_t* tsum, void* stream);

/* dominance.non_dominated_sort + split_fronts, peeling the
 * bit-matrix.  stop_at > 0 stops at the first front whose cumulative size
 * reaches stop_at (later rows get 0x7fffffff = dropped); stop_at <= 0 ranks
 * every valid row.  info: device int32[MO_INFO_COUNT]. */
int mo_front_peel(const uint32_t* bits, int64_t R, const uint8_t* valid, int64_t stop_at,
                  int32_t* ranks, int32_t* info, void* workspace, size_t workspace_bytes,
                  void* stream_);

/* ------------------------------------------------------------- niche (L3) */

/* niche.normalize_objectives, over candidate rows
 * (ranks[i] <= l, l = info[MO_INFO_L]).  ideal (m) is updated in place
 * (running minimum over all R rows); Fn (R x m, may be NULL) receives the
 * normalised objectives of candidate rows; intercepts (m doubles, may be NULL). */
int mo_normalize(const float* F, int64_t R, int32_t m, const int32_t* ranks, const int32_t* info,
                 uint64_t seed, uint32_t generation, float* ideal, float* Fn, double* intercepts,
                 void* workspace, size_t workspace_bytes, void* stream_);

/* niche.perpendicular_distance_matrix + associate, fused and
 * never materialising D: for every candidate row, pi = nearest reference
 * point (canonical FP32 key, lowest shuffled reference position on ties) and
 * d = perpendicular distance.  Fn is R x m, zhat is w x m unit directions. */
int mo_associate(const float* Fn, int64_t R, int32_t m, const float* zhat, int64_t w,
                 const int32_t* ranks, const int32_t* info, uint64_t seed, uint32_t generation,
                 int32_t* pi, float* d, void* workspace, size_t workspace_bytes, void* stream_);

/* niche.niche_counts + nearest_selection + build_cache +
 * batched_random_selection (closed-form water-filling).
 * Promoted individuals get rank l-1 in `ranks`; selected (uint8, R) marks
 * the n survivors. */
int mo_niche_select(const int32_t* pi, const float* d, int64_t R, int64_t w, int64_t n,
                    int32_t* ranks, int32_t* info, uint64_t seed, uint32_t generation,
                    uint8_t* selected, void* workspace, size_t workspace_bytes, void* stream_);

/* ---------------------------------------------------------- engine (L4) */

/* engine.step: one NSGA-III generation.
 *   XR (2n x d), FR (2n x m): rows [0,n) hold the parents on entry;
 *   X_next (n x d), F_next (n x m): survivors, ascending merged index;
 *   ideal (m): running ideal, updated; ranks (2n): merged-population ranks;
 *   info: device int32[MO_INFO_COUNT]; zhat: w x m unit reference directions.
 * Decision variables live in [0,1]^d (the DTLZ domain). */
typedef struct mo_step_args {
  int32_t problem;
  int32_t m;
  int32_t d;
  int32_t pad0;
  int64_t n;
  int64_t w;
  uint64_t seed;
  uint32_t generation;
  uint32_t pad1;
  mo_var_cfg var;
  const float* zhat;
  float* XR;
  float* FR;
  float* X_next;
  float* F_next;
  float* ideal;
  int32_t* ranks;
  int32_t* info;
  void* workspace;
  size_t workspace_bytes;
  /* Optional device uint32 generation counter.  When non-NULL the kernels read
   * the generation from it (instead of `generation`) and the step increments
   * it, so one captured CUDA graph can be replayed generation after generation. */
  uint32_t* generation_dev;
  /* Sort mode: MO_SORT_BITS (0, the default) stores the dominance bit-matrix
   * and peels it inside mo_step; MO_SORT_STREAM (1) never stores it (O(R)
   * memory, for R^2/8 bytes beyond HBM and for sharding) and is driven front
   * by front by the host through mo_sort_stream_begin / _front / _end. */
  int32_t sort_mode;
  /* Shards of the streamed sort and of the association (one process per
   * GPU): this process is shard `shard_rank` of `shard_count` (>= 1). */
  int32_t shard_rank;
  int32_t shard_count;
  int32_t pad2;
  /* Optional lattice pruning of the association (exact; see k_assoc_lattice),
   * for a single-layer Das-Dennis set of H divisions and m <= 5.  Lattice
   * index of k = (k_0, ..., k_{m-2}) in mixed radix H+1, k_0 most significant.
   *   lattice_z:     (H+1)^(m-1) x m FP32: zhat of the point k/H at its
   *                  lattice index (entries outside the simplex unused);
   *   lattice_index: w: lattice index of every reference point;
   *   lattice_pos:   (H+1)^(m-1) int32 scratch (the step writes the shuffled
   *                  position of every point there).
   * NULL lattice_z = full scan.  lattice_r: box radius in lattice steps
   * (0 = default: 6 at m <= 3, 3 at m = 4, 2 at m = 5). */
  const float* lattice_z;
  const int32_t* lattice_index;
  int32_t* lattice_pos;
  int32_t lattice_H;
  int32_t lattice_r;
  int32_t pad3;
  /* Tensor-core filter of the full-scan association (no lattice, one shard,
   * w >= 1024): the unit directions packed by mo_pack_refs_bf16 (device,
   * mo_pack_refs_bytes(w) bytes, static).  NULL = FP32 scan only.  The
   * association stays bit-identical: the bf16 MMA only selects which
   * references get the canonical FP32 key. */
  const void* zhat_frag;
  /* tcgen05 filter of the same full-scan association (k_assoc_umma.cu,
   * preferred over zhat_frag when set): the unit directions as FP16 UMMA
   * tiles packed by mo_pack_refs_f16 (device, mo_pack_refs_f16_bytes(w)
   * bytes, static).  The association stays bit-identical: tcgen05.mma only
   * selects which references get the canonical FP32 key. */
  const void* zhat_umma;
  /* Divisions of the Das-Dennis / two-layer reference set
   * the directions came from (0 = unknown): the tcgen05 filter seeds every
   * row's running maximum with the key of the lattice point nearest to the
   * row's simplex projection, a valid lower bound of its maximum. */
  int32_t ref_H_outer;
  int32_t ref_H_inner;
} mo_step_args;

enum { MO_SORT_BITS = 0, MO_SORT_STREAM = 1 };

int mo_step(const mo_step_args* args, void* stream_);

/* mo_step split into its phases (for per-phase timing):
 * MO_PHASE_VARY = variation + evaluation, MO_PHASE_SORT = dominance bit-matrix
 * + peeling + split, MO_PHASE_NICHE = normalisation + association + niching +
 * survivor compaction.  mo_step == all three in order. */
enum { MO_PHASE_VARY = 1, MO_PHASE_SORT = 2, MO_PHASE_NICHE = 4, MO_PHASE_ALL = 7 };
int mo_step_phases(const mo_step_args* args, uint32_t phase_mask, void* stream_);

/* MO_PHASE_NICHE split for the sharded association:
 *   NICHE_PREP   running ideal, shuffles, candidate list, extremes, intercepts
 *                (replicated on every shard);
 *   NICHE_ASSOC  association keys of every candidate against this shard's
 *                range of reference points (shuffled positions
 *                [rank*w/count, (rank+1)*w/count)) into the akey array
 *                (uint64 per merged row, mo_stream_offsets) -- the host then
 *                max-reduces akey across shards (an exact integer max);
 *   NICHE_FINISH pi, d, niche counts, niching, survivor compaction
 *                (replicated).
 * MO_PHASE_NICHE == the three in order with count == 1. */
enum { MO_PHASE_NICHE_PREP = 8, MO_PHASE_NICHE_ASSOC = 16, MO_PHASE_NICHE_FINISH = 32 };
int mo_niche_phases(const mo_step_args* args, uint32_t phase_mask, void* stream_);

/* ------------------------------------------- streamed / sharded sort (L3) */

/* dominance.non_dominated_sort + split_fronts without the
 * bit-matrix: dominator counts of the shard's rows, then one call per front.
 * Position blocks of 256 presorted rows are dealt round-robin to the shards;
 * each shard writes its slice of the front mask (mask_local, T*8 words,
 * T = ceil(ceil(R/256)/count)) and reads all slices concatenated in shard
 * order (mask_full, count*T*8 words) -- the host all-gathers between the
 * calls (with count == 1 they alias).
 *   begin:      presort, dominator counts, front 0 -> mask_local
 *   front(k):   front k from mask_full (ranks, front list, split decision);
 *               if not done: decrement counts, front k+1 -> mask_local
 *   end:        ranks in row order.
 * After front(k) closed the split, info[MO_INFO_NFRONTS] = k + 1 (0 before)
 * and later front calls are no-ops, so the host may poll lazily.  Needs a
 * workspace sized with sort_mode = MO_SORT_STREAM. */
int mo_sort_stream_begin(const mo_step_args* args, void* stream_);
int mo_sort_stream_front(const mo_step_args* args, int32_t k, void* stream_);
int mo_sort_stream_end(const mo_step_args* args, void* stream_);

/* Zero a workspace (once, before its first mo_step / mo_step_phases / mo_niche_phases): inside a step
 * the kernels keep their own counters and grid barriers consistent instead of re-initialising them with
 * memset nodes, so a captured generation has no memset nodes. */
int mo_workspace_init(void* workspace, size_t workspace_bytes, void* stream_);

/* Workspace bytes for a sort mode and shard count (mo_workspace_bytes ==
 * mode MO_SORT_BITS, 1 shard). */
int mo_workspace_bytes_ex(int64_t n, int32_t m, int32_t d, int64_t w, int32_t sort_mode, int32_t shard_count,
                          size_t* bytes);

/* Byte offset of the streamed sort's uint64[4] pair counters (measurement: (i, j) pairs evaluated by
 * the COUNT sweep with the <= chain / the full dominance chain, then the same for the DEC sweeps of
 * the generation); reset by every mo_sort_stream_begin / streamed mo_step. */
int mo_stream_stats_offset(int64_t n, int32_t m, int64_t w, int32_t sort_mode, int32_t shard_count,
                           int64_t* stats_off);

/* Byte offsets inside that workspace of mask_local / mask_full (uint32),
 * their word counts, and of akey (uint64 per merged row). */
int mo_stream_offsets(int64_t n, int32_t m, int64_t w, int32_t sort_mode, int32_t shard_count,
                      int64_t* mask_local_off, int64_t* mask_local_words, int64_t* mask_full_off,
                      int64_t* akey_off);

/* Survivor selection only (NDS + split + niching + compaction) on merged
 * objectives already in FR -- the part of mo_step after variation. */
int mo_select(const mo_step_args* args, void* stream_);

/* -------------------------------------------------------- metrics (L5) */

/* metrics.igd: mean over the nr reference points (nr x m)
 * of the Euclidean distance to the nearest of the nf front rows (nf x m),
 * FP64 arithmetic; *out (device double) receives the value.  Deterministic.
 * Workspace: mo_igd_workspace_bytes(nr).  Empty input -> MO_ERR_EMPTY. */
size_t mo_igd_workspace_bytes(int64_t nr);
int mo_igd(const float* front, int64_t nf, const float* ref, int64_t nr, int32_t m, double* out, void* workspace,
           size_t workspace_bytes, void* stream_);

/* metrics.hv Monte-Carlo branch (m > 3): `samples`
 * Philox-seeded points uniform in the box [lower, upper] (device double[m]);
 * *hits_out (device uint64) = how many are weakly dominated by some front
 * row.  hv = volume(box) * hits / samples (the caller discards front rows
 * that do not dominate the reference point first).  Workspace:
 * mo_hv_mc_workspace_bytes(samples). */
size_t mo_hv_mc_workspace_bytes(int64_t samples);
int mo_hv_mc(const float* front, int64_t nf, int32_t m, const double* lower, const double* upper, int64_t samples,
             uint64_t seed, unsigned long long* hits_out, void* workspace, size_t workspace_bytes, void* stream_);

/* metrics.hv, exact branch (m <= 3): rows that do not weakly
 * dominate ref (F_i <= ref componentwise) are discarded; the FP64 volume of the
 * region dominated by the rest and bounded by ref is written to out[0] (0 when
 * none is retained).  Deterministic (slab decomposition along f3, fixed-order
 * sums).  Workspace: mo_hv_exact_workspace_bytes(nf).  m outside 1..3 ->
 * MO_ERR_PARAM.  Replaces the reference's exact sweep. */
size_t mo_hv_exact_workspace_bytes(int64_t nf);
int mo_hv_exact(const float* front, int64_t nf, int32_t m, const double* ref, double* out, void* workspace,
                size_t workspace_bytes, void* stream);

/* bf16 hi/lo m16n8k16 B-fragments of the w unit directions zhat (w x m FP32,
 * device) for mo_step_args.zhat_frag, in the packed column order `order`
 * (device int32[w], a permutation of the reference indices; NULL = identity;
 * a random order makes the filter's running maximum converge in a few steps):
 * 544 bytes per 8 columns (fragments + the columns' reference indices).
 * m <= 16. */
size_t mo_pack_refs_bytes(int64_t w);
/* FP16 tiles for the tcgen05 filter: 128 directions x K16 per 4 KB tile in the
 * UMMA K-major no-swizzle core-matrix layout (packed column order `order`,
 * NULL = identity), followed by the reference index of every packed column
 * (int32, -1 = padding).  m <= 16. */
size_t mo_pack_refs_f16_bytes(int64_t w, int32_t m);
int mo_pack_refs_f16(const float* zhat, int64_t w, int32_t m, const int32_t* order, void* out, void* stream);
int mo_pack_refs_bf16(const float* zhat, int64_t w, int32_t m, const int32_t* order, void* out, void* stream);

/* Byte offsets (into a mo_step workspace of the same sizing arguments) of the
 * niche-selection state one step leaves behind -- for the debug bookkeeping
 * check and niche trace of SPEC.md:406, :424 (niche.check_bookkeeping): out11 =
 * {pi, d, rho, rho_p, take, kept, prom, pos_pop, perm_pop, pos_ref, perm_ref}. */
int mo_niche_offsets(int64_t n, int32_t m, int64_t w, int32_t sort_mode, int32_t shard_count, int64_t* out11);

/* ------------------------------------------- op-level API (k_ops.cu)
 * The reference's per-op functions as device kernels, for callers of the
 * per-op API (the engine runs these stages fused inside mo_step).  Index and
 * count arrays are int64 (the reference's integer vectors), outputs follow the
 * reference oracle's order (oracle/manyobj_ref/niche.py:157-278).  Stream
 * ordered; the caller owns every buffer; workspace from
 * mo_ops_workspace_bytes(rows, points). */
int mo_ops_workspace_bytes(int64_t R, int64_t w, size_t* bytes);

/* batchcore.step_mask: out[i] = x[i] > 0. */
int mo_step_mask(const double* x, int64_t n, int8_t* out, void* stream);
/* batchcore.masked_argmin: *out (device int64) = lowest index
 * of the minimum over valid slots (valid NULL = all), -1 when none is valid
 * (the caller raises EmptySelectionError). */
int mo_masked_argmin(const double* values, const uint8_t* valid, int64_t n, int64_t* out, void* workspace,
                     size_t workspace_bytes, void* stream);
/* batchcore.segment_count: counts[j] = valid labels == j;
 * a valid label outside [0, segments) sets *status (device) = MO_ERR_BOUNDS. */
int mo_segment_count(const int64_t* labels, const uint8_t* valid, int64_t n, int64_t segments, int64_t* counts,
                     int32_t* status, void* stream);
/* niche.associate over a materialised distance matrix D
 * (R x w FP64): pi = first column of the row minimum, d = that minimum;
 * invalid rows -> (-1, NaN). */
int mo_associate_matrix(const double* D, const uint8_t* valid, int64_t R, int64_t w, int64_t* pi, double* d,
                        void* stream);
/* niche.niche_counts: rho over rank < l (l > 0), rho' over
 * rank == l, rho = 2^31-1 (infinity) where rho' == 0. */
int mo_niche_counts(const int64_t* pi, const int64_t* ranks, int64_t R, int64_t l, int64_t w, int64_t* rho,
                    int64_t* rho_p, void* stream);
/* niche.nearest_selection: for every point with rho == 0
 * the rank-l candidate of smallest (d, pos_pop); all of them when they are
 * <= k (ascending point order), else the first k by pos_ref.  promoted:
 * device int64[w], *n_promoted (device) entries; rho / rho_p updated in place
 * (rho = 1, rho' - 1, infinity when rho' reaches 0). */
int mo_nearest_selection(const int64_t* pi, const float* d, const int64_t* ranks, int64_t R, int64_t l,
                         int64_t* rho, int64_t* rho_p, int64_t w, int64_t k, const int64_t* pos_pop,
                         const int64_t* pos_ref, int64_t* promoted, int64_t* n_promoted, void* workspace,
                         size_t workspace_bytes, void* stream);
/* niche.build_cache as CSR: offsets[w+1], cand = rank-l
 * rows not flagged in `exclude` (uint8 per row, may be NULL), grouped by pi,
 * shuffled population order inside a point. */
int mo_build_cache(const int64_t* pi, const int64_t* ranks, int64_t R, int64_t l, int64_t w, const int64_t* pos_pop,
                   const uint8_t* exclude, int64_t* offsets, int64_t* cand, void* workspace, size_t workspace_bytes,
                   void* stream);
/* niche.batched_random_selection: the k rows Alg. 2's loop
 * takes from the CSR cache, in the loop's order; info (device int64[3]) =
 * (rows taken, loop iterations, status: MO_ERR_INFEASIBLE when the loop
 * cannot fill k). */
int mo_batched_random_selection(const int64_t* offsets, const int64_t* cand, const int64_t* rho, const int64_t* rho_p,
                                int64_t w, int64_t k, const int64_t* pos_ref, int64_t* taken, int64_t* info,
                                void* workspace, size_t workspace_bytes, void* stream);
/* variation.sbx_pair over npairs pairs of d variables,
 * FP64: with u (npairs x d) SBX on every variable; u == NULL draws the
 * engine's Philox streams (pair Bernoulli(p_c), one u per variable) for
 * (seed, generation).  clamp != 0 clamps to [lo, hi]. */
int mo_sbx_pairs(const double* P1, const double* P2, int64_t npairs, int32_t d, const double* u, double eta_c,
                 float p_c, double lo, double hi, int32_t clamp, uint64_t seed, uint32_t generation, double* C1,
                 double* C2, void* stream);
/* variation.polynomial_mutation, FP64, clamped to [lo, hi]:
 * with u (n x d) mutate where flag (uint8, NULL = everywhere); u == NULL
 * draws the engine's PM stream (flag = u < p_m, then a second draw). */
int mo_polynomial_mutation(const double* X, int64_t n, int32_t d, const double* u, const uint8_t* flag, double eta_m,
                           float p_m, double lo, double hi, uint64_t seed, uint32_t generation, double* out,
                           void* stream);

/* ---------------------------------------------------- measurement helper */

/* Issue-rate microbenchmark for the roofline of the CUDA-core kernels (not a
 * reference op): which = 0 -> 64 FP32 compares (setp.{lt,gt}[.or]) per
 * iteration per thread; which = 1 -> 16 FP32 flops (mul.rn + add.rn) per
 * iteration per thread.  256 threads per block; in64 = 64 floats. */
int mo_peak_issue(int32_t which, int32_t blocks, int32_t iters, const float* in64, void* out, void* stream_);

#ifdef __cplusplus
}
#endif

#endif /* MANYOBJ_B200_H */
