// Argument records + launchers of k_niche.cu, shared with mo_capi.cu.
#pragma once
#include "mo_grid.cuh"

namespace mo {

struct PrepArgs {
  const float* F;
  int R, m, w;
  const int* ranks;
  int* info;
  float* ideal;
  uint64_t seed;
  uint32_t gen;
  const uint32_t* gen_ptr;  // nullable: device generation counter overrides `gen`
  const float* zhat;
  int* pos_pop;
  int* perm_pop;
  int* pos_ref;
  int* perm_ref;
  float* zs;
  int* cand;
  int* ctl;  // ctl[0] = candidate count
  unsigned long long* ext_key;
  unsigned* colmax;
  double* icpt;
  float* a32;
  unsigned long long* akey;
  unsigned* bar;
  double* icpt_out;
  int mode;  // PREP_FULL | PREP_PERMS_CAND | PREP_PERMS
  unsigned long long* trace;  // nullable phase trace (slots 16..19)
  // niche-selection state cleared here for k_assoc_final / k_select
  int* rho;
  int* rho_p;
  int* take;
  int* kept;
  int* fill;
  unsigned long long* near_key;
  uint8_t* prom;
  int* lvl;   // LVL_WORDS: level histograms + level-search accumulators
  int* sctl;  // 16 select counters
  const int* lat_index;  // nullable: lattice index of every reference point (lattice-pruned association)
  int* lat_pos;          // lat_pos[lat_index[j]] = shuffled position of j
  // in_step = 1 (mo_step): no memset nodes -- ctl[0] is zeroed by the previous step's k_select, the
  // barrier is self-resetting, and the lattice fallback counters (nullable) are cleared here
  int in_step;
  int* fb_ctl;
  // mating parents precomputed one generation ahead by the prologue CTAs of k_vary_eval (the mating
  // shuffle depends on (seed, generation, n) only): [4p .. 4p+3] tag of the buffer of parity p =
  // (~generation, seed lo, seed hi, n), [8] completion counter, [16 + p * n ..) parent of slot q.  nullable
  int* mate;
  int pro_done;    // gen_prologue already ran (in k_vary_eval): only the candidate list in phase 0
  int ideal_done;  // the running ideal was already lowered by the offspring (k_vary_eval)
  // wide m (m > 16; nullable otherwise): the FP64 hyperplane system when m > 64 (m x m, global) and the
  // objective-major copy of the shuffled directions, zsT[k * w + p] (written by gen_prologue)
  double* solveA;
  float* zsT;
};

constexpr int LVL_BINS = 1024;
// lvl region: the two level histograms, then 3 x 32 u64 accumulators of the 32-ary level search
// (levels beyond the histogram window)
constexpr int LVL_WORDS = 2 * LVL_BINS + 3 * 32 * 2;
enum { SCTL_M0 = 0, SCTL_ALLOC = 1, SCTL_MAXE = 2, SCTL_NPART = 3 };

enum { PREP_FULL = 0, PREP_PERMS_CAND = 1, PREP_PERMS = 2 };

struct AssocArgs {
  const float* F;        // R x m (raw objectives, or Fn when ideal == a32 == nullptr)
  const float* ideal;    // nullable
  const float* a32;      // nullable
  const float* zs;       // w x m, shuffled order
  const int* cand;
  const int* ctl;        // ctl[0] = candidate count
  const int* info;
  int w;
  int psplit;            // reference points per blockIdx.y
  unsigned long long* akey;
  int zbeg, zend;        // shuffled reference positions handled by this launch (shard range)
  // lattice pruning (k_assoc_lattice): dense (k_0..k_{m-2}) -> reference index table, H, box radius;
  // rows it cannot certify are appended to fb_cand (count fb_ctl[0]) for the full scan
  const float* lat_z;    // (H+1)^(m-1) x m: unit directions in lattice order (static)
  const int* lat_pos;    // (H+1)^(m-1): shuffled position of each lattice point (k_prep, per generation)
  int lat_H, lat_r;
  const int* pos_ref;
  int* fb_cand;
  int* fb_ctl;
  int in_step;           // fb_ctl / info[MO_INFO_ASSOC_FALLBACK] already cleared by k_prep
  // tensor-core filter (k_assoc_hmma): bf16 hi/lo fragments of the unit directions in static reference
  // order (mo_pack_refs_bf16); nullptr = FP32 full scan only
  const uint2* zfrag;
  const float* zsT;      // wide m: m x w objective-major shuffled directions (k_assoc_wide)
  // tcgen05 filter (k_assoc_umma): FP16 reference tiles + packed-column reference indices
  // (mo_pack_refs_f16); preferred over zfrag when set
  const void* zumma;
  int ref_Ho, ref_Hi;    // divisions of the reference set (0 = unknown): lattice seeds of the running maxima
};

struct AssocFinalArgs {
  const float* F;
  const float* ideal;
  const float* a32;
  const float* zs;
  const int* perm_ref;
  const int* cand;
  const int* ctl;
  const int* info;
  int m;
  const unsigned long long* akey;
  int* pi;
  float* d;
  float* Fn_out;  // nullable
  int fn_only;    // write Fn_out and stop (mo_normalize)
  const int* ranks;  // niche counts (nullable: skip): rho over rank < l, rho' over rank == l
  int* rho;
  int* rho_p;
};

struct SelectArgs {
  int R, w, n;
  int* ranks;
  int* info;
  const int* pi;
  const float* d;
  const int* pos_pop;
  const int* perm_pop;
  const int* perm_ref;
  int* rho;       // niche counts over rank < l (k_assoc_final), post-nearest in place
  int* rho_p;     // candidates over rank == l, post-nearest in place
  int* take;      // cache entries taken per reference point
  int* kept;      // marked-and-kept at the last water-fill level
  int* bstart;    // bucket start of partially taken reference points
  int* fill;      // bucket fill cursors
  int* bucket;    // shuffled positions of the bucketed candidates (R)
  unsigned long long* near_key;
  uint8_t* prom;
  int* lvl;       // LVL_WORDS
  int* sctl;
  uint8_t* selected;
  const float* XR;  // compaction sources (nullable)
  const float* FR;
  float* X_next;
  float* F_next;
  int dvars, m;
  int count_inside;   // op-level: compute rho / rho' here (engine: fused in k_assoc_final)
  uint32_t* gen_ptr;  // nullable: incremented once the step is complete
  unsigned long long* trace;  // nullable phase trace (slots 24..40)
  GridCtx g;
  int in_step;        // no barrier memset node (self-resetting barrier)
  int* reset_ctl;     // nullable: k_prep's candidate counter, zeroed here after its last reader
};

int launch_prep(const PrepArgs& a, cudaStream_t s);
int launch_assoc(const AssocArgs& a, int m, int64_t R, cudaStream_t s);
int launch_assoc_hmma(const AssocArgs& a, int m, int64_t R, cudaStream_t s);
int launch_pack_refs(const float* zhat, int64_t w, int m, const int32_t* order, uint2* out, cudaStream_t s);
int launch_assoc_lattice(const AssocArgs& a, int m, int64_t R, cudaStream_t s);
int launch_assoc_fallback(const AssocArgs& a, int m, cudaStream_t s);
int launch_assoc_umma(const AssocArgs& a, int m, int64_t R, cudaStream_t s);
size_t pack_refs_f16_bytes(int64_t w, int m);
int launch_pack_refs_f16(const float* zhat, int64_t w, int m, const int32_t* order, void* out, cudaStream_t s);
int launch_assoc_final(const AssocFinalArgs& a, int64_t R, cudaStream_t s);
int launch_select(const SelectArgs& a, cudaStream_t s);

}  // namespace mo
