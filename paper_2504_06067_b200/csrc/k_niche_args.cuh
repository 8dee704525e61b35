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
};

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
  int* rho;
  int* rho_p;
  int* take;
  int* bstart;
  unsigned long long* near_key;
  uint8_t* prom;
  uint32_t* keyA;
  int* valA;
  uint32_t* keyB;
  int* valB;
  int* ctl;
  uint8_t* selected;
  const float* XR;  // compaction sources (nullable)
  const float* FR;
  float* X_next;
  float* F_next;
  int dvars, m;
  uint32_t* gen_ptr;  // nullable: incremented once the step is complete
  GridCtx g;
};

int launch_prep(const PrepArgs& a, cudaStream_t s);
int launch_assoc(const AssocArgs& a, int m, int64_t R, cudaStream_t s);
int launch_assoc_final(const AssocFinalArgs& a, int64_t R, cudaStream_t s);
int launch_select(const SelectArgs& a, cudaStream_t s);

}  // namespace mo
