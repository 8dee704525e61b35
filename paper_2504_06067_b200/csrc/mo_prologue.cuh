// The rank-independent part of a generation's niche preparation -- keyed
// shuffles of the merged rows and of the reference points, the shuffled
// reference directions, the lattice position scatter and the reset of the
// per-reference niche state -- depends only on (seed, generation), so mo_step
// runs it in extra CTAs of k_vary_eval, concurrently with the variation,
// instead of inside k_prep after the sort (k_prep then builds only the
// candidate list, the extremes and the intercepts).  Same values either way.
#pragma once
#include "mo_common.cuh"
#include "mo_rng.cuh"
#include "k_niche_args.cuh"

namespace mo {

// gtid / gthreads: this thread's index among the threads doing the prologue.
// sK*, sS*, sR*: shared-memory shuffle keys (filled here; __syncthreads inside).
__device__ inline void gen_prologue(const PrepArgs& a, uint32_t gen, int gtid, int gthreads, uint32_t* sKp,
                                    uint32_t* sSp, int* sRp, uint32_t* sKr, uint32_t* sSr, int* sRr) {
  const int R = a.R, m = a.m, w = a.w;
  load_shuffle_keys_smem(sKp, sSp, sRp, (uint32_t)R, a.seed, gen, STREAM_POP_SHUFFLE);
  load_shuffle_keys_smem(sKr, sSr, sRr, (uint32_t)w, a.seed, gen, STREAM_REF_SHUFFLE);
  __syncthreads();
  // one index space over rows then reference points, so a thread runs one shuffle chain (~74 dependent
  // rounds) rather than one of each when the grid covers R + w
  for (int t = gtid; t < R + w; t += gthreads) {
    if (t < R) {
      const int i = t;
      const int p = (int)prp((uint32_t)i, sKp, sSp, *sRp, (uint32_t)R);
      a.pos_pop[i] = p;
      a.perm_pop[p] = i;
      if (a.prom) a.prom[i] = 0;
      if (a.akey) a.akey[i] = 0ull;
      continue;
    }
    const int j = t - R;
    const int p = (int)prp((uint32_t)j, sKr, sSr, *sRr, (uint32_t)w);
    a.pos_ref[j] = p;
    if (a.lat_pos) a.lat_pos[__ldg(a.lat_index + j)] = p;
    a.perm_ref[p] = j;
    if (a.rho) {
      a.rho[j] = 0;
      a.rho_p[j] = 0;
      a.take[j] = 0;
      a.kept[j] = 0;
      a.fill[j] = 0;
      a.near_key[j] = ~0ull;
    }
    if (a.zhat)
      for (int k = 0; k < m; ++k) {
        const float z = a.zhat[(int64_t)j * m + k];
        a.zs[(int64_t)p * m + k] = z;
        if (a.zsT) a.zsT[(int64_t)k * w + p] = z;
      }
  }
  if (a.lvl)
    for (int q = gtid; q < LVL_WORDS; q += gthreads) a.lvl[q] = 0;
  if (a.sctl && gtid < 16) a.sctl[gtid] = 0;
  if (gtid == 0 && a.fb_ctl) {
    a.fb_ctl[0] = 0;
    a.info[MO_INFO_ASSOC_FALLBACK] = 0;
  }
}

}  // namespace mo
