// extern "C" boundary of libmanyobj_b200.so (declared in include/manyobj_b200.h).
//
// Every entry point validates its scalar arguments, carves the caller's
// workspace, and enqueues kernels on the caller's stream.  No allocation, no
// synchronisation, no host round trip: device-side outcomes land in `info`.
#include <stdlib.h>
#include <string.h>

#include "mo_common.cuh"
#include "mo_grid.cuh"
#include "mo_rng.cuh"

namespace mo {
// k_vary.cu
struct PrepArgs;
int launch_vary_eval(int problem, const float* X, int64_t n, int d, int m, uint64_t seed, uint32_t gen,
                     const uint32_t* gen_ptr, const mo_var_cfg& cfg, float* Xo, float* Fo, float* ideal,
                     int* domain_flag, cudaStream_t s, const PrepArgs* pro = nullptr);
int launch_init_population(float* X, int64_t n, int d, uint64_t seed, cudaStream_t s);
int launch_dtlz_eval(int problem, const float* X, int64_t n, int d, int m, float* F, int* domain_flag,
                     cudaStream_t s);
}  // namespace mo

#include "k_niche_args.cuh"

#include "k_dominance_args.cuh"

#include "k_stream_args.cuh"

namespace mo {

thread_local bool g_mo_pdl = false;

struct PdlScope {  // PDL on for the kernels of one generation enqueued by this host thread
  PdlScope() { g_mo_pdl = getenv("MO_NO_PDL") == nullptr; }
  ~PdlScope() { g_mo_pdl = false; }
};

constexpr int MAX_GRID = 1024;  // upper bound on persistent-grid blocks (part/hist sizing)

struct Layout {
  size_t bits, resume, ranked, fsizes, bar, pos_pop, perm_pop, pos_ref, perm_ref, zs, cand, ctl, ext_key,
      colmax, icpt, a32, solve, zsT, tsum, akey, pi, d, rho, rho_p, take, bstart, near_key, prom, keyA, valA, keyB, valB, part,
      hist, sel, FS, SS, perm_sort, wend, hasdom, rank_pos, trace, pcnt, pfill, blkmin, blkmax, pctl, kept, fill,
      lvl, sctl, mate, dtab, fcand, fctl, blkbox, flbox, blkbox32, flbox32, blkS32, flS32, cbox, sstats, tkey, tval, cnt, mask_local, mask_full, fl, flmax, plan, ucnt, stctl, total;
  int64_t T, mask_local_words, mask_full_words;
};

static size_t bump(size_t& cur, size_t bytes) {
  size_t at = (cur + 255) & ~(size_t)255;
  cur = at + bytes;
  return at;
}

static int shards_of(int32_t count) { return count < 1 ? 1 : count; }

// sort_mode LAYOUT_OPS: the per-op entry points (mo_normalize, mo_associate, mo_niche_select, ...) -- no
// bit-matrix (mo_front_peel takes the caller's) and no streamed-sort regions.
constexpr int LAYOUT_OPS = -1;
static Layout make_layout(int64_t R, int64_t w, int m, int sort_mode = MO_SORT_BITS, int G = 1) {
  Layout L;
  size_t c = 0;
  const int64_t W = words_per_row(R);
  L.bits = bump(c, sort_mode == MO_SORT_BITS ? (size_t)R * W * 4 : 0);
  L.resume = bump(c, (size_t)R * 4);
  L.ranked = bump(c, (size_t)W * 4);
  L.fsizes = bump(c, (size_t)(R + 4) * 4);
  L.bar = bump(c, 128 * 4);
  L.pos_pop = bump(c, (size_t)R * 4);
  L.perm_pop = bump(c, (size_t)R * 4);
  L.pos_ref = bump(c, (size_t)w * 4);
  L.perm_ref = bump(c, (size_t)w * 4);
  L.zs = bump(c, (size_t)w * m * 4);
  L.cand = bump(c, (size_t)R * 4);
  L.ctl = bump(c, 64 * 4);
  const int64_t mm = m > 64 ? m : 64;   // per-objective slots (wide m: up to MO_MAX_M)
  L.ext_key = bump(c, (size_t)mm * 8);
  L.colmax = bump(c, (size_t)mm * 4);
  L.icpt = bump(c, (size_t)mm * 8);
  L.a32 = bump(c, (size_t)mm * 4);
  // wide m: the FP64 hyperplane system (m > 64 does not fit k_prep's shared arrays) and the
  // objective-major copy of the shuffled directions read by k_assoc_wide
  L.solve = bump(c, m > 64 ? (size_t)m * m * 8 : 0);
  L.zsT = bump(c, m > 16 ? (size_t)w * m * 4 : 0);
  L.akey = bump(c, (size_t)R * 8);
  L.pi = bump(c, (size_t)R * 4);
  L.d = bump(c, (size_t)R * 4);
  L.rho = bump(c, (size_t)(w + 1) * 4);
  L.rho_p = bump(c, (size_t)(w + 1) * 4);
  L.take = bump(c, (size_t)(w + 1) * 4);
  L.bstart = bump(c, (size_t)(w + 1) * 4);
  L.near_key = bump(c, (size_t)(w + 1) * 8);
  L.prom = bump(c, (size_t)R);
  L.keyA = bump(c, (size_t)R * 4);
  L.valA = bump(c, (size_t)R * 4);
  L.keyB = bump(c, (size_t)R * 4);
  L.valB = bump(c, (size_t)R * 4);
  L.part = bump(c, (size_t)2 * (MAX_GRID + 1) * 4);
  L.hist = bump(c, (size_t)256 * MAX_GRID * 4);
  L.sel = bump(c, (size_t)R);
  L.FS = bump(c, (size_t)R * m * 4);
  L.SS = bump(c, (size_t)R * 4);
  L.perm_sort = bump(c, (size_t)R * 4);
  L.wend = bump(c, (size_t)R * 4);
  L.hasdom = bump(c, (size_t)R);
  L.rank_pos = bump(c, (size_t)R * 4);
  L.trace = bump(c, 64 * 8);
  L.pcnt = bump(c, (size_t)(PRESORT_BUCKETS + 1) * 4);
  L.pfill = bump(c, (size_t)(PRESORT_BUCKETS + 1) * 4);
  L.blkmin = bump(c, (size_t)(R / 256 + 2) * 4);
  L.blkmax = bump(c, (size_t)(R / 256 + 2) * 4);
  L.pctl = bump(c, 16 * 4);
  L.kept = bump(c, (size_t)(w + 1) * 4);
  L.fill = bump(c, (size_t)(w + 1) * 4);
  L.lvl = bump(c, (size_t)LVL_WORDS * 4);
  L.sctl = bump(c, 16 * 4);
  L.mate = bump(c, (size_t)(R + 16) * 4);   // [0..7] two tags, [8] counter, [16..): two n-slot mating buffers
  // rank-mask dominance tables (k_dom_rank.cu): per 256-row block and objective, Eytzinger values +
  // prefix masks (bit-matrix sort, 2 <= m <= MO_MAX_M)
  L.dtab = bump(c, sort_mode == MO_SORT_BITS && m >= 2 && m <= MO_MAX_M ? dom_rank_tables_bytes(R, m) : 0);
  L.tsum = bump(c, sort_mode == MO_SORT_BITS ? (size_t)R * tsum_words(R) * 4 : 0);
  // streamed / sharded sort (sort_mode == MO_SORT_STREAM)
  const bool st = sort_mode == MO_SORT_STREAM;
  const int64_t nb = ceil_div(R, STREAM_BLK);
  L.T = ceil_div(nb, (int64_t)G);
  L.mask_local_words = L.T * (STREAM_BLK / 32);
  L.mask_full_words = L.mask_local_words * G;
  L.fcand = bump(c, (size_t)R * 4);
  L.fctl = bump(c, 64);
  L.blkbox = bump(c, st ? (size_t)(nb + 1) * 2 * m * 4 : 0);
  L.flbox = bump(c, st ? (size_t)(nb + 1) * 2 * m * 4 : 0);
  L.blkbox32 = bump(c, st ? (size_t)(R / 32 + 16) * 2 * m * 4 : 0);
  L.flbox32 = bump(c, st ? (size_t)(R / 32 + 16) * 2 * m * 4 : 0);
  L.blkS32 = bump(c, st ? (size_t)(R / 32 + 16) * 2 * 4 : 0);
  L.flS32 = bump(c, st ? (size_t)(R / 32 + 16) * 2 * 4 : 0);
  L.cbox = bump(c, 32 * 4);
  L.sstats = bump(c, 4 * 8);
  L.tkey = bump(c, st ? (size_t)R * 4 : 0);
  L.tval = bump(c, st ? (size_t)R * 4 : 0);
  L.cnt = bump(c, st ? (size_t)R * 4 : 0);
  L.mask_local = bump(c, st ? (size_t)L.mask_local_words * 4 : 0);
  L.mask_full = G > 1 ? bump(c, st ? (size_t)L.mask_full_words * 4 : 0) : L.mask_local;
  L.fl = bump(c, st ? (size_t)R * 4 : 0);
  L.flmax = bump(c, st ? (size_t)(nb + 2) * 4 : 0);
  L.plan = bump(c, st ? (size_t)(L.T + 1) * 4 : 0);
  L.ucnt = bump(c, st ? (size_t)(L.T + 1) * 4 : 0);
  L.stctl = bump(c, SC_COUNT * 4);
  L.total = (c + 255) & ~(size_t)255;
  return L;
}

template <class T>
static T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(reinterpret_cast<char*>(ws) + off);
}

// Barrier slots inside L.bar (each 2 x u32, 64-byte apart to avoid false sharing)
enum { BAR_PEEL = 0, BAR_PREP = 16, BAR_SELECT = 32, BAR_PRESORT = 48, BAR_STREAM = 64 };

static int check_ws(const Layout& L, void* ws, size_t bytes) {
  if (ws == nullptr || bytes < L.total) return MO_ERR_PARAM;
  if ((reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return MO_ERR_PARAM;
  return MO_OK;
}

static PrepArgs prep_args(const Layout& L, void* ws, const float* F, int64_t R, int m, int64_t w,
                          const int* ranks, int* info, float* ideal, uint64_t seed, uint32_t gen,
                          const float* zhat, double* icpt_out, int mode) {
  PrepArgs a;
  a.F = F;
  a.R = (int)R;
  a.m = m;
  a.w = (int)w;
  a.ranks = ranks;
  a.info = info;
  a.ideal = ideal;
  a.seed = seed;
  a.gen = gen;
  a.gen_ptr = nullptr;
  a.zhat = zhat;
  a.pos_pop = at<int>(ws, L.pos_pop);
  a.perm_pop = at<int>(ws, L.perm_pop);
  a.pos_ref = at<int>(ws, L.pos_ref);
  a.perm_ref = at<int>(ws, L.perm_ref);
  a.zs = at<float>(ws, L.zs);
  a.cand = at<int>(ws, L.cand);
  a.ctl = at<int>(ws, L.ctl);
  a.ext_key = at<unsigned long long>(ws, L.ext_key);
  a.colmax = at<unsigned>(ws, L.colmax);
  a.icpt = at<double>(ws, L.icpt);
  a.a32 = at<float>(ws, L.a32);
  a.akey = at<unsigned long long>(ws, L.akey);
  a.bar = at<unsigned>(ws, L.bar) + BAR_PREP;
  a.icpt_out = icpt_out;
  a.mode = mode;
  a.trace = at<unsigned long long>(ws, L.trace);
  a.rho = at<int>(ws, L.rho);
  a.rho_p = at<int>(ws, L.rho_p);
  a.take = at<int>(ws, L.take);
  a.kept = at<int>(ws, L.kept);
  a.fill = at<int>(ws, L.fill);
  a.near_key = at<unsigned long long>(ws, L.near_key);
  a.prom = at<uint8_t>(ws, L.prom);
  a.lvl = at<int>(ws, L.lvl);
  a.sctl = at<int>(ws, L.sctl);
  a.lat_index = nullptr;
  a.lat_pos = nullptr;
  a.in_step = 0;
  a.fb_ctl = nullptr;
  a.pro_done = 0;
  a.ideal_done = 0;
  a.mate = at<int>(ws, L.mate);
  a.solveA = m > 64 ? at<double>(ws, L.solve) : nullptr;
  a.zsT = m > 16 && zhat ? at<float>(ws, L.zsT) : nullptr;
  return a;
}

static SelectArgs select_args(const Layout& L, void* ws, int64_t R, int64_t w, int64_t n, int* ranks, int* info,
                              const int* pi, const float* d, uint8_t* selected) {
  SelectArgs a;
  a.R = (int)R;
  a.w = (int)w;
  a.n = (int)n;
  a.ranks = ranks;
  a.info = info;
  a.pi = pi;
  a.d = d;
  a.pos_pop = at<int>(ws, L.pos_pop);
  a.perm_pop = at<int>(ws, L.perm_pop);
  a.perm_ref = at<int>(ws, L.perm_ref);
  a.rho = at<int>(ws, L.rho);
  a.rho_p = at<int>(ws, L.rho_p);
  a.take = at<int>(ws, L.take);
  a.kept = at<int>(ws, L.kept);
  a.bstart = at<int>(ws, L.bstart);
  a.fill = at<int>(ws, L.fill);
  a.bucket = at<int>(ws, L.valA);
  a.near_key = at<unsigned long long>(ws, L.near_key);
  a.prom = at<uint8_t>(ws, L.prom);
  a.lvl = at<int>(ws, L.lvl);
  a.sctl = at<int>(ws, L.sctl);
  a.count_inside = 0;
  a.selected = selected;
  a.XR = nullptr;
  a.FR = nullptr;
  a.X_next = nullptr;
  a.F_next = nullptr;
  a.dvars = 0;
  a.m = 0;
  a.gen_ptr = nullptr;
  a.trace = at<unsigned long long>(ws, L.trace);
  a.g.bar = at<unsigned>(ws, L.bar) + BAR_SELECT;
  a.g.part = at<int>(ws, L.part);
  a.g.hist = at<int>(ws, L.hist);
  a.g.parity = 0;
  a.in_step = 0;
  a.reset_ctl = nullptr;
  return a;
}

__global__ void k_permutation(int n, uint64_t seed, uint32_t gen, uint32_t stream, int* perm, int* pos) {
  __shared__ uint32_t sK[MAX_SHUFFLE_ROUNDS], sS[MAX_SHUFFLE_ROUNDS];
  __shared__ int sR;
  load_shuffle_keys_smem(sK, sS, &sR, (uint32_t)n, seed, gen, stream);
  __syncthreads();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (pos) pos[i] = (int)prp((uint32_t)i, sK, sS, sR, (uint32_t)n);
  if (perm) perm[i] = (int)prp_inv((uint32_t)i, sK, sS, sR, (uint32_t)n);
}

static PresortArgs presort_args(const mo_step_args* a, const Layout& L) {
  const int64_t R = 2 * a->n;
  void* ws = a->workspace;
  PresortArgs ps;
  ps.F = a->FR;
  ps.R = (int)R;
  ps.m = a->m;
  ps.keyA = at<uint32_t>(ws, L.keyA);
  ps.valA = at<int>(ws, L.valA);
  ps.keyB = at<uint32_t>(ws, L.keyB);
  ps.valB = at<int>(ws, L.pcnt);
  ps.fill = at<int>(ws, L.pfill);
  ps.blkmin = at<float>(ws, L.blkmin);
  ps.blkmax = at<float>(ws, L.blkmax);
  ps.ctl = at<unsigned>(ws, L.pctl);
  ps.perm = at<int>(ws, L.perm_sort);
  ps.FS = at<float>(ws, L.FS);
  ps.SS = at<float>(ws, L.SS);
  ps.wend = at<int>(ws, L.wend);
  ps.g.bar = at<unsigned>(ws, L.bar) + BAR_PRESORT;
  ps.g.part = at<int>(ws, L.part);
  ps.g.hist = at<int>(ws, L.hist);
  ps.g.parity = 0;
  ps.trace = at<unsigned long long>(ws, L.trace);
  ps.stable = a->sort_mode == MO_SORT_STREAM;
  ps.tkey = ps.stable ? at<uint32_t>(ws, L.tkey) : nullptr;
  ps.tval = ps.stable ? at<int>(ws, L.tval) : nullptr;
  ps.in_step = 0;
  ps.hasdom = nullptr;
  return ps;
}

// rank-mask dominance (k_dom_rank.cu) for 2 <= m <= MO_MAX_M; MO_DOM_PAIRWISE=1 selects the pairwise
// compare-chain tiles (k_dom_tile_sorted) instead
// Tiny populations (R <= 2048, e.g. C1) keep the one-launch pairwise tiles: there the splitter / table
// kernels cost more than the compare chains they replace (C1: 10.8k vs 9.1k generations/s).
static bool use_dom_rank(int m, int64_t R) {
  static int off = -1;
  if (off < 0) {
    const char* e = getenv("MO_DOM_PAIRWISE");
    off = (e && e[0] == '1') ? 1 : 0;
  }
  if (m > 16) return m <= MO_MAX_M;   // the pairwise tiles stop at m = 16
  return !off && m >= 2 && R > 2048;
}

static int sort_phase(const mo_step_args* a, const Layout& L, cudaStream_t s) {
  const int64_t n = a->n, R = 2 * n;
  void* ws = a->workspace;
  uint32_t* bits = at<uint32_t>(ws, L.bits);
  PresortArgs ps = presort_args(a, L);
  uint8_t* hasdom = at<uint8_t>(ws, L.hasdom);
  // no memset nodes inside a step (workspace zero-initialised once, mo_workspace_init)
  ps.in_step = 1;
  ps.hasdom = hasdom;
  MO_TRY(launch_presort(ps, s));
  // rank-mask kernels: only nonzero 256-bit word blocks are stored, flagged in the tile summary that the
  // peel walks (MO_NO_TSUM=1: full stores and the word-by-word peel).  m <= 3 populations have dense
  // dominance (many dominators per row, many fronts: DTLZ3 m=3 N=16k 21 fronts): there the full stores
  // and the contiguous word peel are faster (1,617 vs 928 generations/s), so the summary is for m >= 4
  static int no_tsum = -1;
  if (no_tsum < 0) {
    const char* e = getenv("MO_NO_TSUM");
    no_tsum = (e && e[0] == '1') ? 1 : 0;
  }
  uint32_t* tsum = nullptr;
  if (use_dom_rank(a->m, R)) {
    tsum = (no_tsum || a->m <= 3) ? nullptr : at<uint32_t>(ws, L.tsum);
    MO_TRY(launch_dom_rank(ps.FS, ps.blkmin, ps.blkmax, ps.wend, R, a->m, bits, hasdom, at<uint32_t>(ws, L.dtab), s,
                           tsum));
  } else {
    MO_TRY(launch_dom_tile_sorted(ps.FS, ps.blkmin, ps.blkmax, ps.wend, R, a->m, bits, hasdom, s, false));
  }
  return launch_front_peel(bits, R, nullptr, n, a->ranks, a->info, at<int>(ws, L.resume), at<uint32_t>(ws, L.ranked),
                           at<int>(ws, L.fsizes), at<unsigned>(ws, L.bar) + BAR_PEEL, ps.perm, hasdom, ps.wend,
                           at<int>(ws, L.rank_pos), ps.trace, s, true, tsum);
}

// tensor-core filtered association: full reference range (one shard), packed fragments, enough points
// for the filter to pay (below ~1k points the FP32 scan's smem tiles are as fast); MO_NO_HMMA=1 disables
static bool use_hmma(const AssocArgs& aa, int m) {
  static int off = -1;
  if (off < 0) {
    const char* e = getenv("MO_NO_HMMA");
    off = (e && e[0] == '1') ? 1 : 0;
  }
  return !off && aa.zfrag && m >= 2 && m <= 16 && aa.zbeg == 0 && aa.zend == aa.w && aa.w >= 1024;
}

// tcgen05 association filter (k_assoc_umma.cu): same eligibility, FP16 reference tiles present;
// MO_ASSOC=hmma selects the mma.sync filter, MO_NO_HMMA=1 the FP32 scan
static bool use_umma(const AssocArgs& aa, int m) {
  static int off = -1;
  if (off < 0) {
    const char* e = getenv("MO_ASSOC");
    const char* h = getenv("MO_NO_HMMA");
    off = ((e && strcmp(e, "hmma") == 0) || (h && h[0] == '1')) ? 1 : 0;
  }
  return !off && aa.zumma && m >= 2 && m <= 16 && aa.zbeg == 0 && aa.zend == aa.w && aa.w >= 1024;
}

// box radius of the lattice-pruned association: (2r-1)^(m-1) points per row
static int default_lattice_r(int m) { return m <= 3 ? 6 : (m == 4 ? 3 : 1); }

static PrepArgs niche_prep_args(const mo_step_args* a, const Layout& L) {
  const int64_t R = 2 * a->n;
  void* ws = a->workspace;
  PrepArgs pa = prep_args(L, ws, a->FR, R, a->m, a->w, a->ranks, a->info, a->ideal, a->seed, a->generation, a->zhat,
                          nullptr, PREP_FULL);
  pa.gen_ptr = a->generation_dev;
  pa.in_step = 1;
  pa.fb_ctl = at<int>(ws, L.fctl);
  if (a->lattice_z && a->m >= 2 && a->m <= 5) {
    pa.lat_index = a->lattice_index;
    pa.lat_pos = a->lattice_pos;
  }
  return pa;
}

static int niche_phase(const mo_step_args* a, const Layout& L, uint32_t mask, cudaStream_t s) {
  const int64_t n = a->n, R = 2 * n, w = a->w;
  const int m = a->m;
  void* ws = a->workspace;
  PrepArgs pa = niche_prep_args(a, L);
  pa.pro_done = (mask & MO_PHASE_VARY) ? 1 : 0;
  pa.ideal_done = pa.pro_done;
  if (mask & MO_PHASE_NICHE_PREP) MO_TRY(launch_prep(pa, s));
  if (mask & MO_PHASE_NICHE_ASSOC) {
  const int G = shards_of(a->shard_count);
  AssocArgs aa;
  memset(&aa, 0, sizeof(aa));
  aa.F = a->FR;
  aa.ideal = a->ideal;
  aa.a32 = pa.a32;
  aa.zs = pa.zs;
  aa.cand = pa.cand;
  aa.ctl = pa.ctl;
  aa.info = a->info;
  aa.w = (int)w;
  aa.psplit = (int)w;
  aa.akey = pa.akey;
  aa.zbeg = (int)(w * a->shard_rank / G);
  aa.zend = (int)(w * (a->shard_rank + 1) / G);
  aa.lat_z = a->lattice_z;
  aa.lat_pos = a->lattice_pos;
  aa.lat_H = a->lattice_H;
  aa.lat_r = a->lattice_r > 0 ? a->lattice_r : default_lattice_r(m);
  aa.pos_ref = pa.pos_ref;
  aa.fb_cand = at<int>(ws, L.fcand);
  aa.fb_ctl = at<int>(ws, L.fctl);
  aa.in_step = 1;
  aa.zfrag = reinterpret_cast<const uint2*>(a->zhat_frag);
  aa.zsT = pa.zsT;
  aa.zumma = a->zhat_umma;
  aa.ref_Ho = a->ref_H_outer;
  aa.ref_Hi = a->ref_H_inner;
  if (a->lattice_z && m >= 2 && m <= 5)
    MO_TRY(launch_assoc_lattice(aa, m, R, s));
  else if (use_umma(aa, m))
    MO_TRY(launch_assoc_umma(aa, m, R, s));
  else if (use_hmma(aa, m))
    MO_TRY(launch_assoc_hmma(aa, m, R, s));
  else
    MO_TRY(launch_assoc(aa, m, R, s));
  }
  if (!(mask & MO_PHASE_NICHE_FINISH)) return MO_OK;
  AssocFinalArgs fa;
  memset(&fa, 0, sizeof(fa));
  fa.F = a->FR;
  fa.ideal = a->ideal;
  fa.a32 = pa.a32;
  fa.zs = pa.zs;
  fa.perm_ref = pa.perm_ref;
  fa.cand = pa.cand;
  fa.ctl = pa.ctl;
  fa.info = a->info;
  fa.m = m;
  fa.akey = pa.akey;
  fa.pi = at<int>(ws, L.pi);
  fa.d = at<float>(ws, L.d);
  fa.ranks = a->ranks;
  fa.rho = pa.rho;
  fa.rho_p = pa.rho_p;
  MO_TRY(launch_assoc_final(fa, R, s));
  SelectArgs sa = select_args(L, ws, R, w, n, a->ranks, a->info, fa.pi, fa.d, at<uint8_t>(ws, L.sel));
  sa.XR = a->XR;
  sa.FR = a->FR;
  sa.X_next = a->X_next;
  sa.F_next = a->F_next;
  sa.dvars = a->d;
  sa.m = m;
  sa.gen_ptr = a->generation_dev;
  sa.in_step = 1;
  sa.reset_ctl = pa.ctl;
  return launch_select(sa, s);
}

static int stream_presort(const mo_step_args* a, const Layout& L, cudaStream_t s);
static StreamArgs stream_args(const mo_step_args* a, const Layout& L);

static Layout step_layout(const mo_step_args* a) {
  return make_layout(2 * a->n, a->w, a->m, a->sort_mode, shards_of(a->shard_count));
}

static int run_phases(const mo_step_args* a, uint32_t mask, cudaStream_t s) {
  const int64_t n = a->n;
  PdlScope pdl;
  Layout L = step_layout(a);
  MO_TRY(check_ws(L, a->workspace, a->workspace_bytes));
  if (mask & MO_PHASE_NICHE) mask |= MO_PHASE_NICHE_PREP | MO_PHASE_NICHE_ASSOC | MO_PHASE_NICHE_FINISH;
  // the streamed sort runs device-side in one launch on one shard; sharded fronts are host-driven
  if ((mask & MO_PHASE_SORT) && a->sort_mode != MO_SORT_BITS && shards_of(a->shard_count) > 1) return MO_ERR_PARAM;
  if ((mask & (MO_PHASE_NICHE_ASSOC | MO_PHASE_NICHE_FINISH)) == (MO_PHASE_NICHE_ASSOC | MO_PHASE_NICHE_FINISH) &&
      shards_of(a->shard_count) > 1)
    return MO_ERR_PARAM;  // the akey max-reduction across shards sits between the two
  if (mask & MO_PHASE_VARY) {
    // the generation prologue (shuffles, niche-state reset) runs in extra CTAs of the variation kernel,
    // and the running ideal is lowered by the offspring there (min is idempotent: a later NICHE call
    // without VARY recomputes both, to the same values)
    PrepArgs pa = niche_prep_args(a, L);
    MO_TRY(launch_vary_eval(a->problem, a->XR, n, a->d, a->m, a->seed, a->generation, a->generation_dev, a->var,
                            a->XR + n * a->d, a->FR + n * a->m, a->ideal, nullptr, s, &pa));
  }
  if (mask & MO_PHASE_SORT) {
    if (a->sort_mode == MO_SORT_BITS) {
      MO_TRY(sort_phase(a, L, s));
    } else {
      MO_TRY(stream_presort(a, L, s));
      MO_TRY(launch_stream_fused(stream_args(a, L), s));
    }
  }
  if (mask & (MO_PHASE_NICHE_PREP | MO_PHASE_NICHE_ASSOC | MO_PHASE_NICHE_FINISH))
    MO_TRY(niche_phase(a, L, mask, s));
  return MO_OK;
}

// Boxed (Morton) position space for the streamed sort at m <= 10, S slabs above
// (boxes from a 30-bit Morton key: 3+ bits per coordinate up to m = 10; measured faster than the S slabs
// at every m <= 10 tried, profiles/r01_sort_modes.jsonl)
static int stream_boxed(int m) { return m <= 10 ? 1 : 0; }

static StreamArgs stream_args(const mo_step_args* a, const Layout& L) {
  void* ws = a->workspace;
  StreamArgs sa;
  memset(&sa, 0, sizeof(sa));
  sa.FS = at<float>(ws, L.FS);
  sa.SS = at<float>(ws, L.SS);
  sa.wend = at<int>(ws, L.wend);
  sa.blkmin = at<float>(ws, L.blkmin);
  sa.blkmax = at<float>(ws, L.blkmax);
  sa.perm = at<int>(ws, L.perm_sort);
  sa.R = (int)(2 * a->n);
  sa.m = a->m;
  sa.G = shards_of(a->shard_count);
  sa.g = a->shard_rank;
  sa.T = (int)L.T;
  sa.stop_at = a->n;
  sa.cnt = at<int>(ws, L.cnt);
  sa.rank_pos = at<int>(ws, L.rank_pos);
  sa.mask_local = at<uint32_t>(ws, L.mask_local);
  sa.mask_full = at<uint32_t>(ws, L.mask_full);
  sa.fl = at<int>(ws, L.fl);
  sa.flmax = at<float>(ws, L.flmax);
  sa.plan = at<int>(ws, L.plan);
  sa.ucnt = at<int>(ws, L.ucnt);
  sa.ctl = at<int>(ws, L.stctl);
  sa.info = a->info;
  sa.ranks = a->ranks;
  sa.gc.bar = at<unsigned>(ws, L.bar) + BAR_STREAM;
  sa.gc.part = at<int>(ws, L.part);
  sa.gc.hist = at<int>(ws, L.hist);
  sa.gc.parity = 0;
  sa.boxed = stream_boxed(a->m);
  sa.blkbox = at<float>(ws, L.blkbox);
  sa.flbox = at<float>(ws, L.flbox);
  sa.blkbox32 = at<float>(ws, L.blkbox32);
  sa.flbox32 = at<float>(ws, L.flbox32);
  sa.stats = at<unsigned long long>(ws, L.sstats);
  sa.blkS32 = at<float>(ws, L.blkS32);
  sa.flS32 = at<float>(ws, L.flS32);
  return sa;
}

// Position space of the streamed sort: Morton order + boxes (m <= 4) or S slabs.
static int stream_presort(const mo_step_args* a, const Layout& L, cudaStream_t s) {
  if (!stream_boxed(a->m)) return launch_presort(presort_args(a, L), s);
  void* ws = a->workspace;
  MortonArgs ma;
  ma.F = a->FR;
  ma.R = (int)(2 * a->n);
  ma.m = a->m;
  ma.keyA = at<uint32_t>(ws, L.keyA);
  ma.valA = at<int>(ws, L.valA);
  ma.tkey = at<uint32_t>(ws, L.tkey);
  ma.tval = at<int>(ws, L.tval);
  ma.cbox = at<unsigned>(ws, L.cbox);
  ma.perm = at<int>(ws, L.perm_sort);
  ma.FS = at<float>(ws, L.FS);
  ma.SS = at<float>(ws, L.SS);
  ma.blkmin = at<float>(ws, L.blkmin);
  ma.blkmax = at<float>(ws, L.blkmax);
  ma.blkbox = at<float>(ws, L.blkbox);
  ma.blkbox32 = at<float>(ws, L.blkbox32);
  ma.blkS32 = at<float>(ws, L.blkS32);
  ma.g.bar = at<unsigned>(ws, L.bar) + BAR_PRESORT;
  ma.g.part = at<int>(ws, L.part);
  ma.g.hist = at<int>(ws, L.hist);
  ma.g.parity = 0;
  return launch_presort_morton(ma, s);
}

static int check_stream(const mo_step_args* a, Layout& L) {
  if (a->sort_mode != MO_SORT_STREAM) return MO_ERR_PARAM;
  L = step_layout(a);
  return check_ws(L, a->workspace, a->workspace_bytes);
}

static int check_step_args(const mo_step_args* a) {
  if (a == nullptr) return MO_ERR_PARAM;
  if (a->n < 2 || (a->n & 1) || a->m < 2 || a->m > MO_MAX_M || a->d < a->m || a->w < 1) return MO_ERR_PARAM;
  if (a->m > 16 && a->sort_mode != MO_SORT_BITS) return MO_ERR_PARAM;   // streamed kernels: m <= 16
  if (2 * a->n > (int64_t)0x7fffffff || a->w > (int64_t)0x7fffffff) return MO_ERR_PARAM;
  if (!a->zhat || !a->XR || !a->FR || !a->X_next || !a->F_next || !a->ideal || !a->ranks || !a->info)
    return MO_ERR_PARAM;
  if (a->problem < MO_DTLZ1 || a->problem > MO_DTLZ7) return MO_ERR_PARAM;
  if (a->sort_mode != MO_SORT_BITS && a->sort_mode != MO_SORT_STREAM) return MO_ERR_PARAM;
  if (a->shard_count < 0 || a->shard_rank < 0 || a->shard_rank >= shards_of(a->shard_count)) return MO_ERR_PARAM;
  if (a->lattice_z && (a->lattice_H < 1 || a->lattice_r < 0 || !a->lattice_index || !a->lattice_pos))
    return MO_ERR_PARAM;
  return MO_OK;
}

}  // namespace mo

using namespace mo;

extern "C" {

size_t mo_pack_refs_f16_bytes(int64_t w, int32_t m) { return (w < 1 || m < 1 || m > 16) ? 0 : pack_refs_f16_bytes(w, m); }

int mo_pack_refs_f16(const float* zhat, int64_t w, int32_t m, const int32_t* order, void* out, void* stream_) {
  return launch_pack_refs_f16(zhat, w, m, order, out, (cudaStream_t)stream_);
}

size_t mo_pack_refs_bytes(int64_t w) { return w > 0 ? (size_t)((w + 7) / 8) * 544 : 0; }

int mo_pack_refs_bf16(const float* zhat, int64_t w, int32_t m, const int32_t* order, void* out, void* stream_) {
  if (!zhat || !out) return MO_ERR_PARAM;
  return launch_pack_refs(zhat, w, m, order, reinterpret_cast<uint2*>(out), (cudaStream_t)stream_);
}


const char* mo_version(void) { return "manyobj_b200 0.2.0 (sm_100a)"; }
size_t mo_step_args_bytes(void) { return sizeof(mo_step_args); }

int64_t mo_bits_words_per_row(int64_t R) { return words_per_row(R); }

int64_t mo_trace_offset(int64_t n, int32_t m, int64_t w) { return (int64_t)make_layout(2 * n, w, m).trace; }

int mo_workspace_bytes(int64_t n, int32_t m, int32_t d, int64_t w, size_t* bytes) {
  (void)d;
  if (!bytes || n < 1 || m < 1 || w < 1) return MO_ERR_PARAM;
  *bytes = make_layout(2 * n, w, m).total;
  return MO_OK;
}

int mo_workspace_bytes_rows(int64_t R, int32_t m, int64_t w, size_t* bytes) {
  if (!bytes || R < 1 || m < 1 || w < 0) return MO_ERR_PARAM;
  *bytes = make_layout(R, w > 0 ? w : 1, m, LAYOUT_OPS).total;
  return MO_OK;
}

int mo_permutation(int64_t n, uint64_t seed, uint32_t generation, uint32_t stream, int32_t* perm, int32_t* pos,
                   void* stream_) {
  if (n < 0 || n > (int64_t)0x7fffffff) return MO_ERR_PARAM;
  if (n == 0) return MO_OK;
  k_permutation<<<(unsigned)ceil_div(n, 256), 256, 0, (cudaStream_t)stream_>>>((int)n, seed, generation, stream,
                                                                             perm, pos);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

int mo_init_population(float* X, int64_t n, int32_t d, uint64_t seed, void* stream_) {
  return launch_init_population(X, n, d, seed, (cudaStream_t)stream_);
}

int mo_dtlz_eval(int32_t problem, const float* X, int64_t n, int32_t d, int32_t m, float* F, int32_t* domain_flag,
                 void* stream_) {
  return launch_dtlz_eval(problem, X, n, d, m, F, domain_flag, (cudaStream_t)stream_);
}

int mo_vary_eval(int32_t problem, const float* X, int64_t n, int32_t d, int32_t m, uint64_t seed, uint32_t generation,
                 const mo_var_cfg* cfg, float* Xo, float* Fo, float* ideal, void* stream_) {
  if (!cfg) return MO_ERR_PARAM;
  return launch_vary_eval(problem, X, n, d, m, seed, generation, nullptr, *cfg, Xo, Fo, ideal, nullptr,
                          (cudaStream_t)stream_);
}

int mo_dominance_bits(const float* F, int64_t R, int32_t m, const uint8_t* valid, uint32_t* bits, void* stream_) {
  return launch_dom_tile(F, R, m, valid, bits, (cudaStream_t)stream_);
}

int mo_presort(const float* F, int64_t R, int32_t m, int32_t* perm, float* FS, float* SS, int32_t* wend,
               float* blkmin, float* blkmax, void* workspace, size_t workspace_bytes, void* stream_) {
  if (R < 1 || m < 1 || !F || !perm || !FS || !SS || !wend || !blkmin || !blkmax) return MO_ERR_PARAM;
  Layout L = make_layout(R, 1, m, LAYOUT_OPS);
  MO_TRY(check_ws(L, workspace, workspace_bytes));
  PresortArgs ps;
  ps.F = F;
  ps.R = (int)R;
  ps.m = m;
  ps.keyA = at<uint32_t>(workspace, L.keyA);
  ps.valA = at<int>(workspace, L.valA);
  ps.keyB = at<uint32_t>(workspace, L.keyB);
  ps.valB = at<int>(workspace, L.pcnt);
  ps.fill = at<int>(workspace, L.pfill);
  ps.blkmin = blkmin;
  ps.blkmax = blkmax;
  ps.ctl = at<unsigned>(workspace, L.pctl);
  ps.perm = perm;
  ps.FS = FS;
  ps.SS = SS;
  ps.wend = wend;
  ps.g.bar = at<unsigned>(workspace, L.bar) + BAR_PRESORT;
  ps.g.part = at<int>(workspace, L.part);
  ps.g.hist = at<int>(workspace, L.hist);
  ps.g.parity = 0;
  ps.trace = nullptr;
  ps.stable = 0;
  ps.tkey = nullptr;
  ps.tval = nullptr;
  ps.in_step = 0;
  ps.hasdom = nullptr;
  return launch_presort(ps, (cudaStream_t)stream_);
}

int mo_dominance_bits_sorted(const float* FS, const float* blkmin, const float* blkmax, const int32_t* wend,
                             int64_t R, int32_t m, uint32_t* bits, uint8_t* hasdom, void* stream_) {
  if (!FS || !blkmin || !blkmax || !wend || !bits || !hasdom) return MO_ERR_PARAM;
  return launch_dom_tile_sorted(FS, blkmin, blkmax, wend, R, m, bits, hasdom, (cudaStream_t)stream_);
}

size_t mo_dominance_tables_bytes(int64_t R, int32_t m) {
  return (R < 1 || m < 2 || m > MO_MAX_M) ? 0 : dom_rank_tables_bytes(R, m);
}

int64_t mo_tile_summary_words(int64_t R) { return R < 1 ? 0 : tsum_words(R); }

int mo_dominance_bits_ranked(const float* FS, const float* blkmin, const float* blkmax, const int32_t* wend,
                             int64_t R, int32_t m, uint32_t* bits, uint8_t* hasdom, void* tables,
                             size_t tables_bytes, uint32_t* tsum, void* stream_) {
  if (!FS || !blkmin || !blkmax || !wend || !bits || !hasdom || !tables || m < 2 || m > MO_MAX_M) return MO_ERR_PARAM;
  if (tables_bytes < dom_rank_tables_bytes(R, m)) return MO_ERR_PARAM;
  cudaStream_t s = (cudaStream_t)stream_;
  if (cudaMemsetAsync(hasdom, 0, (size_t)R, s) != cudaSuccess) return MO_ERR_CUDA;
  return launch_dom_rank(FS, blkmin, blkmax, wend, R, m, bits, hasdom, static_cast<uint32_t*>(tables), s, tsum);
}

int mo_front_peel(const uint32_t* bits, int64_t R, const uint8_t* valid, int64_t stop_at, int32_t* ranks,
                  int32_t* info, void* workspace, size_t workspace_bytes, void* stream_) {
  Layout L = make_layout(R, 1, 1, LAYOUT_OPS);
  MO_TRY(check_ws(L, workspace, workspace_bytes));
  return launch_front_peel(bits, R, valid, stop_at, ranks, info, at<int>(workspace, L.resume),
                           at<uint32_t>(workspace, L.ranked), at<int>(workspace, L.fsizes),
                           at<unsigned>(workspace, L.bar) + BAR_PEEL, nullptr, nullptr, nullptr, nullptr,
                           nullptr, (cudaStream_t)stream_);
}

int mo_normalize(const float* F, int64_t R, int32_t m, const int32_t* ranks, const int32_t* info, uint64_t seed,
                 uint32_t generation, float* ideal, float* Fn, double* intercepts, void* workspace,
                 size_t workspace_bytes, void* stream_) {
  if (m < 1 || m > MO_MAX_M || R < 1) return MO_ERR_PARAM;
  Layout L = make_layout(R, 1, m, LAYOUT_OPS);
  MO_TRY(check_ws(L, workspace, workspace_bytes));
  cudaStream_t s = (cudaStream_t)stream_;
  // w = 1 dummy reference point set: only the row shuffle matters here
  // w = 1 and no reference set: only the row shuffle (extreme-point ties) matters here
  PrepArgs pa = prep_args(L, workspace, F, R, m, 1, ranks, const_cast<int*>(info), ideal, seed, generation,
                          nullptr, intercepts, PREP_FULL);
  MO_TRY(launch_prep(pa, s));
  if (Fn) {
    AssocFinalArgs fa;
    memset(&fa, 0, sizeof(fa));
    fa.F = F;
    fa.ideal = ideal;
    fa.a32 = pa.a32;
    fa.cand = pa.cand;
    fa.ctl = pa.ctl;
    fa.info = info;
    fa.m = m;
    fa.Fn_out = Fn;
    fa.fn_only = 1;
    MO_TRY(launch_assoc_final(fa, R, s));
  }
  return MO_OK;
}

int mo_associate(const float* Fn, int64_t R, int32_t m, const float* zhat, int64_t w, const int32_t* ranks,
                 const int32_t* info, uint64_t seed, uint32_t generation, int32_t* pi, float* d, void* workspace,
                 size_t workspace_bytes, void* stream_) {
  if (m < 1 || m > MO_MAX_M || R < 1 || w < 1) return MO_ERR_PARAM;
  Layout L = make_layout(R, w, m, LAYOUT_OPS);
  MO_TRY(check_ws(L, workspace, workspace_bytes));
  cudaStream_t s = (cudaStream_t)stream_;
  PrepArgs pa = prep_args(L, workspace, Fn, R, m, w, ranks, const_cast<int*>(info), nullptr, seed, generation, zhat,
                          nullptr, PREP_PERMS_CAND);
  MO_TRY(launch_prep(pa, s));
  AssocArgs aa;
  memset(&aa, 0, sizeof(aa));
  aa.F = Fn;
  aa.ideal = nullptr;
  aa.a32 = nullptr;
  aa.zs = pa.zs;
  aa.cand = pa.cand;
  aa.ctl = pa.ctl;
  aa.info = info;
  aa.w = (int)w;
  aa.psplit = (int)w;
  aa.akey = pa.akey;
  aa.zbeg = 0;
  aa.zend = (int)w;
  aa.lat_z = nullptr;
  aa.in_step = 0;
  aa.zsT = pa.zsT;
  MO_TRY(launch_assoc(aa, m, R, s));
  AssocFinalArgs fa;
  memset(&fa, 0, sizeof(fa));
  fa.F = Fn;
  fa.zs = pa.zs;
  fa.perm_ref = pa.perm_ref;
  fa.cand = pa.cand;
  fa.ctl = pa.ctl;
  fa.info = info;
  fa.m = m;
  fa.akey = pa.akey;
  fa.pi = pi;
  fa.d = d;
  return launch_assoc_final(fa, R, s);
}

int mo_niche_select(const int32_t* pi, const float* d, int64_t R, int64_t w, int64_t n, int32_t* ranks,
                    int32_t* info, uint64_t seed, uint32_t generation, uint8_t* selected, void* workspace,
                    size_t workspace_bytes, void* stream_) {
  if (R < 1 || w < 1 || n < 1) return MO_ERR_PARAM;
  Layout L = make_layout(R, w, 1, LAYOUT_OPS);
  MO_TRY(check_ws(L, workspace, workspace_bytes));
  cudaStream_t s = (cudaStream_t)stream_;
  // shuffles only (rows and reference points)
  PrepArgs pa = prep_args(L, workspace, nullptr, R, 1, w, ranks, info, nullptr, seed, generation, nullptr, nullptr,
                          PREP_PERMS);
  MO_TRY(launch_prep(pa, s));
  SelectArgs sa = select_args(L, workspace, R, w, n, ranks, info, pi, d, selected);
  sa.count_inside = 1;
  return launch_select(sa, s);
}

int mo_select(const mo_step_args* args, void* stream_) {
  MO_TRY(check_step_args(args));
  return run_phases(args, MO_PHASE_SORT | MO_PHASE_NICHE, (cudaStream_t)stream_);
}

int mo_step(const mo_step_args* a, void* stream_) {
  MO_TRY(check_step_args(a));
  return run_phases(a, MO_PHASE_ALL, (cudaStream_t)stream_);
}

int mo_step_phases(const mo_step_args* a, uint32_t phase_mask, void* stream_) {
  MO_TRY(check_step_args(a));
  if (phase_mask == 0 || (phase_mask & ~(uint32_t)MO_PHASE_ALL)) return MO_ERR_PARAM;
  return run_phases(a, phase_mask, (cudaStream_t)stream_);
}

int mo_niche_phases(const mo_step_args* a, uint32_t phase_mask, void* stream_) {
  MO_TRY(check_step_args(a));
  const uint32_t all = MO_PHASE_NICHE_PREP | MO_PHASE_NICHE_ASSOC | MO_PHASE_NICHE_FINISH;
  if (phase_mask == 0 || (phase_mask & ~all)) return MO_ERR_PARAM;
  return run_phases(a, phase_mask, (cudaStream_t)stream_);
}

int mo_sort_stream_begin(const mo_step_args* a, void* stream_) {
  MO_TRY(check_step_args(a));
  Layout L;
  MO_TRY(check_stream(a, L));
  cudaStream_t s = (cudaStream_t)stream_;
  MO_TRY(stream_presort(a, L, s));
  return launch_stream_begin(stream_args(a, L), s);
}

int mo_sort_stream_front(const mo_step_args* a, int32_t k, void* stream_) {
  MO_TRY(check_step_args(a));
  Layout L;
  MO_TRY(check_stream(a, L));
  if (k < 0) return MO_ERR_PARAM;
  return launch_stream_front(stream_args(a, L), k, (cudaStream_t)stream_);
}

int mo_sort_stream_end(const mo_step_args* a, void* stream_) {
  MO_TRY(check_step_args(a));
  Layout L;
  MO_TRY(check_stream(a, L));
  return launch_stream_end(stream_args(a, L), (cudaStream_t)stream_);
}

int mo_workspace_init(void* workspace, size_t workspace_bytes, void* stream_) {
  if (!workspace) return MO_ERR_PARAM;
  return cudaMemsetAsync(workspace, 0, workspace_bytes, (cudaStream_t)stream_) == cudaSuccess ? MO_OK : MO_ERR_CUDA;
}

int mo_workspace_bytes_ex(int64_t n, int32_t m, int32_t d, int64_t w, int32_t sort_mode, int32_t shard_count,
                          size_t* bytes) {
  (void)d;
  if (!bytes || n < 1 || m < 1 || w < 1 || shard_count < 0) return MO_ERR_PARAM;
  if (sort_mode != MO_SORT_BITS && sort_mode != MO_SORT_STREAM) return MO_ERR_PARAM;
  *bytes = make_layout(2 * n, w, m, sort_mode, shards_of(shard_count)).total;
  return MO_OK;
}

int mo_stream_stats_offset(int64_t n, int32_t m, int64_t w, int32_t sort_mode, int32_t shard_count,
                           int64_t* stats_off) {
  if (n < 1 || m < 1 || w < 1 || shard_count < 0 || !stats_off) return MO_ERR_PARAM;
  *stats_off = (int64_t)make_layout(2 * n, w, m, sort_mode, shards_of(shard_count)).sstats;
  return MO_OK;
}

int mo_stream_offsets(int64_t n, int32_t m, int64_t w, int32_t sort_mode, int32_t shard_count,
                      int64_t* mask_local_off, int64_t* mask_local_words, int64_t* mask_full_off, int64_t* akey_off) {
  if (n < 1 || m < 1 || w < 1 || shard_count < 0) return MO_ERR_PARAM;
  Layout L = make_layout(2 * n, w, m, sort_mode, shards_of(shard_count));
  if (mask_local_off) *mask_local_off = (int64_t)L.mask_local;
  if (mask_local_words) *mask_local_words = L.mask_local_words;
  if (mask_full_off) *mask_full_off = (int64_t)L.mask_full;
  if (akey_off) *akey_off = (int64_t)L.akey;
  return MO_OK;
}

// byte offsets of the niche-selection state a step leaves in its workspace (debug bookkeeping check /
// niche trace): [0] pi (int32 R), [1] d (f32 R), [2] rho, [3] rho_p, [4] take,
// [5] kept (int32 w+1 each), [6] prom (u8 R), [7] pos_pop, [8] perm_pop (int32 R), [9] pos_ref,
// [10] perm_ref (int32 w)
int mo_niche_offsets(int64_t n, int32_t m, int64_t w, int32_t sort_mode, int32_t shard_count, int64_t* out11) {
  if (n < 1 || m < 1 || w < 1 || shard_count < 0 || !out11) return MO_ERR_PARAM;
  Layout L = make_layout(2 * n, w, m, sort_mode, shards_of(shard_count));
  const size_t v[11] = {L.pi, L.d, L.rho, L.rho_p, L.take, L.kept, L.prom, L.pos_pop, L.perm_pop, L.pos_ref,
                        L.perm_ref};
  for (int i = 0; i < 11; ++i) out11[i] = (int64_t)v[i];
  return MO_OK;
}

}  // extern "C"
