// dcopf_dual.cu -- host side of the C ABI declared in include/dcopf_dual.h.
//
// create():  validate + copy the network (SPEC.md:30-50 rules), the angle box
//            (given, or implied by the flow limits), internal numbering
//            (schedule.cpp: DFS tree bus order, branches by larger endpoint,
//            CSR in ascending original branch id, generators per bus).
// set_instance_batch():  choose the path and, for the batched path, the tile
//            width W (instances per CTA, so that #tiles ~ #SMs) and compile
//            the sweep schedule for it; loads -> tile-major device state.
// iterate(): batched: ONE launch of k_sweep running all K iterations and the
//            final evaluation; single: ONE launch of k_single.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <queue>
#include <string>
#include <vector>

#include "../../include/dcopf_dual.h"
#include "cluster.h"
#include "cluster_kernel.cuh"
#include "dual_kernels.cuh"
#include "ptdf.h"
#include "schedule.h"
#include "sweep_kernel.cuh"

using namespace dcopf;

static thread_local std::string g_create_error;

// consumer warps of k_sweep (+1 producer warp): 2 instances per lane 19 (640
// threads, 96 registers), 4 per lane 15 (512 threads, 128 registers)
#ifndef DCOPF_SWEEP_WARPS2
#define DCOPF_SWEEP_WARPS2 19
#endif
constexpr int kSweepWarps2 = DCOPF_SWEEP_WARPS2;
#ifndef DCOPF_SWEEP_WARPS4
#define DCOPF_SWEEP_WARPS4 15
#endif
constexpr int kSweepWarps4 = DCOPF_SWEEP_WARPS4;
// (the optimiser variants spill a little at 96 registers with 19 warps, and
// are still faster than with 15 warps at 128 registers: 2.9e6 vs 3.1e6
// inst-it/s for KVL + Adam on config 4b -- latency hiding wins)
inline int sweep_warps(int V, bool /*opt*/) { return V == 4 ? kSweepWarps4 : kSweepWarps2; }

struct dcopf_dual_s {
  std::string err;
  int device = 0, form = 0, path_opt = 0, single_max = 56, n_sm = 148, dev_smem = 0;
  int opt_parts = 0, opt_lane = 0;
  bool implied_box = false;
  int force_cluster_C = 0;          // configure_cluster: only this cluster size (0: the smallest that fits)         // theta_max was NULL: the library computed the angle box  // dcopf_options tile_parts / lane_instances (0 = chosen per batch)
  int n_bus = 0, n_br = 0, n_gen = 0, ref_int = 0, quadratic = 0, bandwidth = 0;
  std::vector<int> bus_perm, bus_inv, br_perm, br_inv;  // perm: internal -> original
  std::vector<uint8_t> switchable;                      // original ids; empty = all
  NetInternal ni;                                       // internal network (schedule input)
  // device topology (single path)
  int *d_bus_ptr = nullptr, *d_bus_inc = nullptr, *d_gen_ptr = nullptr, *d_br_s = nullptr,
      *d_br_t = nullptr, *d_bus_perm = nullptr, *d_bus_inv = nullptr, *d_br_perm = nullptr,
      *d_br_inv = nullptr;
  double *d_theta = nullptr, *d_gen_c = nullptr, *d_gen_lo = nullptr, *d_gen_hi = nullptr,
         *d_gen_a = nullptr, *d_br_b = nullptr, *d_br_F = nullptr;
  // batch state
  long B = 0, B_pad = 0;
  int T = 1, path = 0, max_out = 0, cur = 0, single_smem = 0, smem_single = 0;
  double *lam[2] = {nullptr, nullptr}, *br[2] = {nullptr, nullptr}, *load = nullptr;
  double *bound = nullptr, *best = nullptr, *value = nullptr;
  int *status = nullptr, *outs = nullptr, *flag = nullptr;
  double *target = nullptr;                           // time-to-gap thresholds [B_pad]
  long long *hit = nullptr;                           // first evaluation index reaching them [B_pad]
  bool has_target = false;
  double tol = 0.0;                                   // stopping rule (set_stop)
  long k_base = 0;                                    // steps taken since set_instance_batch
  double *g_lam = nullptr, *g_br = nullptr;  // evaluate scratch (internal layout)
  double *scratch = nullptr;
  size_t scratch_bytes = 0;
  double *alpha_dev = nullptr, *alpha_pin = nullptr;  // schedule alpha[K]: device + pinned staging
  size_t alpha_cap = 0;
  cudaEvent_t alpha_ev = nullptr;                     // staging reusable once this fired
  // compiled sweep schedule of the batched path (for tile width sched_W,
  // sched_V instances per lane, sched_C parts per tile)
  Schedule sch;
  int sched_W = 0, sched_V = 0, sched_C = 0, sched_nw = 0;
  bool sched_opt = false;  // compiled with the optimiser kernels' shared-memory block
  // the last tiling choice (choose_tiles compiles candidate schedules: ~0.1 s
  // per candidate on the host): reused while the batch size and the variant
  // (warp count, shared-memory block) are unchanged
  int64_t tc_B = -1;
  int tc_opt = -1, tc_V = 0, tc_W = 0, tc_C = 0;
  int tile_V = 2, tile_C = 1;  // loaded batch: instances per lane, parts (CTAs) per tile
  uint8_t *d_prog = nullptr;
  int *d_part_step0 = nullptr;
  std::vector<int> hpos_lam, hpos_d, hpos_br;  // batched layout: storage row of each original entity (host)
  unsigned *d_tile_sync = nullptr;  // split tiles: per-tile arrival counters
  double *d_part_val = nullptr;     // split tiles: per-part partial dual values [2][tiles][C][W]
  size_t tile_sync_cap = 0, part_val_cap = 0;
  long long *d_prog_off = nullptr;
  int *d_prog_bytes = nullptr, *d_tx_bytes = nullptr, *d_ld_ptr = nullptr, *d_ld = nullptr;
  // batched path state layout: storage position <-> original id, per kind
  // ascent-step variant (set_optimizer) and its persistent state (cluster path)
  dcopf_optimizer opt = {DCOPF_OPT_PLAIN, 0, 0.0, 0.0, 0.0, 0.0};
  double *os[4] = {nullptr, nullptr, nullptr, nullptr};  // s1_lam, s2_lam, s1_br, s2_br
  double b1t = 1.0, b2t = 1.0;                            // beta^t after the steps taken so far
  // branch-block multipliers: entities x components (F2: n_br x 1, F1: n_br x 2, KVL: cycles x 1)
  int n_bm_ent = 0, bm_C = 1;
  CycleBasis cyc_orig, cyc_int;                 // KVL: canonical cycle basis (original / internal branch ids)
  int *d_cyc_perm = nullptr, *d_cyc_inv = nullptr;  // KVL: internal cycle order <-> canonical k
  // cluster path: per-rank plan blobs
  ClusterPlan cplan;
  int cplan_C = 0;
  uint8_t *d_cblob = nullptr;
  int *d_lam_perm_b = nullptr, *d_lam_inv_b = nullptr, *d_d_perm_b = nullptr, *d_br_perm_b = nullptr,
      *d_br_inv_b = nullptr, *d_br_pos_b = nullptr;
  // dense-PTDF form (DCOPF_FORM_PTDF): all of its state; the fields above stay unused
  PtdfState *pt = nullptr;
};

namespace {

int fail(dcopf_dual_t h, int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h) h->err = buf;
  else g_create_error = buf;
  return code;
}

#define CK(h, call)                                                                         \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail(h, e_ == cudaErrorMemoryAllocation ? DCOPF_ENOMEM : DCOPF_ECUDA,          \
                  "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

inline int brw(int form) { return form == DCOPF_FORM_LIMIT_ROWS ? 2 : 1; }

template <typename T>
int upload(dcopf_dual_t h, T **dst, const std::vector<T> &src) {
  cudaFree(*dst);
  *dst = nullptr;
  const size_t n = std::max<size_t>(src.size(), 1);
  CK(h, cudaMalloc(dst, n * sizeof(T)));
  if (!src.empty()) CK(h, cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
  return DCOPF_OK;
}

bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

int grid_for(size_t n) {
  const size_t g = (n + 255) / 256;
  return (int)std::min<size_t>(std::max<size_t>(g, 1), 148 * 32);
}

bool connected(int n, const std::vector<int> &fr, const std::vector<int> &to, const std::vector<char> &use) {
  std::vector<std::vector<int>> adj(n);
  for (size_t l = 0; l < fr.size(); ++l)
    if (use[l]) {
      adj[fr[l]].push_back(to[l]);
      adj[to[l]].push_back(fr[l]);
    }
  std::vector<char> seen(n, 0);
  std::vector<int> st{0};
  seen[0] = 1;
  int cnt = 1;
  while (!st.empty()) {
    const int v = st.back();
    st.pop_back();
    for (int u : adj[v])
      if (!seen[u]) {
        seen[u] = 1;
        ++cnt;
        st.push_back(u);
      }
  }
  return cnt == n;
}

int ensure_scratch(dcopf_dual_t h, size_t bytes) {
  if (h->scratch_bytes >= bytes) return DCOPF_OK;
  cudaFree(h->scratch);
  h->scratch = nullptr;
  h->scratch_bytes = 0;
  CK(h, cudaMalloc(&h->scratch, bytes));
  h->scratch_bytes = bytes;
  return DCOPF_OK;
}

void free_batch(dcopf_dual_t h) {
  for (int i = 0; i < 2; ++i) {
    cudaFree(h->lam[i]);
    cudaFree(h->br[i]);
    h->lam[i] = h->br[i] = nullptr;
  }
  double **dp[] = {&h->load, &h->bound, &h->best, &h->value, &h->g_lam, &h->g_br, &h->os[0], &h->os[1], &h->os[2],
                   &h->os[3]};
  for (double **p : dp) {
    cudaFree(*p);
    *p = nullptr;
  }
  cudaFree(h->status);
  cudaFree(h->outs);
  h->status = h->outs = nullptr;
  cudaFree(h->target);
  cudaFree(h->hit);
  h->target = nullptr;
  h->hit = nullptr;
  h->B = h->B_pad = 0;
}

DevNet dev_net(dcopf_dual_t h) {
  DevNet n;
  n.n_bus = h->n_bus;
  n.n_br = h->n_br;
  n.n_gen = h->n_gen;
  n.ref = h->ref_int;
  n.bus_ptr = h->d_bus_ptr;
  n.bus_inc = h->d_bus_inc;
  n.theta = h->d_theta;
  n.gen_ptr = h->d_gen_ptr;
  n.gen_c = h->d_gen_c;
  n.gen_lo = h->d_gen_lo;
  n.gen_hi = h->d_gen_hi;
  n.gen_a = h->d_gen_a;
  n.br_s = h->d_br_s;
  n.br_t = h->d_br_t;
  n.br_b = h->d_br_b;
  n.br_F = h->d_br_F;
  return n;
}

// external [C][n_ent][B] (host or device) -> internal tile-major [tile][n_ent][C][T]
int import_ext(dcopf_dual_t h, const double *ext, double *intl, const int *perm, int n_ent, int C, cudaStream_t s) {
  const double *src = ext;
  const size_t bytes = (size_t)C * n_ent * h->B * sizeof(double);
  if (ext && !is_device_ptr(ext)) {
    int rc = ensure_scratch(h, bytes);
    if (rc) return rc;
    CK(h, cudaMemcpyAsync(h->scratch, ext, bytes, cudaMemcpyDefault, s));
    src = h->scratch;
  }
  const size_t total = (size_t)h->B_pad * n_ent * C;
  k_to_internal<<<grid_for(total), 256, 0, s>>>(src, intl, perm, n_ent, C, h->B, h->B_pad, h->T);
  CK(h, cudaGetLastError());
  return DCOPF_OK;
}

int export_ext(dcopf_dual_t h, const double *intl, double *ext, const int *inv, int n_ent, int C, cudaStream_t s) {
  if (!ext) return DCOPF_OK;
  const size_t bytes = (size_t)C * n_ent * h->B * sizeof(double);
  const bool dev = is_device_ptr(ext);
  double *dst = ext;
  if (!dev) {
    int rc = ensure_scratch(h, bytes);
    if (rc) return rc;
    dst = h->scratch;
  }
  const size_t total = (size_t)C * n_ent * h->B;
  k_to_external<<<grid_for(total), 256, 0, s>>>(intl, dst, inv, n_ent, C, h->B, h->T);
  CK(h, cudaGetLastError());
  if (!dev) {
    CK(h, cudaMemcpyAsync(ext, dst, bytes, cudaMemcpyDefault, s));
    CK(h, cudaStreamSynchronize(s));
  }
  return DCOPF_OK;
}

template <typename T>
int copy_out(dcopf_dual_t h, T *dst, const T *src, cudaStream_t s) {
  if (!dst) return DCOPF_OK;
  CK(h, cudaMemcpyAsync(dst, src, h->B * sizeof(T), cudaMemcpyDefault, s));
  if (!is_device_ptr(dst)) CK(h, cudaStreamSynchronize(s));
  return DCOPF_OK;
}

size_t single_smem(int n_bus, int n_br, int form, bool state) {
  const size_t codes = (size_t)n_bus + n_br;
  const size_t st = state ? (size_t)8 * (n_bus + (size_t)n_br * brw(form)) : 0;
  return 512 + st + ((codes + 15) & ~(size_t)15);
}

// copy alpha[K] to the device through pinned staging (reused only after the
// previous copy has executed)
int stage_alpha(dcopf_dual_t h, int64_t K, const double *alpha, cudaStream_t s) {
  if (!h->alpha_ev) CK(h, cudaEventCreateWithFlags(&h->alpha_ev, cudaEventDisableTiming));
  CK(h, cudaEventSynchronize(h->alpha_ev));
  if ((size_t)K > h->alpha_cap || !h->alpha_dev) {
    // capacity grows geometrically from 64 Ki steps, so a run never allocates
    // (a synchronising call) once its longest schedule has been seen
    size_t cap = std::max<size_t>(65536, h->alpha_cap);
    while (cap < (size_t)K) cap *= 2;
    cudaFree(h->alpha_dev);
    cudaFreeHost(h->alpha_pin);
    h->alpha_dev = h->alpha_pin = nullptr;
    h->alpha_cap = 0;
    CK(h, cudaMalloc(&h->alpha_dev, cap * 8));
    CK(h, cudaMallocHost(&h->alpha_pin, cap * 8));
    h->alpha_cap = cap;
  }
  if (K > 0) {
    memcpy(h->alpha_pin, alpha, K * 8);
    CK(h, cudaMemcpyAsync(h->alpha_dev, h->alpha_pin, K * 8, cudaMemcpyHostToDevice, s));
    CK(h, cudaEventRecord(h->alpha_ev, s));
  }
  return DCOPF_OK;
}

template <typename F>
int set_smem(dcopf_dual_t h, F fn, int bytes) {
  CK(h, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  return DCOPF_OK;
}

// The schedule search for tiles of W instances, V per lane, swept by C parts:
// the largest candidate chunk (48 .. 1 buses) whose kernel shared memory
// fits, at the longest ring life that fits (ch / life > 0: only that one).
// quick (tile choice estimates): a chunk that does not fit at the shortest
// ring life is not tried at the others (shared memory usually grows with the
// ring life).  Returns false (err empty) when nothing fits; err set on a
// compiler error.
bool search_schedule(dcopf_dual_t h, int W, int V, int C, int only_ch, int only_life, Schedule *out,
                     std::string *err, bool quick = false) {
  const int nw = sweep_warps(V, h->opt.variant != DCOPF_OPT_PLAIN);
  const bool optv = h->opt.variant != DCOPF_OPT_PLAIN;
  // program-block stages in flight: 2, except KVL, whose steps are shorter and
  // whose shared memory is better spent on larger chunks (measured on config 4:
  // KVL 1.17e7 at P = 2 / 36-row chunks, 1.21e7 at P = 1 / 48; F2 and F1 best at 2)
#ifndef DCOPF_PREFETCH_F2
#define DCOPF_PREFETCH_F2 2
#endif
#ifndef DCOPF_PREFETCH_KVL
#define DCOPF_PREFETCH_KVL 1
#endif
  const int P = (h->form == DCOPF_FORM_CYCLE) ? DCOPF_PREFETCH_KVL : (h->form == DCOPF_FORM_FLOW_BOX ? DCOPF_PREFETCH_F2 : 2);
  const int chs[] = {48, 40, 36, 34, 32, 30, 28, 26, 24, 22, 20, 18, 16, 14, 12, 10, 8, 6, 4, 2, 1},
            lifes[] = {2, 6, 4};
  const CycleBasis *cy = h->form == DCOPF_FORM_CYCLE ? &h->cyc_int : nullptr;
  err->clear();
  for (int ch : chs) {
    if (only_ch && ch != only_ch) continue;
    Schedule best;
    bool fit = false;
    for (int life : lifes) {  // life 2 first: the smallest footprint of this chunk
      if (only_life && life != only_life) continue;
      Schedule sc;
      sc.ring_life = life;
      sc.pool_gap = 3;  // soft step sync: consumer warps drift by up to two steps
      // optimiser kernels: the tile's state-row byte offsets (16 B) and each
      // consumer warp's step constants (64 B) live in shared memory, not in
      // registers across the step loop (sweep_kernel.cuh)
      sc.opt_bytes = optv ? 16 + 64 * nw : 0;
      *err = build_schedule_split(h->ni, ch, P, W, V, nw, C, {}, &sc, cy);
      if (!err->empty()) return false;
      if (sc.total > h->dev_smem) {
        if (quick && life == 2 && !only_life) break;
        continue;
      }
      if (!fit || life > best.ring_life) best = std::move(sc);
      fit = true;
    }
    if (fit) {
      *out = std::move(best);
      return true;
    }
  }
  return false;
}

// Compile + upload the sweep schedule for tiles of W instances, V per lane,
// swept by C parts: the chunk starts at the largest of the candidate chunks
// (48 .. 1 buses) and ring lives whose kernel shared memory fits; the
// split-tile compiler (split_schedule.cpp; C = 1 is the unsplit sweep).
int compile_schedule(dcopf_dual_t h, int W, int V, int C) {
  const int nw = sweep_warps(V, h->opt.variant != DCOPF_OPT_PLAIN);
  const bool optv = h->opt.variant != DCOPF_OPT_PLAIN;
  if (h->sched_W == W && h->sched_V == V && h->sched_C == C && h->sched_nw == nw && h->sched_opt == optv)
    return DCOPF_OK;
  // the same tiling for another warp count (an optimiser variant switched on
  // or off with a batch loaded): keep the chunk and ring life, so the storage
  // order of the loaded state -- which depends only on them -- stays valid
  const bool keep_layout = h->sched_W == W && h->sched_V == V && h->sched_C == C && h->B > 0;
  const int keep_ch = h->sch.CH, keep_life = h->sch.ring_life;
  Schedule sc;
  std::string err;
  const bool ok = search_schedule(h, W, V, C, keep_layout ? keep_ch : 0, keep_layout ? keep_life : 0, &sc, &err);
  if (!err.empty()) return fail(h, DCOPF_EINVAL, "schedule: %s", err.c_str());
  if (!ok) return fail(h, DCOPF_EINVAL, "batched schedule does not fit shared memory; use the single path");
  h->sched_W = h->sched_V = h->sched_C = h->sched_nw = 0;  // (invalid until every upload succeeded)
  h->sch = sc;
  int rc = upload(h, &h->d_prog, h->sch.prog);
  if (!rc) rc = upload(h, &h->d_prog_off, h->sch.prog_off);
  if (!rc) rc = upload(h, &h->d_prog_bytes, h->sch.prog_bytes);
  if (!rc) rc = upload(h, &h->d_tx_bytes, h->sch.tx_bytes);
  if (!rc) rc = upload(h, &h->d_ld_ptr, h->sch.ld_ptr);
  if (!rc) rc = upload(h, &h->d_part_step0, h->sch.part_step0);
  if (!rc) {
    std::vector<int> ld(4 * h->sch.ld.size());
    for (size_t x = 0; x < h->sch.ld.size(); ++x) {
      ld[4 * x] = h->sch.ld[x].a;
      ld[4 * x + 1] = h->sch.ld[x].b;
      ld[4 * x + 2] = h->sch.ld[x].c;
      ld[4 * x + 3] = h->sch.ld[x].d;
    }
    rc = upload(h, &h->d_ld, ld);
  }
  // storage order of the batched state (per kind) in terms of original ids
  if (!rc) {
    const int nb = h->n_bus, nl = h->n_bm_ent;  // branch-block rows: branches, or cycles (KVL)
    std::vector<int> lam_perm(nb), lam_inv(nb), d_perm(nb), br_perm(nl), br_inv(nl);
    for (int p = 0; p < nb; ++p) {
      lam_perm[p] = h->bus_perm[h->sch.perm_lam[p]];
      lam_inv[lam_perm[p]] = p;
      d_perm[p] = h->bus_perm[h->sch.perm_d[p]];
    }
    for (int p = 0; p < nl; ++p) {
      // KVL: the storage order lists canonical cycle indices directly
      br_perm[p] = (h->form == DCOPF_FORM_CYCLE) ? h->sch.perm_br[p] : h->br_perm[h->sch.perm_br[p]];
      br_inv[br_perm[p]] = p;
    }
    h->hpos_lam = lam_inv;
    h->hpos_d.assign(nb, 0);
    for (int p = 0; p < nb; ++p) h->hpos_d[d_perm[p]] = p;
    h->hpos_br = br_inv;
    if (!rc) rc = upload(h, &h->d_lam_perm_b, lam_perm);
    if (!rc) rc = upload(h, &h->d_lam_inv_b, lam_inv);
    if (!rc) rc = upload(h, &h->d_d_perm_b, d_perm);
    if (!rc) rc = upload(h, &h->d_br_perm_b, br_perm);
    if (!rc) rc = upload(h, &h->d_br_inv_b, br_inv);
    if (h->form == DCOPF_FORM_CYCLE) {  // internal branch -> storage row of the cycle it defines (-1: tree)
      std::vector<int> pos(h->n_br, -1);
      for (int k = 0; k < h->cyc_int.nc; ++k) pos[h->cyc_int.def[k]] = h->sch.pos_br[k];
      if (!rc) rc = upload(h, &h->d_br_pos_b, pos);
    } else if (!rc) {
      rc = upload(h, &h->d_br_pos_b, h->sch.pos_br);
    }
  }
  if (rc) return rc;
  std::vector<uint8_t>().swap(h->sch.prog);  // device copy only
  h->sched_W = W;
  h->sched_V = V;
  h->sched_C = C;
  h->sched_nw = nw;
  h->sched_opt = optv;
  return DCOPF_OK;
}

// Tile configuration of the batched path for B instances: V instances per
// lane, W per tile, C parts (CTAs) per tile.  The sweep is issue-bound and a
// warp instruction costs one issue slot whatever its lane count; measured per
// item, the work of 4 instances per lane is ~2x that of 2 (the fp64 work per
// instance dominates the item), and the time of a CTA's sweep is ~(V / C) x
// (its share of the network's items) plus the halo items of a split tile.
// The batch is covered in ONE wave of tiles x C <= n_sm CTAs at the smallest
// estimated V / C (ties: V = 2, which affords larger chunks); F1 always runs
// V = 2 (its mu rows are twice as wide).  Batches too large for one wave use V = 4, C = 1 and W =
// 128 (several waves of whole-network tiles).  Measured on config 4 (F2 /
// KVL inst-it/s): 8192: V2C1 1.01e7 / 1.22e7, V4C2 1.00e7 /
// 1.20e7; 4096: V2C2 9.5e6 / 1.20e7, V4C4 1.0e7 / 1.21e7; 2048: V2C4 9.2e6 /
// 1.14e7, V4C8 9.5e6 / 1.11e7; 1024: V2C8 8.6e6 / 1.05e7, V4C16 8.6e6 / 1.02e7.
//
// Round 2: the sweep time of a tiling is ~ (pipeline steps of a part) x F +
// (items of a part) x u, F ~ 10 bus items per step (the per-step fixed cost:
// barriers, program header, item ranges), u ~ V / 2; the chunk -- hence the
// steps -- comes from the shared-memory fit of that tiling, which the plain
// V / C x halo model cannot see (F1's halo rows at 9 parts leave 4-bus chunks:
// 2.8e6 inst-it/s at 1024 instances vs 4.7e6 at 6 parts with 18-bus chunks,
// profiles/r2/tiles).  So the best few tilings by the plain model are
// compiled (quick schedule search) and the one with the smallest estimated
// sweep time is taken.  (Checked against the measured table above: the
// choice at 8192 / 4096 / 1024 is unchanged for F2 and KVL.)
void choose_tiles(dcopf_dual_t h, int64_t B, int *V_out, int *W_out, int *C_out) {
  const int optk = h->opt.variant != DCOPF_OPT_PLAIN;
  if (h->tc_B == B && h->tc_opt == optk) {
    *V_out = h->tc_V;
    *W_out = h->tc_W;
    *C_out = h->tc_C;
    return;
  }
  const long nsm = h->n_sm;
  struct Cand {
    int V, W, C;
    double cost;
  };
  std::vector<Cand> cands;
  for (int V : {2, 4})
    for (int C = 1; C <= 16; ++C) {
      if (V == 4 && h->form == DCOPF_FORM_LIMIT_ROWS) break;  // F1: 2 per lane (its mu rows are twice as wide)
      if ((h->opt_lane && V != h->opt_lane) || (h->opt_parts && C != h->opt_parts)) continue;
      if (!h->opt_parts && C > 1 && h->n_bus < 64 * C) break;  // parts of >= 64 buses (halo stays small)
      if (C > h->n_bus) break;
      const long maxt = nsm / C;
      if (maxt < 1) break;
      long W = (B + maxt - 1) / maxt;
      W = std::max<long>(V, (W + V - 1) / V * V);
      if (W > 32L * V) continue;
      const double halo = 1.0 + 0.02 * (C - 1);  // halo items of a split tile (measured ~1-2% per cut)
      cands.push_back({V, (int)W, C, (double)V / C * halo});
    }
  int bV, bW, bC;
  if (cands.empty()) {  // more than one wave (or a forced configuration that cannot cover B in one)
    bV = h->opt_lane ? h->opt_lane : (h->form == DCOPF_FORM_LIMIT_ROWS ? 2 : 4);
    bC = h->opt_parts ? h->opt_parts : 1;
    const long maxt = std::max<long>(1, nsm / bC);
    bW = (int)std::min<long>(32L * bV, std::max<long>(bV, ((B + maxt - 1) / maxt + bV - 1) / bV * bV));
  } else {
    std::stable_sort(cands.begin(), cands.end(), [](const Cand &x, const Cand &y) { return x.cost < y.cost - 1e-9; });
    const Cand *pick = &cands[0];
    double best = 1e300;
    const size_t top = std::min<size_t>(cands.size(), 4);
    for (size_t i = 0; i < top && cands.size() > 1; ++i) {
      const Cand &c = cands[i];
      Schedule sc;
      std::string err;
      if (!search_schedule(h, c.W, c.V, c.C, 0, 0, &sc, &err, /*quick=*/true)) continue;
      int steps = 0;
      for (int p = 0; p < c.C; ++p) steps = std::max(steps, sc.part_step0[p + 1] - sc.part_step0[p]);
      const double halo = 1.0 + 0.02 * (c.C - 1);
      const double t = 10.0 * steps + (double)h->n_bus / c.C * halo * (c.V / 2.0);
      if (t < best) {
        best = t;
        pick = &c;
      }
    }
    bV = pick->V;
    bW = pick->W;
    bC = pick->C;
  }
  *V_out = bV;
  *W_out = bW;
  *C_out = bC;
  h->tc_B = B;
  h->tc_opt = optk;
  h->tc_V = bV;
  h->tc_W = bW;
  h->tc_C = bC;
}

// state-layout permutations of the current path (storage position <-> original id)
struct Perms {
  const int *lam_perm, *lam_inv, *d_perm, *br_perm, *br_inv;
};
Perms perms(dcopf_dual_t h) {
  if (h->path == DCOPF_PATH_BATCHED)
    return Perms{h->d_lam_perm_b, h->d_lam_inv_b, h->d_d_perm_b, h->d_br_perm_b, h->d_br_inv_b};
  if (h->form == DCOPF_FORM_CYCLE)
    return Perms{h->d_bus_perm, h->d_bus_inv, h->d_bus_perm, h->d_cyc_perm, h->d_cyc_inv};
  return Perms{h->d_bus_perm, h->d_bus_inv, h->d_bus_perm, h->d_br_perm, h->d_br_inv};
}

int opt_nstate(dcopf_dual_t h) {
  switch (h->opt.variant) {
    case DCOPF_OPT_PLAIN: return 0;
    case DCOPF_OPT_ADAM: return 2;
    default: return 1;
  }
}

// optimiser state arrays of the loaded batch (cluster path), zeroed
int reset_opt_state(dcopf_dual_t h, cudaStream_t s) {
  h->b1t = h->b2t = 1.0;
  const int ns = opt_nstate(h);
  if (h->B == 0 || h->path == DCOPF_PATH_SINGLE || ns == 0) return DCOPF_OK;
  // same layout as the multipliers (cluster: instance-major; batched: tile-major rows)
  const size_t n[4] = {(size_t)h->B_pad * h->n_bus, (size_t)h->B_pad * h->n_bus,
                       (size_t)h->B_pad * h->n_bm_ent * h->bm_C, (size_t)h->B_pad * h->n_bm_ent * h->bm_C};
  for (int x = 0; x < 4; ++x) {
    if (x == 1 || x == 3) {
      if (ns < 2) continue;
    }
    if (!h->os[x]) CK(h, cudaMalloc(&h->os[x], std::max<size_t>(n[x], 1) * 8));
    CK(h, cudaMemsetAsync(h->os[x], 0, std::max<size_t>(n[x], 1) * 8, s));
  }
  return DCOPF_OK;
}

// Cluster path: the smallest power-of-two cluster (<= 16 CTAs) whose
// partition fits one CTA's shared memory with ~640 buses or fewer per CTA and
// that the device can co-schedule.  Returns DCOPF_EINVAL if none does.
int configure_cluster(dcopf_dual_t h) {
  if (h->cplan_C) return DCOPF_OK;
  int C = 1;
  while (C < 16 && (long)h->n_bus > 640L * C) C *= 2;
  if (h->opt_parts) C = h->opt_parts;  // dcopf_options.tile_parts: the cluster size
  if (h->force_cluster_C) C = h->force_cluster_C;
  std::string err;
  for (; C <= 16; C *= 2) {
    if (h->force_cluster_C && C != h->force_cluster_C) break;
    ClusterPlan pl;
    err = build_cluster_plan(h->ni, C, h->dev_smem, opt_nstate(h), &pl,
                             h->form == DCOPF_FORM_CYCLE ? &h->cyc_int : nullptr);
    if (!err.empty()) continue;
    auto fn = (h->form == DCOPF_FORM_FLOW_BOX)   ? k_cluster<kFormF2, kModeStep>
              : (h->form == DCOPF_FORM_CYCLE) ? k_cluster<kFormKVL, kModeStep>
                                              : k_cluster<kFormF1, kModeStep>;
    const void *fns[9] = {(const void *)k_cluster<kFormF2, kModeStep>,  (const void *)k_cluster<kFormF2, kModeEval>,
                          (const void *)k_cluster<kFormF1, kModeStep>,  (const void *)k_cluster<kFormF1, kModeEval>,
                          (const void *)k_cluster<kFormKVL, kModeStep>, (const void *)k_cluster<kFormKVL, kModeEval>,
                          (const void *)k_cluster<kFormF2, kModeStep, true>,
                          (const void *)k_cluster<kFormF1, kModeStep, true>,
                          (const void *)k_cluster<kFormKVL, kModeStep, true>};
    for (const void *f : fns) {
      CK(h, cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem));
      if (C > 8) CK(h, cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, (const void *)fn, &cfg) != cudaSuccess) {
      cudaGetLastError();
      ncl = 0;
    }
    if (ncl < 1) {
      err = "cluster of " + std::to_string(C) + " CTAs cannot be scheduled";
      continue;
    }
    h->cplan = pl;
    h->cplan_C = C;
    int rc = upload(h, &h->d_cblob, h->cplan.blob);
    if (!rc && h->form == DCOPF_FORM_CYCLE) {  // state order of kappa: internal -> canonical k and back
      std::vector<int> inv(h->n_bm_ent);
      for (int x = 0; x < h->n_bm_ent; ++x) inv[h->cplan.cyc_perm[x]] = x;
      rc = upload(h, &h->d_cyc_perm, h->cplan.cyc_perm);
      if (!rc) rc = upload(h, &h->d_cyc_inv, inv);
    }
    std::vector<uint8_t>().swap(h->cplan.blob);
    return rc;
  }
  return fail(h, DCOPF_EINVAL, "cluster path: %s", err.c_str());
}

ClusterArgs cluster_args(dcopf_dual_t h) {
  ClusterArgs a;
  memset(&a, 0, sizeof a);
  a.blob = h->d_cblob;
  a.blob_stride = h->cplan.blob_stride;
  a.lam = h->lam[0];
  a.br = h->br[0];
  a.d = h->load;
  a.outs = h->outs;
  a.max_out = h->max_out;
  a.bound = h->bound;
  a.best = h->best;
  a.status = h->status;
  a.B = h->B;
  a.target = h->has_target ? h->target : nullptr;
  a.hit = h->hit;
  a.k_base = h->k_base;
  a.n_bus = h->n_bus;
  a.n_br = h->n_br;
  a.n_bm = h->n_bm_ent * h->bm_C;
  a.opt = h->opt.variant;
  a.rho = h->opt.momentum;
  a.beta1 = h->opt.beta1;
  a.beta2 = h->opt.beta2;
  a.eps = h->opt.epsilon;
  a.b1t = h->b1t;
  a.b2t = h->b2t;
  a.tol = h->tol;
  if (const char *e = getenv("DCOPF_CLUSTER_DEBUG")) a.dbg = atoi(e);  // measurement only
  a.s1_lam = h->os[0];
  a.s2_lam = h->os[1];
  a.s1_br = h->os[2];
  a.s2_br = h->os[3];
  return a;
}

template <int MODE>
int launch_cluster(dcopf_dual_t h, const ClusterArgs &a, cudaStream_t s) {
  const int C = h->cplan_C;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)(h->B * C));
  cfg.blockDim = dim3(kClusterThreads);
  cfg.dynamicSmemBytes = h->cplan.smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // (the dynamic shared-memory limit is per function and shared by every
  // handle: set it for this handle's plan right before its launch)
  const bool opt = MODE == kModeStep && h->opt.variant != DCOPF_OPT_PLAIN;
  auto fn = (h->form == DCOPF_FORM_FLOW_BOX) ? (opt ? k_cluster<kFormF2, MODE, true> : k_cluster<kFormF2, MODE>)
            : (h->form == DCOPF_FORM_CYCLE)  ? (opt ? k_cluster<kFormKVL, MODE, true> : k_cluster<kFormKVL, MODE>)
                                             : (opt ? k_cluster<kFormF1, MODE, true> : k_cluster<kFormF1, MODE>);
  CK(h, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, h->cplan.smem));
  CK(h, cudaLaunchKernelEx(&cfg, fn, a));
  CK(h, cudaGetLastError());
  return DCOPF_OK;
}

SweepArgs sweep_args(dcopf_dual_t h) {
  SweepArgs a;
  memset(&a, 0, sizeof a);
  a.lam0 = h->lam[0];
  a.lam1 = h->lam[1];
  a.br0 = h->br[0];
  a.br1 = h->br[1];
  a.d = h->load;
  a.outs = h->outs;
  a.max_out = h->max_out;
  a.cur = h->cur;
  a.bound = h->bound;
  a.best = h->best;
  a.status = h->status;
  a.B = h->B;
  a.target = h->has_target ? h->target : nullptr;
  a.hit = h->hit;
  a.k_base = h->k_base;
  a.n_bus = h->n_bus;
  a.n_br = h->n_br;
  a.n_brows = h->n_bm_ent;
  a.ref = h->ref_int;
  a.W = h->T;
  const Schedule &sc = h->sch;
  a.prog = h->d_prog;
  a.prog_off = h->d_prog_off;
  a.prog_bytes = h->d_prog_bytes;
  a.tx_bytes = h->d_tx_bytes;
  a.ld_ptr = h->d_ld_ptr;
  a.ld = reinterpret_cast<const int4 *>(h->d_ld);
  a.S = sc.S;
  a.row_bytes = sc.row_bytes;
  a.br_row_bytes = sc.br_row_bytes;
  a.off_bar = sc.off_bar;
  a.off_red = sc.off_red;
  a.off_frz = sc.off_frz;
  a.off_obm = sc.off_obm;
  a.off_outs = sc.off_outs;
  a.off_prog = sc.off_prog;
  a.prog_stride = (sc.max_prog_bytes + 127) & ~127;
  a.off_brp = sc.off_brp;
  a.off_lamp = sc.off_lamp;
  a.off_dp = sc.off_dp;
  a.off_th = sc.off_th;
  a.off_fc = sc.off_fc;
  a.parts = h->tile_C;
  for (int p = 0; p <= h->tile_C && p < (int)sc.part_step0.size(); ++p) a.part_step0[p] = sc.part_step0[p];
  a.tile_sync = h->d_tile_sync;
  a.part_val = h->d_part_val;
  a.tiles = (int)(h->B_pad / h->T);
  a.soft = 1;
  a.tol = h->tol;
  a.opt = h->opt.variant;
  a.rho = h->opt.momentum;
  a.beta1 = h->opt.beta1;
  a.beta2 = h->opt.beta2;
  a.eps = h->opt.epsilon;
  a.b1t = h->b1t;
  a.b2t = h->b2t;
  a.s1_lam = h->os[0];
  a.s2_lam = h->os[1];
  a.s1_br = h->os[2];
  a.s2_br = h->os[3];
  return a;
}

// one k_sweep launch: the kernel's dynamic shared-memory limit is set for
// THIS handle's schedule right before the launch (the attribute is per
// function and shared by every handle of the process); a split tile (C > 1)
// is a cooperative launch, so the tile's CTAs are co-resident for the
// once-per-sweep meeting of its parts, whose counters are zeroed first
template <int FORM, bool EVAL, bool OPT, int V, int NW>
int launch_sweep_t(dcopf_dual_t h, const SweepArgs &a, cudaStream_t s) {
  auto fn = k_sweep<FORM, EVAL, NW, true, OPT, V>;
  const int sm = h->sch.total;
  CK(h, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  const int C = h->tile_C;
  if (C > 1) CK(h, cudaMemsetAsync(h->d_tile_sync, 0, (size_t)a.tiles * sizeof(unsigned), s));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.gridDim = dim3((unsigned)(a.tiles * C));
  cfg.blockDim = dim3((NW + 1) * 32);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = (C > 1) ? 1 : 0;
  CK(h, cudaLaunchKernelEx(&cfg, fn, a));
  return DCOPF_OK;
}

template <bool EVAL>
int launch_sweep(dcopf_dual_t h, const SweepArgs &a, cudaStream_t s) {
  constexpr int N2 = kSweepWarps2, N4 = kSweepWarps4;
  const bool opt = !EVAL && h->opt.variant != DCOPF_OPT_PLAIN;  // optimiser variants
  const bool v4 = h->tile_V == 4;
  if (h->sched_nw != sweep_warps(h->tile_V, h->opt.variant != DCOPF_OPT_PLAIN) ||
      h->sched_opt != (h->opt.variant != DCOPF_OPT_PLAIN))
    return fail(h, DCOPF_ESTATE, "batched schedule compiled for another warp count");
  if (h->form == DCOPF_FORM_FLOW_BOX) {
    if (v4) return opt ? launch_sweep_t<kFormF2, false, true, 4, N4>(h, a, s) : launch_sweep_t<kFormF2, EVAL, false, 4, N4>(h, a, s);
    return opt ? launch_sweep_t<kFormF2, false, true, 2, N2>(h, a, s) : launch_sweep_t<kFormF2, EVAL, false, 2, N2>(h, a, s);
  }
  if (h->form == DCOPF_FORM_CYCLE) {
    if (v4) return opt ? launch_sweep_t<kFormKVL, false, true, 4, N4>(h, a, s) : launch_sweep_t<kFormKVL, EVAL, false, 4, N4>(h, a, s);
    return opt ? launch_sweep_t<kFormKVL, false, true, 2, N2>(h, a, s) : launch_sweep_t<kFormKVL, EVAL, false, 2, N2>(h, a, s);
  }
  return opt ? launch_sweep_t<kFormF1, false, true, 2, N2>(h, a, s) : launch_sweep_t<kFormF1, EVAL, false, 2, N2>(h, a, s);
}

SingleArgs single_args(dcopf_dual_t h) {
  SingleArgs a;
  memset(&a, 0, sizeof a);
  a.lam = h->lam[0];
  a.br = h->br[0];
  a.d = h->load;
  a.outs = h->outs;
  a.max_out = h->max_out;
  a.bound = h->bound;
  a.best = h->best;
  a.status = h->status;
  a.B = h->B;
  a.target = h->has_target ? h->target : nullptr;
  a.hit = h->hit;
  a.k_base = h->k_base;
  a.tol = h->tol;
  return a;
}

template <int FORM, bool SM, int MODE>
int launch_single_t(dcopf_dual_t h, const SingleArgs &a, cudaStream_t s) {
  CK(h, cudaFuncSetAttribute(k_single<FORM, SM, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem_single));
  k_single<FORM, SM, MODE><<<(unsigned)h->B, 1024, h->smem_single, s>>>(dev_net(h), a);
  CK(h, cudaGetLastError());
  return DCOPF_OK;
}

template <int MODE>
int launch_single(dcopf_dual_t h, const SingleArgs &a, cudaStream_t s) {
  const bool sm = h->single_smem;
  if (h->form == DCOPF_FORM_FLOW_BOX)
    return sm ? launch_single_t<kFormF2, true, MODE>(h, a, s) : launch_single_t<kFormF2, false, MODE>(h, a, s);
  return sm ? launch_single_t<kFormF1, true, MODE>(h, a, s) : launch_single_t<kFormF1, false, MODE>(h, a, s);
}

}  // namespace

// ============================================================================
extern "C" {

const char *dcopf_dual_last_error(dcopf_dual_t h) { return h ? h->err.c_str() : g_create_error.c_str(); }

void dcopf_dual_destroy(dcopf_dual_t h) {
  if (!h) return;
  cudaSetDevice(h->device);
  ptdf_destroy(h->pt);
  free_batch(h);
  cudaFree(h->d_cyc_perm);
  cudaFree(h->d_cyc_inv);
  int *ip[] = {h->d_bus_ptr, h->d_bus_inc, h->d_gen_ptr,    h->d_br_s,      h->d_br_t,    h->d_bus_perm,
               h->d_bus_inv, h->d_br_perm, h->d_br_inv,     h->d_prog_bytes, h->d_tx_bytes, h->d_ld_ptr,
               h->d_ld,      h->flag,      h->d_lam_perm_b, h->d_lam_inv_b, h->d_d_perm_b, h->d_br_perm_b,
               h->d_br_inv_b, h->d_br_pos_b};
  for (int *p : ip) cudaFree(p);
  double *dp[] = {h->d_theta, h->d_gen_c, h->d_gen_lo, h->d_gen_hi, h->d_gen_a, h->d_br_b, h->d_br_F,
                  h->scratch, h->alpha_dev};
  for (double *p : dp) cudaFree(p);
  cudaFree(h->d_prog);
  cudaFree(h->d_prog_off);
  cudaFree(h->d_part_step0);
  cudaFree(h->d_tile_sync);
  cudaFree(h->d_part_val);
  cudaFree(h->d_cblob);
  cudaFreeHost(h->alpha_pin);
  if (h->alpha_ev) cudaEventDestroy(h->alpha_ev);
  delete h;
}

int dcopf_dual_create(const dcopf_network_desc *net, const dcopf_options *opt, dcopf_dual_t *out) {
  if (!out) return fail(nullptr, DCOPF_EINVAL, "out is NULL");
  *out = nullptr;
  if (!net) return fail(nullptr, DCOPF_EINVAL, "network descriptor is NULL");
  dcopf_options o;
  memset(&o, 0, sizeof o);
  o.precision = 64;
  if (opt) o = *opt;
  if (o.form != DCOPF_FORM_FLOW_BOX && o.form != DCOPF_FORM_LIMIT_ROWS && o.form != DCOPF_FORM_CYCLE &&
      o.form != DCOPF_FORM_PTDF)
    return fail(nullptr, DCOPF_EINVAL, "unknown form %d", o.form);
  if (o.precision != 64 && o.precision != 0)
    return fail(nullptr, DCOPF_EINVAL, "precision %d not supported (fp64 only)", o.precision);
  if (o.path < 0 || o.path > 4) return fail(nullptr, DCOPF_EINVAL, "unknown path %d", o.path);
  if (o.tile_parts < 0 || o.tile_parts > 16) return fail(nullptr, DCOPF_EINVAL, "tile_parts must be in [0, 16]");
  if (o.lane_instances != 0 && o.lane_instances != 2 && o.lane_instances != 4)
    return fail(nullptr, DCOPF_EINVAL, "lane_instances must be 0, 2 or 4");
  if (o.tile_parts & (o.tile_parts - 1) && o.path == DCOPF_PATH_CLUSTER)
    return fail(nullptr, DCOPF_EINVAL, "cluster path: tile_parts (CTAs per instance) must be a power of two");
  if ((o.form == DCOPF_FORM_PTDF) != (o.path == DCOPF_PATH_DENSE) && o.path != DCOPF_PATH_AUTO)
    return fail(nullptr, DCOPF_EINVAL, "the PTDF form runs on DCOPF_PATH_DENSE (and only it)");
  const int nb = net->n_bus, nl = net->n_branch, ng = net->n_gen;
  if (nb < 1 || nl < 0 || ng < 0) return fail(nullptr, DCOPF_EINVAL, "bad sizes n_bus=%d n_branch=%d n_gen=%d", nb, nl, ng);
  if (net->ref_bus < 0 || net->ref_bus >= nb) return fail(nullptr, DCOPF_EINVAL, "ref_bus %d out of range", net->ref_bus);
  if (nl > 0 && (!net->br_from || !net->br_to || !net->br_b || !net->br_fmax))
    return fail(nullptr, DCOPF_EINVAL, "branch arrays missing");
  if (ng > 0 && (!net->gen_bus || !net->gen_pmin || !net->gen_pmax || !net->gen_c))
    return fail(nullptr, DCOPF_EINVAL, "generator arrays missing");
  if (nl >= (1 << 29) || nb >= (1 << 30)) return fail(nullptr, DCOPF_EINVAL, "network too large");
  std::vector<int> fr(nl), to(nl);
  for (int l = 0; l < nl; ++l) {
    fr[l] = net->br_from[l];
    to[l] = net->br_to[l];
    if (fr[l] < 0 || fr[l] >= nb || to[l] < 0 || to[l] >= nb)
      return fail(nullptr, DCOPF_EINVAL, "branch %d endpoint out of range", l);
    if (fr[l] == to[l]) return fail(nullptr, DCOPF_EINVAL, "branch %d is a self loop", l);
    if (!(net->br_b[l] >= 0.0) || !std::isfinite(net->br_b[l]))
      return fail(nullptr, DCOPF_EINVAL, "branch %d susceptance must be finite and >= 0", l);
    if (!(net->br_fmax[l] >= 0.0) || !std::isfinite(net->br_fmax[l]))
      return fail(nullptr, DCOPF_EINVAL, "branch %d flow limit must be finite and >= 0", l);
  }
  for (int g = 0; g < ng; ++g) {
    if (net->gen_bus[g] < 0 || net->gen_bus[g] >= nb) return fail(nullptr, DCOPF_EINVAL, "generator %d bus out of range", g);
    const double lo = net->gen_pmin[g], hi = net->gen_pmax[g], c = net->gen_c[g];
    if (!std::isfinite(lo) || !std::isfinite(hi) || !std::isfinite(c))
      return fail(nullptr, DCOPF_EINVAL, "generator %d data not finite", g);
    if (lo > hi) return fail(nullptr, DCOPF_EINVAL, "generator %d has pmin > pmax", g);
    if (net->gen_a && (!(net->gen_a[g] >= 0.0) || !std::isfinite(net->gen_a[g])))
      return fail(nullptr, DCOPF_EINVAL, "generator %d quadratic cost must be finite and >= 0", g);
  }
  if (net->theta_max && o.form != DCOPF_FORM_PTDF)
    for (int i = 0; i < nb; ++i)
      if (!(net->theta_max[i] >= 0.0) || !std::isfinite(net->theta_max[i]))
        return fail(nullptr, DCOPF_EINVAL, "theta_max[%d] must be finite and >= 0", i);
  std::vector<char> use(nl);
  for (int l = 0; l < nl; ++l) use[l] = net->br_b[l] > 0.0;
  if (!connected(nb, fr, to, use)) return fail(nullptr, DCOPF_ETOPOLOGY, "network is disconnected over branches with b > 0");
  if (o.form == DCOPF_FORM_PTDF) {  // dense PTDF: its own state (ptdf.cu), no internal reordering
    dcopf_dual_t h = new dcopf_dual_s();
    h->device = o.device;
    h->form = o.form;
    h->path_opt = h->path = DCOPF_PATH_DENSE;
    h->n_bus = nb;
    h->n_br = nl;
    h->n_gen = ng;
    PtdfNetIn pn{nb, nl, ng, net->ref_bus, fr.data(), to.data(), net->br_b, net->br_fmax, net->gen_bus,
                 net->gen_pmin, net->gen_pmax, net->gen_c, net->gen_a};
    std::string perr;
    const int prc = ptdf_create(pn, o.device, &h->pt, &perr);
    if (prc) {
      delete h;
      return fail(nullptr, prc, "%s", perr.c_str());
    }
    *out = h;
    return DCOPF_OK;
  }
  if (net->br_switchable) {
    for (int l = 0; l < nl; ++l) use[l] = net->br_b[l] > 0.0 && !net->br_switchable[l];
    if (!connected(nb, fr, to, use))
      return fail(nullptr, DCOPF_ETOPOLOGY, "never-switchable branches do not connect the network");
  }

  // ---- angle box: given, or implied by the flow limits (reading A-2) ----
  std::vector<double> theta(nb, 0.0);
  if (net->theta_max) {
    for (int i = 0; i < nb; ++i) theta[i] = net->theta_max[i];
  } else {
    std::vector<std::vector<std::pair<int, double>>> wadj(nb);
    for (int l = 0; l < nl; ++l) {
      if (!(net->br_b[l] > 0.0)) continue;
      if (net->br_switchable && net->br_switchable[l]) continue;
      const double wgt = net->br_fmax[l] / net->br_b[l];
      wadj[fr[l]].push_back({to[l], wgt});
      wadj[to[l]].push_back({fr[l], wgt});
    }
    std::vector<double> dist(nb, std::numeric_limits<double>::infinity());
    typedef std::pair<double, int> QE;
    std::priority_queue<QE, std::vector<QE>, std::greater<QE>> pq;
    dist[net->ref_bus] = 0.0;
    pq.push({0.0, net->ref_bus});
    while (!pq.empty()) {
      const QE top = pq.top();
      pq.pop();
      if (top.first > dist[top.second]) continue;
      for (auto &e : wadj[top.second]) {
        const double nd = top.first + e.second;
        if (nd < dist[e.first]) {
          dist[e.first] = nd;
          pq.push({nd, e.first});
        }
      }
    }
    theta = dist;
  }
  theta[net->ref_bus] = 0.0;

  dcopf_dual_t h = new dcopf_dual_s();
  h->device = o.device;
  h->form = o.form;
  h->path_opt = o.path;
  // AUTO threshold: measured on config-4 instances of the 10k-bus network
  // (tools/gpu_r2_medium.sh): one 16-CTA cluster per instance
  // runs 9 instances at a time at ~6 us per iteration, the split-tile batched
  // sweep any batch up to ~150 at ~50 us -- equal near B = 60
  h->single_max = o.single_max_batch > 0 ? o.single_max_batch : 56;
  h->opt_parts = o.tile_parts;
  h->opt_lane = o.lane_instances;
  h->n_bus = nb;
  h->n_br = nl;
  h->n_gen = ng;
  if (net->gen_a)
    for (int g = 0; g < ng; ++g) h->quadratic |= net->gen_a[g] > 0.0;
  if (net->br_switchable) h->switchable.assign(net->br_switchable, net->br_switchable + nl);
  h->implied_box = net->theta_max == nullptr;

  // ---- internal numbering: bus order, branch order, CSR, generator map ----
  Internalized in;
  const std::string ierr = internalize(nb, nl, ng, net->ref_bus, fr.data(), to.data(), net->br_b, net->br_fmax,
                                       theta.data(), net->gen_bus, net->gen_pmin, net->gen_pmax, net->gen_c,
                                       net->gen_a, net->br_switchable, h->form, /*rcm=*/false,
                                       &in);
  if (!ierr.empty()) {
    delete h;
    return fail(nullptr, DCOPF_EINVAL, "%s", ierr.c_str());
  }
  h->n_bm_ent = nl;
  h->bm_C = (h->form == DCOPF_FORM_LIMIT_ROWS) ? 2 : 1;
  if (h->form == DCOPF_FORM_CYCLE) {  // the canonical cycle basis (reading A-28), then internal branch ids
    const std::string cerr = build_cycle_basis(nb, nl, net->ref_bus, fr.data(), to.data(), net->br_b,
                                               net->br_switchable, &h->cyc_orig);
    if (!cerr.empty()) {
      delete h;
      return fail(nullptr, DCOPF_ETOPOLOGY, "%s", cerr.c_str());
    }
    h->cyc_int = h->cyc_orig;
    for (int &l : h->cyc_int.def) l = in.br_inv[l];
    for (int &l : h->cyc_int.cb) l = in.br_inv[l];
    h->n_bm_ent = h->cyc_orig.nc;
  }
  h->bus_perm = in.bus_perm;
  h->bus_inv = in.bus_inv;
  h->br_perm = in.br_perm;
  h->br_inv = in.br_inv;
  h->ref_int = in.net.ref;
  h->bandwidth = in.bandwidth;
  h->ni = in.net;

  cudaError_t e = cudaSetDevice(h->device);
  if (e != cudaSuccess) {
    delete h;
    return fail(nullptr, DCOPF_ECUDA, "cudaSetDevice(%d): %s", o.device, cudaGetErrorString(e));
  }
  int rc = DCOPF_OK;
  if (cudaDeviceGetAttribute(&h->n_sm, cudaDevAttrMultiProcessorCount, h->device) != cudaSuccess ||
      cudaDeviceGetAttribute(&h->dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device) != cudaSuccess)
    rc = fail(h, DCOPF_ECUDA, "cudaDeviceGetAttribute failed");
  const NetInternal &ni = h->ni;
  if (!rc) rc = upload(h, &h->d_bus_ptr, ni.bus_ptr);
  if (!rc) rc = upload(h, &h->d_bus_inc, ni.bus_inc);
  if (!rc) rc = upload(h, &h->d_gen_ptr, ni.gen_ptr);
  if (!rc) rc = upload(h, &h->d_br_s, ni.bs);
  if (!rc) rc = upload(h, &h->d_br_t, ni.bt);
  if (!rc) rc = upload(h, &h->d_bus_perm, h->bus_perm);
  if (!rc) rc = upload(h, &h->d_bus_inv, h->bus_inv);
  if (!rc) rc = upload(h, &h->d_br_perm, h->br_perm);
  if (!rc) rc = upload(h, &h->d_br_inv, h->br_inv);
  if (!rc) rc = upload(h, &h->d_theta, ni.theta);
  if (!rc) rc = upload(h, &h->d_gen_c, ni.gc);
  if (!rc) rc = upload(h, &h->d_gen_lo, ni.glo);
  if (!rc) rc = upload(h, &h->d_gen_hi, ni.ghi);
  if (!rc) rc = upload(h, &h->d_gen_a, ni.ga);
  if (!rc) rc = upload(h, &h->d_br_b, ni.b);
  if (!rc) rc = upload(h, &h->d_br_F, ni.F);
  if (!rc) {
    e = cudaMalloc(&h->flag, sizeof(int));
    if (e != cudaSuccess) rc = fail(h, DCOPF_ENOMEM, "cudaMalloc: %s", cudaGetErrorString(e));
  }
  if (rc) {
    g_create_error = h->err;
    dcopf_dual_destroy(h);
    return rc;
  }
  *out = h;
  return DCOPF_OK;
}

int dcopf_dual_set_instance_batch(dcopf_dual_t h, int64_t B, const double *load, const int32_t *outages,
                                  int32_t max_out, void *cuda_stream) {
  if (!h) return fail(nullptr, DCOPF_EINVAL, "null handle");
  if (B < 1) return fail(h, DCOPF_EINVAL, "B must be >= 1 (got %lld)", (long long)B);
  if (!load) return fail(h, DCOPF_EINVAL, "load is NULL");
  if (max_out < 0 || max_out > kMaxOut || (max_out > 0 && !outages))
    return fail(h, DCOPF_EINVAL, "max_out must be in [0, %d] with a non-NULL outage array", kMaxOut);
  CK(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if (h->pt) {
    if (max_out > 0) {
      std::vector<int32_t> raw((size_t)B * max_out);
      CK(h, cudaMemcpy(raw.data(), outages, raw.size() * sizeof(int32_t), cudaMemcpyDefault));
      for (int32_t l : raw)
        if (l != -1)
          return fail(h, DCOPF_EINVAL, "the PTDF form takes load-only batches (one H_a for the batch): no outages");
    }
    std::string perr;
    const int prc = ptdf_set_batch(h->pt, B, load, s, &perr);
    if (prc) return fail(h, prc, "%s", perr.c_str());
    h->B = B;
    return DCOPF_OK;
  }
  int path = h->path_opt;
  if (h->form == DCOPF_FORM_CYCLE && path == DCOPF_PATH_SINGLE)
    return fail(h, DCOPF_EINVAL, "the KVL (cycle) form runs on the cluster and batched paths");
  // outages: validate on the host and convert to internal ids BEFORE anything
  // of the loaded batch (schedule, path, state) is touched, so a rejected call
  // leaves the handle as it was
  std::vector<int> outs_h;
  if (max_out > 0) {
    std::vector<int32_t> raw((size_t)B * max_out);
    CK(h, cudaMemcpy(raw.data(), outages, raw.size() * sizeof(int32_t), cudaMemcpyDefault));
    outs_h.resize(raw.size());
    for (size_t x = 0; x < raw.size(); ++x) {
      const int l = raw[x];
      if (l < -1 || l >= h->n_br) return fail(h, DCOPF_EINVAL, "outage id %d out of range", l);
      if (l >= 0 && !h->switchable.empty() && !h->switchable[l])
        return fail(h, DCOPF_EINVAL, "branch %d is not switchable", l);
      if (l >= 0 && h->implied_box && h->switchable.empty() && h->form != DCOPF_FORM_CYCLE)
        return fail(h, DCOPF_EINVAL,
                    "outage of branch %d with an implied angle box over ALL branches (theta_max and "
                    "br_switchable NULL): the box would not be valid for that instance -- declare the "
                    "switchable branches (br_switchable) or pass theta_max", l);
      if (l >= 0 && h->form == DCOPF_FORM_CYCLE && h->cyc_orig.is_tree[l])
        return fail(h, DCOPF_EINVAL, "branch %d is in the cycle-basis tree (KVL form): declare the switchable "
                                     "branches (br_switchable) so the tree avoids them", l);
      outs_h[x] = l < 0 ? -1 : h->br_inv[l];
    }
  }
  if (path == DCOPF_PATH_AUTO) {
    path = (B <= h->single_max) ? DCOPF_PATH_CLUSTER : DCOPF_PATH_BATCHED;
    if (path == DCOPF_PATH_CLUSTER && configure_cluster(h) != DCOPF_OK) {
      if (h->form == DCOPF_FORM_CYCLE) return DCOPF_EINVAL;  // (message set by configure_cluster)
      path = DCOPF_PATH_SINGLE;
    }
  }
  int W = 1, tV = 2, tC = 1;
  if (path == DCOPF_PATH_BATCHED) {
    if (h->form == DCOPF_FORM_LIMIT_ROWS && h->opt_lane == 4)
      return fail(h, DCOPF_EINVAL, "form F1 runs 2 instances per lane on the batched path");
    choose_tiles(h, B, &tV, &W, &tC);
    // a split tile's parts meet once per sweep, so its launch is cooperative:
    // every CTA resident at once (one per SM)
    if (tC > 1 && (B + W - 1) / W * tC > h->n_sm)
      return fail(h, DCOPF_EINVAL, "tiling of %lld instances with %d parts per tile needs %lld CTAs (> %d SMs, one wave)",
                  (long long)B, tC, (long long)((B + W - 1) / W * tC), h->n_sm);
    // a failed compile leaves sched_* invalid: the old batch (if any) is
    // dropped below before anything can use the new schedule with it
    int rc = compile_schedule(h, W, tV, tC);
    if (rc) {
      free_batch(h);
      return rc;
    }
  } else if (path == DCOPF_PATH_CLUSTER) {
    int rc = configure_cluster(h);
    if (rc) return rc;
  } else {
    const size_t ss_state = single_smem(h->n_bus, h->n_br, h->form, true);
    const size_t ss_nostate = single_smem(h->n_bus, h->n_br, h->form, false);
    if (ss_nostate > (size_t)h->dev_smem)
      return fail(h, DCOPF_EINVAL, "single path needs %zu B shared memory (> %d)", ss_nostate, h->dev_smem);
    h->single_smem = ss_state <= (size_t)h->dev_smem;
    h->smem_single = (int)(h->single_smem ? ss_state : ss_nostate);
  }
  const int64_t B_pad = (B + W - 1) / W * W;
  const bool reuse = h->lam[0] && h->B_pad == B_pad && h->T == W && h->path == path && h->max_out == max_out &&
                     h->tile_V == tV && h->tile_C == tC;
  if (!reuse) free_batch(h);
  h->path = path;
  h->B = B;
  h->T = W;
  h->tile_V = tV;
  h->tile_C = tC;
  h->B_pad = B_pad;
  h->max_out = max_out;
  h->cur = 0;
  const size_t nlam = (size_t)B_pad * h->n_bus, nbr = (size_t)B_pad * h->n_bm_ent * h->bm_C;
  if (!reuse) {
    const int nbuf = (path == DCOPF_PATH_BATCHED) ? 2 : 1;
    for (int i = 0; i < nbuf; ++i) {
      CK(h, cudaMalloc(&h->lam[i], std::max<size_t>(nlam, 1) * 8));
      CK(h, cudaMalloc(&h->br[i], std::max<size_t>(nbr, 1) * 8));
    }
    CK(h, cudaMalloc(&h->load, std::max<size_t>(nlam, 1) * 8));
    CK(h, cudaMalloc(&h->bound, B_pad * 8));
    CK(h, cudaMalloc(&h->best, B_pad * 8));
    CK(h, cudaMalloc(&h->value, B_pad * 8));
    CK(h, cudaMalloc(&h->status, B_pad * 4));
    CK(h, cudaMalloc(&h->outs, std::max<size_t>((size_t)B_pad * max_out, 1) * 4));
    CK(h, cudaMalloc(&h->target, B_pad * 8));
    CK(h, cudaMalloc(&h->hit, B_pad * 8));
  }
  if (path == DCOPF_PATH_BATCHED && tC > 1) {  // split tiles: the parts' meeting place
    const size_t tiles = (size_t)(B_pad / W), nsync = tiles, nval = 2 * tiles * tC * W;
    if (h->tile_sync_cap < nsync) {
      cudaFree(h->d_tile_sync);
      h->d_tile_sync = nullptr;
      h->tile_sync_cap = 0;
      CK(h, cudaMalloc(&h->d_tile_sync, nsync * sizeof(unsigned)));
      h->tile_sync_cap = nsync;
    }
    if (h->part_val_cap < nval) {
      cudaFree(h->d_part_val);
      h->d_part_val = nullptr;
      h->part_val_cap = 0;
      CK(h, cudaMalloc(&h->d_part_val, nval * sizeof(double)));
      h->part_val_cap = nval;
    }
  }
  h->has_target = false;
  h->k_base = 0;
  if (max_out > 0) {
    std::vector<int> padded((size_t)B_pad * max_out, -1);
    std::copy(outs_h.begin(), outs_h.end(), padded.begin());
    CK(h, cudaMemcpyAsync(h->outs, padded.data(), padded.size() * 4, cudaMemcpyHostToDevice, s));
    CK(h, cudaStreamSynchronize(s));  // `padded` dies at scope exit
  }
  int rc = import_ext(h, load, h->load, perms(h).d_perm, h->n_bus, 1, s);
  if (rc) return rc;
  k_fill_d<<<grid_for(nlam), 256, 0, s>>>(h->lam[0], 0.0, nlam);
  k_fill_d<<<grid_for(nbr), 256, 0, s>>>(h->br[0], 0.0, nbr);
  k_fill_d<<<grid_for(B_pad), 256, 0, s>>>(h->best, -std::numeric_limits<double>::infinity(), B_pad);
  k_fill_d<<<grid_for(B_pad), 256, 0, s>>>(h->bound, std::numeric_limits<double>::quiet_NaN(), B_pad);
  k_fill_i<<<grid_for(B_pad), 256, 0, s>>>(h->status, 0, B_pad);
  CK(h, cudaMemsetAsync(h->hit, 0xff, B_pad * 8, s));  // -1
  if (int rc2 = reset_opt_state(h, s)) return rc2;
  CK(h, cudaGetLastError());
  return DCOPF_OK;
}

int dcopf_dual_iterate(dcopf_dual_t h, int64_t K, const double *alpha, double *history, void *cuda_stream) {
  if (!h) return fail(nullptr, DCOPF_EINVAL, "null handle");
  if (h->B == 0) return fail(h, DCOPF_ESTATE, "iterate before set_instance_batch");
  if (K < 0 || (K > 0 && !alpha)) return fail(h, DCOPF_EINVAL, "K must be >= 0 and alpha non-NULL");
  CK(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  double *hist = history;
  const bool hist_host = history && !is_device_ptr(history);
  if (hist_host) {
    int rc = ensure_scratch(h, (size_t)K * h->B * 8 + 8);
    if (rc) return rc;
    hist = h->scratch;
  }
  if (h->opt.variant != DCOPF_OPT_PLAIN && h->path == DCOPF_PATH_SINGLE)
    return fail(h, DCOPF_ESTATE, "optimiser variants run on the cluster and batched paths");
  int rc = stage_alpha(h, K, alpha, s);
  if (rc) return rc;
  if (h->pt) {
    std::string perr;
    rc = ptdf_iterate(h->pt, K, h->alpha_dev, hist, s, &perr);
    if (rc) return fail(h, rc, "%s", perr.c_str());
  } else if (h->path == DCOPF_PATH_BATCHED) {
    SweepArgs a = sweep_args(h);
    a.alpha = h->alpha_dev;
    a.K = K;
    a.hist = hist;
    rc = launch_sweep<false>(h, a, s);
    if (rc) return rc;
    h->cur = (int)((h->cur + K) & 1);
    h->k_base += (long)K;
    if (h->opt.variant == DCOPF_OPT_ADAM)
      for (int64_t k = 0; k < K; ++k) {  // the kernel's repeated products, continued
        h->b1t = h->b1t * h->opt.beta1;
        h->b2t = h->b2t * h->opt.beta2;
      }
  } else if (h->path == DCOPF_PATH_SINGLE) {
    SingleArgs a = single_args(h);
    a.alpha = h->alpha_dev;
    a.K = K;
    a.hist = hist;
    rc = launch_single<kModeStep>(h, a, s);
    if (rc) return rc;
    h->k_base += (long)K;
  } else {
    ClusterArgs a = cluster_args(h);
    a.alpha = h->alpha_dev;
    a.K = K;
    a.hist = hist;
    rc = launch_cluster<kModeStep>(h, a, s);
    if (rc) return rc;
    h->k_base += (long)K;
    if (h->opt.variant == DCOPF_OPT_ADAM)
      for (int64_t k = 0; k < K; ++k) {  // the kernel's repeated products, continued
        h->b1t = h->b1t * h->opt.beta1;
        h->b2t = h->b2t * h->opt.beta2;
      }
  }
  if (hist_host) {
    CK(h, cudaMemcpyAsync(history, hist, (size_t)K * h->B * 8, cudaMemcpyDefault, s));
    CK(h, cudaStreamSynchronize(s));
  }
  return DCOPF_OK;
}

int dcopf_dual_get_bound(dcopf_dual_t h, double *bound, double *best, int32_t *status, void *cuda_stream) {
  if (!h) return fail(nullptr, DCOPF_EINVAL, "null handle");
  if (h->B == 0) return fail(h, DCOPF_ESTATE, "no batch loaded");
  CK(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if (h->pt) {
    std::string perr;
    const int prc = ptdf_get_bound(h->pt, bound, best, status, s, &perr);
    return prc ? fail(h, prc, "%s", perr.c_str()) : DCOPF_OK;
  }
  int rc = copy_out(h, bound, h->bound, s);
  if (!rc) rc = copy_out(h, best, h->best, s);
  if (!rc) rc = copy_out(h, status, h->status, s);
  return rc;
}

int dcopf_dual_get_multipliers(dcopf_dual_t h, double *lambda, double *branch, void *cuda_stream) {
  if (!h) return fail(nullptr, DCOPF_EINVAL, "null handle");
  if (h->B == 0) return fail(h, DCOPF_ESTATE, "no batch loaded");
  CK(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if (h->pt) {
    std::string perr;
    const int prc = ptdf_get_multipliers(h->pt, lambda, branch, s, &perr);
    return prc ? fail(h, prc, "%s", perr.c_str()) : DCOPF_OK;
  }
  const int cur = (h->path == DCOPF_PATH_BATCHED) ? h->cur : 0;
  const Perms pm = perms(h);
  int rc = export_ext(h, h->lam[cur], lambda, pm.lam_inv, h->n_bus, 1, s);
  if (!rc) rc = export_ext(h, h->br[cur], branch, pm.br_inv, h->n_bm_ent, h->bm_C, s);
  return rc;
}

int dcopf_dual_set_multipliers(dcopf_dual_t h, const double *lambda, const double *branch, void *cuda_stream) {
  if (!h) return fail(nullptr, DCOPF_EINVAL, "null handle");
  if (h->B == 0) return fail(h, DCOPF_ESTATE, "no batch loaded");
  CK(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if (h->pt) {
    std::string perr;
    const int prc = ptdf_set_multipliers(h->pt, lambda, branch, s, &perr);
    return prc ? fail(h, prc, "%s", perr.c_str()) : DCOPF_OK;
  }
  const int cur = (h->path == DCOPF_PATH_BATCHED) ? h->cur : 0;
  const size_t nlam = (size_t)h->B_pad * h->n_bus, nbr = (size_t)h->B_pad * h->n_bm_ent * h->bm_C;
  double *tl = nullptr, *tb = nullptr;
  CK(h, cudaMalloc(&tl, std::max<size_t>(nlam, 1) * 8));
  cudaError_t e = cudaMalloc(&tb, std::max<size_t>(nbr, 1) * 8);
  if (e != cudaSuccess) {
    cudaFree(tl);
    return fail(h, DCOPF_ENOMEM, "cudaMalloc: %s", cudaGetErrorString(e));
  }
  int rc = DCOPF_OK;
  const Perms pm = perms(h);
  if (lambda) rc = import_ext(h, lambda, tl, pm.lam_perm, h->n_bus, 1, s);
  if (!rc && branch) rc = import_ext(h, branch, tb, pm.br_perm, h->n_bm_ent, h->bm_C, s);
  if (!rc) {
    int bad = 0;
    cudaMemsetAsync(h->flag, 0, sizeof(int), s);
    if (lambda) k_check_mu<<<grid_for(nlam), 256, 0, s>>>(tl, nlam, h->flag, 0);
    if (branch) {
      k_check_mu<<<grid_for(nbr), 256, 0, s>>>(tb, nbr, h->flag, h->form == DCOPF_FORM_LIMIT_ROWS);
      // the batched F2 kernel holds an outaged branch's nu at exactly 0 (it does
      // not enter that instance's dual); a warm start must respect that
      if (h->form == DCOPF_FORM_FLOW_BOX && h->max_out > 0)
        k_check_outaged<<<grid_for((size_t)h->B * h->max_out), 256, 0, s>>>(
            tb, h->outs, h->path == DCOPF_PATH_BATCHED ? h->d_br_pos_b : nullptr, h->max_out, h->B, h->n_br, h->T,
            h->flag);
      // KVL, batched: kappa of a cycle whose defining branch is out stays 0 (phase B does not mask it)
      if (h->form == DCOPF_FORM_CYCLE && h->path == DCOPF_PATH_BATCHED && h->max_out > 0)
        k_check_outaged<<<grid_for((size_t)h->B * h->max_out), 256, 0, s>>>(
            tb, h->outs, h->d_br_pos_b, h->max_out, h->B, h->n_bm_ent, h->T, h->flag);
    }
    cudaMemcpyAsync(&bad, h->flag, sizeof(int), cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = fail(h, DCOPF_ECUDA, "set_multipliers: %s", cudaGetErrorString(e));
    else if (bad)
      rc = fail(h, DCOPF_EINVAL,
                "multipliers must be finite, mu >= 0 (SPEC.md:239), and nu = 0 on an instance's outaged branches");
  }
  if (!rc) {
    if (lambda) cudaMemcpyAsync(h->lam[cur], tl, nlam * 8, cudaMemcpyDeviceToDevice, s);
    if (branch) cudaMemcpyAsync(h->br[cur], tb, nbr * 8, cudaMemcpyDeviceToDevice, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = fail(h, DCOPF_ECUDA, "set_multipliers: %s", cudaGetErrorString(e));
  }
  cudaFree(tl);
  cudaFree(tb);
  return rc;
}

int dcopf_dual_evaluate(dcopf_dual_t h, double *value, double *grad_lambda, double *grad_branch, void *cuda_stream) {
  if (!h) return fail(nullptr, DCOPF_EINVAL, "null handle");
  if (h->B == 0) return fail(h, DCOPF_ESTATE, "no batch loaded");
  CK(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if (h->pt) {
    std::string perr;
    const int prc = ptdf_evaluate(h->pt, value, grad_lambda, grad_branch, s, &perr);
    return prc ? fail(h, prc, "%s", perr.c_str()) : DCOPF_OK;
  }
  const size_t nlam = (size_t)h->B_pad * h->n_bus, nbr = (size_t)h->B_pad * h->n_bm_ent * h->bm_C;
  if (!h->g_lam) CK(h, cudaMalloc(&h->g_lam, std::max<size_t>(nlam, 1) * 8));
  if (!h->g_br) CK(h, cudaMalloc(&h->g_br, std::max<size_t>(nbr, 1) * 8));
  int rc;
  if (h->path == DCOPF_PATH_BATCHED) {
    SweepArgs a = sweep_args(h);
    a.K = 0;
    a.g_lam = h->g_lam;
    a.g_br = h->g_br;
    a.out_val = h->value;
    rc = launch_sweep<true>(h, a, s);
  } else if (h->path == DCOPF_PATH_SINGLE) {
    SingleArgs a = single_args(h);
    a.grad_lam = h->g_lam;
    a.grad_br = h->g_br;
    a.value = h->value;
    rc = launch_single<kModeEval>(h, a, s);
  } else {
    ClusterArgs a = cluster_args(h);
    a.grad_lam = h->g_lam;
    a.grad_br = h->g_br;
    a.value = h->value;
    rc = launch_cluster<kModeEval>(h, a, s);
  }
  if (rc) return rc;
  rc = copy_out(h, value, h->value, s);
  const Perms pm = perms(h);
  if (!rc) rc = export_ext(h, h->g_lam, grad_lambda, pm.lam_inv, h->n_bus, 1, s);
  if (!rc) rc = export_ext(h, h->g_br, grad_branch, pm.br_inv, h->n_bm_ent, h->bm_C, s);
  return rc;
}

int dcopf_dual_set_optimizer(dcopf_dual_t h, const dcopf_optimizer *opt) {
  if (!h) return fail(nullptr, DCOPF_EINVAL, "null handle");
  dcopf_optimizer o = {DCOPF_OPT_PLAIN, 0, 0.0, 0.0, 0.0, 0.0};
  if (opt) o = *opt;
  if (o.variant < DCOPF_OPT_PLAIN || o.variant > DCOPF_OPT_ADAM)
    return fail(h, DCOPF_EINVAL, "unknown optimiser variant %d", o.variant);
  auto unit = [](double x) { return std::isfinite(x) && x >= 0.0 && x < 1.0; };
  if (!unit(o.momentum) || !unit(o.beta1) || !unit(o.beta2) || !(o.epsilon >= 0.0) || !std::isfinite(o.epsilon))
    return fail(h, DCOPF_EINVAL, "momentum, beta1, beta2 must be in [0, 1) and epsilon finite >= 0");
  // AdaGrad / Adam divide by sqrt(state) + eps, and the state is exactly 0 at
  // the start (and stays 0 on a coordinate whose gradient is 0, e.g. an
  // outaged branch): eps = 0 would give 0/0
  if ((o.variant == DCOPF_OPT_ADAGRAD || o.variant == DCOPF_OPT_ADAM) && !(o.epsilon > 0.0))
    return fail(h, DCOPF_EINVAL, "AdaGrad and Adam need epsilon > 0 (SPEC.md:359 suggests 1e-8)");
  if (h->B > 0 && h->path == DCOPF_PATH_SINGLE && o.variant != DCOPF_OPT_PLAIN)
    return fail(h, DCOPF_EINVAL, "optimiser variants run on the cluster and batched paths");
  CK(h, cudaSetDevice(h->device));
  if (h->pt) {
    h->opt = o;
    std::string perr;
    const int prc = ptdf_set_optimizer(h->pt, o, &perr);
    return prc ? fail(h, prc, "%s", perr.c_str()) : DCOPF_OK;
  }
  const int ns_old = opt_nstate(h);
  const dcopf_optimizer o_old = h->opt;
  h->opt = o;
  if (opt_nstate(h) != ns_old) {  // the shared-memory plan holds the state arrays: rebuild it
    const int C_old = h->cplan_C;
    const ClusterPlan plan_old = h->cplan;
    h->cplan_C = 0;
    if (h->B > 0 && h->path == DCOPF_PATH_CLUSTER) {
      // keep the loaded batch's cluster size: the partition (and the KVL
      // storage order of kappa, cluster.cpp) depends on it
      h->force_cluster_C = C_old;
      int rc = configure_cluster(h);
      h->force_cluster_C = 0;
      if (rc) {  // the variant is not taken: the handle stays as it was
        h->opt = o_old;
        h->cplan = plan_old;
        h->cplan_C = C_old;
        return rc;
      }
    }
  }
  if (h->B > 0 && h->path == DCOPF_PATH_BATCHED) {  // the sweep's warp count follows the variant
    int rc = compile_schedule(h, h->T, h->tile_V, h->tile_C);
    if (rc) {
      h->opt = o_old;
      return rc;
    }
  }
  int rc = reset_opt_state(h, nullptr);
  if (!rc) CK(h, cudaDeviceSynchronize());
  return rc;
}

int dcopf_dual_set_stop(dcopf_dual_t h, double tol) {
  if (!h) return fail(nullptr, DCOPF_EINVAL, "null handle");
  if (!(tol >= 0.0) || !std::isfinite(tol)) return fail(h, DCOPF_EINVAL, "tol must be finite and >= 0");
  h->tol = tol;
  if (h->pt) ptdf_set_stop(h->pt, tol);
  return DCOPF_OK;
}

int dcopf_dual_set_target(dcopf_dual_t h, const double *target, void *cuda_stream) {
  if (!h) return fail(nullptr, DCOPF_EINVAL, "null handle");
  if (h->B == 0) return fail(h, DCOPF_ESTATE, "no batch loaded");
  CK(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if (h->pt) {
    std::string perr;
    const int prc = ptdf_set_target(h->pt, target, s, &perr);
    return prc ? fail(h, prc, "%s", perr.c_str()) : DCOPF_OK;
  }
  if (!target) {
    h->has_target = false;
    return DCOPF_OK;
  }
  std::vector<double> t(h->B_pad, std::numeric_limits<double>::infinity());  // padding never hits
  CK(h, cudaMemcpyAsync(t.data(), target, h->B * 8, cudaMemcpyDefault, s));
  CK(h, cudaStreamSynchronize(s));
  for (long b = 0; b < h->B; ++b)
    if (std::isnan(t[b])) return fail(h, DCOPF_EINVAL, "target[%ld] is NaN", b);
  CK(h, cudaMemcpyAsync(h->target, t.data(), h->B_pad * 8, cudaMemcpyHostToDevice, s));
  CK(h, cudaStreamSynchronize(s));  // `t` dies at scope exit
  h->has_target = true;
  return DCOPF_OK;
}

int dcopf_dual_get_first_hit(dcopf_dual_t h, int64_t *hit, void *cuda_stream) {
  if (!h) return fail(nullptr, DCOPF_EINVAL, "null handle");
  if (h->B == 0) return fail(h, DCOPF_ESTATE, "no batch loaded");
  CK(h, cudaSetDevice(h->device));
  if (h->pt) {
    std::string perr;
    const int prc = ptdf_get_first_hit(h->pt, hit, (cudaStream_t)cuda_stream, &perr);
    return prc ? fail(h, prc, "%s", perr.c_str()) : DCOPF_OK;
  }
  return copy_out(h, reinterpret_cast<long long *>(hit), h->hit, (cudaStream_t)cuda_stream);
}

int dcopf_dual_get_info(dcopf_dual_t h, dcopf_info *info) {
  if (!h || !info) return fail(h, DCOPF_EINVAL, "null argument");
  memset(info, 0, sizeof *info);
  if (h->pt) {
    ptdf_info(h->pt, info);
    return DCOPF_OK;
  }
  info->B = h->B;
  info->B_padded = h->B_pad;
  info->path = h->path;
  info->form = h->form;
  info->n_bus = h->n_bus;
  info->n_branch = h->n_br;
  info->n_gen = h->n_gen;
  info->quadratic = h->quadratic;
  info->alg_bytes_per_inst_iter = 8LL * (3LL * h->n_bus + 2LL * h->n_bm_ent * h->bm_C);
  info->bandwidth = h->bandwidth;
  if (h->path == DCOPF_PATH_BATCHED) {
    info->smem_bytes = h->sch.total;
    info->threads_per_block = (h->sched_nw + 1) * 32;
    info->grid = (int)(h->B_pad / h->T) * h->tile_C;
    info->tile_parts = h->tile_C;
    info->lane_instances = h->tile_V;
    info->halo_items = h->sch.halo_a + h->sch.halo_b;
    {
      int mx = 0;
      for (int p = 0; p + 1 < (int)h->sch.part_step0.size(); ++p)
        mx = std::max(mx, h->sch.part_step0[p + 1] - h->sch.part_step0[p]);
      info->steps_per_sweep = mx;
    }
    info->launches_per_iter = 0;
    info->chunk = h->sch.CH;
    info->ring_bus = h->sch.n_lam_slots;
    info->ring_branch = h->sch.n_br_slots;
    info->copies_per_sweep = h->sch.n_copies;
    info->ring_life = h->sch.ring_life;
    info->tile_width = h->T;
  } else if (h->path == DCOPF_PATH_CLUSTER) {
    info->smem_bytes = h->cplan.smem;
    info->threads_per_block = kClusterThreads;
    info->grid = (int)(h->B * h->cplan_C);
    info->state_on_chip = 1;
    info->tile_width = 1;
    info->cluster_size = h->cplan_C;
  } else if (h->path == DCOPF_PATH_SINGLE) {
    info->smem_bytes = h->smem_single;
    info->threads_per_block = 1024;
    info->grid = (int)h->B;
    info->launches_per_iter = 0;
    info->state_on_chip = h->single_smem;
    info->tile_width = 1;
  }
  if (h->path != DCOPF_PATH_CLUSTER) info->cluster_size = 1;
  return DCOPF_OK;
}

int dcopf_dual_compact(dcopf_dual_t h, int64_t *kept, int64_t *n_kept, void *cuda_stream) {
  if (!h) return fail(nullptr, DCOPF_EINVAL, "null handle");
  if (h->B == 0) return fail(h, DCOPF_ESTATE, "no batch loaded");
  if (h->pt) return fail(h, DCOPF_EINVAL, "compaction runs on the sparse forms' paths");
  CK(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  std::vector<int32_t> st(h->B);
  CK(h, cudaMemcpyAsync(st.data(), h->status, h->B * 4, cudaMemcpyDeviceToHost, s));
  CK(h, cudaStreamSynchronize(s));
  std::vector<long long> act;
  for (long b = 0; b < h->B; ++b)
    if (st[b] == DCOPF_INST_OK) act.push_back(b);
  const long nk = (long)act.size();
  if (n_kept) *n_kept = nk;
  if (nk == 0 || nk == h->B) {  // nothing to drop, or nothing left: the batch stays as it is
    if (kept && nk > 0) {
      std::vector<int64_t> id(act.begin(), act.end());
      CK(h, cudaMemcpyAsync(kept, id.data(), nk * 8, cudaMemcpyDefault, s));
      CK(h, cudaStreamSynchronize(s));
    }
    return DCOPF_OK;
  }
  // the kept instances' tiling: the batched path picks V, W, C again for the
  // smaller batch (a shrinking branch-and-bound batch keeps the SMs busy) and
  // moves every tile-major array into the new layout in one gather
  const int T_old = h->T;
  int T = T_old, nV = h->tile_V, nC = h->tile_C;
  std::vector<int> map_lam, map_d, map_br;  // new storage row -> old storage row (identity if unchanged)
  if (h->path == DCOPF_PATH_BATCHED) {
    choose_tiles(h, nk, &nV, &T, &nC);
    const std::vector<int> old_lam = h->hpos_lam, old_d = h->hpos_d, old_br = h->hpos_br;
    if (T != T_old || nV != h->tile_V || nC != h->tile_C) {
      if (int rc0 = compile_schedule(h, T, nV, nC)) {  // (the batch cannot be kept in either layout)
        free_batch(h);
        return rc0;
      }
    }
    auto mk = [](const std::vector<int> &oldp, const std::vector<int> &newp) {
      std::vector<int> m(newp.size());
      for (size_t e = 0; e < newp.size(); ++e) m[newp[e]] = oldp[e];
      return m;
    };
    map_lam = mk(old_lam, h->hpos_lam);
    map_d = mk(old_d, h->hpos_d);
    map_br = mk(old_br, h->hpos_br);
  } else {
    map_lam.resize(h->n_bus);
    map_d.resize(h->n_bus);
    map_br.resize(h->n_bm_ent);
    for (int x = 0; x < h->n_bus; ++x) map_lam[x] = map_d[x] = x;
    for (int x = 0; x < h->n_bm_ent; ++x) map_br[x] = x;
  }
  const long B_pad = (nk + T - 1) / T * T;
  std::vector<long long> slot(B_pad, -1);
  std::copy(act.begin(), act.end(), slot.begin());
  long long *d_slot = nullptr;
  int *d_map = nullptr;
  CK(h, cudaMalloc(&d_slot, B_pad * 8));
  int rc = DCOPF_OK;
  std::vector<void *> old;  // freed after the gathers have run
  auto done = [&](int code) {
    cudaStreamSynchronize(s);
    for (void *p : old) cudaFree(p);
    cudaFree(d_slot);
    cudaFree(d_map);
    return code;
  };
  if (cudaMemcpyAsync(d_slot, slot.data(), B_pad * 8, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return done(fail(h, DCOPF_ECUDA, "compact: slot upload failed"));
  // row maps on the device: [lambda | d | branch block]
  std::vector<int> maps(map_lam);
  maps.insert(maps.end(), map_d.begin(), map_d.end());
  maps.insert(maps.end(), map_br.begin(), map_br.end());
  if (cudaMalloc(&d_map, maps.size() * sizeof(int)) != cudaSuccess ||
      cudaMemcpyAsync(d_map, maps.data(), maps.size() * sizeof(int), cudaMemcpyHostToDevice, s) != cudaSuccess)
    return done(fail(h, DCOPF_ENOMEM, "compact: map upload failed"));
  const int *m_lam = d_map, *m_d = d_map + map_lam.size(), *m_br = d_map + map_lam.size() + map_d.size();
  // tile-major state: multipliers (current buffer), loads, optimiser state
  const int nbr_ent = h->n_bm_ent;
  struct TA {
    double **p;
    int rows, comps;
    const int *map;
  } tiles[] = {{&h->lam[h->cur], h->n_bus, 1, m_lam}, {&h->br[h->cur], nbr_ent, h->bm_C, m_br},
               {&h->load, h->n_bus, 1, m_d},           {&h->os[0], h->n_bus, 1, m_lam},
               {&h->os[1], h->n_bus, 1, m_lam},         {&h->os[2], nbr_ent, h->bm_C, m_br},
               {&h->os[3], nbr_ent, h->bm_C, m_br}};
  for (auto &ta : tiles) {
    if (!*ta.p) continue;
    double *nw = nullptr;
    if (cudaMalloc(&nw, std::max<size_t>((size_t)B_pad * ta.rows * ta.comps, 1) * 8) != cudaSuccess)
      return done(fail(h, DCOPF_ENOMEM, "compact: cudaMalloc failed"));
    k_retile<<<grid_for((size_t)B_pad * ta.rows * ta.comps), 256, 0, s>>>(*ta.p, nw, ta.map, ta.rows, ta.comps, T_old,
                                                                          T, d_slot, B_pad);
    old.push_back(*ta.p);
    *ta.p = nw;
  }
  if (h->path == DCOPF_PATH_BATCHED) {  // the ping-pong partners: contents dead, sized for the new batch
    const int o = 1 - h->cur;
    double *nl = nullptr, *nb = nullptr;
    if (cudaMalloc(&nl, std::max<size_t>((size_t)B_pad * h->n_bus, 1) * 8) != cudaSuccess ||
        cudaMalloc(&nb, std::max<size_t>((size_t)B_pad * nbr_ent * h->bm_C, 1) * 8) != cudaSuccess)
      return done(fail(h, DCOPF_ENOMEM, "compact: cudaMalloc failed"));
    old.push_back(h->lam[o]);
    old.push_back(h->br[o]);
    h->lam[o] = nl;
    h->br[o] = nb;
    if (nC > 1) {  // split tiles: the parts' meeting place
      const size_t tl = (size_t)(B_pad / T), nval = 2 * tl * nC * T;
      if (h->tile_sync_cap < tl) {
        cudaFree(h->d_tile_sync);
        h->d_tile_sync = nullptr;
        h->tile_sync_cap = 0;
        if (cudaMalloc(&h->d_tile_sync, tl * sizeof(unsigned)) != cudaSuccess)
          return done(fail(h, DCOPF_ENOMEM, "compact: cudaMalloc failed"));
        h->tile_sync_cap = tl;
      }
      if (h->part_val_cap < nval) {
        cudaFree(h->d_part_val);
        h->d_part_val = nullptr;
        h->part_val_cap = 0;
        if (cudaMalloc(&h->d_part_val, nval * sizeof(double)) != cudaSuccess)
          return done(fail(h, DCOPF_ENOMEM, "compact: cudaMalloc failed"));
        h->part_val_cap = nval;
      }
    }
  }
  // per-instance rows: bound, best, status, target, hit, outages
  auto gd = [&](double **p, double fill) -> int {
    double *nw = nullptr;
    if (cudaMalloc(&nw, B_pad * 8) != cudaSuccess) return fail(h, DCOPF_ENOMEM, "compact: cudaMalloc failed");
    k_gather_rows<double><<<grid_for(B_pad), 256, 0, s>>>(*p, nw, 1, d_slot, B_pad, fill);
    old.push_back(*p);
    *p = nw;
    return (int)DCOPF_OK;
  };
  const double inf = std::numeric_limits<double>::infinity();
  if (!rc) rc = gd(&h->bound, std::numeric_limits<double>::quiet_NaN());
  if (!rc) rc = gd(&h->best, -inf);
  if (!rc) rc = gd(&h->target, inf);
  if (!rc) {
    int *ns = nullptr, *no = nullptr;
    long long *nh = nullptr;
    const size_t wo = std::max<size_t>((size_t)B_pad * h->max_out, 1);
    if (cudaMalloc(&ns, B_pad * 4) != cudaSuccess || cudaMalloc(&nh, B_pad * 8) != cudaSuccess ||
        cudaMalloc(&no, wo * 4) != cudaSuccess)
      return done(fail(h, DCOPF_ENOMEM, "compact: cudaMalloc failed"));
    k_gather_rows<int><<<grid_for(B_pad), 256, 0, s>>>(h->status, ns, 1, d_slot, B_pad, 0);
    k_gather_rows<long long><<<grid_for(B_pad), 256, 0, s>>>(h->hit, nh, 1, d_slot, B_pad, -1LL);
    if (h->max_out > 0) k_gather_rows<int><<<grid_for(wo), 256, 0, s>>>(h->outs, no, h->max_out, d_slot, B_pad, -1);
    old.push_back(h->status);
    old.push_back(h->hit);
    old.push_back(h->outs);
    h->status = ns;
    h->hit = nh;
    h->outs = no;
  }
  // scratch sized for the old batch stays valid (larger); value / gradients are recomputed
  if (!rc && cudaGetLastError() != cudaSuccess) rc = fail(h, DCOPF_ECUDA, "compact: kernel launch failed");
  if (!rc && kept) {
    std::vector<int64_t> id(act.begin(), act.end());
    if (cudaMemcpyAsync(kept, id.data(), nk * 8, cudaMemcpyDefault, s) != cudaSuccess)
      rc = fail(h, DCOPF_ECUDA, "compact: kept copy failed");
  }
  if (cudaStreamSynchronize(s) != cudaSuccess && !rc) rc = fail(h, DCOPF_ECUDA, "compact: synchronize failed");
  if (!rc) {
    h->B = nk;
    h->B_pad = B_pad;
    h->T = T;
    h->tile_V = nV;
    h->tile_C = nC;
  }
  return done(rc);
}

int dcopf_dual_get_ptdf(dcopf_dual_t h, double *Ha, void *cuda_stream) {
  if (!h) return fail(nullptr, DCOPF_EINVAL, "null handle");
  if (!h->pt) return fail(h, DCOPF_EINVAL, "dcopf_dual_get_ptdf needs the PTDF form");
  if (!Ha) return fail(h, DCOPF_EINVAL, "Ha is NULL");
  CK(h, cudaSetDevice(h->device));
  std::string perr;
  const int prc = ptdf_get_matrix(h->pt, Ha, (cudaStream_t)cuda_stream, &perr);
  return prc ? fail(h, prc, "%s", perr.c_str()) : DCOPF_OK;
}

}  // extern "C"
