// dcopf_dual.cu -- host side of the C ABI declared in include/dcopf_dual.h.
//
// create(): validate + copy the network (SPEC.md:30-50 rules), reverse
// Cuthill-McKee bus order, branch order by (max, min) internal endpoint,
// bus->branch CSR with entries in ascending ORIGINAL branch id (the summation
// order every per-bus sum uses, reading A-19), generators grouped per bus.
// set_instance_batch(): loads -> tile-major device state, outages -> internal
// ids, multipliers 0, best -inf, status OK.
// iterate(): K launches of k_batched<STEP> + one k_batched<FINAL>, or one
// launch of k_single<STEP> that runs all K iterations on chip.
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
#include "dual_kernels.cuh"
#include "pipe_kernel.cuh"
#include "schedule.h"

using namespace dcopf;

static thread_local std::string g_create_error;

struct dcopf_dual_s {
  std::string err;
  int device = 0, form = 0, path_opt = 0, single_max = 128;
  int n_bus = 0, n_br = 0, n_gen = 0, ref_int = 0, quadratic = 0, bandwidth = 0;
  std::vector<int> bus_perm, bus_inv, br_perm, br_inv;  // perm: internal -> original
  std::vector<uint8_t> switchable;                      // original ids; empty = all
  // device topology
  int *d_bus_ptr = nullptr, *d_bus_inc = nullptr, *d_gen_ptr = nullptr, *d_br_s = nullptr,
      *d_br_t = nullptr, *d_bus_perm = nullptr, *d_bus_inv = nullptr, *d_br_perm = nullptr,
      *d_br_inv = nullptr;
  double *d_theta = nullptr, *d_gen_c = nullptr, *d_gen_lo = nullptr, *d_gen_hi = nullptr,
         *d_gen_a = nullptr, *d_br_b = nullptr, *d_br_F = nullptr;
  // batch state
  long B = 0, B_pad = 0;
  int T = 32, path = 0, max_out = 0, cur = 0, single_smem = 0, smem_batched = 0, smem_single = 0;
  double *lam[2] = {nullptr, nullptr}, *br[2] = {nullptr, nullptr}, *load = nullptr;
  double *bound = nullptr, *best = nullptr, *value = nullptr;
  int *status = nullptr, *outs = nullptr, *flag = nullptr;
  double *scratch = nullptr;
  size_t scratch_bytes = 0;
  double *alpha_dev = nullptr, *alpha_pin = nullptr;  // single path schedule (device + pinned staging)
  size_t alpha_cap = 0;
  cudaEvent_t alpha_ev = nullptr;                     // staging may be reused once this fired
  double *g_lam = nullptr, *g_br = nullptr;  // evaluate scratch (internal layout)
  // compiled sweep schedule of the batched path (per network and form)
  Schedule sch;
  int smem_pipe = 0, sched_ok = 0;
  uint8_t *d_prog = nullptr;
  long long *d_prog_off = nullptr;
  int *d_prog_bytes = nullptr, *d_tx_bytes = nullptr, *d_ld_ptr = nullptr, *d_ld_ent = nullptr,
      *d_ld_slot = nullptr;
  std::string sched_err;
};

static const int kPipeWarps = 8;  // consumer warps of k_pipe (+1 producer warp)

static bool batched_path(int path) { return path == DCOPF_PATH_BATCHED || path == DCOPF_PATH_BATCHED_SIMPLE; }

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
  size_t n = std::max<size_t>(src.size(), 1);
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
  size_t g = (n + 255) / 256;
  return (int)std::min<size_t>(std::max<size_t>(g, 1), 148 * 32);
}

// connectivity over a branch subset
bool connected(int n, const std::vector<int> &fr, const std::vector<int> &to,
               const std::vector<char> &use) {
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
    int v = st.back();
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
  if (h->scratch) cudaFree(h->scratch);
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
  cudaFree(h->load);
  cudaFree(h->bound);
  cudaFree(h->best);
  cudaFree(h->value);
  cudaFree(h->status);
  cudaFree(h->outs);
  cudaFree(h->g_lam);
  cudaFree(h->g_br);
  h->load = h->bound = h->best = h->value = h->g_lam = h->g_br = nullptr;
  h->status = h->outs = nullptr;
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

// external [C][n_ent][B] (host or device) -> internal tile-major
int import_ext(dcopf_dual_t h, const double *ext, double *intl, const int *perm, int n_ent, int C,
               cudaStream_t s) {
  const double *src = ext;
  size_t bytes = (size_t)C * n_ent * h->B * sizeof(double);
  if (ext && !is_device_ptr(ext)) {
    int rc = ensure_scratch(h, bytes);
    if (rc) return rc;
    CK(h, cudaMemcpyAsync(h->scratch, ext, bytes, cudaMemcpyDefault, s));
    src = h->scratch;
  }
  size_t total = (size_t)h->B_pad * n_ent * C;
  k_to_internal<<<grid_for(total), 256, 0, s>>>(src, intl, perm, n_ent, C, h->B, h->B_pad, h->T);
  CK(h, cudaGetLastError());
  return DCOPF_OK;
}

int export_ext(dcopf_dual_t h, const double *intl, double *ext, const int *inv, int n_ent, int C,
               cudaStream_t s) {
  if (!ext) return DCOPF_OK;
  size_t bytes = (size_t)C * n_ent * h->B * sizeof(double);
  bool dev = is_device_ptr(ext);
  double *dst = ext;
  if (!dev) {
    int rc = ensure_scratch(h, bytes);
    if (rc) return rc;
    dst = h->scratch;
  }
  size_t total = (size_t)C * n_ent * h->B;
  k_to_external<<<grid_for(total), 256, 0, s>>>(intl, dst, inv, n_ent, C, h->B, h->T);
  CK(h, cudaGetLastError());
  if (!dev) {
    CK(h, cudaMemcpyAsync(ext, dst, bytes, cudaMemcpyDefault, s));
    CK(h, cudaStreamSynchronize(s));
  }
  return DCOPF_OK;
}

// [B] vectors (no permutation): device->device or device->host
template <typename T>
int copy_out(dcopf_dual_t h, T *dst, const T *src, cudaStream_t s) {
  if (!dst) return DCOPF_OK;
  CK(h, cudaMemcpyAsync(dst, src, h->B * sizeof(T), cudaMemcpyDefault, s));
  if (!is_device_ptr(dst)) CK(h, cudaStreamSynchronize(s));
  return DCOPF_OK;
}

size_t batched_smem(int n_bus, int n_br, int form) {
  return (size_t)8 * n_bus + (form == DCOPF_FORM_FLOW_BOX ? (size_t)8 * n_br : 0) + 8 * 32 * 32;
}

size_t single_smem(int n_bus, int n_br, int form, bool state) {
  size_t codes = (size_t)n_bus + n_br;
  size_t st = state ? (size_t)8 * (n_bus + (size_t)n_br * brw(form)) : 0;
  return 512 + st + ((codes + 15) & ~(size_t)15);
}

template <int FORM, int MODE>
int launch_batched(dcopf_dual_t h, const BatchArgs &a, double alpha, long k, cudaStream_t s) {
  auto fn = k_batched<FORM, MODE>;
  fn<<<(unsigned)(h->B_pad / kTile), kWarps * 32, h->smem_batched, s>>>(dev_net(h), a, alpha, k);
  CK(h, cudaGetLastError());
  return DCOPF_OK;
}

template <int FORM, bool SM, int MODE>
int launch_single_t(dcopf_dual_t h, const SingleArgs &a, cudaStream_t s) {
  auto fn = k_single<FORM, SM, MODE>;
  fn<<<(unsigned)h->B, 1024, h->smem_single, s>>>(dev_net(h), a);
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

template <int MODE>
int launch_batched_form(dcopf_dual_t h, const BatchArgs &a, double alpha, long k, cudaStream_t s) {
  if (h->form == DCOPF_FORM_FLOW_BOX) return launch_batched<kFormF2, MODE>(h, a, alpha, k, s);
  return launch_batched<kFormF1, MODE>(h, a, alpha, k, s);
}

// copy the schedule alpha[K] to the device through pinned staging; the staging
// buffer is reused only after the previous copy has executed (event)
int stage_alpha(dcopf_dual_t h, int64_t K, const double *alpha, cudaStream_t s) {
  if (!h->alpha_ev) CK(h, cudaEventCreateWithFlags(&h->alpha_ev, cudaEventDisableTiming));
  CK(h, cudaEventSynchronize(h->alpha_ev));
  if ((size_t)K > h->alpha_cap) {
    cudaFree(h->alpha_dev);
    cudaFreeHost(h->alpha_pin);
    h->alpha_dev = h->alpha_pin = nullptr;
    h->alpha_cap = 0;
    CK(h, cudaMalloc(&h->alpha_dev, K * 8));
    CK(h, cudaMallocHost(&h->alpha_pin, K * 8));
    h->alpha_cap = K;
  }
  if (K > 0) {
    CK(h, cudaMemcpy(h->alpha_pin, alpha, K * 8, cudaMemcpyDefault));
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

// opt every kernel instantiation into the dynamic shared memory it needs
int configure_kernels(dcopf_dual_t h) {
  int rc = DCOPF_OK;
  if (batched_path(h->path)) {
    const int b = h->smem_batched;
    if (!rc && h->sched_ok) rc = set_smem(h, k_pipe<kFormF2, kPipeWarps>, h->smem_pipe);
    if (!rc && h->sched_ok) rc = set_smem(h, k_pipe<kFormF1, kPipeWarps>, h->smem_pipe);
    if (!rc) rc = set_smem(h, k_batched<kFormF2, kModeStep>, b);
    if (!rc) rc = set_smem(h, k_batched<kFormF2, kModeFinal>, b);
    if (!rc) rc = set_smem(h, k_batched<kFormF2, kModeEval>, b);
    if (!rc) rc = set_smem(h, k_batched<kFormF1, kModeStep>, b);
    if (!rc) rc = set_smem(h, k_batched<kFormF1, kModeFinal>, b);
    if (!rc) rc = set_smem(h, k_batched<kFormF1, kModeEval>, b);
  } else {
    const int b = h->smem_single;
    if (!rc) rc = set_smem(h, k_single<kFormF2, true, kModeStep>, b);
    if (!rc) rc = set_smem(h, k_single<kFormF2, true, kModeEval>, b);
    if (!rc) rc = set_smem(h, k_single<kFormF2, false, kModeStep>, b);
    if (!rc) rc = set_smem(h, k_single<kFormF2, false, kModeEval>, b);
    if (!rc) rc = set_smem(h, k_single<kFormF1, true, kModeStep>, b);
    if (!rc) rc = set_smem(h, k_single<kFormF1, true, kModeEval>, b);
    if (!rc) rc = set_smem(h, k_single<kFormF1, false, kModeStep>, b);
    if (!rc) rc = set_smem(h, k_single<kFormF1, false, kModeEval>, b);
  }
  return rc;
}

BatchArgs batch_args(dcopf_dual_t h) {
  BatchArgs a;
  a.lam = h->lam[h->cur];
  a.br = h->br[h->cur];
  a.lam_o = h->lam[1 - h->cur];
  a.br_o = h->br[1 - h->cur];
  a.d = h->load;
  a.outs = h->outs;
  a.max_out = h->max_out;
  a.out_val = h->bound;
  a.best = h->best;
  a.status = h->status;
  a.hist = nullptr;
  a.B = h->B;
  return a;
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
  return a;
}



// Compile and upload the batched sweep schedule (schedule.h).  The chunk size
// starts at DCOPF_CHUNK (default 32) and halves until the kernel's shared
// memory fits two CTAs per SM (else one).  Failure only disables the batched
// path (sched_err says why).
int compile_schedule(dcopf_dual_t h, const NetInternal &ni) {
  int dev_smem = 0;
  CK(h, cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
  int CH = 32, P = 2;
  if (const char *e = getenv("DCOPF_CHUNK")) CH = std::max(1, atoi(e));
  if (const char *e = getenv("DCOPF_PREFETCH")) P = std::max(1, atoi(e));
  const int two_per_sm = dev_smem / 2 - 1024;
  Schedule best;
  bool have = false;
  for (int ch = CH; ch >= 1; ch /= 2) {
    Schedule sc;
    std::string err = build_schedule(ni, ch, P, kPipeWarps, &sc);
    if (!err.empty()) {
      h->sched_err = err;
      return DCOPF_OK;
    }
    if (sc.total <= dev_smem && !have) {
      best = sc;
      have = true;
    }
    if (sc.total <= two_per_sm) {
      best = sc;
      have = true;
      break;
    }
  }
  if (!have) {
    h->sched_err = "no chunk size fits the shared memory";
    return DCOPF_OK;
  }
  h->sch = best;
  h->smem_pipe = best.total;
  std::vector<uint8_t> &pg = h->sch.prog;
  int rc = upload(h, &h->d_prog, pg);
  if (!rc) rc = upload(h, &h->d_prog_off, h->sch.prog_off);
  if (!rc) rc = upload(h, &h->d_prog_bytes, h->sch.prog_bytes);
  if (!rc) rc = upload(h, &h->d_tx_bytes, h->sch.tx_bytes);
  if (!rc) rc = upload(h, &h->d_ld_ptr, h->sch.ld_ptr);
  if (!rc) rc = upload(h, &h->d_ld_ent, h->sch.ld_ent);
  if (!rc) rc = upload(h, &h->d_ld_slot, h->sch.ld_slot);
  if (!rc) {
    h->sched_ok = 1;
    std::vector<uint8_t>().swap(h->sch.prog);  // device copy only
  }
  return rc;
}

}  // namespace

// ============================================================================
extern "C" {

const char *dcopf_dual_last_error(dcopf_dual_t h) {
  return h ? h->err.c_str() : g_create_error.c_str();
}

void dcopf_dual_destroy(dcopf_dual_t h) {
  if (!h) return;
  cudaSetDevice(h->device);
  free_batch(h);
  int *ip[] = {h->d_bus_ptr, h->d_bus_inc, h->d_gen_ptr, h->d_br_s, h->d_br_t,
               h->d_bus_perm, h->d_bus_inv, h->d_br_perm, h->d_br_inv,
               h->d_prog_bytes, h->d_tx_bytes, h->d_ld_ptr, h->d_ld_ent, h->d_ld_slot};
  for (int *p : ip) cudaFree(p);
  double *dp[] = {h->d_theta, h->d_gen_c, h->d_gen_lo, h->d_gen_hi, h->d_gen_a, h->d_br_b, h->d_br_F,
                  h->scratch, h->alpha_dev};
  for (double *p : dp) cudaFree(p);
  cudaFreeHost(h->alpha_pin);
  cudaFree(h->d_prog);
  cudaFree(h->d_prog_off);
  if (h->alpha_ev) cudaEventDestroy(h->alpha_ev);
  cudaFree(h->flag);
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
  if (o.form != DCOPF_FORM_FLOW_BOX && o.form != DCOPF_FORM_LIMIT_ROWS)
    return fail(nullptr, DCOPF_EINVAL, "unknown form %d", o.form);
  if (o.precision != 64 && o.precision != 0)
    return fail(nullptr, DCOPF_EINVAL, "precision %d not supported (fp64 only)", o.precision);
  if (o.path < 0 || o.path > 3) return fail(nullptr, DCOPF_EINVAL, "unknown path %d", o.path);
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
    double lo = net->gen_pmin[g], hi = net->gen_pmax[g], c = net->gen_c[g];
    if (!std::isfinite(lo) || !std::isfinite(hi) || !std::isfinite(c))
      return fail(nullptr, DCOPF_EINVAL, "generator %d data not finite", g);
    if (lo > hi) return fail(nullptr, DCOPF_EINVAL, "generator %d has pmin > pmax", g);
    if (net->gen_a && (!(net->gen_a[g] >= 0.0) || !std::isfinite(net->gen_a[g])))
      return fail(nullptr, DCOPF_EINVAL, "generator %d quadratic cost must be finite and >= 0", g);
  }
  if (net->theta_max)
    for (int i = 0; i < nb; ++i)
      if (!(net->theta_max[i] >= 0.0) || !std::isfinite(net->theta_max[i]))
        return fail(nullptr, DCOPF_EINVAL, "theta_max[%d] must be finite and >= 0", i);
  std::vector<char> use(nl);
  for (int l = 0; l < nl; ++l) use[l] = net->br_b[l] > 0.0;
  if (!connected(nb, fr, to, use)) return fail(nullptr, DCOPF_ETOPOLOGY, "network is disconnected over branches with b > 0");
  if (net->br_switchable) {
    for (int l = 0; l < nl; ++l) use[l] = net->br_b[l] > 0.0 && !net->br_switchable[l];
    if (!connected(nb, fr, to, use))
      return fail(nullptr, DCOPF_ETOPOLOGY, "never-switchable branches do not connect the network");
  }

  dcopf_dual_t h = new dcopf_dual_s();
  h->device = o.device;
  h->form = o.form;
  h->path_opt = o.path;
  h->single_max = o.single_max_batch > 0 ? o.single_max_batch : 128;
  h->n_bus = nb;
  h->n_br = nl;
  h->n_gen = ng;
  h->quadratic = 0;
  if (net->gen_a)
    for (int g = 0; g < ng; ++g) h->quadratic |= net->gen_a[g] > 0.0;
  if (net->br_switchable) h->switchable.assign(net->br_switchable, net->br_switchable + nl);

  // ---- angle box: given, or implied by the flow limits (reading A-2) ----
  std::vector<double> theta(nb, 0.0);
  if (net->theta_max) {
    for (int i = 0; i < nb; ++i) theta[i] = net->theta_max[i];
  } else {
    std::vector<std::vector<std::pair<int, double>>> wadj(nb);
    for (int l = 0; l < nl; ++l) {
      if (!(net->br_b[l] > 0.0)) continue;
      if (net->br_switchable && net->br_switchable[l]) continue;
      double wgt = net->br_fmax[l] / net->br_b[l];
      wadj[fr[l]].push_back({to[l], wgt});
      wadj[to[l]].push_back({fr[l], wgt});
    }
    std::vector<double> dist(nb, std::numeric_limits<double>::infinity());
    typedef std::pair<double, int> QE;
    std::priority_queue<QE, std::vector<QE>, std::greater<QE>> pq;
    dist[net->ref_bus] = 0.0;
    pq.push({0.0, net->ref_bus});
    while (!pq.empty()) {
      QE top = pq.top();
      pq.pop();
      if (top.first > dist[top.second]) continue;
      for (auto &e : wadj[top.second]) {
        double nd = top.first + e.second;
        if (nd < dist[e.first]) {
          dist[e.first] = nd;
          pq.push({nd, e.first});
        }
      }
    }
    theta = dist;
  }
  theta[net->ref_bus] = 0.0;

  // ---- internal numbering: bus order, branch order, CSR, generator map ----
  const char *ord = getenv("DCOPF_ORDER");
  Internalized in;
  std::string ierr = internalize(nb, nl, ng, net->ref_bus, fr.data(), to.data(), net->br_b, net->br_fmax,
                                 theta.data(), net->gen_bus, net->gen_pmin, net->gen_pmax, net->gen_c,
                                 net->gen_a, h->form, ord && std::string(ord) == "rcm", &in);
  if (!ierr.empty()) {
    int rc = fail(nullptr, DCOPF_EINVAL, "%s", ierr.c_str());
    delete h;
    return rc;
  }
  h->bus_perm = in.bus_perm;
  h->bus_inv = in.bus_inv;
  h->br_perm = in.br_perm;
  h->br_inv = in.br_inv;
  h->ref_int = in.net.ref;
  h->bandwidth = in.bandwidth;
  const NetInternal &ni = in.net;
  const std::vector<int> &bus_ptr = ni.bus_ptr, &bus_inc = ni.bus_inc, &gen_ptr = ni.gen_ptr, &bs = ni.bs,
                         &bt = ni.bt;
  const std::vector<double> &gc = ni.gc, &glo = ni.glo, &ghi = ni.ghi, &ga = ni.ga, &th_int = ni.theta,
                            &bb = ni.b, &FF = ni.F;

  cudaError_t e = cudaSetDevice(h->device);
  if (e != cudaSuccess) {
    int rc = fail(nullptr, DCOPF_ECUDA, "cudaSetDevice(%d): %s", h->device, cudaGetErrorString(e));
    delete h;
    return rc;
  }
  int rc = DCOPF_OK;
  if (!rc) rc = upload(h, &h->d_bus_ptr, bus_ptr);
  if (!rc) rc = upload(h, &h->d_bus_inc, bus_inc);
  if (!rc) rc = upload(h, &h->d_gen_ptr, gen_ptr);
  if (!rc) rc = upload(h, &h->d_br_s, bs);
  if (!rc) rc = upload(h, &h->d_br_t, bt);
  if (!rc) rc = upload(h, &h->d_bus_perm, h->bus_perm);
  if (!rc) rc = upload(h, &h->d_bus_inv, h->bus_inv);
  if (!rc) rc = upload(h, &h->d_br_perm, h->br_perm);
  if (!rc) rc = upload(h, &h->d_br_inv, h->br_inv);
  if (!rc) rc = upload(h, &h->d_theta, th_int);
  if (!rc) rc = upload(h, &h->d_gen_c, gc);
  if (!rc) rc = upload(h, &h->d_gen_lo, glo);
  if (!rc) rc = upload(h, &h->d_gen_hi, ghi);
  if (!rc) rc = upload(h, &h->d_gen_a, ga);
  if (!rc) rc = upload(h, &h->d_br_b, bb);
  if (!rc) rc = upload(h, &h->d_br_F, FF);
  if (!rc) rc = compile_schedule(h, ni);
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
  int path = h->path_opt;
  if (path == DCOPF_PATH_AUTO) path = (B <= h->single_max) ? DCOPF_PATH_SINGLE : DCOPF_PATH_BATCHED;
  // shared-memory budget
  int dev_smem = 0;
  CK(h, cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
  size_t need_b = batched_smem(h->n_bus, h->n_br, h->form);
  if (batched_path(path) && need_b > (size_t)dev_smem)
    return fail(h, DCOPF_EINVAL, "batched path needs %zu B shared memory (> %d); use the single path",
                need_b, dev_smem);
  if (path == DCOPF_PATH_BATCHED && !h->sched_ok)
    return fail(h, DCOPF_EINVAL, "batched schedule unavailable: %s", h->sched_err.c_str());
  size_t ss_state = single_smem(h->n_bus, h->n_br, h->form, true);
  size_t ss_nostate = single_smem(h->n_bus, h->n_br, h->form, false);
  if (path == DCOPF_PATH_SINGLE && ss_nostate > (size_t)dev_smem)
    return fail(h, DCOPF_EINVAL, "single path needs %zu B shared memory (> %d)", ss_nostate, dev_smem);

  // outages: validate on the host, convert to internal ids
  std::vector<int> outs_h;
  if (max_out > 0) {
    std::vector<int32_t> raw((size_t)B * max_out);
    CK(h, cudaMemcpy(raw.data(), outages, raw.size() * sizeof(int32_t), cudaMemcpyDefault));
    outs_h.resize(raw.size());
    for (size_t x = 0; x < raw.size(); ++x) {
      int l = raw[x];
      if (l < -1 || l >= h->n_br) return fail(h, DCOPF_EINVAL, "outage id %d out of range", l);
      if (l >= 0 && !h->switchable.empty() && !h->switchable[l])
        return fail(h, DCOPF_EINVAL, "branch %d is not switchable", l);
      outs_h[x] = l < 0 ? -1 : h->br_inv[l];
    }
  }
  const bool reuse = h->lam[0] && h->B == B && h->path == path && h->max_out == max_out;
  if (!reuse) free_batch(h);
  h->path = path;
  h->B = B;
  h->T = batched_path(path) ? kTile : 1;
  h->B_pad = (B + h->T - 1) / h->T * h->T;
  h->max_out = max_out;
  h->cur = 0;
  h->smem_batched = (int)need_b;
  h->single_smem = ss_state <= (size_t)dev_smem;
  h->smem_single = (int)(h->single_smem ? ss_state : ss_nostate);
  const size_t nlam = (size_t)h->B_pad * h->n_bus, nbr = (size_t)h->B_pad * h->n_br * brw(h->form);
  const int nbuf = batched_path(path) ? 2 : 1;
  if (!reuse) {
    for (int i = 0; i < nbuf; ++i) {
      CK(h, cudaMalloc(&h->lam[i], std::max<size_t>(nlam, 1) * 8));
      CK(h, cudaMalloc(&h->br[i], std::max<size_t>(nbr, 1) * 8));
    }
    CK(h, cudaMalloc(&h->load, std::max<size_t>(nlam, 1) * 8));
    CK(h, cudaMalloc(&h->bound, h->B_pad * 8));
    CK(h, cudaMalloc(&h->best, h->B_pad * 8));
    CK(h, cudaMalloc(&h->value, h->B_pad * 8));
    CK(h, cudaMalloc(&h->status, h->B_pad * 4));
    CK(h, cudaMalloc(&h->outs, std::max<size_t>((size_t)h->B_pad * max_out, 1) * 4));
  }
  if (max_out > 0) {
    std::vector<int> padded((size_t)h->B_pad * max_out, -1);
    std::copy(outs_h.begin(), outs_h.end(), padded.begin());
    CK(h, cudaMemcpyAsync(h->outs, padded.data(), padded.size() * 4, cudaMemcpyHostToDevice, s));
    CK(h, cudaStreamSynchronize(s));  // `padded` dies at scope exit
  }
  int rc = configure_kernels(h);
  if (rc) return rc;
  rc = import_ext(h, load, h->load, h->d_bus_perm, h->n_bus, 1, s);
  if (rc) return rc;
  k_fill_d<<<grid_for(nlam), 256, 0, s>>>(h->lam[0], 0.0, nlam);
  k_fill_d<<<grid_for(nbr), 256, 0, s>>>(h->br[0], 0.0, nbr);
  k_fill_d<<<grid_for(h->B_pad), 256, 0, s>>>(h->best, -std::numeric_limits<double>::infinity(), h->B_pad);
  k_fill_d<<<grid_for(h->B_pad), 256, 0, s>>>(h->bound, std::numeric_limits<double>::quiet_NaN(), h->B_pad);
  k_fill_i<<<grid_for(h->B_pad), 256, 0, s>>>(h->status, 0, h->B_pad);
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
  bool hist_host = history && !is_device_ptr(history);
  if (hist_host) {
    int rc = ensure_scratch(h, (size_t)K * h->B * 8 + 8);
    if (rc) return rc;
    hist = h->scratch;
  }
  if (h->path == DCOPF_PATH_BATCHED_SIMPLE) {
    for (int64_t k = 0; k < K; ++k) {
      BatchArgs a = batch_args(h);
      a.hist = hist;
      int rc = launch_batched_form<kModeStep>(h, a, alpha[k], (long)k, s);
      if (rc) return rc;
      h->cur ^= 1;
    }
    BatchArgs a = batch_args(h);
    int rc = launch_batched_form<kModeFinal>(h, a, 0.0, (long)K, s);
    if (rc) return rc;
  } else {
    int rc = stage_alpha(h, K, alpha, s);
    if (rc) return rc;
    if (h->path == DCOPF_PATH_BATCHED) {
      PipeArgs a;
      a.lam0 = h->lam[0];
      a.lam1 = h->lam[1];
      a.br0 = h->br[0];
      a.br1 = h->br[1];
      a.d = h->load;
      a.outs = h->outs;
      a.max_out = h->max_out;
      a.cur = h->cur;
      a.alpha = h->alpha_dev;
      a.K = K;
      a.bound = h->bound;
      a.best = h->best;
      a.status = h->status;
      a.hist = hist;
      a.B = h->B;
      a.n_bus = h->n_bus;
      a.n_br = h->n_br;
      a.ref = h->ref_int;
      a.prog = h->d_prog;
      a.prog_off = h->d_prog_off;
      a.prog_bytes = h->d_prog_bytes;
      a.tx_bytes = h->d_tx_bytes;
      a.ld_ptr = h->d_ld_ptr;
      a.ld_ent = h->d_ld_ent;
      a.ld_slot = h->d_ld_slot;
      const Schedule &sc = h->sch;
      a.nch = sc.nch;
      a.S = sc.S;
      a.off_bar = sc.off_bar;
      a.off_red = sc.off_red;
      a.off_frz = sc.off_frz;
      a.off_obm = sc.off_obm;
      a.off_prog = sc.off_prog;
      a.prog_stride = (sc.max_prog_bytes + 127) & ~127;
      a.off_brp = sc.off_brp;
      a.off_lamp = sc.off_lamp;
      a.off_dp = sc.off_dp;
      a.off_th = sc.off_th;
      a.off_fc = sc.off_fc;
      a.dbg = nullptr;
      if (getenv("DCOPF_DEBUG_PROGRESS")) {
        static int *dbg_host = nullptr;
        if (!dbg_host) {
          CK(h, cudaHostAlloc(&dbg_host, 64 * sizeof(int), cudaHostAllocMapped));
          memset(dbg_host, 0xff, 64 * sizeof(int));
        }
        int *dev = nullptr;
        CK(h, cudaHostGetDevicePointer(&dev, dbg_host, 0));
        a.dbg = dev;
        fprintf(stderr, "DCOPF_DEBUG_PROGRESS host=%p\n", (void *)dbg_host);
      }
      const unsigned grid = (unsigned)(h->B_pad / kTile);
      const unsigned threads = (kPipeWarps + 1) * 32;
      if (h->form == DCOPF_FORM_FLOW_BOX)
        k_pipe<kFormF2, kPipeWarps><<<grid, threads, h->smem_pipe, s>>>(a);
      else
        k_pipe<kFormF1, kPipeWarps><<<grid, threads, h->smem_pipe, s>>>(a);
      CK(h, cudaGetLastError());
      h->cur = (int)((h->cur + K) & 1);
    } else {
      SingleArgs a = single_args(h);
      a.alpha = h->alpha_dev;
      a.K = K;
      a.hist = hist;
      rc = launch_single<kModeStep>(h, a, s);
      if (rc) return rc;
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
  const int cur = batched_path(h->path) ? h->cur : 0;
  int rc = export_ext(h, h->lam[cur], lambda, h->d_bus_inv, h->n_bus, 1, s);
  if (!rc) rc = export_ext(h, h->br[cur], branch, h->d_br_inv, h->n_br, brw(h->form), s);
  return rc;
}

int dcopf_dual_set_multipliers(dcopf_dual_t h, const double *lambda, const double *branch, void *cuda_stream) {
  if (!h) return fail(nullptr, DCOPF_EINVAL, "null handle");
  if (h->B == 0) return fail(h, DCOPF_ESTATE, "no batch loaded");
  CK(h, cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const int cur = batched_path(h->path) ? h->cur : 0;
  // validate into scratch-free temporaries: import, then check the internal copy
  const size_t nlam = (size_t)h->B_pad * h->n_bus, nbr = (size_t)h->B_pad * h->n_br * brw(h->form);
  double *tl = nullptr, *tb = nullptr;
  CK(h, cudaMalloc(&tl, std::max<size_t>(nlam, 1) * 8));
  CK(h, cudaMalloc(&tb, std::max<size_t>(nbr, 1) * 8));
  int rc = DCOPF_OK;
  if (lambda) rc = import_ext(h, lambda, tl, h->d_bus_perm, h->n_bus, 1, s);
  if (!rc && branch) rc = import_ext(h, branch, tb, h->d_br_perm, h->n_br, brw(h->form), s);
  if (!rc) {
    int bad = 0;
    cudaMemsetAsync(h->flag, 0, sizeof(int), s);
    if (lambda) k_check_mu<<<grid_for(nlam), 256, 0, s>>>(tl, nlam, h->flag, 0);
    if (branch) k_check_mu<<<grid_for(nbr), 256, 0, s>>>(tb, nbr, h->flag, h->form == DCOPF_FORM_LIMIT_ROWS);
    cudaMemcpyAsync(&bad, h->flag, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = fail(h, DCOPF_ECUDA, "set_multipliers: %s", cudaGetErrorString(e));
    else if (bad) rc = fail(h, DCOPF_EINVAL, "multipliers must be finite and mu >= 0 (SPEC.md:239)");
  }
  if (!rc) {
    if (lambda) cudaMemcpyAsync(h->lam[cur], tl, nlam * 8, cudaMemcpyDeviceToDevice, s);
    if (branch) cudaMemcpyAsync(h->br[cur], tb, nbr * 8, cudaMemcpyDeviceToDevice, s);
    cudaError_t e = cudaStreamSynchronize(s);
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
  const size_t nlam = (size_t)h->B_pad * h->n_bus, nbr = (size_t)h->B_pad * h->n_br * brw(h->form);
  if (!h->g_lam) CK(h, cudaMalloc(&h->g_lam, std::max<size_t>(nlam, 1) * 8));
  if (!h->g_br) CK(h, cudaMalloc(&h->g_br, std::max<size_t>(nbr, 1) * 8));
  int rc;
  if (batched_path(h->path)) {
    BatchArgs a = batch_args(h);
    a.lam_o = h->g_lam;
    a.br_o = h->g_br;
    a.out_val = h->value;
    rc = launch_batched_form<kModeEval>(h, a, 0.0, 0, s);
  } else {
    SingleArgs a = single_args(h);
    a.grad_lam = h->g_lam;
    a.grad_br = h->g_br;
    a.value = h->value;
    rc = launch_single<kModeEval>(h, a, s);
  }
  if (rc) return rc;
  rc = copy_out(h, value, h->value, s);
  if (!rc) rc = export_ext(h, h->g_lam, grad_lambda, h->d_bus_inv, h->n_bus, 1, s);
  if (!rc) rc = export_ext(h, h->g_br, grad_branch, h->d_br_inv, h->n_br, brw(h->form), s);
  return rc;
}

int dcopf_dual_get_info(dcopf_dual_t h, dcopf_info *info) {
  if (!h || !info) return fail(h, DCOPF_EINVAL, "null argument");
  memset(info, 0, sizeof *info);
  info->B = h->B;
  info->B_padded = h->B_pad;
  info->path = h->path;
  info->form = h->form;
  info->n_bus = h->n_bus;
  info->n_branch = h->n_br;
  info->n_gen = h->n_gen;
  info->quadratic = h->quadratic;
  info->alg_bytes_per_inst_iter =
      8LL * (3LL * h->n_bus + (h->form == DCOPF_FORM_LIMIT_ROWS ? 4LL : 2LL) * h->n_br);
  info->bandwidth = h->bandwidth;
  info->chunk = h->sch.CH;
  info->ring_bus = h->sch.n_lam_slots;
  info->ring_branch = h->sch.n_br_slots;
  if (h->path == DCOPF_PATH_BATCHED) {
    info->smem_bytes = h->smem_pipe;
    info->threads_per_block = (kPipeWarps + 1) * 32;
    info->grid = (int)(h->B_pad / kTile);
    info->launches_per_iter = 0;
  } else if (h->path == DCOPF_PATH_BATCHED_SIMPLE) {
    info->smem_bytes = h->smem_batched;
    info->threads_per_block = kWarps * 32;
    info->grid = (int)(h->B_pad / kTile);
    info->launches_per_iter = 1;
  } else if (h->path == DCOPF_PATH_SINGLE) {
    info->smem_bytes = h->smem_single;
    info->threads_per_block = 1024;
    info->grid = (int)h->B;
    info->launches_per_iter = 0;  // one launch for all K iterations
    info->state_on_chip = h->single_smem;
  }
  return DCOPF_OK;
}

}  // extern "C"
