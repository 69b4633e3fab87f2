/*
 * dcopf_dual.h -- C ABI of the B200 (sm_100a) projected dual-ascent library
 * for DC optimal power flow, after arXiv 2406.13191 ("PAPER.md").
 *
 * What one iteration computes (PAPER.md line numbers):
 *   S1  inner cost vectors from the multipliers by sparse incidence products:
 *       r_g = c_g + lambda_{bus(g)}, q_l = nu_l - (lambda_s - lambda_t),
 *       w_i = -sum_{l at i} sigma_il b_l nu_l                   (Eq. 3)
 *   S2  closed-form inner minimiser over the generator / flow / angle boxes:
 *       bound selection for linear cost (dual norm, Eq. 7b PAPER.md:157-160,
 *       App. A2), clip(-r/(2a), pmin, pmax) for quadratic
 *       cost (Eq. 15 PAPER.md:230-236 with s maximised out); sign(0) -> midpoint
 *   S3  dual value g (a valid lower bound, Remarks 1-2
 *       PAPER.md:164-172, 237-242) and its gradient = constraint residual at
 *       that minimiser
 *   S4  y <- y + alpha_k grad, then mu <- max(mu, 0) (Alg. 1 line
 *       "mu <- max(mu,0)" PAPER.md:264).  Jacobi: all of S1-S3 read y_k.
 *
 * The primal problem is PAPER.md:94-101 (Eq. 1) in sparse B-theta form:
 *   min sum_g a_g p_g^2 + c_g p_g  s.t.  G p - A^T f = d (lambda),
 *   f = diag(b) A theta, |f| <= F, pmin <= p <= pmax, |theta_i| <= Theta_i,
 *   theta_ref = 0.
 * Form F2 (DCOPF_FORM_FLOW_BOX, default) dualises Kirchhoff with free nu and
 * keeps p, f, theta as boxes.  Form F1 (DCOPF_FORM_LIMIT_ROWS) keeps p, theta
 * as boxes and dualises the 2 n_branch limit rows +-diag(b) A theta <= F with
 * mu+, mu- >= 0 (the C x <= d rows of Eq. 2).
 *
 * Conventions for every call:
 *   - All functions return an int status (DCOPF_OK or a negative code) and
 *     never throw across the ABI; dcopf_dual_last_error() gives the message.
 *   - Numbering in and out is the caller's ORIGINAL numbering; the library
 *     reorders buses and branches internally and never exposes that order.
 *   - "array pointers" may be host or device memory (resolved through CUDA
 *     unified addressing, cudaMemcpyDefault); device pointers avoid a copy.
 *     The caller owns every buffer it passes; the handle owns all device state.
 *   - Every call is ordered on the CUDA stream it is given (NULL = legacy
 *     default stream) and does not synchronise the device, except where a
 *     host buffer forces a synchronous copy or create/set validates inputs.
 *   - Per-instance arrays are instance-contiguous: element (entity e,
 *     instance j) of an [n_entity][B] array is at e*B + j.
 *   - A handle is not thread-safe; independent handles are independent.
 *   - Results are deterministic: identical inputs and schedule give bitwise
 *     identical outputs on the same GPU model.  Multipliers, status and first
 *     hits are also bitwise independent of how a batch is split across
 *     handles / GPUs and of the batched path's tiling (instances never
 *     interact; every per-entity sum has the oracle's fixed order); the dual
 *     value is a fixed-order sum per tiling, so across tilings bound / best
 *     agree to rounding order (reading A-32).
 */
#ifndef DCOPF_DUAL_H
#define DCOPF_DUAL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dcopf_dual_s *dcopf_dual_t; /* opaque; owned by the library */

enum {
  DCOPF_OK = 0,
  DCOPF_EINVAL = -1,    /* bad argument / out-of-range index / malformed data */
  DCOPF_ETOPOLOGY = -2, /* network (or the never-switchable part) disconnected */
  DCOPF_ECUDA = -3,     /* a CUDA runtime call failed (message has the error) */
  DCOPF_ENOMEM = -4,    /* device allocation failed */
  DCOPF_ESTATE = -5     /* call out of order (e.g. iterate before set_instance_batch) */
};

enum {
  DCOPF_FORM_FLOW_BOX = 0,   /* F2 */
  DCOPF_FORM_LIMIT_ROWS = 1, /* F1 */
  DCOPF_FORM_CYCLE = 2,      /* KVL: angle-free cycle-basis twin of the paper's PTDF constraint
                                (Eq. 1): boxes p, |f| <= F; KCL
                                dualised with lambda, Kirchhoff's voltage law on the fundamental
                                cycles of a canonical spanning tree (reading A-28) with
                                free kappa[n_cycles], n_cycles = n_branch - n_bus + 1.  Cluster and
                                batched paths; the branch block of get/set_multipliers and evaluate
                                is kappa[n_cycles][B] in canonical cycle order; outages must be
                                switchable branches (the tree is built from the never-switchable
                                ones) */
  DCOPF_FORM_PTDF = 3        /* the paper's dense-PTDF problem literally (Eq. 1;
                                SURVEY.md NEXT-4), for LOAD-ONLY batches on a fixed topology:
                                  min a p^2 + c p  s.t.  1^T p = 1^T d (lambda, one per instance),
                                  -F <= H_a (G p - d) <= F (mu+, mu- >= 0), pmin <= p <= pmax,
                                H = Omega E (E^T Omega E)^{-1} with a zero slack column,
                                built by the library at create (see dcopf_dual_get_ptdf).  Runs on
                                DCOPF_PATH_DENSE only: per ascent step two fp64 GEMMs over the batch
                                (tensor-core DMMA) with the inner minimiser, dual value, gradient and
                                projected step fused into their epilogues.  Multiplier layouts:
                                lambda[1][B]; branch block mu+[n_branch][B] followed by
                                mu-[n_branch][B] (as F1).  Outages are rejected (EINVAL): one H_a
                                serves the whole batch.  theta_max and br_switchable are ignored. */
};

/* per-instance status: a diverged instance is frozen; the
 * others continue.  DIVERGED = g(y_k) non-finite or |g(y_k)| > 1e15; the step
 * of that iteration is still taken, no later step is (y frozen at y_{k+1}),
 * best keeps only valid values (reading A-23). */
enum { DCOPF_INST_OK = 0, DCOPF_INST_DIVERGED = 1, DCOPF_INST_CONVERGED = 2 };

/* kernel path selection */
enum {
  DCOPF_PATH_AUTO = 0,    /* CLUSTER when B <= single_max_batch (SINGLE if the partition does
                             not fit), else BATCHED */
  DCOPF_PATH_BATCHED = 1, /* tiles of W <= 32 V instances (V = 2 or 4 per lane), each tile swept by
                             C = 1..16 CTAs over contiguous parts of the network (DFS tree bus
                             order), one persistent (cooperative when C > 1) launch for all K
                             iterations: a TMA-fed sweep over a host-compiled schedule; V, W, C
                             chosen per batch so the launch is one wave on the SMs */
  DCOPF_PATH_SINGLE = 2,  /* one persistent CTA per instance running all K iterations on chip */
  DCOPF_PATH_CLUSTER = 3, /* one thread-block cluster of up to 16 CTAs per instance, the network
                             partitioned over the CTAs' shared memories (distributed shared
                             memory), all K iterations in one launch */
  DCOPF_PATH_DENSE = 4    /* DCOPF_FORM_PTDF only (and AUTO resolves to it): batched fp64 GEMMs,
                             3 launches per ascent step, batch padded to a multiple of 128 */
};

/* Network description.  Host pointers,
 * copied and validated at create; the caller keeps ownership. */
typedef struct {
  int32_t n_bus, n_branch, n_gen, ref_bus;
  const int32_t *br_from, *br_to;   /* [n_branch] endpoints, original bus ids, from != to */
  const double *br_b, *br_fmax;     /* [n_branch] susceptance b >= 0, flow limit F >= 0 (p.u.) */
  const double *theta_max;          /* [n_bus] angle-box half widths >= 0 (theta_ref is
                                       pinned to 0 whatever is given); NULL => the library
                                       computes the box implied by the flow limits:
                                       Theta_i = shortest path ref->i with weights F_l/b_l
                                       over never-switchable branches (A-2) */
  const int32_t *gen_bus;           /* [n_gen] bus of each generator (several per bus allowed) */
  const double *gen_pmin, *gen_pmax;/* [n_gen] pmin <= pmax */
  const double *gen_c;              /* [n_gen] linear cost */
  const double *gen_a;              /* [n_gen] quadratic cost a >= 0, or NULL (linear) */
  const uint8_t *br_switchable;     /* [n_branch] nonzero = an instance may take it out,
                                       or NULL (any branch may be out; no check) */
} dcopf_network_desc;

typedef struct {
  int32_t form;             /* DCOPF_FORM_* */
  int32_t precision;        /* 64 (fp64; the only mode in this build) */
  int32_t device;           /* CUDA device ordinal */
  int32_t path;             /* DCOPF_PATH_* */
  int32_t single_max_batch; /* AUTO threshold (cluster path for B <= it); <= 0 means 56 (measured
                               crossover on the 10k-bus network) */
  int32_t tile_parts;       /* batched path: CTAs per instance tile (1..16), each
                               sweeping a contiguous part of the network; cluster path: CTAs per
                               instance cluster (1, 2, 4, 8, 16); 0 = chosen per batch / network.
                               (SURVEY.md §8(b) also lists a "deterministic" flag: every path is
                               deterministic, so it is not an option -- DESIGN.md reading A-31) */
  int32_t lane_instances;   /* batched path: instances per lane, 2 or 4 (F1: 2); 0 = chosen per
                               batch */
  int32_t reserved[1];      /* zero */
} dcopf_options;

/* Create a handle: validates and copies the network, orders the buses
 * internally (depth-first over a breadth-first spanning tree from the
 * reference bus, smallest subtree first: neighbours stay close, which keeps
 * the batched path's shared-memory window and the cluster path's cross-CTA
 * traffic small), builds the bus->branch incidence (CSR, entries in
 * ascending original branch id) and the generator map, and -- KVL form --
 * the canonical cycle basis (reading A-28).
 * Errors: EINVAL (sizes, indices, self loops, negative b/F/Theta/a,
 * pmin > pmax, non-finite data, bad options), ETOPOLOGY (disconnected over
 * b > 0, or over never-switchable branches when br_switchable is given),
 * ECUDA / ENOMEM.  *out is NULL on failure. */
int dcopf_dual_create(const dcopf_network_desc *net, const dcopf_options *opt, dcopf_dual_t *out);

/* Load B instances that share the network: load[n_bus][B] (p.u.), and per
 * instance up to max_out outaged branch ids (original numbering, -1 padded),
 * outages[B][max_out] or NULL (max_out = 0).  An outaged branch has b = F = 0
 * for that instance (A-16).  Resets the multipliers to 0, best to
 * -inf, status to OK.  B >= 1; max_out <= 8.  Errors: EINVAL (B < 1,
 * max_out out of range, an id out of range or not switchable), ECUDA,
 * ENOMEM. */
int dcopf_dual_set_instance_batch(dcopf_dual_t h, int64_t B, const double *load,
                                  const int32_t *outages, int32_t max_out, void *cuda_stream);

/* Run K ascent steps with the explicit schedule alpha[K] (host array, any
 * values; reading A-9), then evaluate once more at y_K:
 *   bound = g(y_K), best = max over valid g(y_k), k in [0, K] (and over
 *   previous calls since set_instance_batch).
 * history: NULL or an [K][B] array that receives g(y_k), k = 0..K-1 (device
 * or host).  K = 0 only evaluates.  Errors: ESTATE (no batch loaded),
 * EINVAL (K < 0, alpha NULL with K > 0), ECUDA. */
int dcopf_dual_iterate(dcopf_dual_t h, int64_t K, const double *alpha, double *history,
                       void *cuda_stream);

/* bound[B] = g(y) at the last evaluation, best[B], status[B]; any may be NULL.
 * The bound is the dual value of Eq. 7b at the current
 * multipliers: a valid lower bound on the optimum of Eq. 1 (weak duality,
 * PAPER.md:135; Remarks 1-2) for any lambda, nu and mu >= 0;
 * best is the running maximum over the iterates (Algorithm 1's gamma,
 * PAPER.md:265).  Layout: instance b at index b (original batch order).
 * Errors: ESTATE (no batch), ECUDA. */
int dcopf_dual_get_bound(dcopf_dual_t h, double *bound, double *best, int32_t *status,
                         void *cuda_stream);

/* The multipliers y_K after the last iterate() (Eq. 3: lambda
 * for the power balance rows, and for the branch rows nu (F2, Kirchhoff
 * f = diag(b) A theta), mu+ / mu- >= 0 (F1 and PTDF, the limit rows of Eq. 2,
 * PAPER.md:111-118) or kappa (KVL)): lambda[n_bus][B] (PTDF: [1][B]); branch:
 * F2 nu[n_branch][B]; F1 / PTDF mu+[n_branch][B] followed by mu-[n_branch][B];
 * KVL kappa[n_cycles][B].  Original numbering, instance-contiguous.  Either
 * may be NULL.  Errors: ESTATE (no batch), ECUDA. */
int dcopf_dual_get_multipliers(dcopf_dual_t h, double *lambda, double *branch, void *cuda_stream);

/* Warm start / checkpoint restore: same layouts as get_multipliers.  Any
 * lambda (and nu) with mu >= 0 is dual feasible, so the anytime-bound property
 * is kept.  Does not reset best or status.
 * Errors: EINVAL (a non-finite value; F1 and some mu < 0; F2 and
 * a nonzero nu on one of the instance's outaged branches -- such a branch has
 * b = F = 0, its nu does not enter the instance's dual, and the batched kernel
 * relies on it staying 0, reading A-24), ESTATE. */
int dcopf_dual_set_multipliers(dcopf_dual_t h, const double *lambda, const double *branch,
                               void *cuda_stream);

/* Value and gradient at the current multipliers, no step and no change to
 * best/status: value[B] = g(y) (Eq. 7b), grad_lambda[n_bus][B]
 * and grad_branch = the constraint residuals at the inner minimiser (the
 * gradient of the dual function, PAPER.md:245 and Alg. 1 PAPER.md:255-256 with
 * the sign of Eq. 7b, reading A-5), in the layout of
 * get_multipliers; for F1 the unprojected d g / d mu.  Any may be NULL.
 * Errors: ESTATE (no batch), ECUDA, ENOMEM. */
int dcopf_dual_evaluate(dcopf_dual_t h, double *value, double *grad_lambda, double *grad_branch,
                        void *cuda_stream);

/* Gradient-based-optimisation variant of the ascent step ("Adam
 * ... AdaGrad ... Gradient with Momentum", Algorithm 1 PAPER.md:247-272;
 * SURVEY.md NEXT-2), per multiplier coordinate y with gradient g and the
 * schedule's step a_k, followed by mu <- max(mu, 0):
 *   PLAIN        y <- y + a_k g                                  (default)
 *   GDM          v <- rho v + a_k g; y <- y + v; y <- y + a_k g   (Algorithm 1 as printed)
 *   GDM_CLASSIC  v <- rho v + a_k g; y <- y + v
 *   ADAGRAD      G <- G + g g; y <- y + (a_k g) / (sqrt(G) + eps)
 *   ADAM         m <- b1 m + (1-b1) g; v <- b2 v + (1-b2)(g g);
 *                y <- y + (a_k (m / (1 - b1^t))) / (sqrt(v / (1 - b2^t)) + eps),
 *                t = steps since the state was reset (b^t by repeated products)
 * Optimiser state starts at 0 and persists across iterate() calls; it is reset
 * by set_instance_batch() and by this call.  Variants other than PLAIN run on
 * the cluster path (state in shared memory) and the batched path (state rows
 * in HBM beside the multipliers, read and written at the update: 1 or 2 more
 * rows per multiplier and iteration); not on DCOPF_PATH_SINGLE (iterate()
 * fails with ESTATE).  Errors: EINVAL (unknown variant, rho/b1/b2 outside
 * [0, 1), eps < 0 (AdaGrad / Adam: eps <= 0), the cluster partition plus the
 * optimiser state does not fit shared memory, or -- a batch loaded on the
 * batched path -- the loaded schedule's chunk does not fit with the optimiser
 * kernels' 1.2 KB shared-memory block; set the variant before
 * set_instance_batch() then).  On an error the handle is unchanged. */
enum { DCOPF_OPT_PLAIN = 0, DCOPF_OPT_GDM = 1, DCOPF_OPT_GDM_CLASSIC = 2, DCOPF_OPT_ADAGRAD = 3, DCOPF_OPT_ADAM = 4 };
typedef struct {
  int32_t variant;   /* DCOPF_OPT_* */
  int32_t reserved;  /* zero */
  double momentum;   /* rho (GDM variants) */
  double beta1, beta2;
  double epsilon;    /* AdaGrad / Adam guard (SPEC.md:359 suggests 1e-8) */
} dcopf_optimizer;
int dcopf_dual_set_optimizer(dcopf_dual_t h, const dcopf_optimizer *opt);

/* Per-instance stopping rule of Algorithm 1 ("if
 * |gamma^(i+1) - gamma^(i)| < tolerance: Stop"): with tol > 0,
 * an instance whose consecutive dual values within one iterate() call differ by
 * less than tol gets status DCOPF_INST_CONVERGED and is frozen exactly like a
 * diverged one (the step of the detecting iteration is taken, no later one;
 * DESIGN.md reading A-29); the other instances of the batch go on.  tol = 0
 * (default) disables it.  Persists until changed.  Errors: EINVAL (tol < 0 or
 * not finite). */
int dcopf_dual_set_stop(dcopf_dual_t h, double tol);

/* Time to gap (BASELINE.json metric "time to 1e-3 gap"):
 * per-instance thresholds target[B] (host or device; NULL clears them).  The
 * kernels then record, per instance, the index k of the FIRST evaluation whose
 * running best bound satisfies best_k >= target, counting the evaluations
 * g(y_0), g(y_1), ... of every iterate() call since set_instance_batch()
 * continuously (a call of K steps covers indices base .. base+K, base = the
 * total number of steps taken before it; its first evaluation re-evaluates the
 * point the previous call ended on).  Cleared (no target, hit = -1) by
 * set_instance_batch().  The threshold is a caller-supplied number (e.g.
 * (1 - 1e-3) x a reference bound); the library never computes one.
 * Errors: EINVAL (a NaN target), ESTATE. */
int dcopf_dual_set_target(dcopf_dual_t h, const double *target, void *cuda_stream);

/* hit[B] (int64): the first evaluation index reaching the target, or -1. */
int dcopf_dual_get_first_hit(dcopf_dual_t h, int64_t *hit, void *cuda_stream);

/* Batch compaction (the branch-and-bound use of the bound,
 * PAPER.md:25, 63): drops every instance whose status is DIVERGED or CONVERGED
 * and packs the remaining (OK) instances, in their current order, into a
 * smaller batch -- fewer tiles / clusters / CTAs per later iterate() call.
 * Each kept instance keeps its multipliers, optimiser state, best, target and
 * first hit, loads and outages, so its later results are bitwise those of an
 * uncompacted run.  kept[j] (host or device, capacity = B before the call, or
 * NULL) receives the pre-compaction index of new instance j; *n_kept (or NULL)
 * their number.  Afterwards every call sees the packed batch (B = n_kept):
 * read the retiring instances' results BEFORE compacting.  If no instance is
 * frozen, or none is OK, the batch is left as it is (n_kept = B, resp. 0).
 * Not for the PTDF form (EINVAL).  Errors: ESTATE (no batch), ENOMEM, ECUDA. */
int dcopf_dual_compact(dcopf_dual_t h, int64_t *kept, int64_t *n_kept, void *cuda_stream);

/* Static facts about the handle, for reporting. */
typedef struct {
  int64_t B;                      /* instances loaded (0 before set_instance_batch) */
  int64_t B_padded;               /* instances actually computed (batched path pads to a multiple of W) */
  int32_t path;                   /* DCOPF_PATH_BATCHED or DCOPF_PATH_SINGLE in use */
  int32_t form;
  int32_t n_bus, n_branch, n_gen, quadratic;
  int64_t alg_bytes_per_inst_iter;/* algorithmic HBM bytes per instance-iteration:
                                     F2 8(3 n_bus + 2 n_branch), F1 8(3 n_bus + 4 n_branch) */
  int32_t bandwidth;              /* bus bandwidth of the internal (RCM) order */
  int32_t smem_bytes;             /* dynamic shared memory of the iteration kernel (dense path,
                                     B <= 4: > 0 only when iterate() takes the B = 1 single-read
                                     step: plain / GDM / GDM-classic steps) */
  int32_t threads_per_block;
  int32_t grid;                   /* CTAs per iteration launch */
  int32_t launches_per_iter;      /* kernel launches per ascent step (0: one launch per call) */
  int32_t state_on_chip;          /* single path: multipliers resident in shared memory */
  int32_t chunk;                  /* batched path: buses per schedule chunk */
  int32_t ring_bus, ring_branch;  /* batched path: shared-memory slots for lambda / branch rows */
  int32_t tile_width;             /* instances per CTA (batched W; 1 for the single path) */
  int32_t copies_per_sweep;       /* batched path: bulk copies per tile per iteration */
  int32_t ring_life;              /* batched path: rows live <= this many steps use the rings */
  int32_t cluster_size;           /* cluster path: CTAs per instance (1 otherwise) */
  int32_t tile_parts;             /* batched path: CTAs per instance tile (each sweeps a part of the
                                     network; the tile's parts meet once per iteration) */
  int32_t lane_instances;         /* batched path: instances per lane (2 or 4) */
  int32_t halo_items;             /* batched path: codes recomputed per sweep by the parts of a tile */
  int32_t steps_per_sweep;        /* batched path: pipeline steps of the longest part */
} dcopf_info;
int dcopf_dual_get_info(dcopf_dual_t h, dcopf_info *info);

/* DCOPF_FORM_PTDF: the PTDF matrix the handle iterates with, H_a[n_branch][n_bus]
 * (row-major, original ids), into a host or device buffer.  The
 * library builds it from a spanning tree and its fundamental cycles (reading
 * A-28): H_a = T - C^T (C X C^T)^{-1} C X T, T the tree flows of "inject 1 at
 * bus i, withdraw at the slack", C the signed cycle incidence, X = diag(1/b);
 * a branch with b = 0 carries no flow (zero row).  Errors: EINVAL (another
 * form, Ha NULL), ECUDA. */
int dcopf_dual_get_ptdf(dcopf_dual_t h, double *Ha, void *cuda_stream);

const char *dcopf_dual_last_error(dcopf_dual_t h); /* never NULL; h may be NULL (last create error) */
void dcopf_dual_destroy(dcopf_dual_t h);           /* NULL is a no-op */

/* Measurement-only environment variables (read by the library; never needed
 * for correct results, each selects among variants that are all
 * parity-tested; DESIGN.md §6 records what they measured):
 *   DCOPF_PTDF_SKINNY=0|1   dense path: force the GEMM or the matrix-vector kernels
 *   DCOPF_PTDF_SPLITK=0     dense path: disable the split-K GEMM1 for medium batches
 *   DCOPF_PTDF_FUSED=0      dense path, B = 1: the two-pass matrix-vector kernels instead of the
 *                           single-read step
 *   DCOPF_PTDF_GROUP=n, DCOPF_PTDF_SPLIT=1|2   dense path: column-group size / stream split
 *   DCOPF_CLUSTER_DEBUG=n   cluster path: skip phases (synchronisation floor, timing only;
 *                           results are NOT the dual iteration when set)
 * The batched path's tiling is an option (dcopf_options tile_parts / lane_instances), not
 * an environment variable. */

#ifdef __cplusplus
}
#endif
#endif /* DCOPF_DUAL_H */
