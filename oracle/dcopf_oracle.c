/*
 * dcopf_oracle.c -- plain, slow, obviously-correct fp64 CPU ORACLE for the
 * projected dual ascent of arXiv 2406.13191, written from the paper
 * and SURVEY.md §8(c).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_2406_13191_b200/csrc, include/), and neither side includes the other.
 *
 * What it computes, per instance, in ORIGINAL numbering, single-threaded
 * (OpenMP only across independent instances):
 *
 *   Primal (Eq. 1 written sparsely, B-theta form):
 *     min  sum_g a_g p_g^2 + c_g p_g
 *     s.t. G p - A^T f = d                    (KCL, multiplier lambda, free)
 *          f = diag(b) A theta                (Kirchhoff, multiplier nu, free)   [F2]
 *          |f| <= F, pmin <= p <= pmax, |theta_i| <= Theta_i, theta_ref = 0
 *     F1 instead keeps theta only and dualises the 2 n_l limit rows
 *     +-diag(b) A theta <= F with mu+, mu- >= 0 (the C x <= d rows
 *     of Eq. 2).
 *
 *   Dual function (Eqs. 3-5): G(y) = inf over the boxes of the
 *   Lagrangian.  The inner minimum over a box is the dual-norm / bound
 *   selection of Eq. 7b (App. A2) for
 *   linear terms, and per-generator clipping for a_g > 0, which is Eq. 15
 *    with the free vector s maximised out (SURVEY F-6).
 *
 *   Gradient: the constraint residual at that minimiser (from Eq. 7b; the
 *   "+b" in Alg. 1 lines 2-3, is read as a sign slip,
 *   DESIGN.md reading A-5).  Tie rule sign(0) -> box midpoint (A-4).
 *
 *   Ascent: y <- y + alpha_k * grad, then mu <- max(mu, 0) (PAPER.md:245,
 *   Alg. 1 line "mu <- max(mu,0)" PAPER.md:264) with an explicit schedule
 *   alpha[K] (A-9).  K+1 evaluations: k = 0..K, no step after the last.
 *
 * Step-by-step order (SURVEY §8(c) oracle algorithm, a-h) is followed
 * literally; every sum runs in ascending index order; no FMA contraction
 * (compile with -ffp-contract=off, reading A-19).
 *
 * Gradient-based-optimisation variants ("Adam ... AdaGrad ...
 * Gradient with Momentum"; Algorithm 1),
 * per multiplier coordinate y with ascent direction g = grad and step a_k:
 *   PLAIN        y <- y + a_k g
 *   GDM          (Algorithm 1 as printed, both updates)
 *                v <- rho v + a_k g;  y <- y + v;  y <- y + a_k g
 *   GDM_CLASSIC  v <- rho v + a_k g;  y <- y + v        (reading A-25)
 *   ADAGRAD      G <- G + g g;  y <- y + (a_k g) / (sqrt(G) + eps)
 *   ADAM         t = steps taken so far + 1; b1t <- b1t beta1, b2t <- b2t beta2
 *                (powers by repeated multiplication from 1);
 *                m <- beta1 m + (1 - beta1) g;  v <- beta2 v + (1 - beta2)(g g);
 *                y <- y + (a_k (m / (1 - b1t))) / (sqrt(v / (1 - b2t)) + eps)
 * then mu <- max(mu, 0).  Optimiser state starts at 0.
 *
 * Divergence (reading A-23 in DESIGN.md): if g(y_k) is not
 * finite or |g(y_k)| > 1e15 the instance is marked DIVERGED; the step of
 * iteration k is still taken, every later step is skipped (y frozen at
 * y_{k+1}) and best never again changes.  best only takes valid values.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_FORM_FLOW_BOX 0   /* F2: boxes p, f, theta; multipliers lambda, nu      */
#define ORC_FORM_LIMIT_ROWS 1 /* F1: boxes p, theta; multipliers lambda, mu+, mu-   */
#define ORC_FORM_CYCLE 2      /* KVL: boxes p, f; multipliers lambda (KCL), kappa (cycle KVL) */
#define ORC_DIVERGED 1
#define ORC_CONVERGED 2  /* stopping rule |g_k - g_{k-1}| < tol (Alg. 1) */

typedef struct {
  int n_bus, n_branch, n_gen, ref_bus;
  const int *br_from, *br_to;
  const double *br_b, *br_fmax, *theta_max;
  const int *gen_bus;
  const double *gen_pmin, *gen_pmax, *gen_c, *gen_a; /* gen_a may be NULL */
} orc_net;

typedef struct {
  double *b, *F;                 /* per-instance susceptance / limit (outages applied) */
  double *r, *p, *q, *f, *w, *th, *phi, *glam, *gbr;
} orc_work;

static void work_alloc(orc_work *W, const orc_net *N, int form) {
  int nb = N->n_bus, nl = N->n_branch, ng = N->n_gen;
  int nbr = (form == ORC_FORM_LIMIT_ROWS) ? 2 * nl : nl;
  W->b = malloc(sizeof(double) * (nl + 1));
  W->F = malloc(sizeof(double) * (nl + 1));
  W->r = malloc(sizeof(double) * (ng + 1));
  W->p = malloc(sizeof(double) * (ng + 1));
  W->q = malloc(sizeof(double) * (nl + 1));
  W->f = malloc(sizeof(double) * (nl + 1));
  W->w = malloc(sizeof(double) * (nb + 1));
  W->th = malloc(sizeof(double) * (nb + 1));
  W->phi = malloc(sizeof(double) * (nl + 1));
  W->glam = malloc(sizeof(double) * (nb + 1));
  W->gbr = malloc(sizeof(double) * (nbr + 1));
}

static void work_free(orc_work *W) {
  free(W->b); free(W->F); free(W->r); free(W->p); free(W->q); free(W->f);
  free(W->w); free(W->th); free(W->phi); free(W->glam); free(W->gbr);
}

/* step 2: outaged branches get b_l = 0 and F_l = 0 (reading A-16) */
static void apply_outages(orc_work *W, const orc_net *N, const int *out, int max_out) {
  int l, j;
  for (l = 0; l < N->n_branch; l++) { W->b[l] = N->br_b[l]; W->F[l] = N->br_fmax[l]; }
  for (j = 0; j < max_out; j++) {
    l = out ? out[j] : -1;
    if (l >= 0 && l < N->n_branch) { W->b[l] = 0.0; W->F[l] = 0.0; }
  }
}

/*
 * Steps 4(a)-(e) and 4(g): value g(y) and its gradient (the residual at the
 * inner minimiser).  lam[n_bus]; br = nu[n_branch] (F2) or mu+[n_branch]
 * followed by mu-[n_branch] (F1).  Gradient left in W->glam, W->gbr.
 */
static double evaluate(const orc_net *N, orc_work *W, int form, const double *d,
                       const double *lam, const double *br) {
  const int nb = N->n_bus, nl = N->n_branch, ng = N->n_gen, ref = N->ref_bus;
  const double *nu = br, *mup = br, *mum = br + nl;
  int i, g, l;
  double s_gen = 0.0, s_br = 0.0, s_th = 0.0, s_ld = 0.0, s_mu = 0.0, val;

  /* (a) r_g = c_g + lambda_{beta(g)}  (argument of Eq. 7b's 1-norm, generator part) */
  for (g = 0; g < ng; g++) W->r[g] = N->gen_c[g] + lam[N->gen_bus[g]];

  /* (b)/(c) branch cost q_l and bus angle cost w_i */
  for (i = 0; i < nb; i++) W->w[i] = 0.0;
  if (form == ORC_FORM_FLOW_BOX) {
    for (l = 0; l < nl; l++) W->q[l] = nu[l] - (lam[N->br_from[l]] - lam[N->br_to[l]]);
    for (l = 0; l < nl; l++) {
      W->w[N->br_from[l]] += -(W->b[l] * nu[l]);
      W->w[N->br_to[l]] += W->b[l] * nu[l];
    }
  } else {
    for (l = 0; l < nl; l++) {
      /* u_l, stored in q */
      W->q[l] = W->b[l] * ((mup[l] - mum[l]) - (lam[N->br_from[l]] - lam[N->br_to[l]]));
    }
    for (l = 0; l < nl; l++) {
      W->w[N->br_from[l]] += W->q[l];
      W->w[N->br_to[l]] -= W->q[l];
    }
  }

  /* (d) closed-form inner minimiser over the boxes */
  for (g = 0; g < ng; g++) {
    double lo = N->gen_pmin[g], hi = N->gen_pmax[g], r = W->r[g];
    if (N->gen_a && N->gen_a[g] > 0.0) {          /* QP: clip(-r/(2a)) */
      double x = -r / (2.0 * N->gen_a[g]);
      W->p[g] = (x < lo) ? lo : ((x > hi) ? hi : x);
    } else if (r > 0.0) {
      W->p[g] = lo;
    } else if (r < 0.0) {
      W->p[g] = hi;
    } else {
      W->p[g] = 0.5 * (lo + hi);
    }
  }
  if (form == ORC_FORM_FLOW_BOX) {
    for (l = 0; l < nl; l++) {
      double q = W->q[l];
      W->f[l] = (q > 0.0) ? -W->F[l] : ((q < 0.0) ? W->F[l] : 0.0);
    }
  }
  for (i = 0; i < nb; i++) {
    double w = W->w[i];
    if (i == ref) W->th[i] = 0.0;
    else W->th[i] = (w > 0.0) ? -N->theta_max[i] : ((w < 0.0) ? N->theta_max[i] : 0.0);
  }
  for (l = 0; l < nl; l++) W->phi[l] = W->b[l] * (W->th[N->br_from[l]] - W->th[N->br_to[l]]);

  /* (e) dual value: brackets in ascending index order, then left to right */
  for (g = 0; g < ng; g++) {
    double t = W->r[g] * W->p[g];
    if (N->gen_a && N->gen_a[g] > 0.0) t = N->gen_a[g] * W->p[g] * W->p[g] + t;
    s_gen += t;
  }
  if (form == ORC_FORM_FLOW_BOX)
    for (l = 0; l < nl; l++) s_br += W->q[l] * W->f[l];
  for (i = 0; i < nb; i++)
    if (i != ref) s_th += W->w[i] * W->th[i];
  for (i = 0; i < nb; i++) s_ld += lam[i] * d[i];
  if (form == ORC_FORM_FLOW_BOX) {
    val = ((s_gen + s_br) + s_th) - s_ld;
  } else {
    for (l = 0; l < nl; l++) s_mu += W->F[l] * (mup[l] + mum[l]);
    val = ((s_gen + s_th) - s_ld) - s_mu;
  }

  /* (g) gradient = residual at the minimiser */
  for (i = 0; i < nb; i++) W->glam[i] = -d[i];
  for (g = 0; g < ng; g++) W->glam[N->gen_bus[g]] += W->p[g];
  if (form == ORC_FORM_FLOW_BOX) {
    for (l = 0; l < nl; l++) {
      W->glam[N->br_from[l]] -= W->f[l];
      W->glam[N->br_to[l]] += W->f[l];
    }
    for (l = 0; l < nl; l++) W->gbr[l] = W->f[l] - W->phi[l];
  } else {
    for (l = 0; l < nl; l++) {
      W->glam[N->br_from[l]] -= W->phi[l];
      W->glam[N->br_to[l]] += W->phi[l];
    }
    for (l = 0; l < nl; l++) {
      W->gbr[l] = W->phi[l] - W->F[l];
      W->gbr[nl + l] = -W->phi[l] - W->F[l];
    }
  }
  return val;
}

static int valid_bound(double g) { return isfinite(g) && fabs(g) <= 1e15; }

#define ORC_OPT_PLAIN 0
#define ORC_OPT_GDM 1
#define ORC_OPT_GDM_CLASSIC 2
#define ORC_OPT_ADAGRAD 3
#define ORC_OPT_ADAM 4

typedef struct {
  int variant;
  double rho, beta1, beta2, eps;
  double tol;  /* stopping rule (0: off) */
} orc_opt;

/* one coordinate of the ascent step (the variants above); s1, s2 = state */
static double opt_step(const orc_opt *o, double y, double g, double a, double *s1, double *s2,
                       double b1t, double b2t) {
  switch (o->variant) {
    case ORC_OPT_GDM:
      *s1 = o->rho * *s1 + a * g;
      y = y + *s1;
      return y + a * g;
    case ORC_OPT_GDM_CLASSIC:
      *s1 = o->rho * *s1 + a * g;
      return y + *s1;
    case ORC_OPT_ADAGRAD:
      *s1 = *s1 + g * g;
      return y + (a * g) / (sqrt(*s1) + o->eps);
    case ORC_OPT_ADAM: {
      *s1 = o->beta1 * *s1 + (1.0 - o->beta1) * g;
      *s2 = o->beta2 * *s2 + (1.0 - o->beta2) * (g * g);
      {
        double mh = *s1 / (1.0 - b1t), vh = *s2 / (1.0 - b2t);
        return y + (a * mh) / (sqrt(vh) + o->eps);
      }
    }
    default:
      return y + a * g;
  }
}

/* ============================================================================
 * Form KVL (reading A-28): the angle-free
 * cycle-basis twin of the paper's PTDF constraint (Eq. 1:
 * f = H(p - d)).  For a connected network, f is the PTDF flow of the
 * injections iff KCL (G p - A^T f = d) holds and Kirchhoff's voltage law
 * holds on every fundamental cycle k of a spanning tree:
 *     sum_l C_kl x_l f_l = 0,   x_l = 1 / b_l,   C_kl in {0, +1, -1}.
 * Dualising KCL (lambda) and KVL (kappa, free) leaves the boxes p, |f| <= F:
 *     q_l    = x_l (sum_k C_kl kappa_k) - (lambda_s - lambda_t)
 *     f*_l   = -F if q > 0, +F if q < 0, 0 on a tie
 *     g      = [sum_g a p*^2 + r p*] + [sum_l q_l f*_l] - [sum_i lambda_i d_i]
 *     dg/dlambda = KCL residual (as F2),  dg/dkappa_k = sum_l C_kl (f*_l x_l).
 * Spanning tree (reading A-28): breadth-first from the reference bus, buses
 * in FIFO order, each bus's incident branches in ascending id, over branches
 * with b > 0 that are never switched.  Cycle k belongs to the k-th non-tree
 * branch l (ascending id): l traversed from s_l to t_l (+1), then the tree
 * path from t_l back to s_l (+1 where a branch is traversed from its from bus
 * to its to bus, -1 otherwise); entries kept in ascending branch id.  A
 * branch with b = 0 (base or outaged) carries no flow (F_eff = 0, x = 0) and
 * the cycle it defines is inactive (kappa_k not used, gradient 0).
 * ========================================================================== */
typedef struct {
  int nc;
  int *is_tree, *def;          /* [nl], [nc] */
  int *cp, *cb, *cs;           /* cycle k: branches cb[cp[k]..cp[k+1]) ascending, signs cs */
  int *bp, *bk, *bs;           /* branch l: cycles bk[bp[l]..bp[l+1]) ascending, signs bs */
} orc_cyc;

static void cyc_free(orc_cyc *Y) {
  free(Y->is_tree); free(Y->def); free(Y->cp); free(Y->cb); free(Y->cs);
  free(Y->bp); free(Y->bk); free(Y->bs);
}

/* returns 0, or -1 if the never-switched branches with b > 0 do not connect the buses */
static int build_cycles(const orc_net *N, const unsigned char *sw, orc_cyc *Y) {
  const int nb = N->n_bus, nl = N->n_branch;
  int *deg = calloc((size_t)nb + 1, sizeof(int)), *ap = calloc((size_t)nb + 1, sizeof(int));
  int *adj = malloc(sizeof(int) * (2 * (size_t)nl + 1));
  int *parent = malloc(sizeof(int) * (nb + 1)), *pbr = malloc(sizeof(int) * (nb + 1));
  int *depth = malloc(sizeof(int) * (nb + 1)), *queue = malloc(sizeof(int) * (nb + 1));
  int *tmpb = malloc(sizeof(int) * (nb + 2)), *tmps = malloc(sizeof(int) * (nb + 2));
  int i, l, k, head = 0, tail = 0, seen = 0, cap, tot = 0;
  for (l = 0; l < nl; l++) { deg[N->br_from[l]]++; deg[N->br_to[l]]++; }
  for (i = 0; i < nb; i++) ap[i + 1] = ap[i] + deg[i];
  for (i = 0; i < nb; i++) deg[i] = 0;
  for (l = 0; l < nl; l++) {                 /* ascending branch id per bus */
    adj[ap[N->br_from[l]] + deg[N->br_from[l]]++] = l;
    adj[ap[N->br_to[l]] + deg[N->br_to[l]]++] = l;
  }
  Y->is_tree = calloc((size_t)nl + 1, sizeof(int));
  for (i = 0; i < nb; i++) parent[i] = -2;
  parent[N->ref_bus] = -1; pbr[N->ref_bus] = -1; depth[N->ref_bus] = 0;
  queue[tail++] = N->ref_bus; seen = 1;
  while (head < tail) {
    int u = queue[head++], e;
    for (e = ap[u]; e < ap[u + 1]; e++) {
      int m = adj[e], v = (N->br_from[m] == u) ? N->br_to[m] : N->br_from[m];
      if (!(N->br_b[m] > 0.0) || (sw && sw[m]) || parent[v] != -2) continue;
      parent[v] = u; pbr[v] = m; depth[v] = depth[u] + 1; Y->is_tree[m] = 1;
      queue[tail++] = v; seen++;
    }
  }
  Y->nc = nl - (nb - 1);
  if (seen != nb || Y->nc < 0) {
    free(deg); free(ap); free(adj); free(parent); free(pbr); free(depth); free(queue); free(tmpb); free(tmps);
    free(Y->is_tree); Y->is_tree = NULL;
    return -1;
  }
  cap = Y->nc * (nb + 1) + 1;
  if (cap > 64 * nl + 1024) cap = 64 * nl + 1024;  /* grown below if needed */
  Y->def = malloc(sizeof(int) * (Y->nc + 1));
  Y->cp = malloc(sizeof(int) * (Y->nc + 2));
  Y->cb = malloc(sizeof(int) * cap);
  Y->cs = malloc(sizeof(int) * cap);
  Y->cp[0] = 0;
  for (k = 0, l = 0; l < nl; l++) {
    int a, b, n = 0, x, y;
    if (Y->is_tree[l]) continue;
    Y->def[k] = l;
    tmpb[n] = l; tmps[n] = 1; n++;            /* l from s to t */
    a = N->br_to[l]; b = N->br_from[l];       /* tree path from t (a) back to s (b) */
    while (a != b) {
      if (depth[a] >= depth[b]) {               /* a climbs: traversed a -> parent(a) */
        int m = pbr[a];
        tmpb[n] = m; tmps[n] = (N->br_from[m] == a) ? 1 : -1; n++;
        a = parent[a];
      } else {                                  /* b climbs: traversed parent(b) -> b */
        int m = pbr[b];
        tmpb[n] = m; tmps[n] = (N->br_to[m] == b) ? 1 : -1; n++;
        b = parent[b];
      }
    }
    for (x = 1; x < n; x++)                     /* ascending branch id (insertion sort) */
      for (y = x; y > 0 && tmpb[y - 1] > tmpb[y]; y--) {
        int tb = tmpb[y], ts = tmps[y];
        tmpb[y] = tmpb[y - 1]; tmps[y] = tmps[y - 1]; tmpb[y - 1] = tb; tmps[y - 1] = ts;
      }
    if (tot + n > cap) {
      cap = 2 * (tot + n);
      Y->cb = realloc(Y->cb, sizeof(int) * cap);
      Y->cs = realloc(Y->cs, sizeof(int) * cap);
    }
    for (x = 0; x < n; x++) { Y->cb[tot + x] = tmpb[x]; Y->cs[tot + x] = tmps[x]; }
    tot += n;
    Y->cp[++k] = tot;
  }
  /* per-branch lists, ascending cycle index */
  Y->bp = calloc((size_t)nl + 2, sizeof(int));
  Y->bk = malloc(sizeof(int) * (tot + 1));
  Y->bs = malloc(sizeof(int) * (tot + 1));
  for (i = 0; i < tot; i++) Y->bp[Y->cb[i] + 1]++;
  for (l = 0; l < nl; l++) Y->bp[l + 1] += Y->bp[l];
  {
    int *fill = calloc((size_t)nl + 1, sizeof(int));
    for (k = 0; k < Y->nc; k++)
      for (i = Y->cp[k]; i < Y->cp[k + 1]; i++) {
        int m = Y->cb[i];
        Y->bk[Y->bp[m] + fill[m]] = k;
        Y->bs[Y->bp[m] + fill[m]] = Y->cs[i];
        fill[m]++;
      }
    free(fill);
  }
  free(deg); free(ap); free(adj); free(parent); free(pbr); free(depth); free(queue); free(tmpb); free(tmps);
  return 0;
}

/* value and gradient of the KVL form; kap[nc]; gradient in W->glam, W->gbr[nc] */
static double evaluate_kvl(const orc_net *N, orc_work *W, const orc_cyc *Y, const double *d,
                           const double *lam, const double *kap) {
  const int nb = N->n_bus, nl = N->n_branch, ng = N->n_gen;
  int i, g, l, k, e;
  double s_gen = 0.0, s_br = 0.0, s_ld = 0.0;
  /* (a) r_g */
  for (g = 0; g < ng; g++) W->r[g] = N->gen_c[g] + lam[N->gen_bus[g]];
  /* (b) q_l = x_l (sum_k C_kl kappa_k) - (lambda_s - lambda_t); active cycles only */
  for (l = 0; l < nl; l++) {
    double x = (W->b[l] > 0.0) ? 1.0 / W->b[l] : 0.0, sum = 0.0;
    for (e = Y->bp[l]; e < Y->bp[l + 1]; e++) {
      k = Y->bk[e];
      if (!(W->b[Y->def[k]] > 0.0)) continue;
      sum = (Y->bs[e] > 0) ? sum + kap[k] : sum - kap[k];
    }
    W->q[l] = x * sum - (lam[N->br_from[l]] - lam[N->br_to[l]]);
  }
  /* (d) minimisers */
  for (g = 0; g < ng; g++) {
    double lo = N->gen_pmin[g], hi = N->gen_pmax[g], r = W->r[g];
    if (N->gen_a && N->gen_a[g] > 0.0) {
      double x = -r / (2.0 * N->gen_a[g]);
      W->p[g] = (x < lo) ? lo : ((x > hi) ? hi : x);
    } else if (r > 0.0) W->p[g] = lo;
    else if (r < 0.0) W->p[g] = hi;
    else W->p[g] = 0.5 * (lo + hi);
  }
  for (l = 0; l < nl; l++) {
    double F = (W->b[l] > 0.0) ? W->F[l] : 0.0, q = W->q[l];
    W->f[l] = (q > 0.0) ? -F : ((q < 0.0) ? F : 0.0);
  }
  /* (e) value */
  for (g = 0; g < ng; g++) {
    double t = W->r[g] * W->p[g];
    if (N->gen_a && N->gen_a[g] > 0.0) t = N->gen_a[g] * W->p[g] * W->p[g] + t;
    s_gen += t;
  }
  for (l = 0; l < nl; l++) s_br += W->q[l] * W->f[l];
  for (i = 0; i < nb; i++) s_ld += lam[i] * d[i];
  /* (g) gradient */
  for (i = 0; i < nb; i++) W->glam[i] = -d[i];
  for (g = 0; g < ng; g++) W->glam[N->gen_bus[g]] += W->p[g];
  for (l = 0; l < nl; l++) {
    W->glam[N->br_from[l]] -= W->f[l];
    W->glam[N->br_to[l]] += W->f[l];
  }
  for (k = 0; k < Y->nc; k++) {
    double acc = 0.0;
    if (W->b[Y->def[k]] > 0.0)
      for (e = Y->cp[k]; e < Y->cp[k + 1]; e++) {
        int m = Y->cb[e];
        double x = (W->b[m] > 0.0) ? 1.0 / W->b[m] : 0.0, t = W->f[m] * x;
        acc = (Y->cs[e] > 0) ? acc + t : acc - t;
      }
    W->gbr[k] = acc;
  }
  return (s_gen + s_br) - s_ld;
}

static void run_instance(const orc_net *N, int form, const double *d, const int *out, int max_out,
                         long K, const double *alpha, double *lam, double *br, double *bound,
                         double *best, int *status, double *hist, int warm, const orc_opt *opt,
                         const orc_cyc *Y) {
  const int nb = N->n_bus, nl = N->n_branch;
  const int nbr = (form == ORC_FORM_LIMIT_ROWS) ? 2 * nl : ((form == ORC_FORM_CYCLE) ? Y->nc : nl);
  orc_work W;
  long k;
  int i, j, frozen = 0;
  double b1t = 1.0, b2t = 1.0;                   /* beta1^t, beta2^t (Adam) */
  double gprev = 0.0;                            /* g(y_{k-1}) for the stopping rule */
  double *s1 = calloc((size_t)(nb + nbr + 1), sizeof(double));   /* optimiser state, y order */
  double *s2 = calloc((size_t)(nb + nbr + 1), sizeof(double));
  work_alloc(&W, N, form);
  apply_outages(&W, N, out, max_out);
  if (!warm) {                                   /* step 3: y_0 = 0 */
    for (i = 0; i < nb; i++) lam[i] = 0.0;
    for (j = 0; j < nbr; j++) br[j] = 0.0;
  }
  *best = -INFINITY;
  *status = 0;
  for (k = 0;; k++) {                            /* step 4: k = 0..K inclusive */
    double g = (form == ORC_FORM_CYCLE) ? evaluate_kvl(N, &W, Y, d, lam, br) : evaluate(N, &W, form, d, lam, br);
    int was_frozen = frozen;
    if (hist) hist[k] = g;
    if (!was_frozen) {                           /* (f) best = max(best, g) */
      if (valid_bound(g)) {
        if (g > *best) *best = g;
        /* Alg. 1 stopping rule: |gamma^(i+1) - gamma^(i)| < tol.
         * Like divergence (reading A-23/A-29) the step of this iteration is
         * still taken and every later one skipped. */
        if (opt->tol > 0.0 && k > 0 && fabs(g - gprev) < opt->tol) { *status = ORC_CONVERGED; frozen = 1; }
      } else { *status = ORC_DIVERGED; frozen = 1; }
    }
    gprev = g;
    if (k == K) { *bound = g; break; }
    if (was_frozen) continue;
    {                                            /* (h) ascent step and projection */
      double a = alpha[k];
      if (opt->variant == ORC_OPT_ADAM) { b1t = b1t * opt->beta1; b2t = b2t * opt->beta2; }
      for (i = 0; i < nb; i++) lam[i] = opt_step(opt, lam[i], W.glam[i], a, &s1[i], &s2[i], b1t, b2t);
      if (form == ORC_FORM_FLOW_BOX || form == ORC_FORM_CYCLE) {   /* nu / kappa: free */
        for (j = 0; j < nbr; j++) br[j] = opt_step(opt, br[j], W.gbr[j], a, &s1[nb + j], &s2[nb + j], b1t, b2t);
      } else {
        for (j = 0; j < 2 * nl; j++) {
          double v = opt_step(opt, br[j], W.gbr[j], a, &s1[nb + j], &s2[nb + j], b1t, b2t);
          br[j] = (v > 0.0) ? v : 0.0;           /* mu <- max(mu, 0) */
        }
      }
    }
  }
  work_free(&W);
  free(s1);
  free(s2);
}

#define NET_ARGS                                                                     \
  int n_bus, int n_branch, int n_gen, int ref_bus, const int *br_from, const int *br_to, \
      const double *br_b, const double *br_fmax, const double *theta_max,             \
      const int *gen_bus, const double *gen_pmin, const double *gen_pmax,             \
      const double *gen_c, const double *gen_a

#define NET_INIT                                                                        \
  orc_net N;                                                                            \
  N.n_bus = n_bus; N.n_branch = n_branch; N.n_gen = n_gen; N.ref_bus = ref_bus;         \
  N.br_from = br_from; N.br_to = br_to; N.br_b = br_b; N.br_fmax = br_fmax;             \
  N.theta_max = theta_max; N.gen_bus = gen_bus; N.gen_pmin = gen_pmin;                  \
  N.gen_pmax = gen_pmax; N.gen_c = gen_c; N.gen_a = gen_a;

/*
 * Run K ascent steps for B independent instances (instance-major arrays).
 *   load[B][n_bus]; outages[B][max_out] (-1 padded) or NULL;
 *   lam[B][n_bus], br[B][nbr] (nbr = n_branch for F2, 2 n_branch for F1):
 *     in: start point if warm != 0; out: y_K;
 *   bound[B] = g(y_K); best[B] = max valid g(y_k), k=0..K; status[B];
 *   hist[B][K+1] (g(y_k)) or NULL.
 * Returns 0, or -1 on bad arguments.
 */
int oracle_solve_opt(NET_ARGS, int form, long B, const double *load, const int *outages, int max_out,
                     long K, const double *alpha, double *lam, double *br, double *bound,
                     double *best, int *status, double *hist, int warm, int n_threads,
                     int variant, double rho, double beta1, double beta2, double eps,
                     const unsigned char *switchable, double tol) {
  NET_INIT
  long j;
  orc_opt opt;
  orc_cyc Y;
  int nbr;
  opt.variant = variant; opt.rho = rho; opt.beta1 = beta1; opt.beta2 = beta2; opt.eps = eps;
  opt.tol = tol;
  memset(&Y, 0, sizeof Y);
  if (variant < ORC_OPT_PLAIN || variant > ORC_OPT_ADAM) return -1;
  /* AdaGrad / Adam divide by sqrt(state) + eps with the state 0 at the start
   * (SPEC.md:359 gives eps = 1e-8): eps <= 0 would divide 0 by 0 */
  if ((variant == ORC_OPT_ADAGRAD || variant == ORC_OPT_ADAM) && !(eps > 0.0)) return -1;
  if (n_bus <= 0 || n_branch < 0 || n_gen < 0 || B < 0 || K < 0) return -1;
  if (form != ORC_FORM_FLOW_BOX && form != ORC_FORM_LIMIT_ROWS && form != ORC_FORM_CYCLE) return -1;
  if (form == ORC_FORM_CYCLE && build_cycles(&N, switchable, &Y) != 0) return -2;
  nbr = (form == ORC_FORM_LIMIT_ROWS) ? 2 * n_branch : ((form == ORC_FORM_CYCLE) ? Y.nc : n_branch);
  (void)n_threads;
#pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads > 0 ? n_threads : 1)
  for (j = 0; j < B; j++) {
    run_instance(&N, form, load + j * (long)n_bus, outages ? outages + j * (long)max_out : NULL,
                 max_out, K, alpha, lam + j * (long)n_bus, br + j * (long)nbr, bound + j,
                 best + j, status + j, hist ? hist + j * (K + 1) : NULL, warm, &opt, &Y);
  }
  if (form == ORC_FORM_CYCLE) cyc_free(&Y);
  return 0;
}

/* KVL form: value and gradient (kap[B][nc], grad_kap[B][nc]); minimiser p, f. */
int oracle_evaluate_kvl(NET_ARGS, const unsigned char *switchable, long B, const double *load,
                        const int *outages, int max_out, const double *lam, const double *kap,
                        double *value, double *grad_lam, double *grad_kap, double *p, double *f) {
  NET_INIT
  long j;
  orc_cyc Y;
  if (n_bus <= 0 || n_branch < 0 || n_gen < 0 || B < 0) return -1;
  if (build_cycles(&N, switchable, &Y) != 0) return -2;
  for (j = 0; j < B; j++) {
    orc_work W;
    work_alloc(&W, &N, ORC_FORM_FLOW_BOX);
    apply_outages(&W, &N, outages ? outages + j * (long)max_out : NULL, max_out);
    value[j] = evaluate_kvl(&N, &W, &Y, load + j * (long)n_bus, lam + j * (long)n_bus, kap + j * (long)Y.nc);
    if (grad_lam) memcpy(grad_lam + j * (long)n_bus, W.glam, sizeof(double) * n_bus);
    if (grad_kap) memcpy(grad_kap + j * (long)Y.nc, W.gbr, sizeof(double) * Y.nc);
    if (p) memcpy(p + j * (long)n_gen, W.p, sizeof(double) * n_gen);
    if (f) memcpy(f + j * (long)n_branch, W.f, sizeof(double) * n_branch);
    work_free(&W);
  }
  cyc_free(&Y);
  return 0;
}

/* The cycle basis (reading A-28): returns the number of entries (or -2 if
 * disconnected); *nc = cycles; def[nc], cp[nc+1], cb/cs[entries] filled when
 * cap >= entries. */
int oracle_cycles(NET_ARGS, const unsigned char *switchable, int *nc, int *def, int *cp, int *cb, int *cs,
                  long cap) {
  NET_INIT
  orc_cyc Y;
  int k, tot;
  if (build_cycles(&N, switchable, &Y) != 0) return -2;
  *nc = Y.nc;
  tot = Y.cp[Y.nc];
  if (cap >= tot && cp != NULL) {   /* cp == NULL: size query only (also when there is no cycle) */
    for (k = 0; k < Y.nc; k++) def[k] = Y.def[k];
    for (k = 0; k <= Y.nc; k++) cp[k] = Y.cp[k];
    for (k = 0; k < tot; k++) { cb[k] = Y.cb[k]; cs[k] = Y.cs[k]; }
  }
  cyc_free(&Y);
  return tot;
}

/* the plain projected step (the north_star path) */
int oracle_solve(NET_ARGS, int form, long B, const double *load, const int *outages, int max_out,
                 long K, const double *alpha, double *lam, double *br, double *bound,
                 double *best, int *status, double *hist, int warm, int n_threads) {
  return oracle_solve_opt(n_bus, n_branch, n_gen, ref_bus, br_from, br_to, br_b, br_fmax, theta_max,
                          gen_bus, gen_pmin, gen_pmax, gen_c, gen_a, form, B, load, outages, max_out, K,
                          alpha, lam, br, bound, best, status, hist, warm, n_threads,
                          ORC_OPT_PLAIN, 0.0, 0.0, 0.0, 0.0, NULL, 0.0);
}

/* Value and gradient at given multipliers (no step). */
int oracle_evaluate(NET_ARGS, int form, long B, const double *load, const int *outages, int max_out,
                    const double *lam, const double *br, double *value, double *grad_lam,
                    double *grad_br) {
  NET_INIT
  long j;
  const int nbr = (form == ORC_FORM_LIMIT_ROWS) ? 2 * n_branch : n_branch;
  if (n_bus <= 0 || n_branch < 0 || n_gen < 0 || B < 0) return -1;
  if (form != ORC_FORM_FLOW_BOX && form != ORC_FORM_LIMIT_ROWS) return -1;
  for (j = 0; j < B; j++) {
    orc_work W;
    work_alloc(&W, &N, form);
    apply_outages(&W, &N, outages ? outages + j * (long)max_out : NULL, max_out);
    value[j] = evaluate(&N, &W, form, load + j * (long)n_bus, lam + j * (long)n_bus,
                        br + j * (long)nbr);
    if (grad_lam) memcpy(grad_lam + j * (long)n_bus, W.glam, sizeof(double) * n_bus);
    if (grad_br) memcpy(grad_br + j * (long)nbr, W.gbr, sizeof(double) * nbr);
    work_free(&W);
  }
  return 0;
}

/* Inner minimiser at given multipliers, for the brute-force pins:
 * p[B][n_gen], flow[B][n_branch] (F2: f*; F1: phi), theta[B][n_bus]. */
int oracle_minimiser(NET_ARGS, int form, long B, const double *load, const int *outages,
                     int max_out, const double *lam, const double *br, double *p, double *flow,
                     double *theta) {
  NET_INIT
  long j;
  const int nbr = (form == ORC_FORM_LIMIT_ROWS) ? 2 * n_branch : n_branch;
  if (n_bus <= 0 || n_branch < 0 || n_gen < 0 || B < 0) return -1;
  for (j = 0; j < B; j++) {
    orc_work W;
    work_alloc(&W, &N, form);
    apply_outages(&W, &N, outages ? outages + j * (long)max_out : NULL, max_out);
    evaluate(&N, &W, form, load + j * (long)n_bus, lam + j * (long)n_bus, br + j * (long)nbr);
    memcpy(p + j * (long)n_gen, W.p, sizeof(double) * n_gen);
    memcpy(flow + j * (long)n_branch, form == ORC_FORM_FLOW_BOX ? W.f : W.phi,
           sizeof(double) * n_branch);
    memcpy(theta + j * (long)n_bus, W.th, sizeof(double) * n_bus);
    work_free(&W);
  }
  return 0;
}
