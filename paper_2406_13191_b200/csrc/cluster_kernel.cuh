// cluster_kernel.cuh -- the cluster path: one thread-block cluster of C CTAs
// (one per SM, C <= 16) runs all K iterations of ONE instance, the network
// partitioned over the CTAs' shared memories (plan: cluster.h).
//
// Per iteration (Eq. 3, 7b, 15, Alg. 1):
//   A   owned buses: w_i over the incidence (neighbours' nu / mu, lambda read
//       over distributed shared memory), theta*_i
//   --- cluster barrier ---
//   B   owned branches: q_l, f*_l, phi_l, residual, nu' / mu' (in place: every
//       reader of nu / mu in this iteration ran in A)
//   --- cluster barrier ---
//   C   owned buses: generators, d/dlambda, lambda' (in place: every reader of
//       lambda in this iteration ran in B, or -- F1 -- in A)
//   (F1 only: --- cluster barrier --- before the next A, which reads lambda')
// The dual value: per-CTA block reduction, then every CTA reads all C partials
// after the next barrier and sums them in rank order (bitwise identical in
// every CTA, so every CTA takes the same best / divergence decision; rank 0
// writes the results).  F2 needs 2 cluster barriers per iteration, F1 3.
//
// Per-entity arithmetic and its operation order are those of the oracle and
// of k_single / k_sweep (reading A-19): sums over a bus's incidence in
// ascending original branch id, generators before branches, y + (alpha*g).
#pragma once
#include "../../include/dcopf_dual.h"
#include "cluster.h"
#include "dual_kernels.cuh"

namespace dcopf {

struct ClusterArgs {
  const uint8_t *blob;          // [C] per-rank blobs (ClusterPlan)
  int blob_stride;
  double *lam, *br;             // instance-major internal state [b][n_bus], [b][n_br * BRW]
  const double *d;              // [b][n_bus]
  const int *outs;              // [B][max_out] internal branch ids, -1 padded
  int max_out;
  const double *alpha;          // [K] device
  long K;
  double *bound, *best;         // [B]
  int *status;                  // [B]
  double *hist;                 // [K][B] or null
  long B;
  const double *target;         // [B] or null (time to gap)
  long long *hit;
  long k_base;
  double *grad_lam, *grad_br, *value;  // EVAL outputs (instance-major) or null
  int n_bus, n_br;
  int n_bm;                     // branch-block multipliers per instance: n_br (F2), 2 n_br (F1), n_cycles (KVL)
  // ascent-step variant (dcopf_dual.h DCOPF_OPT_*) and its persistent state
  int opt;
  double rho, beta1, beta2, eps;
  double b1t, b2t;              // beta1^t, beta2^t at this launch's first step (Adam)
  double *s1_lam, *s2_lam;      // [b][n_bus] instance-major internal, or null
  double *s1_br, *s2_br;        // [b][n_br * BRW]
  double tol;                   // stopping rule (0: off)
  int dbg;                      // measurement only: 1 = skip the phases' work (synchronisation floor)
};

__device__ __forceinline__ double opt_step(const ClusterArgs &a, double y, double g, double al, double *s1,
                                           double *s2, const AdamC &ac) {
  double yv[1] = {y}, s1v[1] = {*s1}, s2v[1] = {*s2};
  const double gv[1] = {g};
  const bool on[1] = {true};
  opt_update_v<1>(a.opt, a.rho, a.beta1, a.beta2, a.eps, yv, gv, al, s1v, s2v, ac, on);
  *s1 = s1v[0];
  *s2 = s2v[0];
  return yv[0];
}

__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_nrank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// (a cluster of one CTA needs only the block barrier)
__device__ __forceinline__ void cl_sync(unsigned C) {
  if (C == 1) __syncthreads();
  else cl_sync();
}
__device__ __forceinline__ unsigned cl_map(unsigned local_addr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
// distributed-shared-memory loads; ordered against the cluster barriers by
// `volatile` (the barriers carry the memory clobber)
__device__ __forceinline__ double cl_ld(unsigned addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ double2 cl_ld2(unsigned addr) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

#ifndef DCOPF_CLUSTER_THREADS
#define DCOPF_CLUSTER_THREADS 1024
#endif
constexpr int kClusterThreads = DCOPF_CLUSTER_THREADS;

// OPT: the optimiser-variant instantiation (the plain step's kernel carries
// none of the variants' code: its registers stay with the plain path)
template <int FORM, int MODE, bool OPT = false>
__global__ void __launch_bounds__(kClusterThreads, 1) k_cluster(const ClusterArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int BRW = (FORM == kFormF2) ? 1 : 2;
  const unsigned rank = cl_rank(), C = cl_nrank();
  const long b = cl_id();
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);

  // ---- plan blob -> shared memory --------------------------------------------
  {
    const ClHeader *g = reinterpret_cast<const ClHeader *>(a.blob + (size_t)rank * a.blob_stride);
    const int n16 = g->blob_bytes / 16;
    const int4 *src = reinterpret_cast<const int4 *>(g);
    int4 *dst = reinterpret_cast<int4 *>(smem);
    for (int x = tid; x < n16; x += nthr) dst[x] = src[x];
  }
  __syncthreads();
  const ClHeader &H = *reinterpret_cast<const ClHeader *>(smem);
  const int nA = H.nA, nB = H.nB;
  double *lam_s = reinterpret_cast<double *>(smem + H.off_lam);
  double *d_s = reinterpret_cast<double *>(smem + H.off_d);
  double *br_s = reinterpret_cast<double *>(smem + H.off_br);
  double *th_s = reinterpret_cast<double *>(smem + H.off_th);
  double *fc_s = reinterpret_cast<double *>(smem + H.off_fc);
  double *red = reinterpret_cast<double *>(smem + H.off_red);        // [0]: this CTA's partial value
  double *wred = red + 8;                                            // [32] per-warp partials
  int *flag = reinterpret_cast<int *>(red + 40);                     // [0]: frozen
  const unsigned red_addr0 = sbase + H.off_red;

  // ---- cluster addresses + this instance's outages (b = F = 0, reading A-16) ---
  const int nout = a.max_out;
  int o[kMaxOut];
#pragma unroll
  for (int j = 0; j < kMaxOut; ++j) o[j] = (j < nout) ? a.outs[b * nout + j] : -1;
  auto cvt = [&](unsigned x) { return cl_map(sbase + (x & ((1u << kClAddrShift) - 1)), x >> kClAddrShift); };
  if (FORM == kFormKVL) {
    const unsigned zero = cl_map(sbase + H.off_zero, rank);  // masked cycle terms read 0.0
    if (tid == 0) reinterpret_cast<double *>(smem + H.off_zero)[0] = 0.0;
    ClBKe *BK = reinterpret_cast<ClBKe *>(smem + H.off_IA);
    for (int e = tid; e < H.nIA; e += nthr) BK[e].kap = is_out(o, nout, BK[e].dbr) ? zero : cvt(BK[e].kap);
    ClBk *Bv = reinterpret_cast<ClBk *>(smem + H.off_B);
    for (int j = tid; j < nB; j += nthr) {
      Bv[j].ls = cvt(Bv[j].ls);
      Bv[j].lt = cvt(Bv[j].lt);
      if (is_out(o, nout, Bv[j].br)) Bv[j].x = Bv[j].F = 0.0;  // an outaged branch: b = F = 0 (A-16)
    }
    ClIC2 *IC = reinterpret_cast<ClIC2 *>(smem + H.off_IC);
    for (int e = tid; e < H.nIC; e += nthr) IC[e].f = cvt(IC[e].f);
    ClCy *Cy = reinterpret_cast<ClCy *>(smem + H.off_Cy);
    for (int c = tid; c < H.nCy; c += nthr)
      if (is_out(o, nout, Cy[c].dbr)) Cy[c].e1 = Cy[c].e0;  // its defining branch is out: no cycle
    ClCe *CE = reinterpret_cast<ClCe *>(smem + H.off_CE);
    for (int e = tid; e < H.nCE; e += nthr) CE[e].f = cvt(CE[e].f);
  } else if (FORM == kFormF2) {
    ClIA2 *IA = reinterpret_cast<ClIA2 *>(smem + H.off_IA);
    ClIC2 *IC = reinterpret_cast<ClIC2 *>(smem + H.off_IC);
    for (int e = tid; e < H.nIA; e += nthr) {
      IA[e].nu = cvt(IA[e].nu);
      IC[e].f = cvt(IC[e].f);
      if (is_out(o, nout, IA[e].br)) IA[e].sb = copysign(0.0, IA[e].sb);
    }
  } else {
    ClIA1 *IA = reinterpret_cast<ClIA1 *>(smem + H.off_IA);
    ClIC1 *IC = reinterpret_cast<ClIC1 *>(smem + H.off_IC);
    for (int e = tid; e < H.nIA; e += nthr) {
      IA[e].mu = cvt(IA[e].mu);
      IA[e].ls = cvt(IA[e].ls);
      IA[e].lt = cvt(IA[e].lt);
      IC[e].ts = cvt(IC[e].ts);
      IC[e].tt = cvt(IC[e].tt);
      if (is_out(o, nout, IA[e].br)) {
        IA[e].sb = copysign(0.0, IA[e].sb);
        IC[e].sb = copysign(0.0, IC[e].sb);
      }
    }
  }
  if (FORM != kFormKVL) {
    ClB *Bv = reinterpret_cast<ClB *>(smem + H.off_B);
    for (int j = tid; j < nB; j += nthr) {
      Bv[j].ts = cvt(Bv[j].ts);
      Bv[j].tt = cvt(Bv[j].tt);
      Bv[j].ls = cvt(Bv[j].ls);
      Bv[j].lt = cvt(Bv[j].lt);
      if (is_out(o, nout, Bv[j].br)) Bv[j].b = Bv[j].F = 0.0;
    }
  }
  // ---- this CTA's state ------------------------------------------------------------
  // branch-block multipliers of this CTA: nu / mu of its branches, or kappa of its cycles (KVL)
  const size_t bm0 = b * (size_t)a.n_bm + (FORM == kFormKVL ? (size_t)H.cy0 : (size_t)H.br0 * BRW);
  const int nbm = (FORM == kFormKVL) ? H.nCy : nB * BRW;
  const double *lam_g = a.lam + b * (size_t)a.n_bus + H.bus0;
  const double *br_g = a.br + bm0;
  const double *d_g = a.d + b * (size_t)a.n_bus + H.bus0;
  for (int i = tid; i < nA; i += nthr) {
    lam_s[i] = lam_g[i];
    d_s[i] = d_g[i];
  }
  for (int j = tid; j < nbm; j += nthr) br_s[j] = br_g[j];
  // optimiser state (same layout as the multipliers)
  const bool ost = OPT && (MODE == kModeStep) && a.opt != DCOPF_OPT_PLAIN;
  const bool ost2 = ost && a.opt == DCOPF_OPT_ADAM;
  double *s1l = reinterpret_cast<double *>(smem + H.off_s1l), *s2l = reinterpret_cast<double *>(smem + H.off_s2l);
  double *s1b = reinterpret_cast<double *>(smem + H.off_s1b), *s2b = reinterpret_cast<double *>(smem + H.off_s2b);
  if (ost) {
    const size_t ol = b * (size_t)a.n_bus + H.bus0;
    for (int i = tid; i < nA; i += nthr) {
      s1l[i] = a.s1_lam[ol + i];
      if (ost2) s2l[i] = a.s2_lam[ol + i];
    }
    for (int j = tid; j < nbm; j += nthr) {
      s1b[j] = a.s1_br[bm0 + j];
      if (ost2) s2b[j] = a.s2_br[bm0 + j];
    }
  }
  double b1t = a.b1t, b2t = a.b2t;
  if (tid == 0) flag[0] = (MODE != kModeEval) ? a.status[b] : 0;
  double best = (MODE != kModeEval) ? a.best[b] : 0.0;
  double gprev = 0.0;  // g(y_{k-1}) within this call (stopping rule; warp 0 lane 0)
  __syncthreads();
  cl_sync();  // every CTA's shared memory is ready for remote reads

  const ClA *Ar = reinterpret_cast<const ClA *>(smem + H.off_A);
  const ClB *Br = reinterpret_cast<const ClB *>(smem + H.off_B);
  const ClC *Cr = reinterpret_cast<const ClC *>(smem + H.off_C);
  const ClG *Gr = reinterpret_cast<const ClG *>(smem + H.off_G);
  const long K = (MODE == kModeEval) ? 0 : a.K;

  // dual value of iteration kk: every CTA sums the C partials in rank order
  auto finish = [&](long kk) {
    if (warp == 0) {
      const double p = (lane < (int)C) ? cl_ld(cl_map(red_addr0, lane)) : 0.0;
      double g = 0.0;
      for (unsigned r = 0; r < C; ++r) g += __shfl_sync(0xffffffffu, p, r);
      if (lane == 0) {
        int frozen = flag[0];
        if (MODE == kModeEval) {
          if (rank == 0) a.value[b] = g;
        } else {
          if (rank == 0) {
            if (kk < K && a.hist) a.hist[(size_t)kk * a.B + b] = g;
            if (kk == K) a.bound[b] = g;
          }
          if (!frozen) {
            if (valid_bound(g)) {
              best = (g > best) ? g : best;
              if (a.tol > 0.0 && kk > 0 && fabs(g - gprev) < a.tol) frozen = 2;  // Alg. 1 stopping rule
            } else {
              frozen = 1;
            }
          }
          gprev = g;
          if (rank == 0 && a.target && a.hit[b] < 0 && best >= a.target[b]) a.hit[b] = a.k_base + kk;
          flag[0] = frozen;
        }
      }
    }
    __syncthreads();
  };

  const int nAw = a.dbg ? 0 : nA, nBw = a.dbg ? 0 : nB, nCyw = a.dbg ? 0 : H.nCy;  // (dbg: measurement)
  // the step of iteration k+1 is fetched during iteration k: every cluster
  // barrier invalidates L1, so a load at the top of the iteration would cost
  // an L2 round trip on the critical path each time
  double alpha_next = (K > 0) ? a.alpha[0] : 0.0;
  for (long k = 0; k <= K; ++k) {
    const double alpha = alpha_next;
    if (k + 1 < K) alpha_next = a.alpha[k + 1];
    if (ost2 && k < K) {  // Adam's beta^t, t = steps since the state was reset
      b1t = b1t * a.beta1;
      b2t = b2t * a.beta2;
    }
    AdamC ac = {1.0, 1.0, 1.0, 1.0};
    if (ost2) ac = adam_consts(b1t, b2t);
    double val = 0.0;
    // ---------------- A: w_i, theta*_i (not in the angle-free KVL form) ----------------
    if (FORM != kFormKVL) {
    for (int i = tid; i < nAw; i += nthr) {
      const ClA r = Ar[i];
      double w = 0.0;
      if (FORM == kFormF2) {
        const ClIA2 *IA = reinterpret_cast<const ClIA2 *>(smem + H.off_IA);
        for (int e = r.e0; e < r.e1; ++e) {
          const ClIA2 x = IA[e];
          w = w + x.sb * cl_ld(x.nu);  // w_s += -(b nu), w_t += b nu
        }
      } else {
        const ClIA1 *IA = reinterpret_cast<const ClIA1 *>(smem + H.off_IA);
        for (int e = r.e0; e < r.e1; ++e) {
          const ClIA1 x = IA[e];
          const double2 m = cl_ld2(x.mu);
          w = w + x.sb * ((m.x - m.y) - (cl_ld(x.ls) - cl_ld(x.lt)));  // w_s += u, w_t -= u
        }
      }
      const bool isref = (i == H.ref_local);
      const double th = isref ? 0.0 : ((w < 0.0) ? r.theta : ((w > 0.0) ? -r.theta : 0.0));
      th_s[i] = th;
      if (!isref) val += w * th;
    }
    cl_sync(C);
    if (FORM == kFormF2 && k > 0) finish(k - 1);
    }
    const bool step = (MODE == kModeStep) && (k < K) && !flag[0];
    // ---------------- B: branches ----------------
    if (FORM == kFormKVL) {
      // q_l = x_l (sum_k C_kl kappa_k) - (lambda_s - lambda_t), cycles in ascending k
      const ClBk *Bk = reinterpret_cast<const ClBk *>(smem + H.off_B);
      const ClBKe *BK = reinterpret_cast<const ClBKe *>(smem + H.off_IA);
      for (int j = tid; j < nBw; j += nthr) {
        const ClBk r = Bk[j];
        double sum = 0.0;
        for (int e = r.e0; e < r.e1; ++e) {
          const ClBKe x = BK[e];
          const double kv = cl_ld(x.kap);
          sum = (x.sgn > 0) ? sum + kv : sum - kv;
        }
        const double q = r.x * sum - (cl_ld(r.ls) - cl_ld(r.lt));
        const double f = (q > 0.0) ? -r.F : ((q < 0.0) ? r.F : 0.0);
        fc_s[j] = f;
        val += q * f;
      }
    } else
    for (int j = tid; j < nBw; j += nthr) {
      const ClB r = Br[j];
      const double phi = r.b * (cl_ld(r.ts) - cl_ld(r.tt));
      if (FORM == kFormF2) {
        const double nu = br_s[j];
        const double q = nu - (cl_ld(r.ls) - cl_ld(r.lt));
        const double f = (q > 0.0) ? -r.F : ((q < 0.0) ? r.F : 0.0);
        fc_s[j] = f;
        const double g = f - phi;  // Kirchhoff residual
        val += q * f;
        if (step) br_s[j] = ost ? opt_step(a, nu, g, alpha, &s1b[j], &s2b[j], ac) : nu + alpha * g;
        if (MODE == kModeEval) a.grad_br[b * (size_t)a.n_br + H.br0 + j] = g;
      } else {
        const double mp = br_s[2 * j], mm = br_s[2 * j + 1];
        const double gp = phi - r.F, gm = -phi - r.F;
        val += -(r.F * (mp + mm));
        if (step) {
          const double vp = ost ? opt_step(a, mp, gp, alpha, &s1b[2 * j], &s2b[2 * j], ac) : mp + alpha * gp;
          const double vm =
              ost ? opt_step(a, mm, gm, alpha, &s1b[2 * j + 1], &s2b[2 * j + 1], ac) : mm + alpha * gm;
          br_s[2 * j] = (vp > 0.0) ? vp : 0.0;  // mu <- max(mu, 0)
          br_s[2 * j + 1] = (vm > 0.0) ? vm : 0.0;
        }
        if (MODE == kModeEval) {
          a.grad_br[(b * (size_t)a.n_br + H.br0 + j) * 2] = gp;
          a.grad_br[(b * (size_t)a.n_br + H.br0 + j) * 2 + 1] = gm;
        }
      }
    }
    cl_sync(C);
    // ---------------- C: generators, d/dlambda, lambda' ----------------
    for (int i = tid; i < nAw; i += nthr) {
      const ClC r = Cr[i];
      const double li = lam_s[i], di = d_s[i];
      double gl = -di;
      for (int gg = r.g0; gg < r.g1; ++gg) {
        const ClG G = Gr[gg];
        const double rc = G.c + li;
        const double p = gen_minimiser(rc, G.lo, G.hi, G.a);
        gl = gl + p;
        val += (G.a > 0.0) ? G.a * p * p + rc * p : rc * p;
      }
      if (FORM == kFormF2 || FORM == kFormKVL) {
        const ClIC2 *IC = reinterpret_cast<const ClIC2 *>(smem + H.off_IC);
        for (int e = r.e0; e < r.e1; ++e) {
          const ClIC2 x = IC[e];
          const double f = cl_ld(x.f);
          gl = (x.sgn > 0) ? gl + f : gl - f;
        }
      } else {
        const ClIC1 *IC = reinterpret_cast<const ClIC1 *>(smem + H.off_IC);
        for (int e = r.e0; e < r.e1; ++e) {
          const ClIC1 x = IC[e];
          gl = gl + x.sb * (cl_ld(x.ts) - cl_ld(x.tt));  // +phi at the to bus, -phi at the from bus
        }
      }
      val += -(li * di);
      if (step) lam_s[i] = ost ? opt_step(a, li, gl, alpha, &s1l[i], &s2l[i], ac) : li + alpha * gl;
      if (MODE == kModeEval) a.grad_lam[b * (size_t)a.n_bus + H.bus0 + i] = gl;
    }
    if (FORM == kFormKVL) {
      // d/dkappa_k = sum_l C_kl (f*_l x_l), branches in ascending id (f * (-x) == -(f x))
      const ClCy *Cy = reinterpret_cast<const ClCy *>(smem + H.off_Cy);
      const ClCe *CE = reinterpret_cast<const ClCe *>(smem + H.off_CE);
      for (int c = tid; c < nCyw; c += nthr) {
        const ClCy r = Cy[c];
        double acc = 0.0;
        for (int e = r.e0; e < r.e1; ++e) {
          const ClCe x = CE[e];
          acc = acc + cl_ld(x.f) * x.sx;
        }
        const double kv = br_s[c];
        if (step) br_s[c] = ost ? opt_step(a, kv, acc, alpha, &s1b[c], &s2b[c], ac) : kv + alpha * acc;
        if (MODE == kModeEval) a.grad_br[b * (size_t)a.n_bm + H.cy0 + c] = acc;
      }
    }
    // ---------------- this CTA's partial of g(y_k) ----------------
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) val += __shfl_xor_sync(0xffffffffu, val, off);
    if (lane == 0) wred[warp] = val;
    __syncthreads();
    if (warp == 0) {
      double v = (lane < (nthr >> 5)) ? wred[lane] : 0.0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) red[0] = v;
    }
    if (FORM != kFormF2 || k == K) {
      cl_sync(C);  // F1 / KVL: the next phase reads lambda' (kappa'); and every partial is published
      finish(k);
    }
  }
  // ---- results -----------------------------------------------------------------
  if (MODE == kModeStep) {
    double *lam_o = a.lam + b * (size_t)a.n_bus + H.bus0;
    double *br_o = a.br + bm0;
    for (int i = tid; i < nAw; i += nthr) lam_o[i] = lam_s[i];
    for (int j = tid; j < nbm; j += nthr) br_o[j] = br_s[j];
    if (ost) {
      const size_t ol = b * (size_t)a.n_bus + H.bus0;
      for (int i = tid; i < nAw; i += nthr) {
        a.s1_lam[ol + i] = s1l[i];
        if (ost2) a.s2_lam[ol + i] = s2l[i];
      }
      for (int j = tid; j < nbm; j += nthr) {
        a.s1_br[bm0 + j] = s1b[j];
        if (ost2) a.s2_br[bm0 + j] = s2b[j];
      }
    }
  }
  if (MODE != kModeEval && rank == 0 && tid == 0) {
    a.best[b] = best;
    a.status[b] = flag[0];
  }
  cl_sync();  // no CTA exits while another may still read its shared memory
}

}  // namespace dcopf
