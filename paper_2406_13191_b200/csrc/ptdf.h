// ptdf.h -- the dense-PTDF form (DCOPF_FORM_PTDF): the
// paper's Eq. 1 literally, for load-only batches on a fixed
// topology.  Internal interface between the ABI (dcopf_dual.cu) and ptdf.cu.
//
// Construction (create): H_a = T - C^T M^{-1} C X T from a spanning tree and
// its fundamental cycles (the canonical basis of cluster.h, reading A-28):
//   T  [n_l][n_b]  tree flows of "inject 1 at bus i, withdraw at the slack"
//                  (+-1 on the tree path i -> ref, 0 elsewhere; slack column 0),
//   C  [n_c][n_l]  signed cycle incidence, X = diag(1/b),
//   M = C X C^T    (SPD, n_c x n_c; Cholesky on the host, L^{-1} explicit),
//   W = L^{-T} (L^{-1} (C X T))   two fp64 GEMMs on the GPU,
//   H_a = T - C^T W               (Kirchhoff's voltage law holds on every cycle
//                                  and the tree part carries the injections).
// This equals Omega E (E^T Omega E)^{-1} with a zero slack column (KCL + KVL
// fix the flows uniquely) but costs O(n_c^3) on the host instead of O(n_b^3).
//
// Iteration (per batch of B load scenarios, instance index contiguous):
//   GEMM1  Q = H_g^T nu        [n_g x B], nu = mu+ - mu-   epilogue: q = c + lambda + Q,
//          p* = argmin (bound selection / clip), per-tile partial sums of a p*^2 + q p* and p*
//   GEMM2  Y = H_g p*          [n_l x B]                    epilogue: grad mu+- = +-(Y - r) - F,
//          partial sums of -mu+ (r + F) + mu- (r - F), projected step of mu+-, nu
//   finish per instance: g, grad lambda = sum p* - 1^T d, best / status / history / first hit,
//          step of lambda
// with r = H_a d computed once per batch (a third GEMM).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/dcopf_dual.h"

namespace dcopf {

struct PtdfState;

struct PtdfNetIn {
  int nb, nl, ng, ref;
  const int *fr, *to;
  const double *b, *F;
  const int *gen_bus;
  const double *lo, *hi, *c, *a;  // a may be null
};

// Every function returns DCOPF_OK or a DCOPF_E* code with *err set.
int ptdf_create(const PtdfNetIn &net, int device, PtdfState **out, std::string *err);
void ptdf_destroy(PtdfState *st);
int ptdf_set_batch(PtdfState *st, int64_t B, const double *load, cudaStream_t s, std::string *err);
// alpha_dev: device copy of alpha[K]; hist: device [K][B] or null
int ptdf_iterate(PtdfState *st, int64_t K, const double *alpha_dev, double *hist, cudaStream_t s, std::string *err);
int ptdf_get_bound(PtdfState *st, double *bound, double *best, int32_t *status, cudaStream_t s, std::string *err);
int ptdf_get_multipliers(PtdfState *st, double *lambda, double *branch, cudaStream_t s, std::string *err);
int ptdf_set_multipliers(PtdfState *st, const double *lambda, const double *branch, cudaStream_t s,
                         std::string *err);
int ptdf_evaluate(PtdfState *st, double *value, double *grad_lambda, double *grad_branch, cudaStream_t s,
                  std::string *err);
int ptdf_set_optimizer(PtdfState *st, const dcopf_optimizer &o, std::string *err);
void ptdf_set_stop(PtdfState *st, double tol);
int ptdf_set_target(PtdfState *st, const double *target, cudaStream_t s, std::string *err);
int ptdf_get_first_hit(PtdfState *st, int64_t *hit, cudaStream_t s, std::string *err);
void ptdf_info(const PtdfState *st, dcopf_info *info);
int64_t ptdf_batch(const PtdfState *st);
// the PTDF matrix H_a [n_l][n_b] (row-major, original ids) into a host or device buffer
int ptdf_get_matrix(PtdfState *st, double *Ha, cudaStream_t s, std::string *err);

}  // namespace dcopf
