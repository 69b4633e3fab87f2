// ptdf.cu -- dense-PTDF form of the dual: the paper's Eq. 1
// with one shared H_a for a batch of load scenarios, iterated
// as two fp64 GEMMs per ascent step on the tensor cores (DMMA, mma.sync
// m8n8k4 f64: sm_100a's fp64 tensor-core instruction; tcgen05 has no fp64
// kind) with the inner minimisation, the dual value, the gradient and the
// projected step fused into the GEMM epilogues.  See ptdf.h for the algebra.
#include "ptdf.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

#include "cluster.h"
#include "fp64_fast.cuh"

namespace dcopf {
namespace {

// ---------------------------------------------------------------------------
// GEMM tiling: C[M][N] = A[M][K] B[K][N], A row-major (K contiguous), B
// row-major (N = instances contiguous).  64 x 128 x 16 CTA tiles of 4 warps
// (warp tile 64 x 32 = 8 x 4 DMMA m8n8k4 tiles, 64 fp64 accumulators per
// thread), two CTAs per SM so one CTA's barrier / epilogue overlaps the
// other's DMMA stream, a 4-stage cp.async pipeline, padded shared-memory rows
// (conflict-free fragment loads: A stride BK+4, B stride 132 doubles).
// Measured on config 4b: 128 x 128 tiles at one CTA per SM
// reached 79% of the DGEMM peak per step, 64 x 128 at two per SM 85%, two
// column groups on two streams 89%, register double-buffered fragments 94%.
// M, N, K are padded to the tile sizes with zeros by the owner of each matrix.
#ifndef PTDF_LINE_STAGE
#define PTDF_LINE_STAGE 1
#endif
#ifndef PTDF_FRAG_DB
#define PTDF_FRAG_DB 1
#endif
#ifndef PTDF_BM
#define PTDF_BM 64
#endif
#ifndef PTDF_BK
#define PTDF_BK 16
#endif
#ifndef PTDF_STAGES
#define PTDF_STAGES 4
#endif
constexpr int BM = PTDF_BM, BN = 128, BK = PTDF_BK, STAGES = PTDF_STAGES;
constexpr int NTHR = (BM / 64) * 4 * 32;  // warps: BM/64 (M) x 4 (N), warp tile 64 x 32
constexpr int CTAS_PER_SM = (BM == 64) ? 2 : 1;
constexpr int WMN = BM / 64;
constexpr int AST = BK + 4, BST = BN + 4;
constexpr int A_STAGE = BM * AST, B_STAGE = BK * BST;  // doubles
constexpr int GEMM_SMEM = STAGES * (A_STAGE + B_STAGE) * 8;

enum { EPI_STORE = 0, EPI_GEN = 1, EPI_LINE_STEP = 2, EPI_LINE_EVAL = 3 };

inline long up(long x, long m) { return (x + m - 1) / m * m; }

struct GemmArgs {
  const double *A;
  long lda;
  const double *Bm;
  long ldb;
  int M, N, K, group;
  int noff;  // first column of this launch (a launch covers columns [noff, noff + N))
  int ktps;          // split-K (EPI_STORE, gridDim.y splits): k-tiles per split (0: all)
  long c_split;      // ... and the distance between the splits' C blocks
  long ld;  // leading dimension of every [rows][B_pad] array (= B_pad) / of C for EPI_STORE
  double *C;
  // EPI_GEN (rows = generators)
  const double *gc, *glo, *ghi, *ga;
  int ng;
  const double *lam;
  double *P, *part_obj, *part_p;
  // EPI_LINE (rows = lines)
  const double *r, *F;
  int nl;
  double *mup, *mum, *nu, *part_line, *gp_out, *gm_out;
  const int *status;
  const double *alpha;
  int k;
  int opt;
  double rho, beta1, beta2, eps, b1t, b2t;
  double *s1p, *s2p, *s1m, *s2m;
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// x / d for a positive finite d, sqrt(x) for x >= 0, skipping the operation
// where x == 0 (the result is x itself; CUDA's zero-operand case is an
// out-of-line slow path taken by the whole warp).  Bitwise the same results.
// (the compiler evaluates both sides of a select and would fold a plain
// (x == 0 ? 1 : x) back into x, so the zero lanes' operand 1 is selected in
// asm: they divide 1 by d -- never the slow path -- and keep x)
__device__ __forceinline__ double nz_or_one(double x) {
  double r;
  asm("{\n\t.reg .pred z;\n\tsetp.eq.f64 z, %1, 0d0000000000000000;\n\tselp.f64 %0, 0d3FF0000000000000, %1, z;\n\t}"
      : "=d"(r)
      : "d"(x));
  return r;
}
__device__ __forceinline__ double div_pos(double x, double d) {
  const double q = nz_or_one(x) / d;
  return x == 0.0 ? x : q;
}
__device__ __forceinline__ double sqrt_nz(double x) {
  const double r = sqrt(nz_or_one(x));
  return x == 0.0 ? x : r;
}

__device__ __forceinline__ double opt_step(const GemmArgs &g, double y, double gr, double al, double &s1,
                                           double &s2) {
  switch (g.opt) {
    case 1: {  // GDM (Algorithm 1 as printed: velocity update, then gradient update; reading A-25)
      const double v = g.rho * s1 + al * gr;
      s1 = v;
      y = y + v;
      return y + al * gr;
    }
    case 2: {  // GDM-classic
      const double v = g.rho * s1 + al * gr;
      s1 = v;
      return y + v;
    }
    case 3: {  // AdaGrad (reading A-26)
      const double G = s1 + gr * gr;
      s1 = G;
      return y + div_pos(al * gr, sqrt_nz(G) + g.eps);
    }
    case 4: {  // Adam (reading A-26)
      const double m = g.beta1 * s1 + (1.0 - g.beta1) * gr;
      const double v = g.beta2 * s2 + (1.0 - g.beta2) * (gr * gr);
      s1 = m;
      s2 = v;
      const double mh = div_pos(m, 1.0 - g.b1t), vh = div_pos(v, 1.0 - g.b2t);
      return y + div_pos(al * mh, sqrt_nz(vh) + g.eps);
    }
    default:
      return y + al * gr;
  }
}

// The adaptive variants (AdaGrad, Adam) on a row's two multipliers (mu+,
// mu-) at once, in opt_step's operation order, every division and square root
// on the branch-free fast paths (fp64_fast.cuh) so the two Newton chains
// overlap, then ONE warp vote: every value passed -- opt_step's bits;
// otherwise opt_step itself.  Other variants: opt_step.
__device__ __forceinline__ void opt_step2(const GemmArgs &g, double yp, double gp, double ym, double gm, double al,
                                          double &s1p, double &s2p, double &s1m, double &s2m, double &vp,
                                          double &vm) {
  if (g.opt == 3 || g.opt == 4) {
    bool ok = true;
    double y[2] = {yp, ym}, gr[2] = {gp, gm}, s1[2] = {s1p, s1m}, s2[2] = {s2p, s2m}, out[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      double num, arg;
      if (g.opt == 4) {
        const double m = g.beta1 * s1[j] + (1.0 - g.beta1) * gr[j];
        const double v = g.beta2 * s2[j] + (1.0 - g.beta2) * (gr[j] * gr[j]);
        s1[j] = m;
        s2[j] = v;
        const double mq = ddiv_fast(nz_or_one(m), 1.0 - g.b1t, ok), vq = ddiv_fast(nz_or_one(v), 1.0 - g.b2t, ok);
        num = al * (m == 0.0 ? m : mq);
        arg = v == 0.0 ? v : vq;
      } else {
        const double G = s1[j] + gr[j] * gr[j];
        s1[j] = G;
        num = al * gr[j];
        arg = G;
      }
      const double sr = dsqrt_fast(nz_or_one(arg), ok);
      const double q = ddiv_fast(nz_or_one(num), (arg == 0.0 ? arg : sr) + g.eps, ok);
      out[j] = y[j] + (num == 0.0 ? num : q);
    }
    if (__all_sync(__activemask(), ok)) {
      vp = out[0];
      vm = out[1];
      s1p = s1[0];
      s1m = s1[1];
      s2p = s2[0];
      s2m = s2[1];
      return;
    }
  }
  vp = opt_step(g, yp, gp, al, s1p, s2p);
  vm = opt_step(g, ym, gm, al, s1m, s2m);
}

// p* = argmin over [lo, hi] of a p^2 + q p: clip(-q / 2a) (reading A-6), else
// bound selection with sign(0) -> midpoint (reading A-4)
__device__ __forceinline__ double minimiser(double q, double lo, double hi, double a) {
  if (a > 0.0) {
    const double x = -q / (2.0 * a);
    return (x < lo) ? lo : ((x > hi) ? hi : x);
  }
  return (q > 0.0) ? lo : ((q < 0.0) ? hi : 0.5 * (lo + hi));
}

// one CTA per 128 x 128 output tile, grouped raster (`group` M-tiles per band,
// M fastest inside a band) so concurrently running CTAs share A and B tiles in L2
template <int EPI>
__global__ void __launch_bounds__(NTHR, CTAS_PER_SM) k_dgemm(const GemmArgs g) {
  extern __shared__ __align__(16) double sm[];
  double *As = sm, *Bs = sm + STAGES * A_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, wm = warp >> 2, wn = warp & 3;
  const int nMt = g.M / BM, nNt = g.N / BN;
  const int t = blockIdx.x, band = t / (g.group * nNt), first_m = band * g.group;
  const int gs = min(nMt - first_m, g.group);
  const int mt = first_m + (t % (g.group * nNt)) % gs, nt = (t % (g.group * nNt)) / gs;
  const int m0 = mt * BM, n0 = g.noff + nt * BN;
  // split-K (gridDim.y > 1, EPI_STORE only): this CTA's k-tile range
  const int KT0 = g.ktps ? blockIdx.y * g.ktps : 0;
  const int KT = g.ktps ? min(g.K / BK - KT0, g.ktps) : g.K / BK;

  auto load_stage = [&](int stage, int kt) {
    const int k0 = (KT0 + kt) * BK;
    double *as = As + stage * A_STAGE, *bs = Bs + stage * B_STAGE;
#pragma unroll
    for (int c = tid; c < BM * BK / 2; c += NTHR) {
      const int row = c / (BK / 2), ch = c % (BK / 2);
      cp_async16(as + row * AST + ch * 2, g.A + (size_t)(m0 + row) * g.lda + k0 + ch * 2);
    }
#pragma unroll
    for (int c = tid; c < BK * BN / 2; c += NTHR) {
      const int row = c >> 6, ch = c & 63;
      cp_async16(bs + row * BST + ch * 2, g.Bm + (size_t)(k0 + row) * g.ldb + n0 + ch * 2);
    }
  };

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }
#if PTDF_FRAG_DB
  // Fragments double-buffered in registers: the next k4 step's fragments are
  // loaded while the current one's DMMAs issue, and at the last k4 step of a
  // tile the next tile's stage is awaited (one barrier per tile) before its
  // first fragments are loaded -- no shared-memory latency after the barrier.
  constexpr int KK = BK / 4;
  static_assert(STAGES >= 3, "the double-buffered main loop waits for stage kt+1 one tile early");
  double fa[2][8], fb[2][4];
  auto ld_frag = [&](int buf, int stage, int kk) {
    const double *as = As + stage * A_STAGE + (wm * 64 + (lane >> 2)) * AST + (lane & 3) + kk * 4;
    const double *bs = Bs + stage * B_STAGE + (lane & 3) * BST + wn * 32 + (lane >> 2) + kk * 4 * BST;
#pragma unroll
    for (int i = 0; i < 8; ++i) fa[buf][i] = as[i * 8 * AST];
#pragma unroll
    for (int j = 0; j < 4; ++j) fb[buf][j] = bs[j * 8];
  };
  if (KT > 0) {
    cp_async_wait<STAGES - 2>();  // stage 0 landed
    __syncthreads();
    ld_frag(0, 0, 0);
  }
  for (int kt = 0; kt < KT; ++kt) {
#pragma unroll
    for (int kk = 0; kk < KK; ++kk) {
      if (kk == KK - 1) {
        cp_async_wait<STAGES - 3>();  // stage kt+1 landed (groups committed: STAGES-1+kt)
        __syncthreads();              // ... for every thread; stage kt-1 is free
        const int nk = kt + STAGES - 1;
        if (nk < KT) load_stage(nk % STAGES, nk);
        cp_async_commit();
        if (kt + 1 < KT) ld_frag((kk + 1) & 1, (kt + 1) % STAGES, 0);
      } else {
        ld_frag((kk + 1) & 1, kt % STAGES, kk + 1);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], fa[kk & 1][i], fb[kk & 1][j]);
    }
  }
#else
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();  // stage kt landed for every thread; stage kt-1 is free
    const int nk = kt + STAGES - 1;
    if (nk < KT) load_stage(nk % STAGES, nk);
    cp_async_commit();
    const double *as = As + (kt % STAGES) * A_STAGE + (wm * 64 + (lane >> 2)) * AST + (lane & 3);
    const double *bs = Bs + (kt % STAGES) * B_STAGE + (lane & 3) * BST + wn * 32 + (lane >> 2);
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double a[8], b[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = as[i * 8 * AST + kk * 4];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bs[kk * 4 * BST + j * 8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    }
  }
#endif
  cp_async_wait<0>();
  __syncthreads();  // pipeline buffers are free: the epilogue reuses them

  // fragment (i, j, e) <-> row m0 + wm*64 + i*8 + lane/4, column n0 + wn*32 + j*8 + 2*(lane%4) + e
  const int rbase = m0 + wm * 64 + (lane >> 2);
  const int cbase = n0 + wn * 32 + 2 * (lane & 3);
  if (EPI == EPI_STORE) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        *reinterpret_cast<double2 *>(g.C + blockIdx.y * g.c_split + (size_t)(rbase + i * 8) * g.ld + cbase + j * 8) =
            make_double2(acc[i][j][0], acc[i][j][1]);
    return;
  }
  double s0[4][2], s1[4][2];  // per-column partial sums over this thread's 8 rows
#pragma unroll
  for (int j = 0; j < 4; ++j) s0[j][0] = s0[j][1] = s1[j][0] = s1[j][1] = 0.0;

  if (EPI == EPI_GEN) {
    double lamv[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double2 l2 = *reinterpret_cast<const double2 *>(g.lam + cbase + j * 8);
      lamv[j][0] = l2.x;
      lamv[j][1] = l2.y;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = rbase + i * 8;
      const bool live = row < g.ng;
      const double c = live ? g.gc[row] : 0.0, lo = live ? g.glo[row] : 0.0, hi = live ? g.ghi[row] : 0.0;
      const double a = (live && g.ga) ? g.ga[row] : 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double pv[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double q = (c + lamv[j][e]) + acc[i][j][e];  // q = c + lambda 1 + H_g^T nu
          double p = minimiser(q, lo, hi, a);
          if (!live) p = 0.0;
          pv[e] = p;
          if (live) {
            s0[j][e] += a * p * p + q * p;
            s1[j][e] += p;
          }
        }
        *reinterpret_cast<double2 *>(g.P + (size_t)row * g.ld + cbase + j * 8) = make_double2(pv[0], pv[1]);
      }
    }
  } else if (PTDF_LINE_STAGE && g.opt != 0) {  // EPI_LINE_* with optimiser state rows: staged
    // (measured: +3% with Adam at config 4b, neutral for the plain step, which keeps the fragment path)
    // The accumulator tile goes to the freed pipeline shared memory; then one
    // thread per column walks the tile's rows with coalesced loads that do not
    // depend on each other (the fragment layout left every row's operands to
    // one dependent chain per thread).  The value partial is per column, rows
    // in order.
    constexpr int CST = BN + 2;
    double *Cs = sm;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        *reinterpret_cast<double2 *>(Cs + (size_t)(wm * 64 + i * 8 + (lane >> 2)) * CST + wn * 32 + j * 8 +
                                     2 * (lane & 3)) = make_double2(acc[i][j][0], acc[i][j][1]);
    __syncthreads();
    for (int c = tid; c < BN; c += NTHR) {
      const int n = n0 + c;
      const double al = (EPI == EPI_LINE_STEP) ? g.alpha[g.k] : 0.0;
      const bool frozen = (EPI == EPI_LINE_STEP) ? g.status[n] != 0 : true;
      double sv = 0.0;
      const int rows = min(BM, g.nl - m0);
#pragma unroll 4
      for (int rr = 0; rr < rows; ++rr) {
        const int row = m0 + rr;
        const size_t o = (size_t)row * g.ld + n;
        const double y = Cs[(size_t)rr * CST + c], F = g.F[row];
        const double rv = g.r[o], mp = g.mup[o], mm = g.mum[o];
        const double gp = (y - rv) - F, gm = (rv - y) - F;  // dg/dmu+-
        sv += mm * (rv - F) - mp * (rv + F);
        if (EPI == EPI_LINE_EVAL) {
          if (g.gp_out) {
            g.gp_out[o] = gp;
            g.gm_out[o] = gm;
          }
        } else if (!frozen) {
          double vp, vm;
          if (g.opt == 0) {
            vp = mp + al * gp;
            vm = mm + al * gm;
          } else {
            double a1 = g.s1p[o], a2 = g.s2p ? g.s2p[o] : 0.0, b1 = g.s1m[o], b2 = g.s2m ? g.s2m[o] : 0.0;
            opt_step2(g, mp, gp, mm, gm, al, a1, a2, b1, b2, vp, vm);
            g.s1p[o] = a1;
            g.s1m[o] = b1;
            if (g.s2p) {
              g.s2p[o] = a2;
              g.s2m[o] = b2;
            }
          }
          const double np = vp > 0.0 ? vp : 0.0, nm = vm > 0.0 ? vm : 0.0;  // mu <- max(mu, 0)
          g.mup[o] = np;
          g.mum[o] = nm;
          g.nu[o] = np - nm;
        }
      }
      g.part_line[(size_t)mt * g.ld + n] = sv;
    }
    return;
  } else {  // EPI_LINE_*
    const double al = (EPI == EPI_LINE_STEP) ? g.alpha[g.k] : 0.0;
    bool frozen[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      frozen[j][0] = (EPI == EPI_LINE_STEP) ? g.status[cbase + j * 8] != 0 : true;
      frozen[j][1] = (EPI == EPI_LINE_STEP) ? g.status[cbase + j * 8 + 1] != 0 : true;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = rbase + i * 8;
      if (row >= g.nl) continue;
      const double F = g.F[row];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const size_t o = (size_t)row * g.ld + cbase + j * 8;
        const double2 r2 = *reinterpret_cast<const double2 *>(g.r + o);
        const double2 p2 = *reinterpret_cast<const double2 *>(g.mup + o);
        const double2 m2 = *reinterpret_cast<const double2 *>(g.mum + o);
        const double rv[2] = {r2.x, r2.y}, mp[2] = {p2.x, p2.y}, mm[2] = {m2.x, m2.y};
        double gp[2], gm[2], np[2], nm[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double y = acc[i][j][e];
          gp[e] = (y - rv[e]) - F;  // dg/dmu+ = H_g p* - r - F
          gm[e] = (rv[e] - y) - F;  // dg/dmu- = r - H_g p* - F
          s0[j][e] += mm[e] * (rv[e] - F) - mp[e] * (rv[e] + F);
          np[e] = mp[e];
          nm[e] = mm[e];
        }
        if (EPI == EPI_LINE_EVAL) {
          if (g.gp_out) {
            *reinterpret_cast<double2 *>(g.gp_out + o) = make_double2(gp[0], gp[1]);
            *reinterpret_cast<double2 *>(g.gm_out + o) = make_double2(gm[0], gm[1]);
          }
        } else {
          if (g.opt == 0) {
#pragma unroll
            for (int e = 0; e < 2; ++e)
              if (!frozen[j][e]) {
                const double vp = mp[e] + al * gp[e], vm = mm[e] + al * gm[e];
                np[e] = vp > 0.0 ? vp : 0.0;  // mu <- max(mu, 0)
                nm[e] = vm > 0.0 ? vm : 0.0;
              }
          } else {
            double2 a1 = *reinterpret_cast<const double2 *>(g.s1p + o);
            double2 a2 = g.s2p ? *reinterpret_cast<const double2 *>(g.s2p + o) : make_double2(0.0, 0.0);
            double2 b1 = *reinterpret_cast<const double2 *>(g.s1m + o);
            double2 b2 = g.s2m ? *reinterpret_cast<const double2 *>(g.s2m + o) : make_double2(0.0, 0.0);
            double sa1[2] = {a1.x, a1.y}, sa2[2] = {a2.x, a2.y}, sb1[2] = {b1.x, b1.y}, sb2[2] = {b2.x, b2.y};
#pragma unroll
            for (int e = 0; e < 2; ++e)
              if (!frozen[j][e]) {
                const double vp = opt_step(g, mp[e], gp[e], al, sa1[e], sa2[e]);
                const double vm = opt_step(g, mm[e], gm[e], al, sb1[e], sb2[e]);
                np[e] = vp > 0.0 ? vp : 0.0;
                nm[e] = vm > 0.0 ? vm : 0.0;
              }
            *reinterpret_cast<double2 *>(g.s1p + o) = make_double2(sa1[0], sa1[1]);
            *reinterpret_cast<double2 *>(g.s1m + o) = make_double2(sb1[0], sb1[1]);
            if (g.s2p) {
              *reinterpret_cast<double2 *>(g.s2p + o) = make_double2(sa2[0], sa2[1]);
              *reinterpret_cast<double2 *>(g.s2m + o) = make_double2(sb2[0], sb2[1]);
            }
          }
          *reinterpret_cast<double2 *>(g.mup + o) = make_double2(np[0], np[1]);
          *reinterpret_cast<double2 *>(g.mum + o) = make_double2(nm[0], nm[1]);
          *reinterpret_cast<double2 *>(g.nu + o) = make_double2(np[0] - nm[0], np[1] - nm[1]);
        }
      }
    }
  }
  // column sums: lanes with the same lane%4 hold the same columns (xor over lane/4),
  // then the two M-warps through shared memory, fixed order (deterministic)
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        s0[j][e] += __shfl_xor_sync(0xffffffffu, s0[j][e], off);
        if (EPI == EPI_GEN) s1[j][e] += __shfl_xor_sync(0xffffffffu, s1[j][e], off);
      }
  double *red = sm;  // [2 sums][WMN][BN]
  if (lane < 4) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = wn * 32 + j * 8 + 2 * lane + e;
        red[wm * BN + col] = s0[j][e];
        if (EPI == EPI_GEN) red[WMN * BN + wm * BN + col] = s1[j][e];
      }
  }
  __syncthreads();
  if (tid < BN) {
    const size_t o = (size_t)mt * g.ld + n0 + tid;
    double so = red[tid], sp = red[WMN * BN + tid];
#pragma unroll
    for (int w = 1; w < WMN; ++w) {  // the M-warps in order
      so += red[w * BN + tid];
      sp += red[WMN * BN + w * BN + tid];
    }
    if (EPI == EPI_GEN) {
      g.part_obj[o] = so;
      g.part_p[o] = sp;
    } else {
      g.part_line[o] = so;
    }
  }
}

// ---------------------------------------------------------------------------
// per instance: the dual value, grad lambda, bookkeeping and the lambda step
struct FinArgs {
  const double *part_obj, *part_p, *part_line;
  int nMt1, nMt2;
  long ld, B;
  long n0, n1;  // instances [n0, n1) of this launch
  const double *D;
  double *lam, *sl1, *sl2;
  int *status;
  double *best, *bound, *value, *gprev, *hist, *glam_out;
  const double *alpha, *target;
  long long *hit;
  long long k_base;
  int k, K, first;
  double tol;
  int opt;
  double rho, beta1, beta2, eps, b1t, b2t;
};

__device__ __forceinline__ bool valid_bound(double g) { return isfinite(g) && fabs(g) <= 1e15; }

template <bool EVAL>
__device__ __forceinline__ void finish_one(const FinArgs &f, long n, double so, double sp, double sl) {
  const double lam = f.lam[n], D = f.D[n];
  const double g = (so - lam * D) + sl;
  const double gl = sp - D;  // dg/dlambda = 1^T p* - 1^T d
  if (EVAL) {
    f.value[n] = g;
    if (f.glam_out) f.glam_out[n] = gl;
    return;
  }
  if (f.hist && f.k < f.K && n < f.B) f.hist[(size_t)f.k * f.B + n] = g;
  if (f.k == f.K) f.bound[n] = g;
  int st = f.status[n];
  const bool was = st != 0;
  double best = f.best[n];
  if (!was) {
    if (valid_bound(g)) {
      if (g > best) best = g;
      if (f.tol > 0.0 && !f.first && fabs(g - f.gprev[n]) < f.tol) st = DCOPF_INST_CONVERGED;  // Alg. 1 stop
    } else {
      st = DCOPF_INST_DIVERGED;
    }
  }
  f.gprev[n] = g;
  f.best[n] = best;
  f.status[n] = st;
  if (f.target && f.hit[n] < 0 && best >= f.target[n]) f.hit[n] = f.k_base + f.k;
  if (f.k < f.K && !was) {
    const double al = f.alpha[f.k];
    double s1 = f.sl1 ? f.sl1[n] : 0.0, s2 = f.sl2 ? f.sl2[n] : 0.0;
    GemmArgs o;
    o.opt = f.opt;
    o.rho = f.rho;
    o.beta1 = f.beta1;
    o.beta2 = f.beta2;
    o.eps = f.eps;
    o.b1t = f.b1t;
    o.b2t = f.b2t;
    f.lam[n] = opt_step(o, lam, gl, al, s1, s2);  // lambda free: no projection
    if (f.sl1) f.sl1[n] = s1;
    if (f.sl2) f.sl2[n] = s2;
  }
}

// GEMM mode: one thread per instance sums its tiles' partials in tile order
template <bool EVAL>
__global__ void k_finish(const FinArgs f) {
  const long n = f.n0 + (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= f.n1) return;
  double so = 0.0, sp = 0.0, sl = 0.0;
  for (int t = 0; t < f.nMt1; ++t) {
    so += f.part_obj[(size_t)t * f.ld + n];
    sp += f.part_p[(size_t)t * f.ld + n];
  }
  for (int t = 0; t < f.nMt2; ++t) sl += f.part_line[(size_t)t * f.ld + n];
  finish_one<EVAL>(f, n, so, sp, sl);
}

// skinny mode: one block per instance, its (many) block partials summed by a
// fixed strided split + tree (deterministic)
template <bool EVAL>
__global__ void __launch_bounds__(256) k_finish_blk(const FinArgs f) {
  __shared__ double red[3][256];
  const long n = f.n0 + blockIdx.x;
  double so = 0.0, sp = 0.0, sl = 0.0;
  for (int t = threadIdx.x; t < f.nMt1; t += 256) {
    so += f.part_obj[(size_t)t * f.ld + n];
    sp += f.part_p[(size_t)t * f.ld + n];
  }
  for (int t = threadIdx.x; t < f.nMt2; t += 256) sl += f.part_line[(size_t)t * f.ld + n];
  red[0][threadIdx.x] = so;
  red[1][threadIdx.x] = sp;
  red[2][threadIdx.x] = sl;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int c = 0; c < 3; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) finish_one<EVAL>(f, n, red[0][0], red[1][0], red[2][0]);
}

// ---------------------------------------------------------------------------
// Medium batches: GEMM1 (K = n_l) split over K when its tiles cannot fill the
// GPU; this kernel sums the splits' Q blocks in split order and applies the
// GEMM1 epilogue -- one thread per column, the 64 rows of an M tile in order.
__global__ void __launch_bounds__(BN) k_gen_reduce(const GemmArgs g, const double *__restrict__ Qs, int S,
                                                   long split) {
  const int mt = blockIdx.x, n = g.noff + blockIdx.y * BN + threadIdx.x;
  double so = 0.0, sp = 0.0;
  const double lam = g.lam[n];
  for (int r = 0; r < BM; ++r) {
    const int row = mt * BM + r;
    const bool live = row < g.ng;
    double Q = 0.0;
    for (int x = 0; x < S; ++x) Q += Qs[x * split + (size_t)row * g.ld + n];
    double p = 0.0;
    if (live) {
      const double a = g.ga ? g.ga[row] : 0.0;
      const double q = (g.gc[row] + lam) + Q;  // q = c + lambda 1 + H_g^T nu
      p = minimiser(q, g.glo[row], g.ghi[row], a);
      so += a * p * p + q * p;
      sp += p;
    }
    g.P[(size_t)row * g.ld + n] = p;
  }
  g.part_obj[(size_t)mt * g.ld + n] = so;
  g.part_p[(size_t)mt * g.ld + n] = sp;
}

// ---------------------------------------------------------------------------
// Skinny batches (B <= 4, e.g. one large instance): the two products are
// matrix-vector shaped, i.e. HBM-bound reads of H_g (254 MB at config 3), not
// tensor work.  One warp per row, coalesced double2 loads along the row, the
// vector in a compact [K][NB] copy (nu_c, p_c: L1/L2 resident), a fixed xor
// tree for the dot product, and the epilogue fused: GEMM1 rows are generators
// (A = H_g^T, row g, K = n_l), GEMM2 rows are lines (A = H_g, row l, K = n_g).
// Each block writes its partial sums per instance to part[block][b] (ld NB).
constexpr int VT = 512, VW = VT / 32;   // threads and warps per block
#ifndef PTDF_LINE_CAP
#define PTDF_LINE_CAP (148 * 3)
#endif
#ifndef PTDF_DU
#define PTDF_DU 1
#endif
#ifndef PTDF_WPR_G
#define PTDF_WPR_G 2
#endif
#ifndef PTDF_WPR_L
#define PTDF_WPR_L 1
#endif
constexpr int WPR_G = PTDF_WPR_G, WPR_L = PTDF_WPR_L;  // warps per row: GEMM1 rows are 100 KB (config 3), GEMM2 rows 20 KB

// resident blocks per SM the register budget is sized for: 3 (<= 42 registers)
// for 1-2 columns -- measured: 116 us/it at 3 blocks vs 118 at 2 and 134 at 1 on
// one config-3 instance -- fewer where the per-column state would spill
constexpr int skinny_minb(int nb) { return nb <= 1 ? 3 : (nb <= 4 ? 2 : 1); }

template <int NB>
__device__ __forceinline__ void warp_dot(const double *__restrict__ row, const double *__restrict__ xc, int k0,
                                         int K, double (&acc)[NB]) {
  const int lane = threadIdx.x & 31;
  // DU independent accumulator sets (k strides of 64, DU deep) keep DU row
  // loads in flight per lane; combined in a fixed order
  constexpr int DU = PTDF_DU;
  double part[DU][NB];
#pragma unroll
  for (int u = 0; u < DU; ++u)
#pragma unroll
    for (int b = 0; b < NB; ++b) part[u][b] = 0.0;
  int k = k0 + 2 * lane;
  for (; k + 64 * (DU - 1) < K; k += 64 * DU) {
    double2 a[DU];
#pragma unroll
    for (int u = 0; u < DU; ++u) a[u] = __ldcs(reinterpret_cast<const double2 *>(row + k + 64 * u));
#pragma unroll
    for (int u = 0; u < DU; ++u) {
      const int kk = k + 64 * u;
#pragma unroll
      if (NB == 1) {  // the vector pair in one 16-byte load
        const double2 x = *reinterpret_cast<const double2 *>(xc + kk);
        part[u][0] += a[u].x * x.x + a[u].y * x.y;
      } else {  // the two vector rows as 16-byte loads (NB even)
#pragma unroll
        for (int b = 0; b < NB; b += 2) {
          const double2 x0 = *reinterpret_cast<const double2 *>(xc + kk * NB + b);
          const double2 x1 = *reinterpret_cast<const double2 *>(xc + (kk + 1) * NB + b);
          part[u][b] += a[u].x * x0.x + a[u].y * x1.x;
          part[u][b + 1] += a[u].x * x0.y + a[u].y * x1.y;
        }
      }
    }
  }
  for (int u = 0; k < K; k += 64, ++u) {
    const double2 a = __ldcs(reinterpret_cast<const double2 *>(row + k));
    if (NB == 1) {
      const double2 x = *reinterpret_cast<const double2 *>(xc + k);
      part[u % DU][0] += a.x * x.x + a.y * x.y;
    } else {
#pragma unroll
      for (int b = 0; b < NB; ++b) part[u % DU][b] += a.x * xc[k * NB + b] + a.y * xc[(k + 1) * NB + b];
    }
  }
#pragma unroll
  for (int u = 1; u < DU; ++u)
#pragma unroll
    for (int b = 0; b < NB; ++b) part[0][b] += part[u][b];
#pragma unroll
  for (int b = 0; b < NB; ++b) acc[b] = part[0][b];
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], off);
}

// block partial sums: per-warp values red[warp][b] summed in warp order
template <int NB>
__device__ __forceinline__ void block_part(double *red, const double (&v)[NB], double *part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane < NB) {
#pragma unroll
    for (int b = 0; b < NB; ++b)
      if (b == lane) red[warp * NB + b] = v[b];
  }
  __syncthreads();
  if (threadIdx.x < NB) {
    double t = 0.0;
    for (int w = 0; w < VW; ++w) t += red[w * NB + threadIdx.x];
    part[(size_t)blockIdx.x * NB + threadIdx.x] = t;
  }
}

// the row's K range split over WPR warps (64-aligned); their dot products are
// combined in warp order through shared memory (deterministic)
template <int NB, int WPR>
__device__ __forceinline__ void row_dot(const GemmArgs &g, int row, bool live, const double *__restrict__ xc,
                                        double (*rp)[NB], double (&acc)[NB]) {
  const int warp = threadIdx.x >> 5, q = warp % WPR;
  const int Kq = ((g.K + WPR * 64 - 1) / (WPR * 64)) * 64;
  const int k0 = q * Kq, k1 = min(g.K, k0 + Kq);
  double a[NB];
  if (live) warp_dot<NB>(g.A + (size_t)row * g.lda, xc, k0, k1, a);
  else
#pragma unroll
    for (int b = 0; b < NB; ++b) a[b] = 0.0;
  if (WPR > 1) {
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int b = 0; b < NB; ++b) rp[warp][b] = a[b];
    __syncthreads();
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      double t = rp[warp - q][b];
      for (int j = 1; j < WPR; ++j) t += rp[warp - q + j][b];
      acc[b] = t;
    }
  } else {
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[b] = a[b];
  }
}

template <int NB>
__global__ void __launch_bounds__(VT, skinny_minb(NB)) k_gen_row(const GemmArgs g, const double *__restrict__ nuc,
                                                double *__restrict__ pc) {
  __shared__ double red[2][VW * NB];
  __shared__ double rp[VW][NB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = blockIdx.x * (VW / WPR_G) + warp / WPR_G;
  const bool live = row < g.ng;
  double so[NB], sp[NB], acc[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) so[b] = sp[b] = 0.0;
  row_dot<NB, WPR_G>(g, row, live, nuc, rp, acc);  // (H_g^T nu)_g
  if (live && warp % WPR_G == 0) {
    const double c = g.gc[row], lo = g.glo[row], hi = g.ghi[row], a = g.ga ? g.ga[row] : 0.0;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const double q = (c + g.lam[b]) + acc[b];
      const double p = minimiser(q, lo, hi, a);
      if (lane == b) pc[(size_t)row * NB + b] = p;
      so[b] += a * p * p + q * p;
      sp[b] += p;
    }
  }
  block_part<NB>(red[0], so, g.part_obj);
  block_part<NB>(red[1], sp, g.part_p);
}

// the last block to finish (atomic ticket) sums every block's partials per
// instance in a fixed order and runs the per-instance finisher: no extra launch
template <int NB, bool STEP, bool FEVAL>
__global__ void __launch_bounds__(VT, skinny_minb(NB)) k_line_row(const GemmArgs g, const double *__restrict__ pcv,
                                                 double *__restrict__ nuc, const FinArgs f, unsigned *ticket) {
  __shared__ double red[VW * NB];
  __shared__ double fred[3][VT];
  __shared__ bool last;
  __shared__ double rp[VW][NB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double sv[NB], acc[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) sv[b] = 0.0;
  // grid-stride over row groups (the grid is capped at the resident blocks, so
  // the rows spread evenly over the SMs instead of a ragged second wave)
  constexpr int RPB = VW / WPR_L;
  const int iters = (g.nl + gridDim.x * RPB - 1) / (gridDim.x * RPB);
  for (int it = 0; it < iters; ++it) {
  const int row = (it * gridDim.x + blockIdx.x) * RPB + warp / WPR_L;
  const bool live = row < g.nl;
  row_dot<NB, WPR_L>(g, row, live, pcv, rp, acc);  // (H_g p*)_l
  if (live && warp % WPR_L == 0) {
    const double al = STEP ? g.alpha[g.k] : 0.0;
    const double F = g.F[row];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const size_t o = (size_t)row * g.ld + b;
      const double y = acc[b];
      const double r = g.r[o], mp = g.mup[o], mm = g.mum[o];
      sv[b] += mm * (r - F) - mp * (r + F);
      if (lane != b) continue;  // lane b owns instance b of this row
      const double gp = (y - r) - F, gm = (r - y) - F;
      if (!STEP) {
        if (g.gp_out) {
          g.gp_out[o] = gp;
          g.gm_out[o] = gm;
        }
      } else if (g.status[b] == 0) {
        double vp, vm;
        if (g.opt == 0) {
          vp = mp + al * gp;
          vm = mm + al * gm;
        } else {
          double a1 = g.s1p[o], a2 = g.s2p ? g.s2p[o] : 0.0, b1 = g.s1m[o], b2 = g.s2m ? g.s2m[o] : 0.0;
          opt_step2(g, mp, gp, mm, gm, al, a1, a2, b1, b2, vp, vm);
          g.s1p[o] = a1;
          g.s1m[o] = b1;
          if (g.s2p) {
            g.s2p[o] = a2;
            g.s2m[o] = b2;
          }
        }
        const double np = vp > 0.0 ? vp : 0.0, nm = vm > 0.0 ? vm : 0.0;  // mu <- max(mu, 0)
        g.mup[o] = np;
        g.mum[o] = nm;
        g.nu[o] = np - nm;
        nuc[(size_t)row * NB + b] = np - nm;
      }
    }
  }
  }  // rows
  block_part<NB>(red, sv, g.part_line);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (long n = f.n0; n < f.n1; ++n) {
    double so = 0.0, sp = 0.0, sl = 0.0;
    for (int t = threadIdx.x; t < f.nMt1; t += VT) {
      so += __ldcg(f.part_obj + (size_t)t * f.ld + n);
      sp += __ldcg(f.part_p + (size_t)t * f.ld + n);
    }
    for (int t = threadIdx.x; t < f.nMt2; t += VT) sl += __ldcg(f.part_line + (size_t)t * f.ld + n);
    fred[0][threadIdx.x] = so;
    fred[1][threadIdx.x] = sp;
    fred[2][threadIdx.x] = sl;
    __syncthreads();
    for (int w = VT / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w)
        for (int c = 0; c < 3; ++c) fred[c][threadIdx.x] += fred[c][threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) finish_one<FEVAL>(f, n, fred[0][0], fred[1][0], fred[2][0]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *ticket = 0u;  // ready for the next launch
}

// compact copy nu_c[l][b] = nu[l][b] (after set_batch / set_multipliers)
__global__ void k_compact_nu(const double *nu, long ld, int nl, int NB, double *nuc) {
  for (long x = (long)blockIdx.x * blockDim.x + threadIdx.x; x < (long)nl * NB; x += (long)gridDim.x * blockDim.x)
    nuc[x] = nu[(x / NB) * ld + x % NB];
}

// ---------------------------------------------------------------------------
// One instance (B = 1): the single-read step.  The two products of a step,
// y = H_g p*_k (line rows) and Q_{k+1} = H_g^T nu_{k+1} (generator columns),
// both read H_g; the skinny kernels above read it twice per step from HBM
// (H_g and H_g^T, 2 x 254 MB at config 3).  Here one pass over the rows of
// H_g does both.  Each CTA streams a contiguous block of rows, R rows (a
// group) at a time, into shared-memory stages with TMA bulk copies (issued by
// the last warp).  The 16 warps own column pairs j = tid + 512 m of every row:
// per group they load their columns of the R rows into registers, form the
// row dots with p*_k (registers) and pass the warp sums through shared memory;
// after one CTA barrier (which also frees the group's stage: S - 1 groups stay
// in flight) every warp adds the 16 warp sums in the same fixed order, takes
// the projected step of the R rows' mu (lane r: row r; bit-identical in every
// warp, warp 0 stores it) and adds H_g[l,:] nu_{k+1,l} into its column
// accumulators from the registers.  The CTAs' column partials are summed in
// CTA order by k_fused_gen, which applies the generator minimiser for k+1.
//   k_fused_line<0>: Q_0 = H_g^T nu (start of a call; no line work)
//   k_fused_line<1>: line step k (+ Q_{k+1} partials); its last CTA runs the
//                    finisher of step k (dual value g_k, the lambda step)
//   k_fused_line<2>: line terms of the final value at y_K (no step, no Q)
// The step sits on each group's path, so the variants whose per-row step is a
// long dependent chain (AdaGrad, Adam: divisions, square roots) keep the
// two-pass kernels (measured on config 3: Adam 105 us/it single-read against
// 99 us two-pass; the plain step 60.5 against 96).
constexpr int FT = 512, FW = FT / 32;  // threads (the last warp also issues the TMA copies)
constexpr int FMAX = 4;                // double2 columns per thread: n_g <= 2 * FT * FMAX
__host__ __device__ constexpr int fused_rows(int M) { return 6 / M; }  // rows per group: 6 double2 held per thread
constexpr int FSMAX = 8;               // stages
// shared memory: the stages (S - 1 groups, >= 120 KB, in flight per SM), the
// warp dots, and the CTA's rows' data (nu, r, F, mu+-, optimiser state: 9 x rpc)
constexpr long kFusedSmemBytes = 220 * 1024;
inline size_t fused_smem(long ldh, int R, int S, int rpc) {
  return (size_t)S * R * ldh * 8 + FSMAX * 8 + 2 * 6 * FW * 8 + FW * 8 + 9 * (size_t)rpc * 8;
}

struct FusedArgs {
  const double *Hg;
  long ldh;           // = ngk (row stride of H_g, doubles; rows 128-byte aligned)
  int S;              // shared-memory stages (groups)
  int rpc;            // >= rows per CTA
  int ng;             // generators (columns of H_g in use)
  const double *pcv;  // p*_k [ngk] (generator order; entries >= n_g unused)
  double *nuc;        // compact nu copy (kept current for the skinny evaluate())
  double *part_q;     // [CTA][ngk] column partials of Q_{k+1}
  double *part_line;  // [CTA] line value terms
  double *part_obj, *part_p;  // [k_fused_gen block]: sum_g (a p^2 + q p), sum_g p at the current point
  int ngb;            // k_fused_gen blocks
  unsigned *ticket;   // k_fused_line's last-CTA ticket (zero between launches)
};

__device__ __forceinline__ unsigned f_smem(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void f_bar_wait(uint64_t *bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(f_smem(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

// M: double2 columns per thread (column pair j = tid + FT m, m < M)
template <int MODE, int M>
__global__ void __launch_bounds__(FT, 1) k_fused_line(const FusedArgs a, const GemmArgs g, const FinArgs f) {
  constexpr int R = fused_rows(M);
  extern __shared__ __align__(128) unsigned char fsm[];
  const int S = a.S, rpc = a.rpc;
  const long ldh = a.ldh;
  double *stage = reinterpret_cast<double *>(fsm);  // [S][R][ldh]
  uint64_t *full = reinterpret_cast<uint64_t *>(stage + (size_t)S * R * ldh);  // [FSMAX]
  double *part = reinterpret_cast<double *>(full + FSMAX);  // [2][R][FW] warp dots, by group parity
  double *svw = part + 2 * 6 * FW;                          // [FW]
  double *rowv = svw + FW;  // [9][rpc]: nu, r, F, mu+, mu-, s1+, s2+, s1-, s2- of the CTA's rows
  __shared__ bool last;
  __shared__ double red[FT];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x, c = blockIdx.x;
  const int r0 = (int)((long)g.nl * c / G), r1 = (int)((long)g.nl * (c + 1) / G);
  const int nrow = r1 - r0, ngr = (nrow + R - 1) / R;
  const int h2 = (int)(ldh / 2);
  if (tid == 0) {
    for (int s = 0; s < S; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(f_smem(&full[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const bool optst = MODE == 1 && g.opt != 0, st2 = g.s2p != nullptr;
  for (int t = tid; t < nrow; t += FT) {  // the rows' data, once (off the per-group path)
    const int row = r0 + t;
    const size_t o = (size_t)row * g.ld;
    rowv[t] = g.nu[o];
    if (MODE != 0) {
      rowv[rpc + t] = g.r[o];
      rowv[2 * rpc + t] = g.F[row];
      rowv[3 * rpc + t] = g.mup[o];
      rowv[4 * rpc + t] = g.mum[o];
      if (optst) {
        rowv[5 * rpc + t] = g.s1p[o];
        rowv[7 * rpc + t] = g.s1m[o];
        if (st2) {
          rowv[6 * rpc + t] = g.s2p[o];
          rowv[8 * rpc + t] = g.s2m[o];
        }
      }
    }
  }
  __syncthreads();
  // the last warp issues the TMA copies: one bulk copy per row, lane r copies row r
  const bool producer = warp == FW - 1;
  const unsigned rowb = (unsigned)(ldh * 8);
  auto issue = [&](int gi) {
    const int st = gi % S, t0 = gi * R, nr = min(R, nrow - t0);
    const unsigned bar = f_smem(&full[st]);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(nr * rowb)
                   : "memory");
    __syncwarp();
    if (lane < nr)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              f_smem(stage + ((size_t)st * R + lane) * ldh)),
          "l"(a.Hg + (size_t)(r0 + t0 + lane) * ldh), "r"(rowb), "r"(bar)
          : "memory");
  };
  if (producer)
    for (int gi = 0; gi < min(S, ngr); ++gi) issue(gi);
  // programmatic dependent launch: everything above (barriers, the rows' data
  // written by the previous line kernel, the first H_g copies) overlaps the
  // tail of the preceding generator pass; p*_k is read after it completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  double2 pv[M], qv[M];
  const bool tail = tid + FT * (M - 1) >= h2;  // this thread's last column pair is past the row
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int j = tid + FT * m;
    double2 p = make_double2(0.0, 0.0);
    if (MODE != 0 && j < h2) {
      if (2 * j < a.ng) p.x = a.pcv[2 * j];
      if (2 * j + 1 < a.ng) p.y = a.pcv[2 * j + 1];
    }
    pv[m] = p;
    qv[m] = make_double2(0.0, 0.0);
  }
  const bool step = MODE == 1 && g.status[0] == 0;
  const double al = MODE == 1 ? g.alpha[g.k] : 0.0;
  double sv = 0.0;  // warp 0: its lanes' rows' value terms
  int s = 0;
  unsigned ph = 0;
  for (int i = 0; i < ngr; ++i) {
    const int t0 = i * R, nr = min(R, nrow - t0);
    f_bar_wait(&full[s], ph);
    const double2 *H = reinterpret_cast<const double2 *>(stage + (size_t)s * R * ldh) + tid;
    double2 h[R][M];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int m = 0; m < M; ++m)
        h[r][m] = (r < nr && (m < M - 1 || !tail)) ? H[(size_t)r * h2 + FT * m] : make_double2(0.0, 0.0);
    double *pp = part + (i & 1) * 6 * FW + warp;
    if (MODE != 0) {  // row dots: each thread's columns, then the warp's xor tree
      double d[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        d[r] = 0.0;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          d[r] = fma(h[r][m].x, pv[m].x, d[r]);
          d[r] = fma(h[r][m].y, pv[m].y, d[r]);
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int r = 0; r < R; ++r) d[r] += __shfl_xor_sync(0xffffffffu, d[r], off);
      if (lane == 0)
#pragma unroll
        for (int r = 0; r < R; ++r) pp[r * FW] = d[r];
    }
    __syncthreads();  // the group's warp dots are in; every warp holds the group: its stage is free
    if (producer && i + S < ngr) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + S);
    }
    if (++s == S) {
      s = 0;
      ph ^= 1u;
    }
    // lane r: row t0 + r's step -- the same arithmetic on the same values in
    // every warp, so every warp holds the same nu_{k+1}; warp 0 stores it
    const bool live = lane < nr;
    const int t = t0 + (live ? lane : 0), crow = r0 + t;
    double nn = rowv[t];
    if (MODE != 0 && live) {
      const double rr = rowv[rpc + t], F = rowv[2 * rpc + t], mp = rowv[3 * rpc + t], mm = rowv[4 * rpc + t];
      const double *pr = part + (i & 1) * 6 * FW + lane * FW;
      // (H_g p*)_l: the 16 warp dots in a fixed order (four interleaved chains)
      double y0 = pr[0], y1 = pr[1], y2 = pr[2], y3 = pr[3];
#pragma unroll
      for (int w = 4; w < FW; w += 4) {
        y0 += pr[w];
        y1 += pr[w + 1];
        y2 += pr[w + 2];
        y3 += pr[w + 3];
      }
      const double y = (y0 + y1) + (y2 + y3);
      if (warp == 0) sv += mm * (rr - F) - mp * (rr + F);
      if (step) {
        const double gp = (y - rr) - F, gm = (rr - y) - F;
        double vp, vm, a1 = 0.0, a2 = 0.0, b1 = 0.0, b2 = 0.0;
        if (g.opt == 0) {
          vp = mp + al * gp;
          vm = mm + al * gm;
        } else {
          a1 = rowv[5 * rpc + t];
          b1 = rowv[7 * rpc + t];
          if (st2) {
            a2 = rowv[6 * rpc + t];
            b2 = rowv[8 * rpc + t];
          }
          opt_step2(g, mp, gp, mm, gm, al, a1, a2, b1, b2, vp, vm);
        }
        const double np = vp > 0.0 ? vp : 0.0, nm = vm > 0.0 ? vm : 0.0;  // mu <- max(mu, 0)
        nn = np - nm;
        if (warp == 0) {
          const size_t o = (size_t)crow * g.ld;
          if (g.opt != 0) {
            g.s1p[o] = a1;
            g.s1m[o] = b1;
            if (st2) {
              g.s2p[o] = a2;
              g.s2m[o] = b2;
            }
          }
          g.mup[o] = np;
          g.mum[o] = nm;
          g.nu[o] = nn;
          a.nuc[crow] = nn;
        }
      }
    }
    if (MODE != 2) {  // Q += H_g[l, :]^T nu_{k+1,l} over the group's rows
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double v = __shfl_sync(0xffffffffu, nn, r);
        if (r < nr)
#pragma unroll
          for (int m = 0; m < M; ++m) {
            qv[m].x = fma(h[r][m].x, v, qv[m].x);
            qv[m].y = fma(h[r][m].y, v, qv[m].y);
          }
      }
    }
  }
  if (MODE != 2) {
    double2 *q = reinterpret_cast<double2 *>(a.part_q + (size_t)c * ldh) + tid;
#pragma unroll
    for (int m = 0; m < M; ++m)
      if (m < M - 1 || !tail) q[FT * m] = qv[m];
  }
  if (MODE == 0) return;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, off);
  if (lane == 0) svw[warp] = sv;
  __syncthreads();
  if (tid == 0) {
    double t = svw[0];
    for (int w = 1; w < FW; ++w) t += svw[w];
    a.part_line[c] = t;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(&a.ticket[0], 1u) == (unsigned)G - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // the last CTA: the CTAs' line terms and the generator pass's block terms,
  // each summed by a fixed tree (loads in parallel)
  double *ro = stage, *rp = stage + FT / 4;  // (the stages are free now: >= 288 doubles)
  red[tid] = tid < G ? __ldcg(a.part_line + tid) : 0.0;
  for (int b = tid + FT; b < G; b += FT) red[tid] += __ldcg(a.part_line + b);
  if (tid < FT / 4) {
    double to = 0.0, tp = 0.0;
    for (int b = tid; b < a.ngb; b += FT / 4) {
      to += __ldcg(a.part_obj + b);
      tp += __ldcg(a.part_p + b);
    }
    ro[tid] = to;
    rp[tid] = tp;
  }
  __syncthreads();
  for (int w = FT / 2; w > 0; w >>= 1) {
    if (tid < w) {
      red[tid] += red[tid + w];
      if (w < FT / 4) {
        ro[tid] += ro[tid + w];
        rp[tid] += rp[tid + w];
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    finish_one<false>(f, 0, ro[0], rp[0], red[0]);
    a.ticket[0] = 0u;
  }
}

// Q_{k+1} = sum over CTAs (in order) of the column partials, then p*_{k+1} and
// the generator value terms; 32 columns per block, the CTA range split over
// 8 warps (combined in warp order); the last block sums the block terms
constexpr int FGW = 16;
__global__ void __launch_bounds__(FGW * 32) k_fused_gen(const FusedArgs a, const GemmArgs g, int G) {
  __shared__ double red[FGW][32];
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the line kernel's partials are complete
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the next line kernel may start its prologue
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col = blockIdx.x * 32 + lane;
  double q = 0.0;
  if (col < g.ng) {  // CTAs [b0, b1) in order, all loads in flight ahead of the adds
    const double *pq = a.part_q + col;
    const int b0 = G * warp / FGW, nb = G * (warp + 1) / FGW - b0;
    constexpr int U = 12;  // >= ceil(CTAs / FGW) for up to 192 CTAs
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = u < nb ? __ldcg(pq + (size_t)(b0 + u) * a.ldh) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (u < nb) q += v[u];
    for (int b = b0 + U; b < b0 + nb; ++b) q += __ldcg(pq + (size_t)b * a.ldh);  // (> 192 CTAs)
  }
  red[warp][lane] = q;
  __syncthreads();
  if (warp == 0) {
    double Q = red[0][lane];
    for (int w = 1; w < FGW; ++w) Q += red[w][lane];
    double so = 0.0, sp = 0.0;
    if (col < g.ng) {
      const double aq = g.ga ? g.ga[col] : 0.0;
      const double qq = (g.gc[col] + g.lam[0]) + Q;
      const double p = minimiser(qq, g.glo[col], g.ghi[col], aq);
      const_cast<double *>(a.pcv)[col] = p;
      so = aq * p * p + qq * p;
      sp = p;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      so += __shfl_xor_sync(0xffffffffu, so, off);
      sp += __shfl_xor_sync(0xffffffffu, sp, off);
    }
    if (lane == 0) {  // the block's generator terms (summed by the next line kernel's finisher)
      a.part_obj[blockIdx.x] = so;
      a.part_p[blockIdx.x] = sp;
    }
  }
}

// ---------------------------------------------------------------------------
// construction kernels (tree flows, cycle sums, H_a assembly, generator columns)
struct TreeDev {
  const int *tin, *tout;   // DFS entry / exit times per bus
  const int *child;        // per branch: the deeper endpoint of a tree branch, -1 otherwise
  const double *sig;       // per branch: +1 if the flow child -> parent runs from -> to, else -1
};

__device__ __forceinline__ double tflow(const TreeDev &T, const int *tin_bus, int l, int i) {
  const int c = T.child[l];
  if (c < 0) return 0.0;
  const int ti = tin_bus[i];
  return (T.tin[c] <= ti && ti < T.tout[c]) ? T.sig[l] : 0.0;
}

// S[k][i] = sum_{l in cycle k} C_kl x_l T[l][i]
__global__ void k_cycle_tree(TreeDev T, const int *cp, const int *cb, const double *cs, const double *x, int nc,
                             int nb, double *S, long lds) {
  for (long id = (long)blockIdx.x * blockDim.x + threadIdx.x; id < (long)nc * nb; id += (long)gridDim.x * blockDim.x) {
    const int k = (int)(id / nb), i = (int)(id % nb);
    double s = 0.0;
    for (int e = cp[k]; e < cp[k + 1]; ++e) {
      const int l = cb[e];
      s += cs[e] * x[l] * tflow(T, T.tin, l, i);
    }
    S[(size_t)k * lds + i] = s;
  }
}

// H_a[l][i] = T[l][i] - sum_{k containing l} C_kl W[k][i]  (0 for an open branch, b = 0).
// PTDF entries are flow fractions, |H| <= 1; an entry below 1e-12 is a
// rounding residue of a structural zero (no path from bus i to the slack runs
// through l, e.g. a line into a part of the network with no injection) and is
// stored as the exact 0 it is (reading A-30)
__global__ void k_assemble(TreeDev T, const int *bp, const int *bk, const double *bs, const double *W, long ldw,
                           const double *b, int nl, int nb, double *Ha, long ldh) {
  for (long id = (long)blockIdx.x * blockDim.x + threadIdx.x; id < (long)nl * nb; id += (long)gridDim.x * blockDim.x) {
    const int l = (int)(id / nb), i = (int)(id % nb);
    double h = 0.0;
    if (b[l] > 0.0) {
      h = tflow(T, T.tin, l, i);
      for (int e = bp[l]; e < bp[l + 1]; ++e) h -= bs[e] * W[(size_t)bk[e] * ldw + i];
    }
    Ha[(size_t)l * ldh + i] = (fabs(h) < 1e-12) ? 0.0 : h;
  }
}

// HgT[g][l] = Hg[l][g] = H_a[l][bus(g)]
__global__ void k_gen_cols(const double *Ha, long ldh, const int *gbus, int ng, int nl, double *HgT, long ldt,
                           double *Hg, long ldg) {
  for (long id = (long)blockIdx.x * blockDim.x + threadIdx.x; id < (long)ng * nl; id += (long)gridDim.x * blockDim.x) {
    const int g = (int)(id / nl), l = (int)(id % nl);
    const double v = Ha[(size_t)l * ldh + gbus[g]];
    HgT[(size_t)g * ldt + l] = v;
    Hg[(size_t)l * ldg + g] = v;
  }
}

__global__ void k_colsum(const double *Dm, int nb, long ld, double *D) {
  const long n = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= ld) return;  // (launched with ld threads)
  double s = 0.0;
  for (int i = 0; i < nb; ++i) s += Dm[(size_t)i * ld + n];  // 1^T d, ascending bus
  D[n] = s;
}

__global__ void k_fill(double *p, double v, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_sub(const double *a, const double *b, double *c, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    c[i] = a[i] - b[i];
}

// set_multipliers validation: finite, and mu >= 0 where `nonneg`
__global__ void k_check(const double *p, size_t rows, long ld, long B, int nonneg, int *flag) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows * B; i += (size_t)gridDim.x * blockDim.x) {
    const double v = p[(i / B) * ld + i % B];
    if (!isfinite(v) || (nonneg && v < 0.0)) *flag = 1;
  }
}

int blocks_for(size_t n) { return (int)std::min<size_t>(std::max<size_t>((n + 255) / 256, 1), 148 * 64); }

}  // namespace

// ===========================================================================
struct PtdfState {
  int device = 0, nb = 0, nl = 0, ng = 0, nc = 0;
  long nlp = 0, nlk = 0, ngp = 0, ngk = 0, nbk = 0;  // padded sizes (M: 128, K: 16)
  int quadratic = 0;
  int group = 8;
  // network (device)
  double *Ha = nullptr, *HgT = nullptr, *Hg = nullptr, *F = nullptr, *gc = nullptr, *glo = nullptr, *ghi = nullptr,
         *ga = nullptr;
  // batch
  long B = 0, Bp = 0;
  double *r = nullptr, *D = nullptr, *lam = nullptr, *mup = nullptr, *mum = nullptr, *nu = nullptr, *P = nullptr;
  double *part_obj = nullptr, *part_p = nullptr, *part_line = nullptr;
  double *best = nullptr, *bound = nullptr, *value = nullptr, *gprev = nullptr, *target = nullptr;
  double *gp = nullptr, *gm = nullptr, *glam = nullptr;
  int *status = nullptr, *flag = nullptr;
  long long *hit = nullptr;
  bool has_target = false;
  long long k_base = 0;
  double tol = 0.0;
  dcopf_optimizer opt = {DCOPF_OPT_PLAIN, 0, 0.0, 0.0, 0.0, 0.0};
  double b1t = 1.0, b2t = 1.0;
  double *os[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // s1p s2p s1m s2m sl1 sl2
  double *scratch = nullptr;
  size_t scratch_bytes = 0;
  // iterate(): the batch's column blocks in `nsplit` groups on their own streams,
  // so one group's GEMM tail overlaps the other's (instances are independent)
  int nsplit = 2;
  // skinny batches (B <= 4): matrix-vector kernels; nbv = instance columns computed (0: GEMM mode)
  int nbv = 0;
  double *nuc = nullptr, *pcv = nullptr, *sp_obj = nullptr, *sp_p = nullptr, *sp_line = nullptr;
  unsigned *ticket = nullptr;  // [2] last-block tickets of the skinny / single-read kernels (zero between launches)
  // B = 1: the single-read step (k_fused_line / k_fused_gen); fG CTAs, fS stages, fR rows per
  // group, frpc >= rows per CTA
  bool fused = false;
  int nsm = 148, fG = 0, fS = 0, fR = 0, fgb = 0, frpc = 0;
  double *fq = nullptr, *fline = nullptr, *fobj = nullptr, *fp = nullptr;
  // medium batches: split-K scratch of GEMM1 ([S][n_g pad][B_pad]), CTA slots of the GPU
  double *qsplit = nullptr;
  size_t qsplit_n = 0;
  int n_slots = 296;
  cudaStream_t sub[2] = {nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr};
};

namespace {

#define PCK(call)                                                                                           \
  do {                                                                                                      \
    cudaError_t e_ = (call);                                                                                \
    if (e_ != cudaSuccess) {                                                                                \
      *err = std::string(#call) + " failed: " + cudaGetErrorString(e_);                                     \
      return e_ == cudaErrorMemoryAllocation ? DCOPF_ENOMEM : DCOPF_ECUDA;                                  \
    }                                                                                                       \
  } while (0)

int dalloc(double **p, size_t n, std::string *err) {
  cudaFree(*p);
  *p = nullptr;
  PCK(cudaMalloc(p, std::max<size_t>(n, 1) * 8));
  PCK(cudaMemset(*p, 0, std::max<size_t>(n, 1) * 8));
  return DCOPF_OK;
}

bool is_dev(const void *p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

template <int EPI>
int launch_gemm(const GemmArgs &g, cudaStream_t s, std::string *err) {
  if (g.M == 0 || g.N == 0) return DCOPF_OK;
  const int tiles = (g.M / BM) * (g.N / BN);
  const int splits = (EPI == EPI_STORE && g.ktps) ? (g.K / BK + g.ktps - 1) / g.ktps : 1;
  k_dgemm<EPI><<<dim3(tiles, splits), NTHR, GEMM_SMEM, s>>>(g);
  PCK(cudaGetLastError());
  return DCOPF_OK;
}

int set_gemm_attrs(std::string *err) {
  PCK(cudaFuncSetAttribute(k_dgemm<EPI_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM));
  PCK(cudaFuncSetAttribute(k_dgemm<EPI_GEN>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM));
  PCK(cudaFuncSetAttribute(k_dgemm<EPI_LINE_STEP>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM));
  PCK(cudaFuncSetAttribute(k_dgemm<EPI_LINE_EVAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM));
  return DCOPF_OK;
}

GemmArgs plain_gemm(const double *A, long lda, const double *Bm, long ldb, double *C, long ldc, long M, long N,
                    long K, int group) {
  GemmArgs g;
  memset(&g, 0, sizeof g);
  g.A = A;
  g.lda = lda;
  g.Bm = Bm;
  g.ldb = ldb;
  g.C = C;
  g.ld = ldc;
  g.M = (int)M;
  g.N = (int)N;
  g.K = (int)K;
  g.group = group;
  return g;
}

// Host: Cholesky M = L L^T (row-major lower) and X = L^{-1}; returns false if not SPD.
bool chol_inverse(std::vector<double> &M, int n, std::vector<double> *Linv) {
  for (int j = 0; j < n; ++j) {
    double *Lj = &M[(size_t)j * n];
    for (int i = j; i < n; ++i) {
      double *Li = &M[(size_t)i * n];
      double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
      int k = 0;
      for (; k + 4 <= j; k += 4) {
        s0 += Li[k] * Lj[k];
        s1 += Li[k + 1] * Lj[k + 1];
        s2 += Li[k + 2] * Lj[k + 2];
        s3 += Li[k + 3] * Lj[k + 3];
      }
      for (; k < j; ++k) s0 += Li[k] * Lj[k];
      const double v = Li[j] - ((s0 + s1) + (s2 + s3));
      if (i == j) {
        if (!(v > 0.0)) return false;
        Lj[j] = std::sqrt(v);
      } else {
        Li[j] = v / Lj[j];
      }
    }
  }
  // L^{-1}: column j solves L x = e_j; columns are independent (threads)
  Linv->assign((size_t)n * n, 0.0);
  std::vector<double> &X = *Linv;
  const int nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  auto work = [&](int t0) {
    std::vector<double> x(n);
    for (int j = t0; j < n; j += nt) {
      x[j] = 1.0 / M[(size_t)j * n + j];
      for (int i = j + 1; i < n; ++i) {
        const double *Li = &M[(size_t)i * n];
        double s = 0.0;
        for (int k = j; k < i; ++k) s += Li[k] * x[k];
        x[i] = -s / Li[i];
      }
      for (int i = j; i < n; ++i) X[(size_t)i * n + j] = x[i];
    }
  };
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) th.emplace_back(work, t);
  for (auto &t : th) t.join();
  return true;
}

int ensure_scratch(PtdfState *st, size_t bytes, std::string *err) {
  if (st->scratch_bytes >= bytes) return DCOPF_OK;
  cudaFree(st->scratch);
  st->scratch = nullptr;
  st->scratch_bytes = 0;
  PCK(cudaMalloc(&st->scratch, bytes));
  st->scratch_bytes = bytes;
  return DCOPF_OK;
}

void free_batch(PtdfState *st) {
  double **dp[] = {&st->r,     &st->D,      &st->lam,    &st->mup,   &st->mum,   &st->nu,     &st->P,
                   &st->part_obj, &st->part_p, &st->part_line, &st->best, &st->bound, &st->value, &st->gprev,
                   &st->target, &st->gp,    &st->gm,     &st->glam,  &st->os[0], &st->os[1], &st->os[2],
                   &st->os[3],  &st->os[4], &st->os[5]};
  for (double **p : dp) {
    cudaFree(*p);
    *p = nullptr;
  }
  cudaFree(st->status);
  cudaFree(st->hit);
  st->status = nullptr;
  st->hit = nullptr;
  st->B = st->Bp = 0;
}

int nstate(const dcopf_optimizer &o) {
  return o.variant == DCOPF_OPT_ADAM ? 2 : (o.variant == DCOPF_OPT_PLAIN ? 0 : 1);
}

int reset_opt(PtdfState *st, std::string *err) {
  for (double *&p : st->os) {
    cudaFree(p);
    p = nullptr;
  }
  st->b1t = st->b2t = 1.0;
  const int ns = nstate(st->opt);
  if (st->Bp == 0 || ns == 0) return DCOPF_OK;
  const size_t nm = (size_t)st->nlp * st->Bp;
  int rc = dalloc(&st->os[0], nm, err);
  if (!rc) rc = dalloc(&st->os[2], nm, err);
  if (!rc) rc = dalloc(&st->os[4], st->Bp, err);
  if (!rc && ns == 2) rc = dalloc(&st->os[1], nm, err);
  if (!rc && ns == 2) rc = dalloc(&st->os[3], nm, err);
  if (!rc && ns == 2) rc = dalloc(&st->os[5], st->Bp, err);
  return rc;
}

GemmArgs gen_args(PtdfState *st) {
  GemmArgs g = plain_gemm(st->HgT, st->nlk, st->nu, st->Bp, nullptr, st->Bp, st->ngp, st->Bp, st->nlk, st->group);
  g.gc = st->gc;
  g.glo = st->glo;
  g.ghi = st->ghi;
  g.ga = st->quadratic ? st->ga : nullptr;
  g.ng = st->ng;
  g.lam = st->lam;
  g.P = st->P;
  g.part_obj = st->part_obj;
  g.part_p = st->part_p;
  return g;
}

GemmArgs line_args(PtdfState *st) {
  GemmArgs g = plain_gemm(st->Hg, st->ngk, st->P, st->Bp, nullptr, st->Bp, st->nlp, st->Bp, st->ngk, st->group);
  g.r = st->r;
  g.F = st->F;
  g.nl = st->nl;
  g.mup = st->mup;
  g.mum = st->mum;
  g.nu = st->nu;
  g.part_line = st->part_line;
  g.status = st->status;
  g.opt = st->opt.variant;
  g.rho = st->opt.momentum;
  g.beta1 = st->opt.beta1;
  g.beta2 = st->opt.beta2;
  g.eps = st->opt.epsilon;
  g.s1p = st->os[0];
  g.s2p = st->os[1];
  g.s1m = st->os[2];
  g.s2m = st->os[3];
  return g;
}

FinArgs fin_args(PtdfState *st) {
  FinArgs f;
  memset(&f, 0, sizeof f);
  f.part_obj = st->part_obj;
  f.part_p = st->part_p;
  f.part_line = st->part_line;
  f.nMt1 = (int)(st->ngp / BM);
  f.nMt2 = (int)(st->nlp / BM);
  f.ld = st->Bp;
  f.B = st->B;
  f.n0 = 0;
  f.n1 = st->Bp;
  f.D = st->D;
  f.lam = st->lam;
  f.sl1 = st->os[4];
  f.sl2 = st->os[5];
  f.status = st->status;
  f.best = st->best;
  f.bound = st->bound;
  f.value = st->value;
  f.gprev = st->gprev;
  f.opt = st->opt.variant;
  f.rho = st->opt.momentum;
  f.beta1 = st->opt.beta1;
  f.beta2 = st->opt.beta2;
  f.eps = st->opt.epsilon;
  f.tol = st->tol;
  return f;
}

// rows x B (ld Bp, device) <-> rows x B (ld B, host or device)
int copy_rows_out(PtdfState *st, double *dst, const double *src, long rows, cudaStream_t s, std::string *err) {
  if (!dst || rows == 0) return DCOPF_OK;
  PCK(cudaMemcpy2DAsync(dst, st->B * 8, src, st->Bp * 8, st->B * 8, rows, cudaMemcpyDefault, s));
  if (!is_dev(dst)) PCK(cudaStreamSynchronize(s));
  return DCOPF_OK;
}

int skinny_blocks_g(int rows) { return std::max(1, (rows + VW / WPR_G - 1) / (VW / WPR_G)); }
int skinny_blocks_l(int rows) {  // capped at the blocks resident on 148 SMs (the kernel strides over rows)
  return std::max(1, std::min((rows + VW / WPR_L - 1) / (VW / WPR_L), PTDF_LINE_CAP));
}

template <int NB>
int skinny_pass_t(PtdfState *st, const GemmArgs &g1, const GemmArgs &g2, bool step, const FinArgs &f, bool feval,
                  cudaStream_t s, std::string *err) {
  GemmArgs a = g1, b = g2;
  a.A = st->HgT;  // row g of H_g^T, K = n_l
  a.lda = st->nlk;
  a.K = st->nl;
  a.part_obj = st->sp_obj;
  a.part_p = st->sp_p;
  b.A = st->Hg;   // row l of H_g, K = n_g
  b.lda = st->ngk;
  b.K = st->ng;
  b.part_line = st->sp_line;
  if (st->ng > 0) k_gen_row<NB><<<skinny_blocks_g(st->ng), VT, 0, s>>>(a, st->nuc, st->pcv);
  const int lb = skinny_blocks_l(st->nl);
  if (st->nl > 0) {  // the line kernel's last block runs the finisher
    if (step)
      k_line_row<NB, true, false><<<lb, VT, 0, s>>>(b, st->pcv, st->nuc, f, st->ticket);
    else if (!feval)
      k_line_row<NB, false, false><<<lb, VT, 0, s>>>(b, st->pcv, st->nuc, f, st->ticket);
    else
      k_line_row<NB, false, true><<<lb, VT, 0, s>>>(b, st->pcv, st->nuc, f, st->ticket);
  } else if (feval) {
    k_finish_blk<true><<<(int)st->B, 256, 0, s>>>(f);
  } else {
    k_finish_blk<false><<<(int)st->B, 256, 0, s>>>(f);
  }
  PCK(cudaGetLastError());
  return DCOPF_OK;
}

int skinny_pass(PtdfState *st, const GemmArgs &g1, const GemmArgs &g2, bool step, const FinArgs &f, bool feval,
                cudaStream_t s, std::string *err) {
  switch (st->nbv) {
    case 1: return skinny_pass_t<1>(st, g1, g2, step, f, feval, s, err);
    case 2: return skinny_pass_t<2>(st, g1, g2, step, f, feval, s, err);
    case 4: return skinny_pass_t<4>(st, g1, g2, step, f, feval, s, err);
    case 8: return skinny_pass_t<8>(st, g1, g2, step, f, feval, s, err);
    default: return skinny_pass_t<16>(st, g1, g2, step, f, feval, s, err);
  }
}

// skinny mode: the finisher reads the per-block partials [block][NB]
void fin_tiles(const PtdfState *st, FinArgs *f) {
  if (st->nbv) {
    f->part_obj = st->sp_obj;
    f->part_p = st->sp_p;
    f->part_line = st->sp_line;
    f->nMt1 = st->ng > 0 ? skinny_blocks_g(st->ng) : 0;
    f->nMt2 = st->nl > 0 ? skinny_blocks_l(st->nl) : 0;
    f->ld = st->nbv;
    f->n0 = 0;
    f->n1 = st->B;
  }
}

// GEMM1 of one launch: fused epilogue, or -- when its tiles cannot fill the
// GPU (medium batches) -- split over K into scratch + k_gen_reduce
// (ncon: launches of this shape running concurrently, one per column group)
int launch_gen(PtdfState *st, const GemmArgs &g1, cudaStream_t s, std::string *err, int ncon = 1) {
  if (g1.M == 0 || g1.N == 0) return DCOPF_OK;
  const int tiles = (g1.M / BM) * (g1.N / BN), ktiles = g1.K / BK;
  int S = 1;
  const char *ev = getenv("DCOPF_PTDF_SPLITK");  // measurement: 0 disables
  // measured on config 3: B = 128 1.67 -> 0.91 ms/it, B = 512 +13%, B = 1024 (320 tiles) better unsplit
  if (tiles * ncon < st->n_slots && ktiles >= 32 && !(ev && atoi(ev) == 0))
    S = std::min((2 * st->n_slots + tiles * ncon - 1) / (tiles * ncon), ktiles / 16);
  if (S <= 1) return launch_gemm<EPI_GEN>(g1, s, err);
  GemmArgs gs = g1;
  gs.ktps = (ktiles + S - 1) / S;
  S = (ktiles + gs.ktps - 1) / gs.ktps;
  const long split = (long)st->ngp * st->Bp;
  // sized once for the most splits any launch of this batch can use, so the two
  // column groups of iterate() (two streams) never see it reallocated
  const size_t need = (size_t)std::max(1, ktiles / 16) * split;
  if (st->qsplit_n < need) {
    cudaFree(st->qsplit);
    st->qsplit = nullptr;
    st->qsplit_n = 0;
    PCK(cudaMalloc(&st->qsplit, need * 8));
    st->qsplit_n = need;
  }
  gs.C = st->qsplit;
  gs.c_split = split;
  int rc = launch_gemm<EPI_STORE>(gs, s, err);
  if (rc) return rc;
  k_gen_reduce<<<dim3(g1.M / BM, g1.N / BN), BN, 0, s>>>(g1, st->qsplit, S, split);
  PCK(cudaGetLastError());
  return DCOPF_OK;
}

int skinny_sync_nu(PtdfState *st, cudaStream_t s, std::string *err) {
  if (!st->nbv || st->nl == 0) return DCOPF_OK;
  k_compact_nu<<<blocks_for((size_t)st->nl * st->nbv), 256, 0, s>>>(st->nu, st->Bp, st->nl, st->nbv, st->nuc);
  PCK(cudaGetLastError());
  return DCOPF_OK;
}

}  // namespace

// ===========================================================================
int ptdf_create(const PtdfNetIn &net, int device, PtdfState **out, std::string *err) {
  *out = nullptr;
  CycleBasis cb;
  std::string e = build_cycle_basis(net.nb, net.nl, net.ref, net.fr, net.to, net.b, nullptr, &cb);
  if (!e.empty()) {
    *err = e;
    return DCOPF_ETOPOLOGY;
  }
  PtdfState *st = new PtdfState();
  st->device = device;
  st->nb = net.nb;
  st->nl = net.nl;
  st->ng = net.ng;
  if (net.a)
    for (int g = 0; g < net.ng; ++g) st->quadratic |= net.a[g] > 0.0;
  if (const char *ev = getenv("DCOPF_PTDF_GROUP")) st->group = std::max(1, atoi(ev));
  if (const char *ev = getenv("DCOPF_PTDF_SPLIT")) st->nsplit = std::max(1, std::min(2, atoi(ev)));  // measurement
  st->nlp = up(net.nl, BM);
  st->nlk = up(net.nl, BK);
  st->ngp = up(net.ng, BM);
  st->ngk = up(net.ng, BK);
  st->nbk = up(net.nb, BK);
  auto fail = [&](int rc) {
    ptdf_destroy(st);
    return rc;
  };

  // ---- tree: parent / child per branch, DFS times ----
  const int nb = net.nb, nl = net.nl;
  std::vector<std::vector<int>> adj(nb);
  for (int l = 0; l < nl; ++l)
    if (cb.is_tree[l]) {
      adj[net.fr[l]].push_back(l);
      adj[net.to[l]].push_back(l);
    }
  std::vector<int> tin(nb, 0), tout(nb, 0), child(nl, -1);
  std::vector<double> sig(nl, 0.0);
  {
    std::vector<int> parent(nb, -1), it(nb, 0), stack{net.ref};
    std::vector<char> seen(nb, 0);
    seen[net.ref] = 1;
    int clock = 0;
    tin[net.ref] = clock++;
    while (!stack.empty()) {
      const int u = stack.back();
      if (it[u] < (int)adj[u].size()) {
        const int l = adj[u][it[u]++];
        const int v = net.fr[l] == u ? net.to[l] : net.fr[l];
        if (seen[v]) continue;
        seen[v] = 1;
        parent[v] = u;
        child[l] = v;
        sig[l] = (net.fr[l] == v) ? 1.0 : -1.0;  // flow v -> u (towards the slack) runs from -> to?
        tin[v] = clock++;
        stack.push_back(v);
      } else {
        tout[u] = clock;
        stack.pop_back();
      }
    }
  }
  // ---- cycles of the branches with b > 0 (the others carry no flow) ----
  std::vector<int> ccp{0}, ccb;
  std::vector<double> ccs;
  for (int k = 0; k < cb.nc; ++k) {
    if (!(net.b[cb.def[k]] > 0.0)) continue;
    for (int x = cb.cp[k]; x < cb.cp[k + 1]; ++x) {
      ccb.push_back(cb.cb[x]);
      ccs.push_back((double)cb.cs[x]);
    }
    ccp.push_back((int)ccb.size());
  }
  const int nc = (int)ccp.size() - 1;
  st->nc = nc;
  std::vector<double> x(nl, 0.0);
  for (int l = 0; l < nl; ++l) x[l] = net.b[l] > 0.0 ? 1.0 / net.b[l] : 0.0;
  // branch -> (cycle, sign) lists, ascending cycle
  std::vector<int> bp(nl + 1, 0), bk;
  std::vector<double> bsg;
  {
    std::vector<std::vector<std::pair<int, double>>> per(nl);
    for (int k = 0; k < nc; ++k)
      for (int q = ccp[k]; q < ccp[k + 1]; ++q) per[ccb[q]].push_back({k, ccs[q]});
    for (int l = 0; l < nl; ++l) {
      for (auto &pr : per[l]) {
        bk.push_back(pr.first);
        bsg.push_back(pr.second);
      }
      bp[l + 1] = (int)bk.size();
    }
  }
  // ---- M = C X C^T, Cholesky, L^{-1} (host) ----
  std::vector<double> Linv;
  if (nc > 0) {
    std::vector<double> M((size_t)nc * nc, 0.0);
    for (int l = 0; l < nl; ++l)
      for (int u = bp[l]; u < bp[l + 1]; ++u)
        for (int v = bp[l]; v < bp[l + 1]; ++v)
          M[(size_t)bk[u] * nc + bk[v]] += bsg[u] * bsg[v] * x[l];
    if (!chol_inverse(M, nc, &Linv)) {
      *err = "PTDF: the cycle matrix C X C^T is not positive definite";
      return fail(DCOPF_EINVAL);
    }
  }
  cudaError_t ce = cudaSetDevice(device);
  if (ce != cudaSuccess) {
    *err = std::string("cudaSetDevice: ") + cudaGetErrorString(ce);
    return fail(DCOPF_ECUDA);
  }
  if (int arc = set_gemm_attrs(err)) return fail(arc);
  {
    int nsm = 148;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device) == cudaSuccess)
      st->n_slots = CTAS_PER_SM * nsm;
    st->nsm = nsm;
  }
  // ---- device: S = C X T, W = L^{-T} (L^{-1} S), H_a = T - C^T W ----
  int *d_tin = nullptr, *d_tout = nullptr, *d_child = nullptr, *d_cp = nullptr, *d_cb = nullptr, *d_bp = nullptr,
      *d_bk = nullptr, *d_gbus = nullptr;
  double *d_sig = nullptr, *d_cs = nullptr, *d_x = nullptr, *d_bs = nullptr, *d_b = nullptr, *d_S = nullptr,
         *d_V = nullptr, *d_W = nullptr, *d_L = nullptr, *d_LT = nullptr;
  int rc = DCOPF_OK;
  auto upi = [&](int **d, const std::vector<int> &v) {
    if (rc) return;
    if (cudaMalloc(d, std::max<size_t>(v.size(), 1) * 4) != cudaSuccess ||
        (!v.empty() && cudaMemcpy(*d, v.data(), v.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)) {
      *err = "PTDF: device upload failed";
      rc = DCOPF_ENOMEM;
    }
  };
  auto upd = [&](double **d, const std::vector<double> &v) {
    if (rc) return;
    if (cudaMalloc(d, std::max<size_t>(v.size(), 1) * 8) != cudaSuccess ||
        (!v.empty() && cudaMemcpy(*d, v.data(), v.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess)) {
      *err = "PTDF: device upload failed";
      rc = DCOPF_ENOMEM;
    }
  };
  std::vector<int> gbus(net.gen_bus, net.gen_bus + net.ng);
  upi(&d_tin, tin);
  upi(&d_tout, tout);
  upi(&d_child, child);
  upi(&d_cp, ccp);
  upi(&d_cb, ccb);
  upi(&d_bp, bp);
  upi(&d_bk, bk);
  upi(&d_gbus, gbus);
  upd(&d_sig, sig);
  upd(&d_cs, ccs);
  upd(&d_x, x);
  upd(&d_bs, bsg);
  upd(&d_b, std::vector<double>(net.b, net.b + nl));
  const long ncp = up(std::max(nc, 1), BM), nck = up(std::max(nc, 1), BK), nbN = up(nb, BN);
  if (!rc) rc = dalloc(&st->Ha, (size_t)st->nlp * st->nbk, err);
  if (!rc) rc = dalloc(&d_W, (size_t)ncp * nbN, err);
  TreeDev T{d_tin, d_tout, d_child, d_sig};
  if (!rc && nc > 0) {
    rc = dalloc(&d_S, (size_t)ncp * nbN, err);
    if (!rc) rc = dalloc(&d_V, (size_t)ncp * nbN, err);
    std::vector<double> Lp((size_t)ncp * nck, 0.0), LTp((size_t)ncp * nck, 0.0);
    for (int i = 0; i < nc; ++i)
      for (int j = 0; j < nc; ++j) {
        Lp[(size_t)i * nck + j] = Linv[(size_t)i * nc + j];
        LTp[(size_t)i * nck + j] = Linv[(size_t)j * nc + i];
      }
    upd(&d_L, Lp);
    upd(&d_LT, LTp);
    if (!rc) {
      k_cycle_tree<<<blocks_for((size_t)nc * nb), 256>>>(T, d_cp, d_cb, d_cs, d_x, nc, nb, d_S, nbN);
      rc = launch_gemm<EPI_STORE>(plain_gemm(d_L, nck, d_S, nbN, d_V, nbN, ncp, nbN, nck, st->group), nullptr, err);
    }
    // the rows of V beyond nc are zero (zero rows of L^{-1}); K of the second product is nck
    if (!rc)
      rc = launch_gemm<EPI_STORE>(plain_gemm(d_LT, nck, d_V, nbN, d_W, nbN, ncp, nbN, nck, st->group), nullptr, err);
  }
  if (!rc) {
    k_assemble<<<blocks_for((size_t)nl * nb), 256>>>(T, d_bp, d_bk, d_bs, d_W, nbN, d_b, nl, nb, st->Ha, st->nbk);
    if (!rc) rc = dalloc(&st->HgT, (size_t)st->ngp * st->nlk, err);
    if (!rc) rc = dalloc(&st->Hg, (size_t)st->nlp * st->ngk, err);
    if (!rc)
      k_gen_cols<<<blocks_for((size_t)net.ng * nl), 256>>>(st->Ha, st->nbk, d_gbus, net.ng, nl, st->HgT, st->nlk,
                                                           st->Hg, st->ngk);
    ce = cudaDeviceSynchronize();
    if (!rc && ce != cudaSuccess) {
      *err = std::string("PTDF construction: ") + cudaGetErrorString(ce);
      rc = DCOPF_ECUDA;
    }
  }
  int *ip[] = {d_tin, d_tout, d_child, d_cp, d_cb, d_bp, d_bk, d_gbus};
  for (int *p : ip) cudaFree(p);
  double *dp[] = {d_sig, d_cs, d_x, d_bs, d_b, d_S, d_V, d_W, d_L, d_LT};
  for (double *p : dp) cudaFree(p);
  if (rc) return fail(rc);
  // ---- generators and limits ----
  auto padv = [&](const double *src, int n, long np) {
    std::vector<double> v(np, 0.0);
    if (src) std::copy(src, src + n, v.begin());
    return v;
  };
  upd(&st->F, padv(net.F, nl, st->nlp));
  upd(&st->gc, padv(net.c, net.ng, st->ngp));
  upd(&st->glo, padv(net.lo, net.ng, st->ngp));
  upd(&st->ghi, padv(net.hi, net.ng, st->ngp));
  upd(&st->ga, padv(net.a, net.ng, st->ngp));
  if (rc) return fail(rc);
  ce = cudaMalloc(&st->flag, sizeof(int));
  if (ce != cudaSuccess) {
    *err = "cudaMalloc failed";
    return fail(DCOPF_ENOMEM);
  }
  *out = st;
  return DCOPF_OK;
}

void ptdf_destroy(PtdfState *st) {
  if (!st) return;
  cudaSetDevice(st->device);
  free_batch(st);
  double *dp[] = {st->Ha, st->HgT, st->Hg, st->F, st->gc, st->glo, st->ghi, st->ga, st->scratch, st->nuc, st->pcv,
                  st->sp_obj, st->sp_p, st->sp_line, st->qsplit, st->fq, st->fline, st->fobj, st->fp};
  for (double *p : dp) cudaFree(p);
  for (int c = 0; c < 2; ++c) {
    if (st->sub[c]) cudaStreamDestroy(st->sub[c]);
    if (st->ev_join[c]) cudaEventDestroy(st->ev_join[c]);
  }
  if (st->ev_fork) cudaEventDestroy(st->ev_fork);
  cudaFree(st->flag);
  cudaFree(st->ticket);
  delete st;
}

int64_t ptdf_batch(const PtdfState *st) { return st->B; }

int ptdf_set_batch(PtdfState *st, int64_t B, const double *load, cudaStream_t s, std::string *err) {
  const long Bp = up(B, BN);
  const bool reuse = st->B > 0 && st->Bp == Bp;
  if (!reuse) {
    free_batch(st);
    const size_t nm = (size_t)st->nlp * Bp;
    int rc = DCOPF_OK;
    double **rows_l[] = {&st->r, &st->mup, &st->mum, &st->nu};
    for (double **p : rows_l)
      if (!rc) rc = dalloc(p, nm, err);
    if (!rc) rc = dalloc(&st->P, (size_t)st->ngp * Bp, err);
    if (!rc) rc = dalloc(&st->part_obj, (size_t)(st->ngp / BM) * Bp, err);
    if (!rc) rc = dalloc(&st->part_p, (size_t)(st->ngp / BM) * Bp, err);
    if (!rc) rc = dalloc(&st->part_line, (size_t)(st->nlp / BM) * Bp, err);
    double **vec[] = {&st->D, &st->lam, &st->best, &st->bound, &st->value, &st->gprev, &st->target, &st->glam};
    for (double **p : vec)
      if (!rc) rc = dalloc(p, Bp, err);
    if (rc) return rc;
    PCK(cudaMalloc(&st->status, Bp * 4));
    PCK(cudaMalloc(&st->hit, Bp * 8));
  }
  st->B = B;
  st->Bp = Bp;
  // skinny mode for B <= 4 (DCOPF_PTDF_SKINNY=0 forces the GEMMs; measurement).  Measured on
  // config 3 (us per step): skinny 100 / 157 / 379 at B = 1 / 2 / 4 (2369 at B = 8), the
  // split-K GEMMs a flat 934 for any B <= 128
  st->nbv = 0;
  const char *sk = getenv("DCOPF_PTDF_SKINNY");
  if (B <= 4 && !(sk && atoi(sk) == 0)) {
    st->nbv = B <= 1 ? 1 : (B <= 2 ? 2 : (B <= 4 ? 4 : (B <= 8 ? 8 : 16)));
    // compact vectors padded to the row padding (the double2 loads read one past an odd K)
    int rc0 = dalloc(&st->nuc, (size_t)st->nlk * 16 + 16, err);
    if (!rc0) rc0 = dalloc(&st->pcv, (size_t)st->ngk * 16 + 16, err);
    if (!rc0) rc0 = dalloc(&st->sp_obj, (size_t)skinny_blocks_g(st->ng) * 16, err);
    if (!rc0) rc0 = dalloc(&st->sp_p, (size_t)skinny_blocks_g(st->ng) * 16, err);
    if (!rc0) rc0 = dalloc(&st->sp_line, (size_t)skinny_blocks_l(st->nl) * 16, err);
    if (!rc0 && !st->ticket) {
      PCK(cudaMalloc(&st->ticket, 2 * sizeof(unsigned)));
      PCK(cudaMemset(st->ticket, 0, 2 * sizeof(unsigned)));
    }
    if (rc0) return rc0;
    // B = 1: the single-read step when a group of rows fits the shared-memory
    // stages (DCOPF_PTDF_FUSED=0 keeps the two-pass kernels; measurement)
    const char *fe = getenv("DCOPF_PTDF_FUSED");
    const long rowb = st->ngk * 8;
    st->fused = false;
    if (st->nbv == 1 && st->nl > 0 && st->ng > 0 && st->ngk <= 2L * FT * FMAX && !(fe && atoi(fe) == 0)) {
      const int M = (int)((st->ngk / 2 + FT - 1) / FT);
      st->fR = fused_rows(M);
      st->fG = std::min(st->nsm, st->nl);
      st->frpc = (st->nl + st->fG - 1) / st->fG + 1;
      const long fixed = (long)fused_smem(0, 0, 0, st->frpc);
      st->fS = (int)std::max<long>(0, std::min<long>(FSMAX, (kFusedSmemBytes - fixed) / (st->fR * rowb)));
      st->fgb = (st->ng + 31) / 32;
      if (st->fS >= 3) {  // >= 2 groups in flight ahead of the one being read
        st->fused = true;
        rc0 = dalloc(&st->fq, (size_t)st->fG * st->ngk, err);
        if (!rc0) rc0 = dalloc(&st->fline, st->fG, err);
        if (!rc0) rc0 = dalloc(&st->fobj, st->fgb, err);
        if (!rc0) rc0 = dalloc(&st->fp, st->fgb, err);
        if (rc0) return rc0;
      }
    }
  }
  // loads: [n_bus][B] -> Dm [nbk][Bp] (zero padded), r = H_a Dm, D = 1^T d
  const size_t dm = (size_t)st->nbk * Bp;
  int rc = ensure_scratch(st, dm * 8, err);
  if (rc) return rc;
  PCK(cudaMemsetAsync(st->scratch, 0, dm * 8, s));
  PCK(cudaMemcpy2DAsync(st->scratch, Bp * 8, load, B * 8, B * 8, st->nb, cudaMemcpyDefault, s));
  rc = launch_gemm<EPI_STORE>(plain_gemm(st->Ha, st->nbk, st->scratch, Bp, st->r, Bp, st->nlp, Bp, st->nbk, st->group),
                              s, err);
  if (rc) return rc;
  k_colsum<<<blocks_for(Bp), 256, 0, s>>>(st->scratch, st->nb, Bp, st->D);
  const size_t nm = (size_t)st->nlp * Bp;
  k_fill<<<blocks_for(nm), 256, 0, s>>>(st->mup, 0.0, nm);
  k_fill<<<blocks_for(nm), 256, 0, s>>>(st->mum, 0.0, nm);
  k_fill<<<blocks_for(nm), 256, 0, s>>>(st->nu, 0.0, nm);
  k_fill<<<blocks_for(Bp), 256, 0, s>>>(st->lam, 0.0, Bp);
  k_fill<<<blocks_for(Bp), 256, 0, s>>>(st->best, -std::numeric_limits<double>::infinity(), Bp);
  k_fill<<<blocks_for(Bp), 256, 0, s>>>(st->bound, std::numeric_limits<double>::quiet_NaN(), Bp);
  PCK(cudaMemsetAsync(st->status, 0, Bp * 4, s));
  PCK(cudaMemsetAsync(st->hit, 0xff, Bp * 8, s));
  PCK(cudaGetLastError());
  st->has_target = false;
  st->k_base = 0;
  PCK(cudaStreamSynchronize(s));  // the load scratch is reused by the next call
  return reset_opt(st, err);
}

template <int M>
int fused_loop(PtdfState *st, int64_t K, const FusedArgs &a, GemmArgs g, const GemmArgs &gg, FinArgs f,
               size_t smem, cudaStream_t s, std::string *err);

// B = 1: Q_0 pass + generator pass, then per step the single-read line pass
// (its last CTA runs the finisher) and the generator pass, then the final
// evaluation's line terms
int fused_iterate(PtdfState *st, int64_t K, GemmArgs g, FinArgs f, cudaStream_t s, std::string *err) {
  FusedArgs a;
  a.Hg = st->Hg;
  a.ldh = st->ngk;
  a.S = st->fS;
  a.rpc = st->frpc;
  a.ng = st->ng;
  a.pcv = st->pcv;
  a.nuc = st->nuc;
  a.part_q = st->fq;
  a.part_line = st->fline;
  a.part_obj = st->fobj;
  a.part_p = st->fp;
  a.ngb = st->fgb;
  a.ticket = st->ticket;
  GemmArgs gg = gen_args(st);
  const size_t smem = fused_smem(a.ldh, st->fR, a.S, a.rpc);
  const int M = (int)((a.ldh / 2 + FT - 1) / FT);
  switch (M) {
    case 1: return fused_loop<1>(st, K, a, g, gg, f, smem, s, err);
    case 2: return fused_loop<2>(st, K, a, g, gg, f, smem, s, err);
    case 3: return fused_loop<3>(st, K, a, g, gg, f, smem, s, err);
    default: return fused_loop<4>(st, K, a, g, gg, f, smem, s, err);
  }
}

template <int M>
int fused_loop(PtdfState *st, int64_t K, const FusedArgs &a, GemmArgs g, const GemmArgs &gg, FinArgs f,
               size_t smem, cudaStream_t s, std::string *err) {
  PCK(cudaFuncSetAttribute(k_fused_line<0, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  PCK(cudaFuncSetAttribute(k_fused_line<1, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  PCK(cudaFuncSetAttribute(k_fused_line<2, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int G = st->fG, T = FT;
  // both kernels launched with programmatic stream serialization (each waits
  // for its predecessor with griddepcontrol.wait where it reads its results)
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cl = {}, cg = {};
  cl.gridDim = dim3(G);
  cl.blockDim = dim3(T);
  cl.dynamicSmemBytes = smem;
  cl.stream = s;
  cl.attrs = at;
  cl.numAttrs = 1;
  cg = cl;
  cg.gridDim = dim3(st->fgb);
  cg.blockDim = dim3(FGW * 32);
  cg.dynamicSmemBytes = 0;
  PCK(cudaLaunchKernelEx(&cl, k_fused_line<0, M>, a, g, f));
  PCK(cudaLaunchKernelEx(&cg, k_fused_gen, a, gg, G));
  for (int64_t k = 0; k <= K; ++k) {
    const bool step = k < K;
    if (step && st->opt.variant == DCOPF_OPT_ADAM) {  // beta^t by repeated products (reading A-26)
      st->b1t = st->b1t * st->opt.beta1;
      st->b2t = st->b2t * st->opt.beta2;
    }
    g.k = f.k = (int)k;
    g.b1t = f.b1t = st->b1t;
    g.b2t = f.b2t = st->b2t;
    f.first = k == 0;
    if (step) {
      PCK(cudaLaunchKernelEx(&cl, k_fused_line<1, M>, a, g, f));
      PCK(cudaLaunchKernelEx(&cg, k_fused_gen, a, gg, G));
    } else {
      PCK(cudaLaunchKernelEx(&cl, k_fused_line<2, M>, a, g, f));
    }
  }
  st->k_base += K;
  return DCOPF_OK;
}

// the single-read step serves this batch and step variant
#ifndef DCOPF_PTDF_FUSED_ADAPTIVE
#define DCOPF_PTDF_FUSED_ADAPTIVE 1
#endif
static bool fused_for(const PtdfState *st) {
  return st->fused && (DCOPF_PTDF_FUSED_ADAPTIVE ||
                       (st->opt.variant != DCOPF_OPT_ADAGRAD && st->opt.variant != DCOPF_OPT_ADAM));
}

int ptdf_iterate(PtdfState *st, int64_t K, const double *alpha_dev, double *hist, cudaStream_t s, std::string *err) {
  GemmArgs g1 = gen_args(st), g2 = line_args(st);
  g2.alpha = alpha_dev;
  FinArgs f = fin_args(st);
  f.alpha = alpha_dev;
  f.hist = hist;
  f.K = (int)K;
  f.k_base = st->k_base;
  f.target = st->has_target ? st->target : nullptr;
  f.hit = st->hit;
  // B = 1: the single-read step (every variant since the adaptive steps run
  // on the branch-free division / square root, opt_step2; before that their
  // per-row chain kept AdaGrad / Adam on the two-pass kernels)
  if (fused_for(st)) return fused_iterate(st, K, g2, f, s, err);
  if (st->nbv) {  // skinny batch: matrix-vector passes on the caller's stream
    fin_tiles(st, &f);
    for (int64_t k = 0; k <= K; ++k) {
      const bool step = k < K;
      if (step && st->opt.variant == DCOPF_OPT_ADAM) {  // beta^t by repeated products (reading A-26)
        st->b1t = st->b1t * st->opt.beta1;
        st->b2t = st->b2t * st->opt.beta2;
      }
      g2.k = (int)k;
      g2.b1t = f.b1t = st->b1t;
      g2.b2t = f.b2t = st->b2t;
      f.k = (int)k;
      f.first = k == 0;
      int rc = skinny_pass(st, g1, g2, step, f, false, s, err);
      if (rc) return rc;
    }
    st->k_base += K;
    return DCOPF_OK;
  }
  // column groups: nsplit contiguous ranges of whole N tiles, one stream each
  const int ntiles = (int)(st->Bp / BN);
  const int ns = std::max(1, std::min(st->nsplit, ntiles));
  if (ns > 1 && !st->ev_fork) {
    for (int c = 0; c < 2; ++c) {
      PCK(cudaStreamCreateWithFlags(&st->sub[c], cudaStreamNonBlocking));
      PCK(cudaEventCreateWithFlags(&st->ev_join[c], cudaEventDisableTiming));
    }
    PCK(cudaEventCreateWithFlags(&st->ev_fork, cudaEventDisableTiming));
  }
  GemmArgs G1[2], G2[2];
  FinArgs Fc[2];
  cudaStream_t ss[2] = {s, s};
  for (int c = 0; c < ns; ++c) {
    const int t0 = ntiles * c / ns, t1 = ntiles * (c + 1) / ns;
    G1[c] = g1;
    G2[c] = g2;
    Fc[c] = f;
    G1[c].noff = G2[c].noff = t0 * BN;
    G1[c].N = G2[c].N = (t1 - t0) * BN;
    Fc[c].n0 = (long)t0 * BN;
    Fc[c].n1 = (long)t1 * BN;
    if (ns > 1) ss[c] = st->sub[c];
  }
  if (ns > 1) {
    PCK(cudaEventRecord(st->ev_fork, s));
    for (int c = 0; c < ns; ++c) PCK(cudaStreamWaitEvent(st->sub[c], st->ev_fork, 0));
  }
  for (int64_t k = 0; k <= K; ++k) {
    const bool step = k < K;
    if (step && st->opt.variant == DCOPF_OPT_ADAM) {  // beta^t by repeated products (reading A-26)
      st->b1t = st->b1t * st->opt.beta1;
      st->b2t = st->b2t * st->opt.beta2;
    }
    for (int c = 0; c < ns; ++c) {
      int rc = launch_gen(st, G1[c], ss[c], err, ns);
      if (rc) return rc;
      G2[c].k = (int)k;
      G2[c].b1t = Fc[c].b1t = st->b1t;
      G2[c].b2t = Fc[c].b2t = st->b2t;
      if (step) {
        rc = launch_gemm<EPI_LINE_STEP>(G2[c], ss[c], err);
      } else {  // the final evaluation at y_K: the value's line terms only, no step
        rc = launch_gemm<EPI_LINE_EVAL>(G2[c], ss[c], err);
      }
      if (rc) return rc;
      Fc[c].k = (int)k;
      Fc[c].first = k == 0;
      k_finish<false><<<blocks_for(Fc[c].n1 - Fc[c].n0), 256, 0, ss[c]>>>(Fc[c]);
      PCK(cudaGetLastError());
    }
  }
  if (ns > 1)
    for (int c = 0; c < ns; ++c) {
      PCK(cudaEventRecord(st->ev_join[c], st->sub[c]));
      PCK(cudaStreamWaitEvent(s, st->ev_join[c], 0));
    }
  st->k_base += K;
  return DCOPF_OK;
}

int ptdf_get_bound(PtdfState *st, double *bound, double *best, int32_t *status, cudaStream_t s, std::string *err) {
  const size_t n = st->B;
  if (bound) PCK(cudaMemcpyAsync(bound, st->bound, n * 8, cudaMemcpyDefault, s));
  if (best) PCK(cudaMemcpyAsync(best, st->best, n * 8, cudaMemcpyDefault, s));
  if (status) PCK(cudaMemcpyAsync(status, st->status, n * 4, cudaMemcpyDefault, s));
  if ((bound && !is_dev(bound)) || (best && !is_dev(best)) || (status && !is_dev(status)))
    PCK(cudaStreamSynchronize(s));
  return DCOPF_OK;
}

int ptdf_get_multipliers(PtdfState *st, double *lambda, double *branch, cudaStream_t s, std::string *err) {
  int rc = copy_rows_out(st, lambda, st->lam, 1, s, err);
  if (!rc) rc = copy_rows_out(st, branch, st->mup, st->nl, s, err);
  if (!rc && branch) rc = copy_rows_out(st, branch + (size_t)st->nl * st->B, st->mum, st->nl, s, err);
  return rc;
}

int ptdf_set_multipliers(PtdfState *st, const double *lambda, const double *branch, cudaStream_t s,
                         std::string *err) {
  const size_t nm = (size_t)st->nlp * st->Bp;
  // stage into scratch: [lambda Bp][mu+ nlp x Bp][mu- nlp x Bp], validate, then commit
  int rc = ensure_scratch(st, (2 * nm + st->Bp) * 8, err);
  if (rc) return rc;
  double *tl = st->scratch, *tp = tl + st->Bp, *tm = tp + nm;
  PCK(cudaMemsetAsync(st->scratch, 0, (2 * nm + st->Bp) * 8, s));
  if (lambda) PCK(cudaMemcpyAsync(tl, lambda, st->B * 8, cudaMemcpyDefault, s));
  if (branch && st->nl > 0) {
    PCK(cudaMemcpy2DAsync(tp, st->Bp * 8, branch, st->B * 8, st->B * 8, st->nl, cudaMemcpyDefault, s));
    PCK(cudaMemcpy2DAsync(tm, st->Bp * 8, branch + (size_t)st->nl * st->B, st->B * 8, st->B * 8, st->nl,
                          cudaMemcpyDefault, s));
  }
  PCK(cudaMemsetAsync(st->flag, 0, sizeof(int), s));
  if (lambda) k_check<<<blocks_for(st->B), 256, 0, s>>>(tl, 1, st->Bp, st->B, 0, st->flag);
  if (branch && st->nl > 0) k_check<<<blocks_for(2 * nm), 256, 0, s>>>(tp, 2 * st->nlp, st->Bp, st->B, 1, st->flag);
  int bad = 0;
  PCK(cudaMemcpyAsync(&bad, st->flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  PCK(cudaStreamSynchronize(s));
  if (bad) {
    *err = "multipliers must be finite and mu >= 0 (SPEC.md:239)";
    return DCOPF_EINVAL;
  }
  if (lambda) PCK(cudaMemcpyAsync(st->lam, tl, st->B * 8, cudaMemcpyDeviceToDevice, s));
  if (branch) {
    PCK(cudaMemcpyAsync(st->mup, tp, nm * 8, cudaMemcpyDeviceToDevice, s));
    PCK(cudaMemcpyAsync(st->mum, tm, nm * 8, cudaMemcpyDeviceToDevice, s));
    k_sub<<<blocks_for(nm), 256, 0, s>>>(st->mup, st->mum, st->nu, nm);
    if (int rc2 = skinny_sync_nu(st, s, err)) return rc2;
  }
  PCK(cudaStreamSynchronize(s));
  return DCOPF_OK;
}

int ptdf_evaluate(PtdfState *st, double *value, double *grad_lambda, double *grad_branch, cudaStream_t s,
                  std::string *err) {
  int rc = DCOPF_OK;
  if (!st->gp) rc = dalloc(&st->gp, (size_t)st->nlp * st->Bp, err);
  if (!rc && !st->gm) rc = dalloc(&st->gm, (size_t)st->nlp * st->Bp, err);
  if (rc) return rc;
  GemmArgs g2 = line_args(st);
  g2.gp_out = st->gp;
  g2.gm_out = st->gm;
  FinArgs f = fin_args(st);
  fin_tiles(st, &f);
  f.glam_out = st->glam;
  if (st->nbv) {
    rc = skinny_pass(st, gen_args(st), g2, false, f, true, s, err);
  } else {
    rc = launch_gen(st, gen_args(st), s, err);
    if (!rc) rc = launch_gemm<EPI_LINE_EVAL>(g2, s, err);
    if (!rc) k_finish<true><<<blocks_for(st->Bp), 256, 0, s>>>(f);
  }
  if (rc) return rc;
  PCK(cudaGetLastError());
  if (value) PCK(cudaMemcpyAsync(value, st->value, st->B * 8, cudaMemcpyDefault, s));
  rc = copy_rows_out(st, grad_lambda, st->glam, 1, s, err);
  if (!rc) rc = copy_rows_out(st, grad_branch, st->gp, st->nl, s, err);
  if (!rc && grad_branch) rc = copy_rows_out(st, grad_branch + (size_t)st->nl * st->B, st->gm, st->nl, s, err);
  if (!rc) PCK(cudaStreamSynchronize(s));
  return rc;
}

int ptdf_set_optimizer(PtdfState *st, const dcopf_optimizer &o, std::string *err) {
  st->opt = o;
  int rc = reset_opt(st, err);
  if (!rc) PCK(cudaDeviceSynchronize());
  return rc;
}

void ptdf_set_stop(PtdfState *st, double tol) { st->tol = tol; }

int ptdf_set_target(PtdfState *st, const double *target, cudaStream_t s, std::string *err) {
  if (!target) {
    st->has_target = false;
    return DCOPF_OK;
  }
  std::vector<double> t(st->Bp, std::numeric_limits<double>::infinity());
  PCK(cudaMemcpyAsync(t.data(), target, st->B * 8, cudaMemcpyDefault, s));
  PCK(cudaStreamSynchronize(s));
  for (long b = 0; b < st->B; ++b)
    if (std::isnan(t[b])) {
      *err = "target is NaN";
      return DCOPF_EINVAL;
    }
  PCK(cudaMemcpyAsync(st->target, t.data(), st->Bp * 8, cudaMemcpyHostToDevice, s));
  PCK(cudaStreamSynchronize(s));
  st->has_target = true;
  return DCOPF_OK;
}

int ptdf_get_first_hit(PtdfState *st, int64_t *hit, cudaStream_t s, std::string *err) {
  if (!hit) return DCOPF_OK;
  PCK(cudaMemcpyAsync(hit, st->hit, st->B * 8, cudaMemcpyDefault, s));
  if (!is_dev(hit)) PCK(cudaStreamSynchronize(s));
  return DCOPF_OK;
}

int ptdf_get_matrix(PtdfState *st, double *Ha, cudaStream_t s, std::string *err) {
  if (!Ha || st->nl == 0) return DCOPF_OK;
  PCK(cudaMemcpy2DAsync(Ha, (size_t)st->nb * 8, st->Ha, st->nbk * 8, (size_t)st->nb * 8, st->nl, cudaMemcpyDefault,
                        s));
  PCK(cudaStreamSynchronize(s));
  return DCOPF_OK;
}

void ptdf_info(const PtdfState *st, dcopf_info *info) {
  info->B = st->B;
  info->B_padded = st->Bp;
  info->path = DCOPF_PATH_DENSE;
  info->form = DCOPF_FORM_PTDF;
  info->n_bus = st->nb;
  info->n_branch = st->nl;
  info->n_gen = st->ng;
  info->quadratic = st->quadratic;
  // per instance-iteration, algorithmic: the two GEMMs' shares of H_g (read once per
  // iteration for the whole batch, so ~0 per instance) + nu, p*, r, mu+-, nu rows
  info->alg_bytes_per_inst_iter = 8LL * (2LL * st->nl + 2LL * st->ng + 6LL * st->nl);
  info->smem_bytes = GEMM_SMEM;
  info->threads_per_block = NTHR;
  info->grid = (int)((st->nlp / BM) * (st->Bp / BN));
  info->launches_per_iter = 3;
  info->tile_width = BN;
  if (st->nbv) {  // skinny batch: warp-per-row matrix-vector kernels (grid of the line kernel)
    info->smem_bytes = 0;
    info->threads_per_block = VT;
    info->grid = skinny_blocks_l(st->nl);
    info->launches_per_iter = 2;
    info->tile_width = st->nbv;
    if (fused_for(st)) {
      // B = 1, the single-read step (with this step variant): its line kernel's stages and grid
      info->smem_bytes = (int)fused_smem(st->ngk, st->fR, st->fS, st->frpc);
      info->threads_per_block = FT;
      info->grid = st->fG;
    }
  }
  info->cluster_size = 1;
}

}  // namespace dcopf
