// sweep_kernel.cuh -- the batched path: one persistent, warp-specialised,
// TMA-fed sweep kernel per dcopf_dual_iterate() call (sm_100a).
//
// Layout: instances are grouped in tiles of W (even, <= 64) -- the tile width
// is chosen per batch so the number of tiles is about the SM count -- and
// every per-instance array is tile-major [tile][entity][W] (F1 mu:
// [tile][branch][2][W]).  A row (one entity of one tile) is 8 W contiguous
// bytes.  Lane l of a warp owns instances 2l and 2l+1 of its tile, so every
// shared-memory / global access of a row is one 16-byte vector per lane and
// every topology record is a warp-uniform broadcast shared by 2*32 instances.
//
// One CTA = one tile, for all K iterations (instances never interact: no grid
// synchronisation, one launch per call).  Each iteration is a sweep over a
// host-compiled schedule (schedule.h) of nch chunks in nch+2 skewed steps;
// step s runs, between two barriers,
//     A(s)    buses of chunk s: w_i over the incidence -> theta* codes
//     B(s-1)  branches whose larger endpoint is in chunk s-1: q_l, f* codes,
//             phi_l, Kirchhoff (F2) / limit (F1) residual, nu' / mu' -> HBM
//     C(s-2)  buses whose last neighbour is in chunk s-2: generators,
//             d/dlambda, lambda' -> HBM
// (the three read only codes produced in earlier steps, so they need no
// barrier between them).  A producer warp streams each step's program block
// and state rows into interval-coloured shared-memory slots with
// cp.async.bulk (TMA 1-D bulk copies) P steps ahead, synchronised by
// full/empty mbarriers.  Every HBM byte of the iteration is read once and
// written once: the traffic is the algorithmic 8 (3 n_b + 2 n_l) B per
// instance-iteration (F2).  Between sweeps the pipeline drains (y_{k+1} rows
// are read by TMA in sweep k+1, so writers fence generic -> async proxy).
//
// Outages (F2): an outaged branch's nu is held at exactly zero (it starts at
// 0 and its gradient f* - phi is +-0), so b nu vanishes in phase A without a
// check; phase B applies b = F = 0 per lane (a per-tile bitmap makes the
// check one broadcast load for unflagged branches) and forces the f* code to
// the tie, so phase C decodes +-0 without a check.  F1 checks in all phases.
//
// Per-entity arithmetic and operation order match dual_kernels.cuh and the
// oracle (reading A-19); only the dual value is summed in another fixed order.
#pragma once
#include <type_traits>

#include "dual_kernels.cuh"
#include "schedule.h"

namespace dcopf {

struct SweepArgs {
  double *lam0, *lam1, *br0, *br1;  // ping-pong state (tile-major)
  const double *d;
  const int *outs;                  // [B_pad][max_out] internal ids, -1 padded
  int max_out;
  int cur;
  const double *alpha;              // [K] device
  long K;
  double *bound, *best;             // [B_pad]
  int *status;
  double *hist;                     // [K][B] or null
  long B;
  const double *target;             // [B_pad] time-to-gap thresholds or null
  long long *hit;                   // [B_pad] first evaluation index with best >= target (-1: none)
  long k_base;                      // evaluation index of this launch's k = 0
  double *out_val;                  // EVAL: value [B_pad]
  double *g_lam, *g_br;             // EVAL: gradients (tile-major)
  int n_bus, n_br, ref, W;
  int n_brows;                      // branch-block rows per tile: n_br (F2 / F1), n_cycles (KVL)
  const uint8_t *prog;
  const long long *prog_off;
  const int *prog_bytes, *tx_bytes;
  const int *ld_ptr;
  const int4 *ld;                   // load entries {kind, first storage position, rows, first slot}
  int nsteps, S, row_bytes, br_row_bytes;
  int off_bar, off_red, off_frz, off_obm, off_outs, off_prog, prog_stride, off_brp, off_lamp, off_dp, off_th,
      off_fc;
  int soft;                         // 1: consumer warps drift by <= 1 step (pool_gap 2); 0: lock-step
  double tol;                       // stopping rule (0: off)
  // ascent-step variant (OPT kernels): DCOPF_OPT_* and its state, stored like
  // the multipliers (tile-major rows in storage order), updated in place
  int opt;
  double rho, beta1, beta2, eps, b1t, b2t;  // b1t, b2t: beta^t before this launch's first step
  double *s1_lam, *s2_lam, *s1_br, *s2_br;
  int debug_mode;                   // 0; 1 = data movement only; 2 = no row copies (measurement only)
};

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// one arrival for the whole warp: __syncwarp orders every lane's shared-memory
// accesses before lane 0's release-arrive (the count of such barriers is the
// number of warps)
__device__ __forceinline__ void warp_arrive(uint64_t *bar, int lane) {
  __syncwarp();
  if (lane == 0) mbar_arrive(bar);
}
// try_wait suspend-time hint: a waiting warp sleeps in hardware until the phase
// completes (or this many ns pass) instead of re-polling, so waiting warps do
// not take issue slots from the working ones
constexpr unsigned kSuspendNs = 1000000;
#ifndef DCOPF_BACKOFF_NS0
#define DCOPF_BACKOFF_NS0 32
#endif
#ifndef DCOPF_BACKOFF_NSMAX
#define DCOPF_BACKOFF_NSMAX 256
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(kSuspendNs)
        : "memory");
  } while (!done);
}
// consumer-to-consumer waits (A-done / B-done): test, then back off with
// nanosleep so a waiting warp issues a handful of instructions instead of
// re-polling (its SM sub-partition's other warps keep the issue slots)
__device__ __forceinline__ void mbar_wait_backoff(uint64_t *bar, unsigned parity) {
  unsigned done = 0, ns = DCOPF_BACKOFF_NS0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(ns);
    ns = ns < DCOPF_BACKOFF_NSMAX ? 2 * ns : ns;
  }
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// the two instances of a lane
struct D2 {
  double x, y;
};
struct OState {  // optimiser state of a lane's two instances (one row)
  double2 s1, s2;
};
__device__ __forceinline__ D2 ld2(const uint8_t *base, int off) {
  const double2 v = *reinterpret_cast<const double2 *>(base + off);
  return D2{v.x, v.y};
}
__device__ __forceinline__ void st2(double *p, double x, double y) {
  *reinterpret_cast<double2 *>(p) = make_double2(x, y);
}
// minimiser codes: one signed byte per instance (+1 / -1 / 0), a lane's two
// instances in one 16-bit word; value = code * bound, exact for codes in {-1, 0, 1}
__device__ __forceinline__ int code_of(bool up, bool down) { return up ? 1 : (down ? -1 : 0); }
__device__ __forceinline__ void st_code2(uint8_t *p, int c0, int c1) {
  *reinterpret_cast<unsigned short *>(p) = (unsigned short)((c0 & 0xff) | ((c1 & 0xff) << 8));
}
__device__ __forceinline__ D2 ld_code2(const uint8_t *base, int off, double x) {
  const unsigned c = *reinterpret_cast<const unsigned short *>(base + off);
  const int c0 = (int)(signed char)(c & 0xffu), c1 = (int)(signed char)(c >> 8);
  return D2{(double)c0 * x, (double)c1 * x};
}

template <int FORM, bool EVAL, int NW, bool SOFT, bool OPT = false>
#ifndef DCOPF_SWEEP_MAXREG
#define DCOPF_SWEEP_MAXREG 96  // 20 warps x 32 x 96 + allocation granularity fit the 64K register file
#endif
__global__ void __maxnreg__(DCOPF_SWEEP_MAXREG) k_sweep(const SweepArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + a.off_bar);
  uint64_t *empty = full + a.S;
  uint64_t *adone = empty + a.S;  // [4] all consumer threads finished phase A of step g (slot g & 3)
  uint64_t *bdone = adone + 4;    // [4] ... phase B of step g
  double *red = reinterpret_cast<double *>(smem + a.off_red);   // [NW][64]
  int *frz = reinterpret_cast<int *>(smem + a.off_frz);         // [64]
  double *bst = reinterpret_cast<double *>(smem + a.off_frz + 256);  // [64] running best (no registers held)
  double *gpv = bst + 64;                                              // [64] previous g (stopping rule)
  unsigned *obm = reinterpret_cast<unsigned *>(smem + a.off_obm);
  int *outs_s = reinterpret_cast<int *>(smem + a.off_outs);     // [64][kMaxOut]
  constexpr int BRW = (FORM == kFormF2) ? 1 : 2;
  constexpr int CT = NW * 32;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W = a.W, L = W >> 1;
  const bool act = lane < L;
  const size_t tile = blockIdx.x;
  const long ib = (long)tile * W;          // first instance of the tile
  const int S = a.S, nst = a.nsteps;
  const long K = EVAL ? 0 : a.K;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SOFT ? NW : 1);  // soft: one arrival per consumer warp
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(&adone[s], NW);
      mbar_init(&bdone[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int x = threadIdx.x; x < (a.n_br + 31) / 32; x += blockDim.x) obm[x] = 0u;
  for (int t = threadIdx.x; t < 64; t += blockDim.x) {
    frz[t] = (!EVAL && t < W) ? a.status[ib + t] : 0;
    bst[t] = (!EVAL && t < W) ? a.best[ib + t] : 0.0;
  }
  for (int x = threadIdx.x; x < 64 * kMaxOut; x += blockDim.x) {
    const int t = x / kMaxOut, j = x % kMaxOut;
    outs_s[x] = (t < W && j < a.max_out) ? a.outs[(ib + t) * a.max_out + j] : -1;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < 64 * kMaxOut; x += blockDim.x)
    if (outs_s[x] >= 0) atomicOr(&obm[outs_s[x] >> 5], 1u << (outs_s[x] & 31));
  __syncthreads();

  if (warp == NW) {
    // =========================== producer ===========================
    const int RB = a.row_bytes, BR = a.br_row_bytes;
    int pst = 0;           // stage of the next step
    unsigned pph = 0;      // its use parity
    bool pused = false;    // every stage used at least once
    for (long k = 0; k <= K; ++k) {
      if (k > 0) named_bar(2, (NW + 1) * 32);  // sweep k-1 written and fenced
      const int par = (a.cur + (int)(k & 1)) & 1;
      const uint8_t *lam_src = reinterpret_cast<const uint8_t *>(par ? a.lam1 : a.lam0) + tile * (size_t)a.n_bus * RB;
      const uint8_t *br_src = reinterpret_cast<const uint8_t *>(par ? a.br1 : a.br0) + tile * (size_t)a.n_brows * BR;
      const uint8_t *d_src = reinterpret_cast<const uint8_t *>(a.d) + tile * (size_t)a.n_bus * RB;
      for (int c = 0; c < nst; ++c) {
        const int st = pst;
        const unsigned pu = pph;  // parity of this use of stage st
        if (++pst == S) {
          pst = 0;
          pph ^= 1u;
        }
        if (pused) mbar_wait(&empty[st], pu ^ 1u);  // previous use of the stage released
        if (pst == 0) pused = true;
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[st], (unsigned)(a.debug_mode == 2 ? a.prog_bytes[c] : a.tx_bytes[c]));
          tma_load_1d(smem + a.off_prog + st * a.prog_stride, a.prog + a.prog_off[c], (unsigned)a.prog_bytes[c],
                      &full[st]);
        }
        __syncwarp();
        // each entry is one bulk copy of `rows` consecutive rows (storage
        // order = load order) into consecutive slots
        const int e1 = (a.debug_mode == 2) ? a.ld_ptr[c] : a.ld_ptr[c + 1];
        for (int e = a.ld_ptr[c] + lane; e < e1; e += 32) {
          const int4 x = a.ld[e];
          if (x.x == LD_LAM)
            tma_load_1d(smem + a.off_lamp + x.w * RB, lam_src + (size_t)x.y * RB, x.z * RB, &full[st]);
          else if (x.x == LD_D)
            tma_load_1d(smem + a.off_dp + x.w * RB, d_src + (size_t)x.y * RB, x.z * RB, &full[st]);
          else
            tma_load_1d(smem + a.off_brp + x.w * BR, br_src + (size_t)x.y * BR, x.z * BR, &full[st]);
        }
      }
    }
    return;
  }

  // =========================== consumers ===========================
  const int RB = a.row_bytes, BR = a.br_row_bytes;
  // lanes past the tile width (W < 64) read the pools' tail padding and never
  // store (mirroring lane 0 instead would put them in lane 0's banks)
  const int lofs = lane * 16;
  const uint8_t *brp = smem + a.off_brp + lofs;
  const uint8_t *lamp = smem + a.off_lamp + lofs;
  const uint8_t *dp = smem + a.off_dp + lofs;
  // optimiser state rows of this tile (OPT kernels)
  uint8_t *os1l = OPT ? reinterpret_cast<uint8_t *>(a.s1_lam) + tile * (size_t)a.n_bus * RB + lofs : nullptr;
  uint8_t *os2l = OPT ? reinterpret_cast<uint8_t *>(a.s2_lam) + tile * (size_t)a.n_bus * RB + lofs : nullptr;
  uint8_t *os1b = OPT ? reinterpret_cast<uint8_t *>(a.s1_br) + tile * (size_t)a.n_brows * BR + lofs : nullptr;
  uint8_t *os2b = OPT ? reinterpret_cast<uint8_t *>(a.s2_br) + tile * (size_t)a.n_brows * BR + lofs : nullptr;
  const bool ost2 = OPT && a.opt == 4;  // Adam: two state arrays
  double ob1t = a.b1t, ob2t = a.b2t;
  uint8_t *thp = smem + a.off_th + 2 * lane;  // theta*_i code rows
  uint8_t *fcp = smem + a.off_fc + 2 * lane;  // f*_l code rows (F2)
  // Consumer warps are not stepped in lock-step.  In step g a warp waits on
  //   full[stage]   before anything: the step's program block and rows landed;
  //   A-done(g-1)   after its A(g) items, before B: the theta* codes of chunk
  //                 g-1 exist (every warp finished A(g-1), hence step g-2);
  //   B-done(g-1)   after its B items, before C: the f* codes C reads exist.
  // A(g) itself waits on no warp: the theta* slots it writes were last read
  // 3 or more steps earlier (schedule pool_gap = 3) and the A-done(g-2) wait of
  // the previous step already guarantees every warp finished step g-3.  (KVL:
  // B(g) likewise, then B-done(g-1) before C and D.)  Warps drift by <= 2 steps.
  unsigned gs = 0;  // global step counter (continues across sweeps; only gs mod 8 matters)
  const int nout = a.max_out;
  const int *my_outs0 = outs_s + (2 * lane) * kMaxOut, *my_outs1 = my_outs0 + kMaxOut;
  auto flagged = [&](int l) { return (obm[l >> 5] >> (l & 31)) & 1u; };
  auto out_t = [&](const int *lst, int l) {
    bool r = false;
    for (int j = 0; j < nout; ++j) r |= (lst[j] == l);
    return r;
  };
  int cst = 0;         // stage of the next step
  unsigned cph = 0;    // parity of its full barrier

  for (long k = 0; k <= K; ++k) {
    const bool last = (k == K);
    const bool write = EVAL || !last;
    const int par = (a.cur + (int)(k & 1)) & 1;
    uint8_t *lam_o = reinterpret_cast<uint8_t *>(EVAL ? a.g_lam : (par ? a.lam0 : a.lam1)) + tile * (size_t)a.n_bus * RB +
                     lofs;
    uint8_t *br_o = reinterpret_cast<uint8_t *>(EVAL ? a.g_br : (par ? a.br0 : a.br1)) + tile * (size_t)a.n_brows * BR +
                    lofs;
    const bool step0 = !EVAL && !last && !frz[2 * lane], step1 = !EVAL && !last && !frz[2 * lane + 1];
    const double alpha = (EVAL || last) ? 0.0 : a.alpha[k];
    if (OPT && !EVAL && !last) {  // Adam's beta^t, t = steps since the state was reset
      ob1t = ob1t * a.beta1;
      ob2t = ob2t * a.beta2;
    }
    // optimiser-variant update of one row of the lane's two instances (the
    // state row sits at the same offset of the state arrays)
    // (oload issues the state loads at the start of an item so their latency
    // overlaps the item's work; ostep updates and stores them)
    auto oload = [&](size_t off, bool lam_side, bool on) -> OState {
      OState o{make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
      if (on) {
        o.s1 = *reinterpret_cast<const double2 *>((lam_side ? os1l : os1b) + off);
        if (ost2) o.s2 = *reinterpret_cast<const double2 *>((lam_side ? os2l : os2b) + off);
      }
      return o;
    };
    auto ostep = [&](OState &o, double y0, double y1, double g0, double g1, size_t off, bool lam_side, bool do0,
                     bool do1) -> D2 {
      if (do0) y0 = opt_update(a.opt, a.rho, a.beta1, a.beta2, a.eps, y0, g0, alpha, o.s1.x, o.s2.x, ob1t, ob2t);
      if (do1) y1 = opt_update(a.opt, a.rho, a.beta1, a.beta2, a.eps, y1, g1, alpha, o.s1.y, o.s2.y, ob1t, ob2t);
      *reinterpret_cast<double2 *>((lam_side ? os1l : os1b) + off) = o.s1;
      if (ost2) *reinterpret_cast<double2 *>((lam_side ? os2l : os2b) + off) = o.s2;
      return D2{y0, y1};
    };
    double v0 = 0.0, v1 = 0.0;

    // the step loop, instantiated twice: CHK = some instance of the tile is
    // frozen (diverged) and its state must be carried over unchanged
    auto run_steps = [&](auto chk_tag) {
    constexpr bool CHK = decltype(chk_tag)::value;
    for (int c = 0; c < nst; ++c) {
      const int st = cst;
      mbar_wait(&full[st], cph);
      if (++cst == S) {
        cst = 0;
        cph ^= 1u;
      }
      const uint8_t *prog = smem + a.off_prog + st * a.prog_stride;
      const int4 h0 = *reinterpret_cast<const int4 *>(prog);       // nA nIA nB nC
      const int4 h1 = *reinterpret_cast<const int4 *>(prog + 16);  // nIC nG a0 b0
      const int4 h2 = *reinterpret_cast<const int4 *>(prog + 32);  // offA offIA offB offC
      const int4 h3 = *reinterpret_cast<const int4 *>(prog + 48);  // offG offIC bytes -
      const int4 h4 = *reinterpret_cast<const int4 *>(prog + 64);  // - - offW -
      const unsigned short *wt = reinterpret_cast<const unsigned short *>(prog + h4.z);  // [3][NW+1] item ranges
      const int nA = h0.x, nB = h0.z, nC = h0.w;

      // ---------------- C: ready buses (F2 / F1: C(s-2), warp table 2; KVL: C(s-1), table 1) ----
      auto phaseC = [&](int tbl) {
        const RecC *Cv = reinterpret_cast<const RecC *>(prog + h2.w);
        const RecG *G = reinterpret_cast<const RecG *>(prog + h3.x);
        for (int j = wt[tbl * (NW + 1) + warp], je = wt[tbl * (NW + 1) + warp + 1]; j < je; ++j) {
          const RecC r = Cv[j];
          OState ost = oload((size_t)r.wpos * RB, true, OPT && !EVAL && write && act);
          const D2 li = ld2(lamp, r.ls), di = ld2(dp, r.ds);
          double gl0 = -di.x, gl1 = -di.y;
#pragma unroll 1
          for (int gg = r.g0; gg < r.g1; ++gg) {  // mostly 0 or 1 generator
            const RecG gr = G[gg];
            const double r0 = gr.c + li.x, r1 = gr.c + li.y;
            const double p0 = gen_minimiser(r0, gr.lo, gr.hi, gr.a), p1 = gen_minimiser(r1, gr.lo, gr.hi, gr.a);
            gl0 = gl0 + p0;
            gl1 = gl1 + p1;
            if (gr.a > 0.0) {
              v0 += gr.a * p0 * p0 + r0 * p0;
              v1 += gr.a * p1 * p1 + r1 * p1;
            } else {
              v0 += r0 * p0;
              v1 += r1 * p1;
            }
          }
          if (FORM != kFormF1) {
            const RecIC2 *IC = reinterpret_cast<const RecIC2 *>(prog + h3.y) + r.e0;
            const int n = r.e1 - r.e0;
            auto acc = [&](const RecIC2 &x) {
              const D2 f = ld_code2(fcp, x.f, x.sF);  // +-f* (c * (+-F) == +-(c * F) exactly)
              gl0 = gl0 + f.x;  // +f* at the to bus, -f* at the from bus
              gl1 = gl1 + f.y;
            };
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (e < n) acc(IC[e]);
#pragma unroll 1
            for (int e = 4; e < n; ++e) acc(IC[e]);
          } else {
            const RecIC1 *IC = reinterpret_cast<const RecIC1 *>(prog + h3.y);
#pragma unroll 1
            for (int e = r.e0; e < r.e1; ++e) {
              const RecIC1 x = IC[e];
              double sb0 = x.sb, sb1 = x.sb;
              if (x.br >= 0 && flagged(x.br)) {
                if (out_t(my_outs0, x.br)) sb0 = copysign(0.0, sb0);
                if (out_t(my_outs1, x.br)) sb1 = copysign(0.0, sb1);
              }
              const D2 ts = ld_code2(thp, x.ts, x.ths), tt = ld_code2(thp, x.tt, x.tht);
              gl0 = gl0 + sb0 * (ts.x - tt.x);
              gl1 = gl1 + sb1 * (ts.y - tt.y);
            }
          }
          v0 += -(li.x * di.x);
          v1 += -(li.y * di.y);
          if (write && act) {
            double *dst = reinterpret_cast<double *>(lam_o + (size_t)r.wpos * RB);
            if (EVAL) {
              st2(dst, gl0, gl1);
            } else if constexpr (OPT) {
              const D2 y = ostep(ost, li.x, li.y, gl0, gl1, (size_t)r.wpos * RB, true, !CHK || step0, !CHK || step1);
              st2(dst, y.x, y.y);
            } else {
              st2(dst, (!CHK || step0) ? li.x + alpha * gl0 : li.x, (!CHK || step1) ? li.y + alpha * gl1 : li.y);
            }
          }
        }
      };
      if constexpr (FORM == kFormKVL) {
      if (a.debug_mode != 1) {
      // B(s) needs no other warp: its rows come by TMA, and the f* code slots
      // it writes were last read 3+ steps ago (pool_gap 3), by which time every
      // warp has finished (this warp waited B-done(s-2) in the previous step)
      // ---------------- B(s): q_l = x_l (sum_k C_kl kappa_k) - (lambda_s - lambda_t), f* ----------------
      {
        const RecBK *Bv = reinterpret_cast<const RecBK *>(prog + h2.z);
        const RecBKe *BKe = reinterpret_cast<const RecBKe *>(prog + h3.w);
        for (int j = wt[warp], je = wt[warp + 1]; j < je; ++j) {
          const RecBK r = Bv[j];
          double x0 = r.x, x1 = r.x, F0 = r.F, F1v = r.F;
          bool o0 = false, o1 = false;
          if (r.obr >= 0 && flagged(r.obr)) {  // an outaged lane: b = F = 0
            o0 = out_t(my_outs0, r.obr);
            o1 = out_t(my_outs1, r.obr);
            if (o0) x0 = F0 = 0.0;
            if (o1) x1 = F1v = 0.0;
          }
          double s0 = 0.0, s1 = 0.0;  // cycles in ascending k (the oracle's order)
#pragma unroll 1
          for (int e = r.e0; e < r.e1; ++e) {
            const RecBKe t = BKe[e];
            const D2 kv = ld2(brp, t.ks);
            s0 = (t.sgn > 0) ? s0 + kv.x : s0 - kv.x;
            s1 = (t.sgn > 0) ? s1 + kv.y : s1 - kv.y;
          }
          const D2 ls = ld2(lamp, r.ls), lt = ld2(lamp, r.lt);
          const double q0 = x0 * s0 - (ls.x - lt.x), q1 = x1 * s1 - (ls.y - lt.y);
          const double f0 = (q0 > 0.0) ? -F0 : ((q0 < 0.0) ? F0 : 0.0);
          const double f1 = (q1 > 0.0) ? -F1v : ((q1 < 0.0) ? F1v : 0.0);
          if (act) st_code2(fcp + r.fs, o0 ? 0 : code_of(q0 < 0.0, q0 > 0.0), o1 ? 0 : code_of(q1 < 0.0, q1 > 0.0));
          v0 += q0 * f0;
          v1 += q1 * f1;
        }
      }
      if (SOFT) {  // C and D read the f* codes of B(<= s-1)
        warp_arrive(&bdone[gs & 3], lane);
        if (gs > 0) mbar_wait_backoff(&bdone[(gs - 1) & 3], ((gs - 1) >> 2) & 1u);
      }
      phaseC(1);
      // ---------------- D(s-1): d/dkappa_k = sum_l C_kl x_l f*_l, kappa' ----------------
      {
        const RecD *Dv = reinterpret_cast<const RecD *>(prog + h2.x);
        const RecDe *De = reinterpret_cast<const RecDe *>(prog + h2.y);
        for (int j = wt[2 * (NW + 1) + warp], je = wt[2 * (NW + 1) + warp + 1]; j < je; ++j) {
          const RecD r = Dv[j];
          OState ost = oload((size_t)r.wpos * BR, false, OPT && !EVAL && write && act);
          const D2 kv = ld2(brp, r.ks);
          double acc0 = 0.0, acc1 = 0.0;
#pragma unroll 1
          for (int e = r.e0; e < r.e1; ++e) {
            const RecDe d = De[e];
            const unsigned c = *reinterpret_cast<const unsigned short *>(fcp + d.fs);
            // index 0 / 1 / 2 for code -1 / 0 / +1 (lanes past the tile width read
            // padding bytes: clamp so they never index outside the record)
            const int c0 = (int)(signed char)(c & 0xffu), c1 = (int)(signed char)(c >> 8);
            const int i0 = (c0 > 0) ? 2 : ((c0 < 0) ? 0 : 1), i1 = (c1 > 0) ? 2 : ((c1 < 0) ? 0 : 1);
            acc0 = acc0 + d.t[i0];  // (c F) sx: the oracle's C_kl (f*_l x_l), exact
            acc1 = acc1 + d.t[i1];
          }
          if (r.dbr >= 0 && flagged(r.dbr)) {  // defining branch out: no cycle, gradient 0
            if (out_t(my_outs0, r.dbr)) acc0 = 0.0;
            if (out_t(my_outs1, r.dbr)) acc1 = 0.0;
          }
          if (write && act) {
            double *dst = reinterpret_cast<double *>(br_o + (size_t)r.wpos * BR);
            if (EVAL) {
              st2(dst, acc0, acc1);
            } else if constexpr (OPT) {
              const D2 y = ostep(ost, kv.x, kv.y, acc0, acc1, (size_t)r.wpos * BR, false, !CHK || step0, !CHK || step1);
              st2(dst, y.x, y.y);
            } else {
              st2(dst, (!CHK || step0) ? kv.x + alpha * acc0 : kv.x, (!CHK || step1) ? kv.y + alpha * acc1 : kv.y);
            }
          }
        }
      }
      }  // debug_mode
      } else {
      if (a.debug_mode != 1) {  // (1: data movement only -- measurement)
      // A(s) needs no other warp: its rows come by TMA, and the theta* code
      // slots it writes were last read 3+ steps ago (pool_gap 3), by which time
      // every warp has finished (this warp waited A-done(s-2) in step s-1)
      // ---------------- A(s): w_i, theta* codes ----------------
      {
        const RecA *A = reinterpret_cast<const RecA *>(prog + h2.x);
        for (int j = wt[warp], je = wt[warp + 1]; j < je; ++j) {
          const RecA ra = A[j];
          const int bus = ra.bus;
          double w0 = 0.0, w1 = 0.0;
          if (FORM == kFormF2) {
            // incidence entries in ascending original branch id (the oracle's
            // order); degree <= 4 for ~97% of buses: a fixed 4-way body with
            // warp-uniform guards instead of a counted loop, the rest in a tail
            const RecIA2 *IA = reinterpret_cast<const RecIA2 *>(prog + h2.y) + ra.e0;
            const int n = ra.e1 - ra.e0;
            auto acc = [&](const RecIA2 &r) {
              const D2 nu = ld2(brp, r.row);
              w0 = w0 + r.sb * nu.x;  // w_s += -(b nu), w_t += b nu (outaged: nu == 0)
              w1 = w1 + r.sb * nu.y;
            };
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (e < n) acc(IA[e]);
#pragma unroll 1
            for (int e = 4; e < n; ++e) acc(IA[e]);
          } else {
            const RecIA1 *IA = reinterpret_cast<const RecIA1 *>(prog + h2.y);
#pragma unroll 1
            for (int e = ra.e0; e < ra.e1; ++e) {
              const RecIA1 r = IA[e];
              double sb0 = r.sb, sb1 = r.sb;
              if (r.br >= 0 && flagged(r.br)) {  // br < 0: branch never taken out
                if (out_t(my_outs0, r.br)) sb0 = copysign(0.0, sb0);
                if (out_t(my_outs1, r.br)) sb1 = copysign(0.0, sb1);
              }
              const D2 mp = ld2(brp, r.row), mm = ld2(brp, r.row + RB);
              const D2 ls = ld2(lamp, r.ls), lt = ld2(lamp, r.lt);
              w0 = w0 + sb0 * ((mp.x - mm.x) - (ls.x - lt.x));  // w_s += u, w_t -= u
              w1 = w1 + sb1 * ((mp.y - mm.y) - (ls.y - lt.y));
            }
          }
          // theta* = -Theta if w > 0, +Theta if w < 0, 0 on a tie and at the reference bus
          const bool nr = (bus != a.ref);
          const double t0 = (nr && w0 < 0.0) ? ra.theta : ((nr && w0 > 0.0) ? -ra.theta : 0.0);
          const double t1 = (nr && w1 < 0.0) ? ra.theta : ((nr && w1 > 0.0) ? -ra.theta : 0.0);
          if (act) st_code2(thp + ra.th, code_of(nr && w0 < 0.0, nr && w0 > 0.0), code_of(nr && w1 < 0.0, nr && w1 > 0.0));
          if (nr) {
            v0 += w0 * t0;
            v1 += w1 * t1;
          }
        }
      }
      if (SOFT) {  // B(s-1) reads the theta* codes of A(<= s-1); the f* slots it writes
        // were last read 2+ steps ago, and A-done(s-1) implies every warp finished step s-2
        warp_arrive(&adone[gs & 3], lane);
        if (gs > 0) mbar_wait_backoff(&adone[(gs - 1) & 3], ((gs - 1) >> 2) & 1u);
      }
      // ---------------- B(s-1): branches ----------------
      {
        const RecB *Bv = reinterpret_cast<const RecB *>(prog + h2.z);
        for (int j = wt[NW + 1 + warp], je = wt[NW + 2 + warp]; j < je; ++j) {
          const RecB r = Bv[j];
          OState ost = oload((size_t)r.wpos * BR, false, OPT && !EVAL && write && act);
          OState ost_m = oload((size_t)r.wpos * BR + RB, false, FORM == kFormF1 && OPT && !EVAL && write && act);
          double b0 = r.b, b1 = r.b, F0 = r.F, F1v = r.F;
          bool o0 = false, o1 = false;
          if (r.obr >= 0 && flagged(r.obr)) {  // obr < 0: branch never taken out
            o0 = out_t(my_outs0, r.obr);
            o1 = out_t(my_outs1, r.obr);
            if (o0) b0 = F0 = 0.0;
            if (o1) b1 = F1v = 0.0;
          }
          const D2 ths = ld_code2(thp, r.ts, r.ths), tht = ld_code2(thp, r.tt, r.tht);
          const double phi0 = b0 * (ths.x - tht.x);
          const double phi1 = b1 * (ths.y - tht.y);
          double* dst = reinterpret_cast<double *>(br_o + (size_t)r.wpos * BR);
          if (FORM == kFormF2) {
            const D2 nu = ld2(brp, r.row), ls = ld2(lamp, r.ls), lt = ld2(lamp, r.lt);
            const double q0 = nu.x - (ls.x - lt.x), q1 = nu.y - (ls.y - lt.y);
            // f* = -F if q > 0, +F if q < 0, 0 on a tie (an outaged lane has F = 0)
            const double f0 = (q0 > 0.0) ? -F0 : ((q0 < 0.0) ? F0 : 0.0);
            const double f1 = (q1 > 0.0) ? -F1v : ((q1 < 0.0) ? F1v : 0.0);
            // code for C (an outaged lane stores the tie: its f* = +-0)
            if (act) st_code2(fcp + r.fs, o0 ? 0 : code_of(q0 < 0.0, q0 > 0.0), o1 ? 0 : code_of(q1 < 0.0, q1 > 0.0));
            const double g0 = f0 - phi0, g1 = f1 - phi1;  // Kirchhoff residual
            v0 += q0 * f0;
            v1 += q1 * f1;
            if (write && act) {
              if (EVAL) {
                st2(dst, g0, g1);
              } else if constexpr (OPT) {
                const D2 y = ostep(ost, nu.x, nu.y, g0, g1, (size_t)r.wpos * BR, false, !CHK || step0, !CHK || step1);
                st2(dst, y.x, y.y);
              } else {
                st2(dst, (!CHK || step0) ? nu.x + alpha * g0 : nu.x, (!CHK || step1) ? nu.y + alpha * g1 : nu.y);
              }
            }
          } else {
            const D2 mp = ld2(brp, r.row), mm = ld2(brp, r.row + RB);
            const double gp0 = phi0 - F0, gm0 = -phi0 - F0, gp1 = phi1 - F1v, gm1 = -phi1 - F1v;
            v0 += -(F0 * (mp.x + mm.x));
            v1 += -(F1v * (mp.y + mm.y));
            if (write && act) {
              double* dst2 = reinterpret_cast<double *>(br_o + (size_t)r.wpos * BR + RB);
              if (EVAL) {
                st2(dst, gp0, gp1);
                st2(dst2, gm0, gm1);
              } else {
                double p0 = mp.x, m0 = mm.x, p1 = mp.y, m1 = mm.y;
                if constexpr (OPT) {
                  const bool d0 = !CHK || step0, d1 = !CHK || step1;
                  const D2 yp = ostep(ost, mp.x, mp.y, gp0, gp1, (size_t)r.wpos * BR, false, d0, d1);
                  const D2 ym = ostep(ost_m, mm.x, mm.y, gm0, gm1, (size_t)r.wpos * BR + RB, false, d0, d1);
                  if (d0) {
                    p0 = (yp.x > 0.0) ? yp.x : 0.0;  // mu <- max(mu, 0)
                    m0 = (ym.x > 0.0) ? ym.x : 0.0;
                  }
                  if (d1) {
                    p1 = (yp.y > 0.0) ? yp.y : 0.0;
                    m1 = (ym.y > 0.0) ? ym.y : 0.0;
                  }
                } else {
                if (!CHK || step0) {
                  p0 = mp.x + alpha * gp0;
                  m0 = mm.x + alpha * gm0;
                  p0 = (p0 > 0.0) ? p0 : 0.0;  // mu <- max(mu, 0)
                  m0 = (m0 > 0.0) ? m0 : 0.0;
                }
                if (!CHK || step1) {
                  p1 = mp.y + alpha * gp1;
                  m1 = mm.y + alpha * gm1;
                  p1 = (p1 > 0.0) ? p1 : 0.0;
                  m1 = (m1 > 0.0) ? m1 : 0.0;
                }
                }
                st2(dst, p0, p1);
                st2(dst2, m0, m1);
              }
            }
          }
        }
      }
      if (SOFT) {
        warp_arrive(&bdone[gs & 3], lane);
        if (gs > 0) mbar_wait_backoff(&bdone[(gs - 1) & 3], ((gs - 1) >> 2) & 1u);
      }
      phaseC(2);
      }  // debug_mode
      }  // FORM
      if (SOFT) {
        warp_arrive(&empty[st], lane);
      } else {  // lock-step mode: every warp finished the step
        named_bar(1, CT);
        if (threadIdx.x == 0) mbar_arrive(&empty[st]);
      }
      ++gs;
    }
    };
    const bool anyf = __any_sync(0xffffffffu, (frz[2 * lane] | frz[2 * lane + 1]) != 0);
    if (anyf) run_steps(std::integral_constant<bool, true>{});
    else run_steps(std::integral_constant<bool, false>{});
    // ---------------- dual value, best, status ----------------
    named_bar(1, CT);  // every warp is past the sweep's last step: the pools red aliases are dead
    red[warp * 64 + 2 * lane] = v0;
    red[warp * 64 + 2 * lane + 1] = v1;
    named_bar(1, CT);
    if (warp == 0 && act) {
      double g0 = 0.0, g1 = 0.0;
      for (int w = 0; w < NW; ++w) {
        g0 += red[w * 64 + 2 * lane];
        g1 += red[w * 64 + 2 * lane + 1];
      }
      const long b0i = ib + 2 * lane, b1i = b0i + 1;
      if (EVAL) {
        a.out_val[b0i] = g0;
        a.out_val[b1i] = g1;
      } else {
        if (!last && a.hist) {
          if (b0i < a.B) a.hist[(size_t)k * a.B + b0i] = g0;
          if (b1i < a.B) a.hist[(size_t)k * a.B + b1i] = g1;
        }
        if (last) {
          a.bound[b0i] = g0;
          a.bound[b1i] = g1;
        }
        double best0 = bst[2 * lane], best1 = bst[2 * lane + 1];
        // (stopping rule: |g_k - g_{k-1}| < tol within this call; status 2)
        const bool chk = a.tol > 0.0 && k > 0;
        if (!frz[2 * lane]) {
          if (valid_bound(g0)) {
            best0 = (g0 > best0) ? g0 : best0;
            if (chk && fabs(g0 - gpv[2 * lane]) < a.tol) frz[2 * lane] = 2;
          } else {
            frz[2 * lane] = 1;
          }
        }
        if (!frz[2 * lane + 1]) {
          if (valid_bound(g1)) {
            best1 = (g1 > best1) ? g1 : best1;
            if (chk && fabs(g1 - gpv[2 * lane + 1]) < a.tol) frz[2 * lane + 1] = 2;
          } else {
            frz[2 * lane + 1] = 1;
          }
        }
        bst[2 * lane] = best0;
        bst[2 * lane + 1] = best1;
        gpv[2 * lane] = g0;
        gpv[2 * lane + 1] = g1;
        if (a.target) {  // time to gap: first evaluation whose running best reaches the target
          // (state kept in global memory, touched once per sweep: no registers held)
          if (a.hit[b0i] < 0 && best0 >= a.target[b0i]) a.hit[b0i] = a.k_base + k;
          if (a.hit[b1i] < 0 && best1 >= a.target[b1i]) a.hit[b1i] = a.k_base + k;
        }
      }
    }
    if (!last) {
      // y_{k+1} rows must be visible to the async proxy before the producer
      // issues sweep k+1's bulk copies
      __threadfence();
      asm volatile("fence.proxy.async.global;" ::: "memory");
      named_bar(2, (NW + 1) * 32);
    } else {
      named_bar(1, CT);
    }
  }
  if (!EVAL && warp == 0 && act) {
    a.best[ib + 2 * lane] = bst[2 * lane];
    a.best[ib + 2 * lane + 1] = bst[2 * lane + 1];
    a.status[ib + 2 * lane] = frz[2 * lane];
    a.status[ib + 2 * lane + 1] = frz[2 * lane + 1];
  }
}

}  // namespace dcopf
