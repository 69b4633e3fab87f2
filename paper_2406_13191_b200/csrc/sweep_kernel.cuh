// sweep_kernel.cuh -- the batched path: one persistent, warp-specialised,
// TMA-fed sweep kernel per dcopf_dual_iterate() call (sm_100a).
//
// Layout: instances are grouped in tiles of W (a multiple of V <= 32 V) and
// every per-instance array is tile-major [tile][entity][W] (F1 mu:
// [tile][branch][2][W]).  A row (one entity of one tile) is 8 W contiguous
// bytes.  Lane l of a warp owns V instances of its tile: 2l and 2l+1 (V = 2),
// plus W/2 + 2l and W/2 + 2l + 1 (V = 4), so every shared-memory / global
// access of a row is one (V = 2) or two (V = 4) 16-byte vectors per lane, and
// every topology record is a warp-uniform broadcast shared by 32 V instances.
// The issue cost of an item (record decode, addressing, loop control) is per
// warp, so V = 4 halves it per instance; only the fp64 arithmetic scales
// with V.
//
// A tile is swept by C CTAs ("parts", split_schedule.cpp), part p owning a
// contiguous range of the network (C = 1: the whole network).  Instances
// never interact: there is no grid synchronisation, only the tile's parts
// meet once per sweep (below).  Each iteration is a sweep over the part's
// host-compiled steps (schedule.h); for F2 / F1 step s runs, between
// barriers,
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
// instance-iteration (F2), plus the few halo rows of a split tile.  Between
// sweeps the pipeline drains (y_{k+1} rows are read by TMA in sweep k+1, so
// writers fence generic -> async proxy).
//
// Split tiles (C > 1): halo items recompute the codes a part reads but does
// not own (RecA kAFlagHalo, RecB wpos < 0, RecBK halo) and count nothing
// toward the value.  At the end of a sweep every part publishes its partial
// dual value of each instance, arrives on the tile's counter in global
// memory (release) and waits for all C arrivals (acquire); then every part
// sums the C partials in part order, so all parts take the same best /
// divergence / stopping decisions, and the y_{k+1} rows each part wrote are
// visible to the other parts' TMA copies of sweep k+1.  The launch is
// cooperative: all CTAs are co-resident.
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
#include <cstddef>
#include <type_traits>

#include "dual_kernels.cuh"
#include "schedule.h"

namespace dcopf {

// (byte offsets of the records' wpos field: the optimiser kernels read the next
// item's wpos alone to prefetch its state rows)
static_assert(offsetof(RecC, wpos) == 0 && offsetof(RecB, wpos) == 24 && offsetof(RecD, wpos) == 4,
              "record layout");

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
  int S, row_bytes, br_row_bytes;
  int off_bar, off_red, off_frz, off_obm, off_outs, off_prog, prog_stride, off_brp, off_lamp, off_dp, off_th,
      off_fc;
  // split tiles
  int parts;                        // C: CTAs per tile (blockIdx.x = tile * C + part)
  int part_step0[kMaxParts + 1];    // first global step of each part (kernel parameter space: the
                                    // per-step loop bound is a constant-bank operand, never spilled)
  unsigned *tile_sync;              // [tiles] arrival counters, zero at launch (C > 1)
  double *part_val;                 // [2][tiles][C][W] partial dual values (C > 1)
  int tiles;
  int soft;                         // 1: consumer warps drift by <= 2 steps (pool_gap 3); 0: lock-step
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
#ifdef DCOPF_CW_SUSPEND
  mbar_wait(bar, parity);
  return;
#endif
  unsigned done = 0, ns = 32;
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
    ns = ns < 256 ? 2 * ns : ns;
  }
}
// (the same operations on 32-bit shared addresses, precomputed once per kernel)
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity), "r"(kSuspendNs)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_wait_backoff(unsigned bar, unsigned parity) {
#ifdef DCOPF_CW_SUSPEND
  mbar_wait(bar, parity);
  return;
#endif
#ifndef DCOPF_CW_NS0
#define DCOPF_CW_NS0 32
#define DCOPF_CW_NSMAX 256
#endif
  unsigned done = 0, ns = DCOPF_CW_NS0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(ns);
    ns = ns < DCOPF_CW_NSMAX ? 2 * ns : ns;
  }
}
__device__ __forceinline__ void tma_load_1d(unsigned dst, const void *src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void l2_prefetch(const void *src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_l1(const void *p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// branch-free select (selp.f64): the bound selections below differ per lane,
// and written as nested conditionals nvcc may compile them into divergent
// branches (BSSY / BSYNC around both paths) instead of selects
__device__ __forceinline__ double sel(bool p, double a, double b) {
  double r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\tselp.f64 %0, %1, %2, q;\n\t}"
      : "=d"(r)
      : "d"(a), "d"(b), "r"((unsigned)p));
  return r;
}
// x on "up", -x on "down", 0 otherwise (x >= 0: the upper / lower box bound)
__device__ __forceinline__ double bound_sel(bool up, bool down, double x) { return sel(up, x, sel(down, -x, 0.0)); }
// the flow-box minimiser and its code from the sign of q in one go (shared
// predicates): f = +F, code +1 if q < 0; f = -F (nF), code -1 if q > 0; else 0
// (a NaN q is a tie, as in the oracle's comparisons)
__device__ __forceinline__ double flow_min(double q, double F, double nF, int &code) {
  double f;
  asm("{\n\t.reg .pred pu, pd;\n\t.reg .f64 t;\n\t"
      "setp.lt.f64 pu, %2, 0d0000000000000000;\n\t"
      "setp.gt.f64 pd, %2, 0d0000000000000000;\n\t"
      "selp.f64 t, %4, 0d0000000000000000, pd;\n\t"
      "selp.f64 %0, %3, t, pu;\n\t"
      "selp.s32 %1, -1, 0, pd;\n\t"
      "selp.s32 %1, 1, %1, pu;\n\t}"
      : "=d"(f), "=r"(code)
      : "d"(q), "d"(F), "d"(nF));
  return f;
}

// the V instances of a lane
template <int V>
struct DV {
  double v[V];
};
template <int V>
struct OState {  // optimiser state of a lane's instances (one row)
  double s1[V], s2[V];
};
// Shared memory is addressed by 32-bit shared-window addresses held in
// registers (`sa` arguments) and read / written with explicit ld.shared /
// st.shared: from generic pointers into the dynamic shared array nvcc
// re-derives the window base (S2UR SR_CgaCtaId + ULEA) at many accesses of the
// item loops, and the S2UR latency stalled ~5% of the warps' time.  The asm is
// volatile (never moved across the mbarrier waits, which are volatile asm).
__device__ __forceinline__ double2 lds_f64x2(unsigned sa) {
  return *reinterpret_cast<const double2 *>(__cvta_shared_to_generic((size_t)sa));
}
__device__ __forceinline__ uint4 lds_u32x4(unsigned sa) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(sa));
  return r;
}
__device__ __forceinline__ uint2 lds_u32x2(unsigned sa) {
  uint2 r;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(sa));
  return r;
}
__device__ __forceinline__ unsigned lds_u16(unsigned sa) {
  return *reinterpret_cast<const unsigned short *>(__cvta_shared_to_generic((size_t)sa));
}
__device__ __forceinline__ unsigned lds_u32(unsigned sa) {
  return *reinterpret_cast<const unsigned *>(__cvta_shared_to_generic((size_t)sa));
}
__device__ __forceinline__ void sts_u16(unsigned sa, unsigned v) {
  *reinterpret_cast<unsigned short *>(__cvta_shared_to_generic((size_t)sa)) = (unsigned short)v;
}
__device__ __forceinline__ void sts_u64(unsigned sa, unsigned long long v) {
  *reinterpret_cast<unsigned long long *>(__cvta_shared_to_generic((size_t)sa)) = v;
}
__device__ __forceinline__ unsigned long long lds_u64(unsigned sa) {
  return *reinterpret_cast<const unsigned long long *>(__cvta_shared_to_generic((size_t)sa));
}
__device__ __forceinline__ void sts_f64(unsigned sa, double v) {
  *reinterpret_cast<double *>(__cvta_shared_to_generic((size_t)sa)) = v;
}
__device__ __forceinline__ double lds_f64(unsigned sa) {
  return *reinterpret_cast<const double *>(__cvta_shared_to_generic((size_t)sa));
}
__device__ __forceinline__ void sts_u32(unsigned sa, unsigned v) {
  *reinterpret_cast<unsigned *>(__cvta_shared_to_generic((size_t)sa)) = v;
}
// a program-block record by value: a plain load through a generic pointer
// formed from the 32-bit shared address (the compiler folds the conversion
// back into shared loads of just the fields used, with the window base kept
// in a uniform register)
template <class T>
__device__ __forceinline__ T lds_rec(unsigned sa) {
  return *reinterpret_cast<const T *>(__cvta_shared_to_generic((size_t)sa));
}

// row loads / stores: instances 2l, 2l+1 at byte 16 l of the row (folded into
// the base address), instances W/2 + 2l, W/2 + 2l + 1 hb = 4 W bytes further
template <int V>
__device__ __forceinline__ DV<V> ldsv(unsigned base, int off, int hb) {
  DV<V> r;
  const double2 a = lds_f64x2(base + off);
  r.v[0] = a.x;
  r.v[1] = a.y;
  if constexpr (V == 4) {
    const double2 b = lds_f64x2(base + off + hb);
    r.v[2] = b.x;
    r.v[3] = b.y;
  }
  return r;
}
template <int V>
__device__ __forceinline__ DV<V> ldv(const uint8_t *base, int off, int hb) {
  DV<V> r;
  const double2 a = *reinterpret_cast<const double2 *>(base + off);
  r.v[0] = a.x;
  r.v[1] = a.y;
  if constexpr (V == 4) {
    const double2 b = *reinterpret_cast<const double2 *>(base + off + hb);
    r.v[2] = b.x;
    r.v[3] = b.y;
  }
  return r;
}
template <int V>
__device__ __forceinline__ void stv(void *p, const double (&x)[V], int hb) {
  *reinterpret_cast<double2 *>(p) = make_double2(x[0], x[1]);
  if constexpr (V == 4) *reinterpret_cast<double2 *>(reinterpret_cast<uint8_t *>(p) + hb) = make_double2(x[2], x[3]);
}
// minimiser codes: one signed byte per instance (+1 / -1 / 0), a lane's V
// instances in one 2- or 4-byte word at byte V l of the code row (folded into
// the base pointer); value = code * bound, exact for codes in {-1, 0, 1}
__device__ __forceinline__ int code_of(bool up, bool down) { return up ? 1 : (down ? -1 : 0); }
template <int V>
__device__ __forceinline__ void st_codes(unsigned sa, const int (&c)[V]) {
  if constexpr (V == 2) {
    sts_u16(sa, (unsigned)((c[0] & 0xff) | ((c[1] & 0xff) << 8)));
  } else {
    sts_u32(sa, (unsigned)(c[0] & 0xff) | ((unsigned)(c[1] & 0xff) << 8) | ((unsigned)(c[2] & 0xff) << 16) |
                    ((unsigned)(c[3] & 0xff) << 24));
  }
}
template <int V>
__device__ __forceinline__ void ld_codes(unsigned base, int off, int (&c)[V]) {
  if constexpr (V == 2) {
    const unsigned u = lds_u16(base + off);
    c[0] = (int)(signed char)(u & 0xffu);
    c[1] = (int)(signed char)(u >> 8);
  } else {
    const unsigned u = lds_u32(base + off);
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = (int)(signed char)((u >> (8 * j)) & 0xffu);
  }
}
template <int V>
__device__ __forceinline__ DV<V> ld_code(unsigned base, int off, double x) {
  int c[V];
  ld_codes<V>(base, off, c);
  DV<V> r;
#pragma unroll
  for (int j = 0; j < V; ++j) r.v[j] = (double)c[j] * x;
  return r;
}

// registers per thread: (NW + 1) warps share the 64K register file
template <int NW>
struct SweepRegs {  // the largest multiple of 8 registers with which NW + 1 warps fit the register
  // file: 16K registers per SM sub-partition, warps spread round-robin over the 4
  static constexpr int per_smsp = (NW + 1 + 3) / 4;
  static constexpr int r = 16384 / (per_smsp * 32) / 8 * 8;
  static constexpr int value = r > 168 ? 168 : r;
};

template <int FORM, bool EVAL, int NW, bool SOFT, bool OPT, int V>
__global__ void __maxnreg__(SweepRegs<NW>::value) k_sweep(const SweepArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + a.off_bar);
  uint64_t *empty = full + a.S;
  uint64_t *adone = empty + a.S;  // [4] all consumer threads finished phase A of step g (slot g & 3)
  uint64_t *bdone = adone + 4;    // [4] ... phase B of step g
  const unsigned sbase = smem_u32(smem);  // 32-bit shared addresses of the pools and barriers
  const unsigned full_sa = sbase + a.off_bar, empty_sa = full_sa + 8 * a.S, adone_sa = empty_sa + 8 * a.S,
                 bdone_sa = adone_sa + 32;
  constexpr int TS = 32 * V;  // per-tile instance slots (schedule.cpp layout_smem)
  double *red = reinterpret_cast<double *>(smem + a.off_red);   // [NW][TS]
  int *frz = reinterpret_cast<int *>(smem + a.off_frz);         // [TS]
  double *bst = reinterpret_cast<double *>(smem + a.off_frz + 4 * TS);  // [TS] running best
  double *gpv = bst + TS;                                                // [TS] previous g
  unsigned *obm = reinterpret_cast<unsigned *>(smem + a.off_obm);
  int *outs_s = reinterpret_cast<int *>(smem + a.off_outs);     // [TS][kMaxOut]
  constexpr int CT = NW * 32;
  static_assert(V == 2 || V == 4, "2 or 4 instances per lane");

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W = a.W, L = W / V, hW = W >> 1, hb = 4 * W;
  const bool act = lane < L;
  // the tile, the part and the part's step range are recomputed where they
  // are used (per sweep) or read from shared memory (per step) instead of
  // being held in registers across the step loop: at this register budget
  // they are what ptxas spills first, and a spilled loop bound or stage
  // address is a round trip to L1/L2 per step on the critical path
  const int C = a.parts;
#define DCOPF_PART ((int)(blockIdx.x % (unsigned)a.parts))
#define DCOPF_TILE ((size_t)(blockIdx.x / (unsigned)a.parts))
  const int S = a.S;
  int *s_rng = reinterpret_cast<int *>(bdone + 4);  // [2] the part's first step, last step + 1
#define DCOPF_S0 ((int)lds_u32(bdone_sa + 32))
#define DCOPF_S1 ((int)lds_u32(bdone_sa + 36))
  const long K = EVAL ? 0 : a.K;
  // instance (within the tile) of this lane's j-th value
  auto inst = [&](int j) { return (j < 2) ? 2 * lane + j : hW + 2 * lane + (j - 2); };

  // optimiser kernels (schedule opt_bytes): after the step range, the tile's
  // byte offsets of its lambda-side / branch-side state rows, then per consumer
  // warp [1 - beta1^t, 1 - beta2^t, their reciprocals, beta1^t, beta2^t] -- kept
  // here rather than in registers across the step loop, where they spilled
  const unsigned opt_sa = bdone_sa + 48;
  if (threadIdx.x == 0) {
    s_rng[0] = a.part_step0[DCOPF_PART];
    s_rng[1] = a.part_step0[DCOPF_PART + 1];
    if (OPT) {
      sts_u64(opt_sa, (unsigned long long)(DCOPF_TILE * (size_t)a.n_bus * a.row_bytes));
      sts_u64(opt_sa + 8, (unsigned long long)(DCOPF_TILE * (size_t)a.n_brows * a.br_row_bytes));
    }
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SOFT ? CT : 1);  // soft: one arrival per consumer thread
    }
    for (int s = 0; s < 4; ++s) {  // (every consumer thread arrives: no __syncwarp before one lane's arrive)
      mbar_init(&adone[s], CT);
      mbar_init(&bdone[s], CT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int x = threadIdx.x; x < (a.n_br + 31) / 32; x += blockDim.x) obm[x] = 0u;
  for (int t = threadIdx.x; t < TS; t += blockDim.x) {
    const long ib = (long)DCOPF_TILE * W;  // first instance of the tile
    frz[t] = (!EVAL && t < W) ? a.status[ib + t] : 0;
    bst[t] = (!EVAL && t < W) ? a.best[ib + t] : 0.0;
  }
  for (int x = threadIdx.x; x < TS * kMaxOut; x += blockDim.x) {
    const int t = x / kMaxOut, j = x % kMaxOut;
    outs_s[x] = (t < W && j < a.max_out) ? a.outs[((long)DCOPF_TILE * W + t) * a.max_out + j] : -1;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < TS * kMaxOut; x += blockDim.x)
    if (outs_s[x] >= 0) atomicOr(&obm[outs_s[x] >> 5], 1u << (outs_s[x] & 31));
  __syncthreads();

  if (warp == NW) {
    // =========================== producer ===========================
    const int RB = a.row_bytes, BR = a.br_row_bytes;
    int pst = 0;           // stage of the next step
    unsigned pph = 0;      // its use parity
    bool pused = false;    // every stage used at least once
    for (long k = 0; k <= K; ++k) {
      if (k > 0) {
        named_bar(2, (NW + 1) * 32);  // sweep k-1 written and fenced (all parts of the tile)
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      const int par = (a.cur + (int)(k & 1)) & 1;
      const size_t tile = DCOPF_TILE;
      const uint8_t *lam_src = reinterpret_cast<const uint8_t *>(par ? a.lam1 : a.lam0) + tile * (size_t)a.n_bus * RB;
      const uint8_t *br_src = reinterpret_cast<const uint8_t *>(par ? a.br1 : a.br0) + tile * (size_t)a.n_brows * BR;
      const uint8_t *d_src = reinterpret_cast<const uint8_t *>(a.d) + tile * (size_t)a.n_bus * RB;
      for (int c = DCOPF_S0; c < DCOPF_S1; ++c) {
        const int st = pst;
        const unsigned pu = pph;  // parity of this use of stage st
        if (++pst == S) {
          pst = 0;
          pph ^= 1u;
        }
        if (pused) mbar_wait(empty_sa + 8 * st, pu ^ 1u);  // previous use of the stage released
        if (pst == 0) pused = true;
        if (lane == 0) {
          mbar_arrive_expect_tx(full_sa + 8 * st, (unsigned)(a.debug_mode == 2 ? a.prog_bytes[c] : a.tx_bytes[c]));
          tma_load_1d(sbase + a.off_prog + st * a.prog_stride, a.prog + a.prog_off[c], (unsigned)a.prog_bytes[c],
                      full_sa + 8 * st);
        }
        __syncwarp();
        // each entry is one bulk copy of `rows` consecutive rows (storage
        // order = load order) into consecutive slots
        const int e1 = (a.debug_mode == 2) ? a.ld_ptr[c] : a.ld_ptr[c + 1];
        for (int e = a.ld_ptr[c] + lane; e < e1; e += 32) {
          const int4 x = a.ld[e];
          if (x.x == LD_LAM)
            tma_load_1d(sbase + a.off_lamp + x.w * RB, lam_src + (size_t)x.y * RB, x.z * RB, full_sa + 8 * st);
          else if (x.x == LD_D)
            tma_load_1d(sbase + a.off_dp + x.w * RB, d_src + (size_t)x.y * RB, x.z * RB, full_sa + 8 * st);
          else
            tma_load_1d(sbase + a.off_brp + x.w * BR, br_src + (size_t)x.y * BR, x.z * BR, full_sa + 8 * st);
#ifndef DCOPF_NO_OPT_L2PF
          if (OPT && k < K && x.x != LD_D) {
            // the optimiser state rows of these multiplier rows (same storage
            // positions) into L2, P steps before their update reads them
            const bool lam = x.x == LD_LAM;
            const size_t rb = lam ? RB : BR, rows = lam ? a.n_bus : a.n_brows;
            const size_t off = (tile * rows + (size_t)x.y) * rb;
            l2_prefetch(reinterpret_cast<const uint8_t *>(lam ? a.s1_lam : a.s1_br) + off, (unsigned)(x.z * rb));
            if (a.opt == 4)
              l2_prefetch(reinterpret_cast<const uint8_t *>(lam ? a.s2_lam : a.s2_br) + off, (unsigned)(x.z * rb));
          }
#endif
        }
      }
    }
    return;
  }

  // =========================== consumers ===========================
  const int RB = a.row_bytes, BR = a.br_row_bytes;
  // lanes past the tile width read the pools' tail padding and never store
  const int lofs = lane * 16;
  const unsigned brp = sbase + a.off_brp + lofs;
  const unsigned lamp = sbase + a.off_lamp + lofs;
  const unsigned dp = sbase + a.off_dp + lofs;
  // optimiser state rows of this tile (OPT kernels): base + the tile offset
  // from shared memory + the lane's 16 bytes, formed at each use
  auto obase = [&](bool lam_side, bool second) -> uint8_t * {
    const double *b = lam_side ? (second ? a.s2_lam : a.s1_lam) : (second ? a.s2_br : a.s1_br);
    return reinterpret_cast<uint8_t *>(const_cast<double *>(b)) + lds_u64(opt_sa + (lam_side ? 0 : 8)) + lofs;
  };
  const bool ost2 = OPT && a.opt == 4;  // Adam: two state arrays
  const unsigned oc_sa = opt_sa + 16 + 64 * warp;  // this warp's step constants
  if (OPT && lane == 0) {
    sts_f64(oc_sa + 32, a.b1t);
    sts_f64(oc_sa + 40, a.b2t);
  }
  const unsigned thp = sbase + a.off_th + V * lane;  // theta*_i code rows
  const unsigned fcp = sbase + a.off_fc + V * lane;  // f*_l code rows (F2)
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
  // (a lane's outage lists: outs_s + inst(q) * kMaxOut, formed at the rare use
  // sites -- outaged branches only -- rather than held in registers)
#define my_outs(q) (outs_s + inst(q) * kMaxOut)
  auto flagged = [&](int l) { return (obm[l >> 5] >> (l & 31)) & 1u; };
  auto out_t = [&](const int *lst, int l) {
    bool r = false;
    for (int j = 0; j < nout; ++j) r |= (lst[j] == l);
    return r;
  };
  // consumer-to-consumer waits: nanosleep back-off in the plain kernels,
  // try_wait with a suspend hint in the optimiser kernels (A/B on config 4 /
  // 4b, K = 100: plain F2 -1% with the suspend, F2 + Adam +1.2%, KVL + Adam
  // +0.4%; profiles/r2/fastdiv/ab_wait)
  auto cwait = [&](unsigned bar, unsigned parity) {
    if constexpr (OPT) mbar_wait(bar, parity);
    else mbar_wait_backoff(bar, parity);
  };
  int cst = 0;         // stage of the next step
  unsigned cph = 0;    // parity of its full barrier

  for (long k = 0; k <= K; ++k) {
    const bool last = (k == K);
    const bool write = EVAL || !last;
    // the launch's final sweep only evaluates g(y_K) (Algorithm 1's value of
    // the last iteration): the work that only forms the gradient
    // -- the f* / theta* sums of phase C, phi of phase B, the whole of phase D
    // (KVL) -- is skipped there (not in EVAL launches, which return it).  Only
    // where it measured faster (A/B against the kernel without it, config 4 /
    // 4b, profiles/r2/tried/final_sweep_gskip*): the plain KVL kernel (+2.2% at
    // the driver's K = 20) and the F2 optimiser kernel (+1.6%); in the plain
    // F2 / F1 kernels the extra branches cost the other sweeps more than the
    // final one saves (F2 -3.5%), KVL + Adam -0.5%, F1 + Adam unchanged
    const bool gskip = ((FORM == kFormKVL && !OPT) || (FORM == kFormF2 && OPT)) && !EVAL && last;
    const int par = (a.cur + (int)(k & 1)) & 1;
    uint8_t *lam_o = reinterpret_cast<uint8_t *>(EVAL ? a.g_lam : (par ? a.lam0 : a.lam1)) +
                     DCOPF_TILE * (size_t)a.n_bus * RB + lofs;
    uint8_t *br_o = reinterpret_cast<uint8_t *>(EVAL ? a.g_br : (par ? a.br0 : a.br1)) +
                    DCOPF_TILE * (size_t)a.n_brows * BR + lofs;
    bool stp[V];
#pragma unroll
    for (int j = 0; j < V; ++j) stp[j] = !EVAL && !last && !frz[inst(j)];
    const double alpha = (EVAL || last) ? 0.0 : a.alpha[k];
    if (OPT && a.opt == 4 && !last && lane == 0) {  // Adam's beta^t, t = steps since the state was reset
      const double b1t = lds_f64(oc_sa + 32) * a.beta1, b2t = lds_f64(oc_sa + 40) * a.beta2;
      const AdamC c = adam_consts(b1t, b2t);
      sts_f64(oc_sa, c.d1);
      sts_f64(oc_sa + 8, c.d2);
      sts_f64(oc_sa + 16, c.r1);
      sts_f64(oc_sa + 24, c.r2);
      sts_f64(oc_sa + 32, b1t);
      sts_f64(oc_sa + 40, b2t);
    }
    if (OPT) __syncwarp();
    // optimiser-variant update of one row of the lane's instances (the state
    // row sits at the same offset of the state arrays); oload issues the
    // state loads at the start of an item so their latency overlaps the item's
    // work, ostep updates and stores them
    auto oload = [&](size_t off, bool lam_side, bool on) -> OState<V> {
      OState<V> o;
#pragma unroll
      for (int j = 0; j < V; ++j) o.s1[j] = o.s2[j] = 0.0;
      if (on) {
        const DV<V> x = ldv<V>(obase(lam_side, false), (int)off, hb);
#pragma unroll
        for (int j = 0; j < V; ++j) o.s1[j] = x.v[j];
        if (ost2) {
          const DV<V> y = ldv<V>(obase(lam_side, true), (int)off, hb);
#pragma unroll
          for (int j = 0; j < V; ++j) o.s2[j] = y.v[j];
        }
      }
      return o;
    };
    // y[j] <- update (only where do_[j]); state stored back
    auto ostep = [&](OState<V> &o, double (&y)[V], const double (&g)[V], size_t off, bool lam_side,
                     const bool (&do_)[V]) {
      AdamC oac = {1.0, 1.0, 1.0, 1.0};
      if (ost2) {
        const double2 c01 = lds_f64x2(oc_sa), c23 = lds_f64x2(oc_sa + 16);
        oac = AdamC{c01.x, c01.y, c23.x, c23.y};
      }
      opt_update_v<V>(a.opt, a.rho, a.beta1, a.beta2, a.eps, y, g, alpha, o.s1, o.s2, oac, do_);
      stv<V>(obase(lam_side, false) + off, o.s1, hb);
      if (ost2) stv<V>(obase(lam_side, true) + off, o.s2, hb);
    };
    // the NEXT item's optimiser state rows into L1 (OPT kernels, F2 / F1): its
    // oload at the item's start then hits L1 instead of waiting the L2 latency
    // (the producer already brought the rows into L2); rec_sa: the record's
    // wpos.  Measured (config 4b, Adam, K = 100, profiles/r2/fastdiv): F2 +1.8%;
    // KVL -7% (its 48-bus steps' prefetches overrun the L1 left beside the
    // 220 KB of shared memory), so KVL does without
    auto opf = [&](unsigned rec_sa, bool lam_side, int rb, bool two) {
#ifndef DCOPF_NO_OPT_L1PF
      if (OPT && FORM != kFormKVL && !EVAL && write && act) {
        const int wpos = (int)lds_u32(rec_sa);
        if (wpos >= 0) {
          const size_t off = (size_t)wpos * rb;
          uint8_t *p1 = obase(lam_side, false) + off;
          prefetch_l1(p1);
          if (V == 4) prefetch_l1(p1 + hb);
          if (two) prefetch_l1(p1 + RB);
          if (ost2) {
            uint8_t *p2 = obase(lam_side, true) + off;
            prefetch_l1(p2);
            if (V == 4) prefetch_l1(p2 + hb);
            if (two) prefetch_l1(p2 + RB);
          }
        }
      }
#endif
    };
    double v[V];
#pragma unroll
    for (int j = 0; j < V; ++j) v[j] = 0.0;

    // the step loop, instantiated twice: CHK = some instance of the tile is
    // frozen (diverged / converged) and its state must be carried over unchanged
    auto run_steps = [&](auto chk_tag) {
    constexpr bool CHK = decltype(chk_tag)::value;
    bool dos[V];  // the step is taken for instance j
#pragma unroll
    for (int j = 0; j < V; ++j) dos[j] = !CHK || stp[j];
    for (int c = DCOPF_S0; c < DCOPF_S1; ++c) {
      const int st = cst;
      mbar_wait(full_sa + 8 * st, cph);
      if (++cst == S) {
        cst = 0;
        cph ^= 1u;
      }
      const unsigned prog = sbase + a.off_prog + st * a.prog_stride;
      const int4 h0 = lds_rec<int4>(prog);       // nA nIA nB nC (KVL: nD nDe nB nC)
      const int4 h2 = lds_rec<int4>(prog + 32);  // offA offIA offB offC
      const int4 h3 = lds_rec<int4>(prog + 48);  // offG offIC bytes PH_PAD (KVL: cycle terms of B)
      const int4 h4 = lds_rec<int4>(prog + 64);  // - - offW -
      // this warp's item ranges of the step's three phases, one 16-byte load
      const uint4 wr = lds_u32x4(prog + h4.z + 16 * warp);
      auto rng0 = [](unsigned x) { return (int)(x & 0xffffu); };
      auto rng1 = [](unsigned x) { return (int)(x >> 16); };
      // (the phase index argument is unused: items come from static LPT ranges;
      // dynamic grabbing by a shared-memory counter was measured 10% slower)
#define ITEM_LOOP(ph, r, n) for (int j = rng0(r), je = rng1(r); j < je; ++j)

      // ---------------- C: ready buses (F2 / F1: C(s-2), warp table 2; KVL: C(s-1), table 1) ----
      auto phaseC = [&](unsigned tr, int ph) {
        const unsigned Cv = prog + h2.w, G = prog + h3.x;
        ITEM_LOOP(ph, tr, h0.w) {
          const RecC r = lds_rec<RecC>(Cv + j * (unsigned)sizeof(RecC));
          if (OPT && j + 1 < je) opf(Cv + (j + 1) * (unsigned)sizeof(RecC), true, RB, false);
          OState<V> ost = oload((size_t)r.wpos * RB, true, OPT && !EVAL && write && act);
          const DV<V> li = ldsv<V>(lamp, r.ls, hb), di = ldsv<V>(dp, r.ds, hb);
          double gl[V];
#pragma unroll
          for (int q = 0; q < V; ++q) gl[q] = -di.v[q];
#pragma unroll 1
          for (int gg = r.g0; gg < r.g1; ++gg) {  // mostly 0 or 1 generator
            const RecG gr = lds_rec<RecG>(G + gg * (unsigned)sizeof(RecG));
#pragma unroll
            if (gr.a > 0.0) {  // (warp-uniform: one generator record per warp)
#pragma unroll
              for (int q = 0; q < V; ++q) {
                const double rr = gr.c + li.v[q];
                const double x = -rr / (2.0 * gr.a);
                const double p = sel(x < gr.lo, gr.lo, sel(x > gr.hi, gr.hi, x));  // clip(-r / (2a), lo, hi)
                gl[q] = gl[q] + p;
                v[q] += gr.a * p * p + rr * p;
              }
            } else {
              const double mid = 0.5 * (gr.lo + gr.hi);
#pragma unroll
              for (int q = 0; q < V; ++q) {
                const double rr = gr.c + li.v[q];
                const double p = sel(rr > 0.0, gr.lo, sel(rr < 0.0, gr.hi, mid));  // bound selection, tie -> midpoint
                gl[q] = gl[q] + p;
                v[q] += rr * p;
              }
            }
          }
          if (gskip) {
            // (value only: the incidence sums feed the gradient alone)
          } else if (FORM != kFormF1) {
            const unsigned IC = prog + h3.y + r.e0 * (unsigned)sizeof(RecIC2);
            const int n = r.e1 - r.e0;
            auto acc = [&](const RecIC2 &x) {
              const DV<V> f = ld_code<V>(fcp, x.f, x.sF);  // +-f* (c * (+-F) == +-(c * F) exactly)
#pragma unroll
              for (int q = 0; q < V; ++q) gl[q] = gl[q] + f.v[q];  // +f* at the to bus, -f* at the from bus
            };
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (e < n) acc(lds_rec<RecIC2>(IC + e * (unsigned)sizeof(RecIC2)));
#pragma unroll 1
            for (int e = 4; e < n; ++e) acc(lds_rec<RecIC2>(IC + e * (unsigned)sizeof(RecIC2)));
          } else {
            const unsigned IC = prog + h3.y;
#pragma unroll 1
            for (int e = r.e0; e < r.e1; ++e) {
              const RecIC1 x = lds_rec<RecIC1>(IC + e * (unsigned)sizeof(RecIC1));
              double sb[V];
#pragma unroll
              for (int q = 0; q < V; ++q) sb[q] = x.sb;
              if (x.br >= 0 && flagged(x.br)) {
#pragma unroll
                for (int q = 0; q < V; ++q)
                  if (out_t(my_outs(q), x.br)) sb[q] = copysign(0.0, sb[q]);
              }
              const DV<V> ts = ld_code<V>(thp, x.ts, x.ths), tt = ld_code<V>(thp, x.tt, x.tht);
#pragma unroll
              for (int q = 0; q < V; ++q) gl[q] = gl[q] + sb[q] * (ts.v[q] - tt.v[q]);
            }
          }
#pragma unroll
          for (int q = 0; q < V; ++q) v[q] += -(li.v[q] * di.v[q]);
          if (write && act) {
            uint8_t *dst = lam_o + (size_t)r.wpos * RB;
            if (EVAL) {
              stv<V>(dst, gl, hb);
            } else if constexpr (OPT) {
              double y[V];
#pragma unroll
              for (int q = 0; q < V; ++q) y[q] = li.v[q];
              ostep(ost, y, gl, (size_t)r.wpos * RB, true, dos);
              stv<V>(dst, y, hb);
            } else {
              double y[V];
#pragma unroll
              for (int q = 0; q < V; ++q) y[q] = dos[q] ? li.v[q] + alpha * gl[q] : li.v[q];
              stv<V>(dst, y, hb);
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
        const unsigned Bv = prog + h2.z, BKe = prog + h3.w;
        auto bkitem = [&](const RecBK &r, auto out_tag) {
          constexpr bool OUT = decltype(out_tag)::value;
          double x[V], F[V];
          bool o[V];
#pragma unroll
          for (int q = 0; q < V; ++q) {
            x[q] = r.x;
            F[q] = r.F;
            o[q] = false;
          }
          if constexpr (OUT) {  // an outaged lane: b = F = 0
#pragma unroll
            for (int q = 0; q < V; ++q) {
              o[q] = out_t(my_outs(q), r.obr);
              if (o[q]) x[q] = F[q] = 0.0;
            }
          }
          double s[V];  // cycles in ascending k (the oracle's order)
#pragma unroll
          for (int q = 0; q < V; ++q) s[q] = 0.0;
#pragma unroll 1
          for (int e = r.e0; e < r.e1; ++e) {
            const RecBKe t = lds_rec<RecBKe>(BKe + e * (unsigned)sizeof(RecBKe));
            const DV<V> kv = ldsv<V>(brp, t.ks, hb);
#pragma unroll
            for (int q = 0; q < V; ++q) s[q] = (t.sgn > 0) ? s[q] + kv.v[q] : s[q] - kv.v[q];
          }
          const DV<V> ls = ldsv<V>(lamp, r.ls, hb), lt = ldsv<V>(lamp, r.lt, hb);
          int cd[V];
#pragma unroll
          for (int q = 0; q < V; ++q) {
            const double qq = x[q] * s[q] - (ls.v[q] - lt.v[q]);
            int c;
            const double f = flow_min(qq, F[q], -F[q], c);  // -F if q > 0, +F if q < 0, 0 on a tie
            cd[q] = (OUT && o[q]) ? 0 : c;
            if (!r.halo) v[q] += qq * f;
          }
          if (act) st_codes<V>(fcp + r.fs, cd);
        };
        ITEM_LOOP(0, wr.x, h0.z) {
          const RecBK r = lds_rec<RecBK>(Bv + j * (unsigned)sizeof(RecBK));
          if (r.obr >= 0 && flagged(r.obr)) bkitem(r, std::integral_constant<bool, true>{});
          else bkitem(r, std::integral_constant<bool, false>{});
        }
      }
      if (SOFT) {  // C and D read the f* codes of B(<= s-1)
        mbar_arrive(bdone_sa + 8 * (gs & 3));
        if (gs > 0) cwait(bdone_sa + 8 * ((gs - 1) & 3), ((gs - 1) >> 2) & 1u);
      }
      phaseC(wr.y, 1);
      // ---------------- D(s-1): d/dkappa_k = sum_l C_kl x_l f*_l, kappa' ----------------
      if (!gskip) {  // (gradient and step only)
        const unsigned Dv = prog + h2.x, De = prog + h2.y;
        ITEM_LOOP(2, wr.z, h0.x) {
          const RecD r = lds_rec<RecD>(Dv + j * (unsigned)sizeof(RecD));
          if (OPT && j + 1 < je) opf(Dv + (j + 1) * (unsigned)sizeof(RecD) + 4, false, BR, false);
          OState<V> ost = oload((size_t)r.wpos * BR, false, OPT && !EVAL && write && act);
          const DV<V> kv = ldsv<V>(brp, r.ks, hb);
          double acc[V];
#pragma unroll
          for (int q = 0; q < V; ++q) acc[q] = 0.0;
#pragma unroll 1
          for (int e = r.e0; e < r.e1; ++e) {
            const RecDe d = lds_rec<RecDe>(De + e * (unsigned)sizeof(RecDe));
            int cd[V];
            ld_codes<V>(fcp, d.fs, cd);
            // index 0 / 1 / 2 for code -1 / 0 / +1 (lanes past the tile width read
            // padding bytes: clamp so they never index outside the record)
#pragma unroll
            for (int q = 0; q < V; ++q) {
              const int i = (cd[q] > 0) ? 2 : ((cd[q] < 0) ? 0 : 1);
              acc[q] = acc[q] + d.t[i];  // (c F) sx: the oracle's C_kl (f*_l x_l), exact
            }
          }
          if (r.dbr >= 0 && flagged(r.dbr)) {  // defining branch out: no cycle, gradient 0
#pragma unroll
            for (int q = 0; q < V; ++q)
              if (out_t(my_outs(q), r.dbr)) acc[q] = 0.0;
          }
          if (write && act) {
            uint8_t *dst = br_o + (size_t)r.wpos * BR;
            if (EVAL) {
              stv<V>(dst, acc, hb);
            } else if constexpr (OPT) {
              double y[V];
#pragma unroll
              for (int q = 0; q < V; ++q) y[q] = kv.v[q];
              ostep(ost, y, acc, (size_t)r.wpos * BR, false, dos);
              stv<V>(dst, y, hb);
            } else {
              double y[V];
#pragma unroll
              for (int q = 0; q < V; ++q) y[q] = dos[q] ? kv.v[q] + alpha * acc[q] : kv.v[q];
              stv<V>(dst, y, hb);
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
        const unsigned A = prog + h2.x;
        ITEM_LOOP(0, wr.x, h0.x) {
          const RecA ra = lds_rec<RecA>(A + j * (unsigned)sizeof(RecA));
          double w[V];
#pragma unroll
          for (int q = 0; q < V; ++q) w[q] = 0.0;
          if (FORM == kFormF2) {
            // incidence entries in ascending original branch id (the oracle's
            // order); degree <= 4 for ~97% of buses: a fixed 4-way body with
            // warp-uniform guards instead of a counted loop, the rest in a tail
            const unsigned IA = prog + h2.y + ra.e0 * (unsigned)sizeof(RecIA2);
            const int n = ra.e1 - ra.e0;
            auto acc = [&](const RecIA2 &r) {
              const DV<V> nu = ldsv<V>(brp, r.row, hb);
#pragma unroll
              for (int q = 0; q < V; ++q) w[q] = w[q] + r.sb * nu.v[q];  // w_s += -(b nu), w_t += b nu (outaged: nu == 0)
            };
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (e < n) acc(lds_rec<RecIA2>(IA + e * (unsigned)sizeof(RecIA2)));
#pragma unroll 1
            for (int e = 4; e < n; ++e) acc(lds_rec<RecIA2>(IA + e * (unsigned)sizeof(RecIA2)));
          } else {
            const unsigned IA = prog + h2.y;
#pragma unroll 1
            for (int e = ra.e0; e < ra.e1; ++e) {
              const RecIA1 r = lds_rec<RecIA1>(IA + e * (unsigned)sizeof(RecIA1));
              double sb[V];
#pragma unroll
              for (int q = 0; q < V; ++q) sb[q] = r.sb;
              if (r.br >= 0 && flagged(r.br)) {  // br < 0: branch never taken out
#pragma unroll
                for (int q = 0; q < V; ++q)
                  if (out_t(my_outs(q), r.br)) sb[q] = copysign(0.0, sb[q]);
              }
              const DV<V> mp = ldsv<V>(brp, r.row, hb), mm = ldsv<V>(brp, r.row + RB, hb);
              const DV<V> ls = ldsv<V>(lamp, r.ls, hb), lt = ldsv<V>(lamp, r.lt, hb);
#pragma unroll
              for (int q = 0; q < V; ++q)
                w[q] = w[q] + sb[q] * ((mp.v[q] - mm.v[q]) - (ls.v[q] - lt.v[q]));  // w_s += u, w_t -= u
            }
          }
          // theta* = -Theta if w > 0, +Theta if w < 0, 0 on a tie and at the reference bus
          int cd[V];
          if (ra.flags & kAFlagRef) {  // (warp-uniform)
#pragma unroll
            for (int q = 0; q < V; ++q) cd[q] = 0;
          } else {
            const bool val = !(ra.flags & kAFlagHalo);  // a halo bus: code only
            const double nth = -ra.theta;
#pragma unroll
            for (int q = 0; q < V; ++q) {
              const double t = flow_min(w[q], ra.theta, nth, cd[q]);
              if (val) v[q] += w[q] * t;
            }
          }
          if (act) st_codes<V>(thp + ra.th, cd);
        }
      }
      if (SOFT) {  // B(s-1) reads the theta* codes of A(<= s-1); the f* slots it writes
        // were last read 2+ steps ago, and A-done(s-1) implies every warp finished step s-2
        mbar_arrive(adone_sa + 8 * (gs & 3));
        if (gs > 0) cwait(adone_sa + 8 * ((gs - 1) & 3), ((gs - 1) >> 2) & 1u);
      }
      // ---------------- B(s-1): branches ----------------
      {
        const unsigned Bv = prog + h2.z;
        // one branch; OUT: some instance of the tile has it out (per-lane b = F
        // = 0), else the warp-uniform fast path with no per-lane outage state
        auto bitem = [&](const RecB &r, auto out_tag) {
          constexpr bool OUT = decltype(out_tag)::value;
          double b[V], F[V];
          bool o[V];
#pragma unroll
          for (int q = 0; q < V; ++q) {
            b[q] = r.b;
            F[q] = r.F;
            o[q] = false;
          }
          if constexpr (OUT) {
#pragma unroll
            for (int q = 0; q < V; ++q) {
              o[q] = out_t(my_outs(q), r.obr);
              if (o[q]) b[q] = F[q] = 0.0;
            }
          }
          if (FORM == kFormF2 && r.wpos < 0) {
            // lite halo branch (split tiles): its f* code for this part's C items
            const DV<V> nu = ldsv<V>(brp, r.row, hb), ls = ldsv<V>(lamp, r.ls, hb), lt = ldsv<V>(lamp, r.lt, hb);
            int cd[V];
#pragma unroll
            for (int q = 0; q < V; ++q) {
              const double qq = nu.v[q] - (ls.v[q] - lt.v[q]);
              cd[q] = o[q] ? 0 : code_of(qq < 0.0, qq > 0.0);
            }
            if (act) st_codes<V>(fcp + r.fs, cd);
            return;
          }
          OState<V> ost = oload((size_t)r.wpos * BR, false, OPT && !EVAL && write && act);
          OState<V> ost_m = oload((size_t)r.wpos * BR + RB, false, FORM == kFormF1 && OPT && !EVAL && write && act);
          double phi[V];  // (the gradient's flow term; not needed by the final sweep's value)
          if (gskip) {
#pragma unroll
            for (int q = 0; q < V; ++q) phi[q] = 0.0;
          } else {
            const DV<V> ths = ld_code<V>(thp, r.ts, r.ths), tht = ld_code<V>(thp, r.tt, r.tht);
#pragma unroll
            for (int q = 0; q < V; ++q) phi[q] = b[q] * (ths.v[q] - tht.v[q]);
          }
          uint8_t *dst = br_o + (size_t)r.wpos * BR;
          if (FORM == kFormF2) {
            const DV<V> nu = ldsv<V>(brp, r.row, hb), ls = ldsv<V>(lamp, r.ls, hb), lt = ldsv<V>(lamp, r.lt, hb);
            double g[V];
            int cd[V];
#pragma unroll
            for (int q = 0; q < V; ++q) {
              const double qq = nu.v[q] - (ls.v[q] - lt.v[q]);
              // f* = -F if q > 0, +F if q < 0, 0 on a tie (an outaged lane has F = 0);
              // code for C (an outaged lane stores the tie: its f* = +-0)
              int c;
              const double f = flow_min(qq, F[q], -F[q], c);
              cd[q] = (OUT && o[q]) ? 0 : c;
              g[q] = f - phi[q];  // Kirchhoff residual
              v[q] += qq * f;
            }
            if (act) st_codes<V>(fcp + r.fs, cd);
            if (write && act) {
              if (EVAL) {
                stv<V>(dst, g, hb);
              } else if constexpr (OPT) {
                double y[V];
#pragma unroll
                for (int q = 0; q < V; ++q) y[q] = nu.v[q];
                ostep(ost, y, g, (size_t)r.wpos * BR, false, dos);
                stv<V>(dst, y, hb);
              } else {
                double y[V];
#pragma unroll
                for (int q = 0; q < V; ++q) y[q] = dos[q] ? nu.v[q] + alpha * g[q] : nu.v[q];
                stv<V>(dst, y, hb);
              }
            }
          } else {
            const DV<V> mp = ldsv<V>(brp, r.row, hb), mm = ldsv<V>(brp, r.row + RB, hb);
            double gp[V], gm[V];
#pragma unroll
            for (int q = 0; q < V; ++q) {
              gp[q] = phi[q] - F[q];
              gm[q] = -phi[q] - F[q];
              v[q] += -(F[q] * (mp.v[q] + mm.v[q]));
            }
            if (write && act) {
              uint8_t *dst2 = br_o + (size_t)r.wpos * BR + RB;
              if (EVAL) {
                stv<V>(dst, gp, hb);
                stv<V>(dst2, gm, hb);
              } else {
                double pp[V], mq[V];
#pragma unroll
                for (int q = 0; q < V; ++q) {
                  pp[q] = mp.v[q];
                  mq[q] = mm.v[q];
                }
                if constexpr (OPT) {
                  double yp[V], ym[V];
#pragma unroll
                  for (int q = 0; q < V; ++q) {
                    yp[q] = mp.v[q];
                    ym[q] = mm.v[q];
                  }
                  ostep(ost, yp, gp, (size_t)r.wpos * BR, false, dos);
                  ostep(ost_m, ym, gm, (size_t)r.wpos * BR + RB, false, dos);
#pragma unroll
                  for (int q = 0; q < V; ++q)
                    if (dos[q]) {
                      pp[q] = sel(yp[q] > 0.0, yp[q], 0.0);  // mu <- max(mu, 0)
                      mq[q] = sel(ym[q] > 0.0, ym[q], 0.0);
                    }
                } else {
#pragma unroll
                  for (int q = 0; q < V; ++q)
                    if (dos[q]) {
                      const double p0 = mp.v[q] + alpha * gp[q], m0 = mm.v[q] + alpha * gm[q];
                      pp[q] = sel(p0 > 0.0, p0, 0.0);  // mu <- max(mu, 0)
                      mq[q] = sel(m0 > 0.0, m0, 0.0);
                    }
                }
                stv<V>(dst, pp, hb);
                stv<V>(dst2, mq, hb);
              }
            }
          }
        };
        ITEM_LOOP(1, wr.y, h0.z) {
          const RecB r = lds_rec<RecB>(Bv + j * (unsigned)sizeof(RecB));
          if (OPT && j + 1 < je) opf(Bv + (j + 1) * (unsigned)sizeof(RecB) + 24, false, BR, FORM == kFormF1);
          if (r.obr >= 0 && flagged(r.obr)) bitem(r, std::integral_constant<bool, true>{});  // (obr < 0: never out)
          else bitem(r, std::integral_constant<bool, false>{});
        }
      }
      if (SOFT) {
        mbar_arrive(bdone_sa + 8 * (gs & 3));
        if (gs > 0) cwait(bdone_sa + 8 * ((gs - 1) & 3), ((gs - 1) >> 2) & 1u);
      }
      phaseC(wr.z, 2);
      }  // debug_mode
      }  // FORM
      if (SOFT) {
        mbar_arrive(empty_sa + 8 * st);
      } else {  // lock-step mode: every warp finished the step
        named_bar(1, CT);
        if (threadIdx.x == 0) mbar_arrive(empty_sa + 8 * st);
      }
      ++gs;
    }
    };
    bool anyf_l = false;
#pragma unroll
    for (int j = 0; j < V; ++j) anyf_l |= frz[inst(j)] != 0;
    const bool anyf = __any_sync(0xffffffffu, anyf_l);
    if (anyf) run_steps(std::integral_constant<bool, true>{});
    else run_steps(std::integral_constant<bool, false>{});
    // ---------------- dual value, best, status ----------------
    named_bar(1, CT);  // every warp is past the sweep's last step: the pools red aliases are dead
#pragma unroll
    for (int j = 0; j < V; ++j) red[warp * TS + inst(j)] = v[j];
    named_bar(1, CT);
    double g[V];
    const int part = DCOPF_PART;
    const size_t tile = DCOPF_TILE;
    const long ib = (long)tile * W;
    if (warp == 0 && act) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        double s = 0.0;
        for (int w = 0; w < NW; ++w) s += red[w * TS + inst(j)];
        g[j] = s;
        if (C > 1) a.part_val[((size_t)((k & 1) * a.tiles + tile) * C + part) * W + inst(j)] = s;
      }
    }
    if (!last || C > 1) __threadfence();  // y_{k+1} rows (and the partials) visible device-wide
    if (!last) asm volatile("fence.proxy.async.global;" ::: "memory");  // ... and to the TMA copies of sweep k+1
    if (C > 1) {
      // the tile's parts meet: arrive (release) and wait for all C (acquire)
      named_bar(1, CT);
      if (threadIdx.x == 0) {
        atomicAdd(&a.tile_sync[tile], 1u);
        const unsigned want = (unsigned)C * (unsigned)(k + 1);
        while (ld_acquire_gpu(&a.tile_sync[tile]) < want) __nanosleep(64);
      }
      named_bar(1, CT);
      if (warp == 0 && act) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
          double s = 0.0;  // the parts' partials in part order: the same sum on every part
          for (int p = 0; p < C; ++p) s += __ldcg(&a.part_val[((size_t)((k & 1) * a.tiles + tile) * C + p) * W + inst(j)]);
          g[j] = s;
        }
      }
    }
    if (warp == 0 && act) {
      const bool out = part == 0;  // every part takes the same decisions; part 0 writes the outputs
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int t = inst(j);
        const long bi = ib + t;
        if (EVAL) {
          if (out) a.out_val[bi] = g[j];
        } else {
          if (out && !last && a.hist && bi < a.B) a.hist[(size_t)k * a.B + bi] = g[j];
          if (out && last) a.bound[bi] = g[j];
          double best = bst[t];
          // (stopping rule: |g_k - g_{k-1}| < tol within this call; status 2)
          const bool chk = a.tol > 0.0 && k > 0;
          if (!frz[t]) {
            if (valid_bound(g[j])) {
              best = (g[j] > best) ? g[j] : best;
              if (chk && fabs(g[j] - gpv[t]) < a.tol) frz[t] = 2;
            } else {
              frz[t] = 1;
            }
          }
          bst[t] = best;
          gpv[t] = g[j];
          // time to gap: first evaluation whose running best reaches the target
          // (state kept in global memory, touched once per sweep: no registers held)
          if (out && a.target && a.hit[bi] < 0 && best >= a.target[bi]) a.hit[bi] = a.k_base + k;
        }
      }
    }
    if (!last) named_bar(2, (NW + 1) * 32);  // the producer may start sweep k+1
    else named_bar(1, CT);
  }
  if (!EVAL && warp == 0 && act && DCOPF_PART == 0) {
    const long ib = (long)DCOPF_TILE * W;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      a.best[ib + inst(j)] = bst[inst(j)];
      a.status[ib + inst(j)] = frz[inst(j)];
    }
  }
}

#undef my_outs
#undef ITEM_LOOP
#undef DCOPF_S0
#undef DCOPF_S1
#undef DCOPF_PART
#undef DCOPF_TILE

}  // namespace dcopf
