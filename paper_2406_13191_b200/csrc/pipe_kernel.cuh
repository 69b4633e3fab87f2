// pipe_kernel.cuh -- the batched path: a persistent, warp-specialised,
// TMA-fed sweep kernel for sm_100a.
//
// One CTA owns one 32-instance tile (lane = instance) for all K iterations of
// a dcopf_dual_iterate() call (instances never interact: no grid sync, one
// launch per call).  Each iteration is one sweep over the chunks of a
// host-compiled schedule (schedule.h):
//
//   producer warp (warp NW):  for chunk j, once chunk j-S has been consumed
//     (empty[j%S] mbarrier), arm full[j%S] with the chunk's byte count and
//     issue cp.async.bulk (TMA 1-D bulk copies) for (a) the chunk's program
//     block and (b) every state row (lambda, d, nu / mu pair) whose first use
//     is chunk j, into its interval-coloured shared-memory slot.
//   consumer warps (0..NW-1): wait full[j%S]; then from shared memory only
//     A  buses of the chunk:  w_i = gather over the incidence, theta* codes
//     B  branches whose larger endpoint is in the chunk: q_l, f* codes, phi_l,
//        Kirchhoff (F2) / limit (F1) residual, nu' / mu' stored to HBM
//     C  buses whose last neighbour is in the chunk: generators, d/dlambda,
//        lambda' stored to HBM
//   with a named barrier (consumers only) after each phase, then release
//   empty[j%S].
//
// Every HBM byte of the iteration is read once (TMA) and written once
// (coalesced 256 B row stores), i.e. the traffic is the algorithmic
// 8 (3 n_b + 2 n_l) B per instance-iteration (F2); the re-reads of the
// method (nu at both endpoints and at the branch, lambda at every incident
// branch and at the bus) are served from shared memory.  Between sweeps the
// pipeline drains: y_{k+1} rows written in sweep k are read by TMA in sweep
// k+1, so every writer fences (generic -> async proxy) before the producer
// restarts.
//
// Per-entity arithmetic and its operation order are those of
// dual_kernels.cuh and of the oracle (reading A-19); only the dual value is
// summed in a different (fixed) order.
#pragma once
#include "dual_kernels.cuh"
#include "schedule.h"

namespace dcopf {

struct PipeArgs {
  double *lam0, *lam1, *br0, *br1;  // ping-pong state (tile-major)
  const double *d;
  const int *outs;
  int max_out;
  int cur;
  const double *alpha;              // [K] device
  long K;
  double *bound, *best;
  int *status;
  double *hist;
  long B;
  int n_bus, n_br, ref;
  // schedule
  const uint8_t *prog;              // program blocks
  const long long *prog_off;        // [nch]
  const int *prog_bytes, *tx_bytes; // [nch]
  const int *ld_ptr, *ld_ent, *ld_slot;
  int nch, S;
  int off_bar, off_red, off_frz, off_prog, prog_stride, off_brp, off_lamp, off_dp, off_th, off_fc;
  volatile int *dbg;                // debug progress (mapped host memory) or null
};

__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
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
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
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

template <typename T>
__device__ __forceinline__ const T *sec(const uint8_t *prog, int field) {
  return reinterpret_cast<const T *>(prog + reinterpret_cast<const int *>(prog)[field]);
}

template <int FORM, int NW>
__global__ void __launch_bounds__((NW + 1) * 32, 2) k_pipe(const PipeArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + a.off_bar);
  uint64_t *empty = full + a.S;
  double *red = reinterpret_cast<double *>(smem + a.off_red);
  int *frz = reinterpret_cast<int *>(smem + a.off_frz);
  constexpr int BRW = (FORM == kFormF2) ? 1 : 2;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t tile = blockIdx.x;
  const long b = (long)tile * kTile + lane;
  const int nch = a.nch, S = a.S;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) frz[lane] = a.status[b];
  __syncthreads();

  if (warp == NW) {
    // =========================== producer ===========================
    for (long k = 0; k <= a.K; ++k) {
      if (k > 0) named_bar(2, (NW + 1) * 32);  // sweep k-1 fully written and fenced
      const int par = (a.cur + (int)(k & 1)) & 1;
      const uint8_t *lam_src = reinterpret_cast<const uint8_t *>((par ? a.lam1 : a.lam0) + tile * (size_t)a.n_bus * kTile);
      const uint8_t *br_src = reinterpret_cast<const uint8_t *>((par ? a.br1 : a.br0) + tile * (size_t)a.n_br * BRW * kTile);
      const uint8_t *d_src = reinterpret_cast<const uint8_t *>(a.d + tile * (size_t)a.n_bus * kTile);
      for (int c = 0; c < nch; ++c) {
        const long g = k * nch + c;
        const int st = (int)(g % S);
        const long u = g / S;
        if (a.dbg && lane == 0 && tile == 0) a.dbg[0] = (int)(2 * g);
        if (u > 0) mbar_wait(&empty[st], (unsigned)((u - 1) & 1));
        if (a.dbg && lane == 0 && tile == 0) a.dbg[0] = (int)(2 * g + 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[st], (unsigned)a.tx_bytes[c]);
          tma_load_1d(smem + a.off_prog + st * a.prog_stride, a.prog + a.prog_off[c], (unsigned)a.prog_bytes[c],
                      &full[st]);
        }
        __syncwarp();
        if (a.dbg && lane == 0 && tile == 0) a.dbg[9] = (int)(g);
        const int e0 = a.ld_ptr[c], e1 = a.ld_ptr[c + 1];
        for (int e = e0 + lane; e < e1; e += 32) {
          const int x = a.ld_ent[e], slot = a.ld_slot[e];
          const int kind = (int)((unsigned)x >> 30), ent = x & 0x3fffffff;
          if (kind == LD_LAM)
            tma_load_1d(smem + a.off_lamp + slot * 256, lam_src + (size_t)ent * 256, 256, &full[st]);
          else if (kind == LD_D)
            tma_load_1d(smem + a.off_dp + slot * 256, d_src + (size_t)ent * 256, 256, &full[st]);
          else
            tma_load_1d(smem + a.off_brp + slot * 256 * BRW, br_src + (size_t)ent * 256 * BRW, 256 * BRW, &full[st]);
        }
      }
    }
    return;
  }

  // =========================== consumers ===========================
  const double *brp = reinterpret_cast<const double *>(smem + a.off_brp) + lane;
  const double *lamp = reinterpret_cast<const double *>(smem + a.off_lamp) + lane;
  const double *dp = reinterpret_cast<const double *>(smem + a.off_dp) + lane;
  uint2 *th = reinterpret_cast<uint2 *>(smem + a.off_th);
  uint2 *fc = reinterpret_cast<uint2 *>(smem + a.off_fc);
  int o[kMaxOut];
  const int nout = a.max_out;
#pragma unroll
  for (int j = 0; j < kMaxOut; ++j) o[j] = (j < nout) ? a.outs[b * nout + j] : -1;
  double best = a.best[b];
  constexpr int CT = NW * 32;

  for (long k = 0; k <= a.K; ++k) {
    const bool last = (k == a.K);
    const int par = (a.cur + (int)(k & 1)) & 1;
    double *__restrict__ lam_o = (par ? a.lam0 : a.lam1) + tile * (size_t)a.n_bus * kTile + lane;
    double *__restrict__ br_o = (par ? a.br0 : a.br1) + tile * (size_t)a.n_br * BRW * kTile + lane;
    const bool frozen = frz[lane] != 0;
    const bool step = !last && !frozen;
    const double alpha = last ? 0.0 : a.alpha[k];
    double val = 0.0;

    for (int c = 0; c < nch; ++c) {
      const long g = k * nch + c;
      const int st = (int)(g % S);
      if (a.dbg && lane == 0 && tile == 0) a.dbg[1 + warp] = (int)(4 * g);
      if (a.dbg) {
        long spins = 0;
        unsigned done = 0;
        do {
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
              "selp.u32 %0, 1, 0, p;\n\t}"
              : "=r"(done)
              : "r"(smem_u32(&full[st])), "r"((unsigned)((g / S) & 1))
              : "memory");
          if (++spins == 2000000 && lane == 0 && warp == 0 && tile == 0) {
            const unsigned long long raw = *reinterpret_cast<volatile unsigned long long *>(&full[st]);
            a.dbg[10] = (int)(raw & 0xffffffffu);
            a.dbg[11] = (int)(raw >> 32);
            a.dbg[12] = st;
            a.dbg[13] = a.tx_bytes[c];
            a.dbg[14] = a.prog_bytes[c];
            a.dbg[15] = a.ld_ptr[c + 1] - a.ld_ptr[c];
          }
        } while (!done);
      }
      mbar_wait(&full[st], (unsigned)((g / S) & 1));
      if (a.dbg && lane == 0 && tile == 0) a.dbg[1 + warp] = (int)(4 * g + 1);
      const uint8_t *prog = smem + a.off_prog + st * a.prog_stride;
      const int *hd = reinterpret_cast<const int *>(prog);

      // ---------------- A: w_i, theta* codes ----------------
      {
        const int nA = hd[PH_NA], a0 = hd[PH_A0];
        const int *A_ptr = sec<int>(prog, PH_A_PTR), *A_ths = sec<int>(prog, PH_A_THS);
        const double *A_th = sec<double>(prog, PH_A_TH);
        const int *IA_row = sec<int>(prog, PH_IA_ROW), *IA_br = sec<int>(prog, PH_IA_BR);
        const double *IA_b = sec<double>(prog, PH_IA_B);
        const int *IA_ls = sec<int>(prog, PH_IA_LS), *IA_lt = sec<int>(prog, PH_IA_LT);
        for (int j = warp; j < nA; j += NW) {
          const int bus = a0 + j;
          double w = 0.0;
          const int e1 = A_ptr[j + 1];
          for (int e = A_ptr[j]; e < e1; ++e) {
            const unsigned code = (unsigned)IA_row[e];
            const int slot = (int)(code & 0x7fffffffu);
            const bool to = code >> 31;
            const double bl = is_out(o, nout, IA_br[e]) ? 0.0 : IA_b[e];
            if (FORM == kFormF2) {
              const double t = bl * brp[slot * 32];
              w = to ? w + t : w + (-t);
            } else {
              const double u = bl * ((brp[slot * 64] - brp[slot * 64 + 32]) - (lamp[IA_ls[e] * 32] - lamp[IA_lt[e] * 32]));
              w = to ? w - u : w + u;
            }
          }
          const bool notref = (bus != a.ref);
          const bool pos = notref && (w < 0.0), neg = notref && (w > 0.0);
          const unsigned mp = __ballot_sync(0xffffffffu, pos), mn = __ballot_sync(0xffffffffu, neg);
          if (lane == 0) th[A_ths[j]] = make_uint2(mp, mn);
          const double tv = A_th[j];
          if (notref) val += w * (pos ? tv : (neg ? -tv : 0.0));
        }
      }
      if (a.dbg && lane == 0 && tile == 0) a.dbg[1 + warp] = (int)(4 * g + 2);
      named_bar(1, CT);
      // ---------------- B: branches ----------------
      {
        const int nB = hd[PH_NB], b0 = hd[PH_B0];
        const int *B_row = sec<int>(prog, PH_B_ROW), *B_ts = sec<int>(prog, PH_B_TS), *B_tt = sec<int>(prog, PH_B_TT);
        const double *B_b = sec<double>(prog, PH_B_B), *B_F = sec<double>(prog, PH_B_F);
        const double *B_Ts = sec<double>(prog, PH_B_THS), *B_Tt = sec<double>(prog, PH_B_THT);
        const int *B_ls = sec<int>(prog, PH_B_LS), *B_lt = sec<int>(prog, PH_B_LT), *B_fs = sec<int>(prog, PH_B_FS);
        for (int j = warp; j < nB; j += NW) {
          const int l = b0 + j;
          const bool out = is_out(o, nout, l);
          const double bl = out ? 0.0 : B_b[j];
          const double Fl = out ? 0.0 : B_F[j];
          const double ths = decode(th[B_ts[j]], lane, B_Ts[j]);
          const double tht = decode(th[B_tt[j]], lane, B_Tt[j]);
          const double phi = bl * (ths - tht);
          const int row = B_row[j];
          if (FORM == kFormF2) {
            const double nu = brp[row * 32];
            const double q = nu - (lamp[B_ls[j] * 32] - lamp[B_lt[j] * 32]);
            const bool fneg = q > 0.0, fpos = q < 0.0;
            const unsigned mp = __ballot_sync(0xffffffffu, fpos), mn = __ballot_sync(0xffffffffu, fneg);
            if (lane == 0) fc[B_fs[j]] = make_uint2(mp, mn);
            const double f = fneg ? -Fl : (fpos ? Fl : 0.0);
            const double gv = f - phi;
            val += q * f;
            if (!last) br_o[(size_t)l * kTile] = step ? nu + alpha * gv : nu;
          } else {
            const double mp = brp[row * 64], mm = brp[row * 64 + 32];
            const double gp = phi - Fl, gm = -phi - Fl;
            val += -(Fl * (mp + mm));
            if (!last) {
              double vp = mp, vm = mm;
              if (step) {
                vp = mp + alpha * gp;
                vm = mm + alpha * gm;
                vp = (vp > 0.0) ? vp : 0.0;
                vm = (vm > 0.0) ? vm : 0.0;
              }
              br_o[(size_t)(2 * l) * kTile] = vp;
              br_o[(size_t)(2 * l + 1) * kTile] = vm;
            }
          }
        }
      }
      named_bar(1, CT);
      // ---------------- C: ready buses ----------------
      {
        const int nC = hd[PH_NC];
        const int *C_bus = sec<int>(prog, PH_C_BUS), *C_ls = sec<int>(prog, PH_C_LS), *C_ds = sec<int>(prog, PH_C_DS);
        const int *C_gp = sec<int>(prog, PH_C_GP), *C_ip = sec<int>(prog, PH_C_IP);
        const double *G_c = sec<double>(prog, PH_G_C), *G_lo = sec<double>(prog, PH_G_LO);
        const double *G_hi = sec<double>(prog, PH_G_HI), *G_a = sec<double>(prog, PH_G_A);
        const int *IC_a = sec<int>(prog, PH_IC_A), *IC_br = sec<int>(prog, PH_IC_BR), *IC_tt = sec<int>(prog, PH_IC_TT);
        const double *IC_x = sec<double>(prog, PH_IC_X), *IC_Ts = sec<double>(prog, PH_IC_THS),
                     *IC_Tt = sec<double>(prog, PH_IC_THT);
        for (int j = warp; j < nC; j += NW) {
          const int i = C_bus[j];
          const double li = lamp[C_ls[j] * 32];
          const double di = dp[C_ds[j] * 32];
          double gl = -di;
          const int g1 = C_gp[j + 1];
          for (int gg = C_gp[j]; gg < g1; ++gg) {
            const double r = G_c[gg] + li;
            const double ag = G_a[gg];
            const double p = gen_minimiser(r, G_lo[gg], G_hi[gg], ag);
            gl = gl + p;
            val += (ag > 0.0) ? ag * p * p + r * p : r * p;
          }
          const int e1 = C_ip[j + 1];
          for (int e = C_ip[j]; e < e1; ++e) {
            const unsigned code = (unsigned)IC_a[e];
            const int sl = (int)(code & 0x7fffffffu);
            const bool to = code >> 31;
            const bool out = is_out(o, nout, IC_br[e]);
            double fl;
            if (FORM == kFormF2) {
              fl = decode(fc[sl], lane, out ? 0.0 : IC_x[e]);
            } else {
              const double bl = out ? 0.0 : IC_x[e];
              fl = bl * (decode(th[sl], lane, IC_Ts[e]) - decode(th[IC_tt[e]], lane, IC_Tt[e]));
            }
            gl = to ? gl + fl : gl - fl;
          }
          val += -(li * di);
          if (!last) lam_o[(size_t)i * kTile] = step ? li + alpha * gl : li;
        }
      }
      named_bar(1, CT);
      if (threadIdx.x == 0) mbar_arrive(&empty[st]);
    }
    // ---------------- dual value, best, status ----------------
    red[warp * 32 + lane] = val;
    named_bar(1, CT);
    if (warp == 0) {
      double gsum = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) gsum += red[w * 32 + lane];
      if (!last && a.hist && b < a.B) a.hist[(size_t)k * a.B + b] = gsum;
      if (last) a.bound[b] = gsum;
      if (!frozen) {
        if (valid_bound(gsum)) {
          if (gsum > best) best = gsum;
        } else {
          frz[lane] = 1;
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
  if (warp == 0) {
    a.best[b] = best;
    a.status[b] = frz[lane];
  }
}

}  // namespace dcopf
