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
  int off_bar, off_red, off_frz, off_obm, off_prog, prog_stride, off_brp, off_lamp, off_dp, off_th, off_fc;
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
  const uint8_t *brp = smem + a.off_brp + lane * 8;   // + row byte offset
  const uint8_t *lamp = smem + a.off_lamp + lane * 8;
  const uint8_t *dp = smem + a.off_dp + lane * 8;
  uint2 *th = reinterpret_cast<uint2 *>(smem + a.off_th);
  uint2 *fc = reinterpret_cast<uint2 *>(smem + a.off_fc);
  unsigned *obm = reinterpret_cast<unsigned *>(smem + a.off_obm);
  constexpr int CT = NW * 32;
  auto ld = [](const uint8_t *base, int off) { return *reinterpret_cast<const double *>(base + off); };
  int o[kMaxOut];
  const int nout = a.max_out;
#pragma unroll
  for (int j = 0; j < kMaxOut; ++j) o[j] = (j < nout) ? a.outs[b * nout + j] : -1;
  // per-tile outage bitmap: bit l set if some instance of the tile has branch l
  // out; the per-lane check only runs for flagged branches (rare)
  for (int x = threadIdx.x; x < (a.n_br + 31) / 32; x += CT) obm[x] = 0u;
  named_bar(1, CT);
#pragma unroll
  for (int j = 0; j < kMaxOut; ++j)
    if (o[j] >= 0) atomicOr(&obm[o[j] >> 5], 1u << (o[j] & 31));
  named_bar(1, CT);
  auto flagged = [&](int l) { return (obm[l >> 5] >> (l & 31)) & 1u; };
  double best = a.best[b];

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
      mbar_wait(&full[st], (unsigned)((g / S) & 1));
      const uint8_t *prog = smem + a.off_prog + st * a.prog_stride;
      const int4 h0 = *reinterpret_cast<const int4 *>(prog);        // nA nIA nB nC
      const int4 h1 = *reinterpret_cast<const int4 *>(prog + 16);   // nIC nG a0 b0
      const int4 h2 = *reinterpret_cast<const int4 *>(prog + 32);   // offA offIA offB offC
      const int4 h3 = *reinterpret_cast<const int4 *>(prog + 48);   // offG offIC

      // ---------------- A: w_i, theta* codes ----------------
      {
        const RecA *A = reinterpret_cast<const RecA *>(prog + h2.x);
        for (int j = warp; j < h0.x; j += NW) {
          const RecA ra = A[j];
          const int bus = h1.z + j;
          double w = 0.0;
          if (FORM == kFormF2) {
            const RecIA2 *IA = reinterpret_cast<const RecIA2 *>(prog + h2.y);
            for (int e = ra.e0; e < ra.e1; ++e) {
              const RecIA2 r = IA[e];
              double sb = r.sb;
              if (flagged(r.br) && is_out(o, nout, r.br)) sb = copysign(0.0, sb);
              w = w + sb * ld(brp, r.row);                  // w_s += -(b nu), w_t += b nu
            }
          } else {
            const RecIA1 *IA = reinterpret_cast<const RecIA1 *>(prog + h2.y);
            for (int e = ra.e0; e < ra.e1; ++e) {
              const RecIA1 r = IA[e];
              double sb = r.sb;
              if (flagged(r.br) && is_out(o, nout, r.br)) sb = copysign(0.0, sb);
              const double x = (ld(brp, r.row) - ld(brp, r.row + 256)) - (ld(lamp, r.ls) - ld(lamp, r.lt));
              w = w + sb * x;                                // w_s += u, w_t -= u
            }
          }
          const bool notref = (bus != a.ref);
          const bool pos = notref && (w < 0.0), neg = notref && (w > 0.0);
          const unsigned mp = __ballot_sync(0xffffffffu, pos), mn = __ballot_sync(0xffffffffu, neg);
          if (lane == 0) th[ra.th] = make_uint2(mp, mn);
          if (notref) val += w * (pos ? ra.theta : (neg ? -ra.theta : 0.0));
        }
      }
      named_bar(1, CT);
      // ---------------- B: branches ----------------
      {
        const RecB *Bv = reinterpret_cast<const RecB *>(prog + h2.z);
        for (int j = warp; j < h0.z; j += NW) {
          const RecB r = Bv[j];
          const int l = h1.w + j;
          double bl = r.b, Fl = r.F;
          if (flagged(l) && is_out(o, nout, l)) {
            bl = 0.0;
            Fl = 0.0;
          }
          const double ths = decode(th[r.ts], lane, r.Ts);
          const double tht = decode(th[r.tt], lane, r.Tt);
          const double phi = bl * (ths - tht);
          if (FORM == kFormF2) {
            const double nu = ld(brp, r.row);
            const double q = nu - (ld(lamp, r.ls) - ld(lamp, r.lt));
            const bool fneg = q > 0.0, fpos = q < 0.0;
            const unsigned mp = __ballot_sync(0xffffffffu, fpos), mn = __ballot_sync(0xffffffffu, fneg);
            if (lane == 0) fc[r.fs] = make_uint2(mp, mn);
            const double f = fneg ? -Fl : (fpos ? Fl : 0.0);
            const double gv = f - phi;
            val += q * f;
            if (!last) br_o[(size_t)l * kTile] = step ? nu + alpha * gv : nu;
          } else {
            const double mp = ld(brp, r.row), mm = ld(brp, r.row + 256);
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
        const RecC *Cv = reinterpret_cast<const RecC *>(prog + h2.w);
        const RecG *G = reinterpret_cast<const RecG *>(prog + h3.x);
        for (int j = warp; j < h0.w; j += NW) {
          const RecC r = Cv[j];
          const double li = ld(lamp, r.ls);
          const double di = ld(dp, r.ds);
          double gl = -di;
          for (int gg = r.g0; gg < r.g1; ++gg) {
            const RecG gr = G[gg];
            const double rr = gr.c + li;
            const double p = gen_minimiser(rr, gr.lo, gr.hi, gr.a);
            gl = gl + p;
            val += (gr.a > 0.0) ? gr.a * p * p + rr * p : rr * p;
          }
          if (FORM == kFormF2) {
            const RecIC2 *IC = reinterpret_cast<const RecIC2 *>(prog + h3.y);
            for (int e = r.e0; e < r.e1; ++e) {
              const RecIC2 x = IC[e];
              double sF = x.sF;
              if (flagged(x.br) && is_out(o, nout, x.br)) sF = copysign(0.0, sF);
              const uint2 cw = fc[x.fs];
              // +f* at the to bus, -f* at the from bus (sign folded into sF)
              const double v = ((cw.x >> lane) & 1u) ? sF : (((cw.y >> lane) & 1u) ? -sF : sF * 0.0);
              gl = gl + v;
            }
          } else {
            const RecIC1 *IC = reinterpret_cast<const RecIC1 *>(prog + h3.y);
            for (int e = r.e0; e < r.e1; ++e) {
              const RecIC1 x = IC[e];
              double sb = x.sb;
              if (flagged(x.br) && is_out(o, nout, x.br)) sb = copysign(0.0, sb);
              gl = gl + sb * (decode(th[x.ts], lane, x.Ts) - decode(th[x.tt], lane, x.Tt));
            }
          }
          val += -(li * di);
          if (!last) lam_o[(size_t)r.bus * kTile] = step ? li + alpha * gl : li;
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
