// Host-only checker of the batched sweep schedule (paper_2406_13191_b200/csrc/split_schedule.cpp):
// replays every part's producer/consumer order of k_sweep with worst-case
// (instant) TMA landing and verifies that every shared-memory slot read holds
// the row or code the program expects, that codes are read only in a later
// step than the one writing them, and that the owned items cover every bus /
// branch / cycle exactly once per phase.  Input on stdin: nb nl ref form CH P,
// then nl lines "s t" (original ids).  Arguments: order(dfs|rcm) W life
// [pool_gap [V C]].
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <string>
#include <vector>

#include "../paper_2406_13191_b200/csrc/cluster.h"
#include "../paper_2406_13191_b200/csrc/schedule.h"

using namespace dcopf;


// Split-tile replay (build_schedule_split, forms F2 / KVL): every part runs its
// steps with its own pools; worst-case (instant) copy landing; a code read at
// step c must see a code written at a step <= c - 1 of the same part, and a
// code slot may be rewritten only GAP steps after its previous occupant's
// last read.  Owned items must cover every bus / branch (/ cycle) exactly
// once over the parts; halo items may repeat.
static int check_split(const NetInternal &n, const Schedule &S, const CycleBasis *Y, int P, int GAP) {
  const bool kvl = n.form == 2, f1 = n.form == 1;
  const int RB = S.row_bytes, BR = S.br_row_bytes, CRB = S.code_row_bytes;
  const int nrows_br = kvl ? Y->nc : n.nl;
  std::vector<int> seenA(n.nb, 0), seenB(n.nl, 0), seenC(n.nb, 0), seenD(kvl ? Y->nc : 0, 0);
  int bad = 0, halo = 0;
  auto BADF = [&](const char *m, int c, int x) { if (bad < 12) printf("BAD %s step %d ent %d\n", m, c, x); ++bad; };
  // positions form permutations
  for (int k = 0; k < 3; ++k) {
    const std::vector<int> &perm = k == 0 ? S.perm_lam : k == 1 ? S.perm_d : S.perm_br;
    const int nn = k == 2 ? nrows_br : n.nb;
    std::vector<int> seen(nn, 0);
    if ((int)perm.size() != nn) { printf("BAD perm size\n"); return 1; }
    for (int x : perm) if (x < 0 || x >= nn || seen[x]++) { printf("BAD perm\n"); return 1; }
  }
  for (int p = 0; p < S.C; ++p) {
    const int s0 = S.part_step0[p], s1 = S.part_step0[p + 1], b0 = S.part_bus0[p], b1 = S.part_bus0[p + 1];
    auto own = [&](int i) { return i >= b0 && i < b1; };
    std::vector<int> brp(S.n_br_slots, -1), lamp(S.n_lam_slots, -1), dp(S.n_d_slots, -1);
    std::vector<int> th(S.n_th_slots, -1), thw(S.n_th_slots, -100), thr(S.n_th_slots, -100);
    std::vector<int> fc(S.n_f_slots, -1), fw(S.n_f_slots, -100), fr(S.n_f_slots, -100);
    auto issue = [&](int c) {
      if (c >= s1) return;
      for (int e = S.ld_ptr[c]; e < S.ld_ptr[c + 1]; ++e) {
        const int4_t x = S.ld[e];
        std::vector<int> &pool = x.a == LD_LAM ? lamp : x.a == LD_D ? dp : brp;
        const std::vector<int> &perm = x.a == LD_LAM ? S.perm_lam : x.a == LD_D ? S.perm_d : S.perm_br;
        for (int r = 0; r < x.c; ++r) {
          if (x.d + r >= (int)pool.size() || x.b + r >= (int)perm.size()) { printf("BAD slot range\n"); ++bad; continue; }
          pool[x.d + r] = perm[x.b + r];
        }
      }
    };
    auto want = [&](std::vector<int> &pool, int off, int unit, int ent, const char *what, int c) {
      const int slot = off / unit;
      if (off % unit || slot < 0 || slot >= (int)pool.size() || pool[slot] != ent) BADF(what, c, ent);
    };
    auto code_w = [&](std::vector<int> &pool, std::vector<int> &w, std::vector<int> &r, int off, int ent, int c,
                      const char *what) {
      const int slot = off / CRB;
      if (off % CRB || slot < 0 || slot >= (int)pool.size()) { BADF(what, c, ent); return; }
      if (pool[slot] != -1 && pool[slot] != ent && r[slot] > c - GAP) BADF("code slot reused too early", c, ent);
      pool[slot] = ent;
      w[slot] = c;
    };
    auto code_r = [&](std::vector<int> &pool, std::vector<int> &w, std::vector<int> &r, int off, int ent, int c,
                      const char *what) {
      const int slot = off / CRB;
      if (off % CRB || slot < 0 || slot >= (int)pool.size() || pool[slot] != ent) { BADF(what, c, ent); return; }
      if (w[slot] > c - 1) BADF("code read in the step that writes it", c, ent);
      r[slot] = std::max(r[slot], c);
    };
    for (int c = s0; c <= s0 + P; ++c) issue(c);
    for (int c = s0; c < s1; ++c) {
      long bytes = S.prog_bytes[c];
      for (int e = S.ld_ptr[c]; e < S.ld_ptr[c + 1]; ++e)
        bytes += (long)S.ld[e].c * ((S.ld[e].a == LD_BR) ? BR : RB);
      if (bytes != S.tx_bytes[c]) BADF("tx bytes", c, 0);
      const uint8_t *pg = S.prog.data() + S.prog_off[c];
      const int *h = reinterpret_cast<const int *>(pg);
      const RecC *Cv = reinterpret_cast<const RecC *>(pg + h[PH_OFF_C]);
      const RecIC2 *IC = reinterpret_cast<const RecIC2 *>(pg + h[PH_OFF_IC]);
      const RecIC1 *IC1 = reinterpret_cast<const RecIC1 *>(pg + h[PH_OFF_IC]);
      if (!kvl) {
        const RecA *A = reinterpret_cast<const RecA *>(pg + h[PH_OFF_A]);
        const RecIA2 *IA = reinterpret_cast<const RecIA2 *>(pg + h[PH_OFF_IA]);
        const RecIA1 *IA1 = reinterpret_cast<const RecIA1 *>(pg + h[PH_OFF_IA]);
        const RecB *Bv = reinterpret_cast<const RecB *>(pg + h[PH_OFF_B]);
        for (int j = 0; j < h[PH_NA]; ++j) {
          const int bus = A[j].bus;
          const bool hl = A[j].flags & kAFlagHalo;
          if (hl) { ++halo; if (own(bus)) BADF("halo A of an owned bus", c, bus); }
          else { seenA[bus]++; if (!own(bus)) BADF("A of a foreign bus", c, bus); }
          if (((A[j].flags & kAFlagRef) != 0) != (bus == n.ref)) BADF("A ref flag", c, bus);
          if (A[j].e1 - A[j].e0 != n.bus_ptr[bus + 1] - n.bus_ptr[bus]) BADF("A degree", c, bus);
          for (int e = A[j].e0; e < A[j].e1; ++e) {
            const int k = n.bus_ptr[bus] + e - A[j].e0, l = n.bus_inc[k] >> 1, to = n.bus_inc[k] & 1;
            if (f1) {
              if ((IA1[e].br < 0 ? l : IA1[e].br) != l) BADF("A order", c, bus);
              if (IA1[e].sb != (to ? -n.b[l] : n.b[l])) BADF("A sign", c, bus);
              want(brp, IA1[e].row, BR, l, "A mu", c);
              want(lamp, IA1[e].ls, RB, n.bs[l], "A lam_s", c);
              want(lamp, IA1[e].lt, RB, n.bt[l], "A lam_t", c);
              continue;
            }
            if (IA[e].br != l) BADF("A order", c, bus);
            if (IA[e].sb != (to ? n.b[l] : -n.b[l])) BADF("A sign", c, bus);
            want(brp, IA[e].row, BR, l, "A nu", c);
          }
        }
        for (int j = 0; j < h[PH_NB]; ++j) {
          const bool lite = Bv[j].wpos < 0;
          const int l = lite ? -1 - Bv[j].wpos : S.perm_br[Bv[j].wpos];
          const int hi = std::max(n.bs[l], n.bt[l]), lo = std::min(n.bs[l], n.bt[l]);
          if (lite) { ++halo; if (!(own(lo) && hi >= b1)) BADF("lite B not a halo branch", c, l); }
          else { seenB[l]++; if (!own(hi)) BADF("B of a foreign branch", c, l); }
          want(brp, Bv[j].row, BR, l, "B nu", c);
          if (!f1) {
            want(lamp, Bv[j].ls, RB, n.bs[l], "B lam_s", c);
            want(lamp, Bv[j].lt, RB, n.bt[l], "B lam_t", c);
          }
          if (Bv[j].b != n.b[l] || Bv[j].F != n.F[l]) BADF("B data", c, l);
        }
        // theta* reads (own B) see codes of earlier steps; then this step's A writes land
        for (int j = 0; j < h[PH_NB]; ++j)
          if (Bv[j].wpos >= 0) {
            const int l = S.perm_br[Bv[j].wpos];
            code_r(th, thw, thr, Bv[j].ts, n.bs[l], c, "B th_s");
            code_r(th, thw, thr, Bv[j].tt, n.bt[l], c, "B th_t");
          }
        // (C's reads: F1 theta* codes of both endpoints, F2 f* codes -- before this step's writes land)
        for (int j = 0; j < h[PH_NC]; ++j) {
          const int bus = S.perm_lam[Cv[j].wpos];
          for (int e = Cv[j].e0; e < Cv[j].e1; ++e) {
            const int l = n.bus_inc[n.bus_ptr[bus] + e - Cv[j].e0] >> 1;
            if (f1) {
              code_r(th, thw, thr, IC1[e].ts, n.bs[l], c, "C th_s");
              code_r(th, thw, thr, IC1[e].tt, n.bt[l], c, "C th_t");
            } else {
              code_r(fc, fw, fr, IC[e].f, IC[e].br, c, "C f");
            }
          }
        }
        for (int j = 0; j < h[PH_NA]; ++j) code_w(th, thw, thr, A[j].th, A[j].bus, c, "A th write");
        if (!f1)
          for (int j = 0; j < h[PH_NB]; ++j) {
            const int l = Bv[j].wpos < 0 ? -1 - Bv[j].wpos : S.perm_br[Bv[j].wpos];
            code_w(fc, fw, fr, Bv[j].fs, l, c, "B f write");
          }
      } else {
        const RecBK *Bv = reinterpret_cast<const RecBK *>(pg + h[PH_OFF_B]);
        const RecBKe *BK = reinterpret_cast<const RecBKe *>(pg + h[PH_PAD]);
        const RecD *Dv = reinterpret_cast<const RecD *>(pg + h[PH_OFF_A]);
        const RecDe *De = reinterpret_cast<const RecDe *>(pg + h[PH_OFF_IA]);
        for (int j = 0; j < h[PH_NB]; ++j) {
          const int l = Bv[j].br, hi = std::max(n.bs[l], n.bt[l]);
          if (Bv[j].halo) { ++halo; if (own(hi)) BADF("halo B of an owned branch", c, l); }
          else { seenB[l]++; if (!own(hi)) BADF("B of a foreign branch", c, l); }
          want(lamp, Bv[j].ls, RB, n.bs[l], "B lam_s", c);
          want(lamp, Bv[j].lt, RB, n.bt[l], "B lam_t", c);
          int cnt = 0;
          for (int k = 0; k < Y->nc; ++k)
            for (int e = Y->cp[k]; e < Y->cp[k + 1]; ++e)
              if (Y->cb[e] == l && n.b[Y->def[k]] > 0.0) {
                if (Bv[j].e0 + cnt >= Bv[j].e1) { BADF("B terms", c, l); break; }
                want(brp, BK[Bv[j].e0 + cnt].ks, RB, k, "B kappa", c);
                if (BK[Bv[j].e0 + cnt].sgn != Y->cs[e]) BADF("B sign", c, l);
                ++cnt;
              }
          if (cnt != Bv[j].e1 - Bv[j].e0) BADF("B term count", c, l);
        }
        for (int j = 0; j < h[PH_NC]; ++j)
          for (int e = Cv[j].e0; e < Cv[j].e1; ++e) code_r(fc, fw, fr, IC[e].f, IC[e].br, c, "C f");
        for (int j = 0; j < h[PH_NA]; ++j) {
          const int k = S.perm_br[Dv[j].wpos];
          seenD[k]++;
          want(brp, Dv[j].ks, RB, k, "D kappa", c);
          const bool active = n.b[Y->def[k]] > 0.0;
          if (Dv[j].e1 - Dv[j].e0 != (active ? Y->cp[k + 1] - Y->cp[k] : 0)) { BADF("D length", c, k); continue; }
          for (int e = Dv[j].e0; e < Dv[j].e1; ++e) {
            const int q = Y->cp[k] + e - Dv[j].e0, l = Y->cb[q];
            code_r(fc, fw, fr, De[e].fs, l, c, "D f");
            const double sx = (Y->cs[q] > 0 ? 1.0 : -1.0) / n.b[l];
            if (De[e].t[2] != n.F[l] * sx || De[e].t[0] != -n.F[l] * sx) BADF("D coefficient", c, k);
          }
        }
        for (int j = 0; j < h[PH_NB]; ++j) code_w(fc, fw, fr, Bv[j].fs, Bv[j].br, c, "B f write");
      }
      for (int j = 0; j < h[PH_NC]; ++j) {
        const int bus = S.perm_lam[Cv[j].wpos];
        seenC[bus]++;
        if (!own(bus)) BADF("C of a foreign bus", c, bus);
        want(lamp, Cv[j].ls, RB, bus, "C lam", c);
        want(dp, Cv[j].ds, RB, bus, "C d", c);
        if (Cv[j].e1 - Cv[j].e0 != n.bus_ptr[bus + 1] - n.bus_ptr[bus]) BADF("C degree", c, bus);
        for (int e = Cv[j].e0; e < Cv[j].e1; ++e) {
          const int k = n.bus_ptr[bus] + e - Cv[j].e0, l = n.bus_inc[k] >> 1, to = n.bus_inc[k] & 1;
          if (f1) {
            if ((IC1[e].br < 0 ? l : IC1[e].br) != l || IC1[e].sb != (to ? n.b[l] : -n.b[l])) BADF("C order / sign", c, bus);
            continue;
          }
          const double F = (!kvl || n.b[l] > 0.0) ? n.F[l] : 0.0;
          if (IC[e].br != l || IC[e].sF != (to ? F : -F)) BADF("C order / sign", c, bus);
        }
      }
      issue(c + P + 1);
    }
  }
  if (!kvl) for (int i = 0; i < n.nb; ++i) if (seenA[i] != 1) { printf("BAD cover A bus %d\n", i); ++bad; break; }
  for (int i = 0; i < n.nb; ++i) if (seenC[i] != 1) { printf("BAD cover C bus %d\n", i); ++bad; break; }
  for (int l = 0; l < n.nl; ++l) if (seenB[l] != 1) { printf("BAD cover br %d\n", l); ++bad; break; }
  if (kvl) for (int k = 0; k < Y->nc; ++k) if (seenD[k] != 1) { printf("BAD cover cycle %d\n", k); ++bad; break; }
  int mx = 0;
  for (int p = 0; p < S.C; ++p) mx = std::max(mx, S.part_step0[p + 1] - S.part_step0[p]);
  printf("parts %d steps %d slots br %d lam %d d %d th %d f %d smem %d copies %d sticky %d halo %d bad %d\n", S.C, mx,
         S.n_br_slots, S.n_lam_slots, S.n_d_slots, S.n_th_slots, S.n_f_slots, S.total, S.n_copies,
         S.n_sticky_copies, halo, bad);
  return bad ? 1 : 0;
}

int main(int argc, char **argv) {
  int nb, nl, ref, form, CH, P;
  if (scanf("%d %d %d %d %d %d", &nb, &nl, &ref, &form, &CH, &P) != 6) return 2;
  std::vector<int> fr(nl), to(nl);
  for (int l = 0; l < nl; ++l) if (scanf("%d %d", &fr[l], &to[l]) != 2) return 2;
  std::vector<double> b(nl), F(nl), theta(nb, 1.0);
  for (int l = 0; l < nl; ++l) { b[l] = 1.0 + (l % 7); F[l] = 0.5 * (l % 5); }
  Internalized in;
  bool rcm = argc > 1 && std::string(argv[1]) == "rcm";
  std::string e0 = internalize(nb, nl, 0, ref, fr.data(), to.data(), b.data(), F.data(), theta.data(), nullptr,
                               nullptr, nullptr, nullptr, nullptr, nullptr, form, rcm, &in);
  if (!e0.empty()) { printf("ERR %s\n", e0.c_str()); return 1; }
  NetInternal &n = in.net;
  Schedule S;
  const int W = argc > 2 ? atoi(argv[2]) : 32;
  if (argc > 3) S.ring_life = atoi(argv[3]);
  if (argc > 4) S.pool_gap = atoi(argv[4]);
  CycleBasis Y, Yi;
  if (form == 2) {  // KVL: the canonical basis (every non-tree branch switchable for this check)
    std::vector<uint8_t> none(nl, 0);
    std::string e1 = build_cycle_basis(nb, nl, ref, fr.data(), to.data(), b.data(), none.data(), &Y);
    if (!e1.empty()) { printf("ERR %s\n", e1.c_str()); return 1; }
    Yi = Y;
    for (int &l : Yi.def) l = in.br_inv[l];
    for (int &l : Yi.cb) l = in.br_inv[l];
  }
  // argv[5], argv[6]: instances per lane and parts (default 2, 1: the unsplit sweep)
  const int V = argc > 6 ? atoi(argv[5]) : 2, C = argc > 6 ? atoi(argv[6]) : 1;
  std::string e2 = build_schedule_split(n, CH, P, W, V, 8, C, {}, &S, form == 2 ? &Yi : nullptr);
  if (!e2.empty()) { printf("ERR %s\n", e2.c_str()); return 1; }
  return check_split(n, S, form == 2 ? &Yi : nullptr, P, S.pool_gap);
}
