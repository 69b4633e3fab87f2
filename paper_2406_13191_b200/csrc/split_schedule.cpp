// split_schedule.cpp -- the split-tile sweep schedule of the batched path
// (schedule.h build_schedule_split; forms F2, F1 and KVL).
//
// A tile of W instances is swept by C CTAs ("parts").  Part p owns the
// internal buses [cuts[p], cuts[p+1]) (a contiguous range of the DFS tree
// order), the branches whose larger endpoint it owns and (KVL) the cycles
// whose largest branch endpoint it owns; it runs the unsplit sweep's items
// for what it owns, in skewed steps over its own chunks of CH buses, and
// writes exactly the multipliers it owns.  The few minimiser codes it reads
// but does not own come from HALO items that recompute them from the y_k rows
// in HBM -- the same arithmetic on the same inputs, so bitwise the owner's
// code -- and contribute nothing to the dual value:
//   F2   halo A(j): theta*_j of a lower-part endpoint j of an owned branch;
//        lite B(l): f*_l of a branch from an owned bus to a higher part
//   F1   halo A(j): theta*_j of every bus of another part adjacent to an owned
//        bus (read by B of owned branches and by C, whose d/dlambda uses phi)
//   KVL  halo B(l): f*_l of a branch from an owned bus to a higher part (read
//        by C) or of a lower-part branch of an owned cycle (read by D)
// Rows the part owns are stored in HBM in its load order inside its segment
// of the tile (ring runs = one bulk copy); halo rows are individual copies
// from the owner's segment.  The tile's parts meet once per sweep (the
// kernel's inter-part barrier, sweep_kernel.cuh): y_{k+1} rows are written by
// their owners and read by the other parts' halo items only in sweep k+1.
//
// Step semantics are those of the unsplit schedule (schedule.cpp):
//   F2  step s: A items, [A-done(s-1)], B items, [B-done(s-1)], C items; a B
//       item at s reads theta* codes written at steps <= s-1, a C item f*
//       codes written at <= s-1.
//   KVL step s: B items, [B-done(s-1)], C and D items (same rule for f*).
#include <algorithm>
#include <climits>
#include <cstring>
#include <numeric>
#include <string>
#include <type_traits>
#include <vector>

#include "schedule.h"
#include "schedule_detail.h"

namespace dcopf {

using detail::Interval;

namespace {

struct Use {  // steps at which a row is read
  int first = INT_MAX, last = -1;
  void at(int s) {
    first = std::min(first, s);
    last = std::max(last, s);
  }
  bool used() const { return last >= 0; }
};
struct CodeUse {  // step a code is written at, last step it is read at
  int w = -1, last = -1;
};

enum { K_LAM = 0, K_D = 1, K_BR = 2 };

struct Part {
  int b0 = 0, b1 = 0, nch = 0, nst = 0;
  // items per local step: entity, halo flag
  std::vector<std::vector<std::pair<int, int>>> A, B, Cc, D;
  std::vector<Use> use[3];     // per kind, per entity
  std::vector<CodeUse> th, fc;  // theta* (per bus), f* (per branch)
  std::vector<int> slot[3], th_slot, f_slot;
  std::vector<int> own_order[3];  // own rows in local storage order (ring rows first)
  int nring[3] = {0, 0, 0}, R[3] = {1, 1, 1}, nslots[3] = {0, 0, 0}, nth = 0, nf = 0;
  std::vector<int> lpos[3];   // local storage position of an own row (-1: not own)
};

// per-bus / per-branch estimated issue cost (instructions per warp), the
// weights of the unsplit schedule's warp balancing
long bus_cost_f2(const NetInternal &n, int i) {
  const int deg = n.bus_ptr[i + 1] - n.bus_ptr[i], gens = n.gen_ptr[i + 1] - n.gen_ptr[i];
  return (30 + 12 * deg) + (35 + 12 * deg + 25 * gens);
}

}  // namespace

std::string build_schedule_split(const NetInternal &net, int CH, int P, int W, int V, int nw, int C,
                                 std::vector<int> cuts, Schedule *out, const CycleBasis *cyc) {
  Schedule &S = *out;
  const bool kvl = net.form == 2, f1 = net.form == 1;
  if (kvl && !cyc) return "KVL form needs its cycle basis";
  if (V != 2 && V != 4) return "instances per lane must be 2 or 4";
  if (f1 && V != 2) return "form F1 runs 2 instances per lane";
  if (W < V || W > 32 * V || W % V) return "tile width must be a multiple of V in [V, 32 V]";
  const int nb = net.nb, nl = net.nl, nc = kvl ? cyc->nc : 0;
  const int nrow[3] = {nb, nb, kvl ? nc : nl};
  if (C < 1 || C > nb) return "bad part count";
  if (CH < 1) return "bad chunk";
  std::vector<int> hi(nl), lo(nl);
  for (int l = 0; l < nl; ++l) {
    hi[l] = std::max(net.bs[l], net.bt[l]);
    lo[l] = std::min(net.bs[l], net.bt[l]);
    if (l > 0 && hi[l] < hi[l - 1]) return "internal branch order not sorted by larger endpoint";
  }
  // cycles through each branch (KVL), ascending k; a cycle is active when its
  // defining branch has b > 0 (an open circuit has no loop)
  std::vector<std::vector<std::pair<int, int>>> bcyc(kvl ? nl : 0);
  std::vector<int> cyc_hi(nc, -1);
  if (kvl) {
    for (int k = 0; k < nc; ++k)
      for (int e = cyc->cp[k]; e < cyc->cp[k + 1]; ++e) {
        const int l = cyc->cb[e];
        bcyc[l].push_back({k, cyc->cs[e]});
        cyc_hi[k] = std::max(cyc_hi[k], hi[l]);
      }
  }
  // ---- part boundaries: balanced by estimated cost ----
  if (cuts.empty()) {
    std::vector<long> cost(nb, 0);
    for (int i = 0; i < nb; ++i) {
      const long deg = net.bus_ptr[i + 1] - net.bus_ptr[i], gens = net.gen_ptr[i + 1] - net.gen_ptr[i];
      cost[i] = kvl ? 35 + 12 * deg + 25 * gens : (f1 ? 65 + 40 * deg + 25 * gens : bus_cost_f2(net, i));
    }
    for (int l = 0; l < nl; ++l) cost[hi[l]] += kvl ? 50 + 10L * (long)bcyc[l].size() : (f1 ? 60 : 70);
    if (kvl)
      for (int k = 0; k < nc; ++k) cost[cyc_hi[k]] += 30 + 10L * (cyc->cp[k + 1] - cyc->cp[k]);
    const long tot = std::accumulate(cost.begin(), cost.end(), 0L);
    cuts.assign(C + 1, nb);
    cuts[0] = 0;
    long acc = 0;
    for (int i = 0, p = 1; i < nb && p < C; ++i) {
      acc += cost[i];
      if (acc * C >= tot * p) cuts[p++] = i + 1;
    }
  }
  if ((int)cuts.size() != C + 1 || cuts[0] != 0 || cuts[C] != nb) return "bad part cuts";
  for (int p = 0; p < C; ++p)
    if (cuts[p + 1] <= cuts[p]) return "empty part";

  S.CH = CH;
  S.P = P;
  S.S = P + 1;
  S.W = W;
  S.V = V;
  S.C = C;
  S.row_bytes = 8 * W;
  S.br_row_bytes = f1 ? 16 * W : 8 * W;  // F1: mu+ then mu- in one row
  S.code_row_bytes = 32 * V;
  S.part_bus0 = cuts;
  const int RB = S.row_bytes, BR = S.br_row_bytes, CRB = S.code_row_bytes, LIFE = S.ring_life, GAP = S.pool_gap;
  const int off_B = kvl ? 0 : 1;  // step of an item of chunk c: F2 A c, B c+1, C c+2; KVL B c, C / D c+1
  const int off_C = kvl ? 1 : 2;

  std::vector<Part> parts(C);
  std::vector<int> owner_bus(nb), owner_row[3];
  for (int p = 0; p < C; ++p)
    for (int i = cuts[p]; i < cuts[p + 1]; ++i) owner_bus[i] = p;
  owner_row[K_LAM] = owner_bus;
  owner_row[K_D] = owner_bus;
  owner_row[K_BR].resize(nrow[K_BR]);
  for (int x = 0; x < nrow[K_BR]; ++x) owner_row[K_BR][x] = owner_bus[kvl ? cyc_hi[x] : hi[x]];
  S.halo_a = S.halo_b = 0;

  // ================= pass 1: items, uses, slots, local storage order =================
  for (int p = 0; p < C; ++p) {
    Part &Pt = parts[p];
    Pt.b0 = cuts[p];
    Pt.b1 = cuts[p + 1];
    const int b0 = Pt.b0, b1 = Pt.b1;
    Pt.nch = (b1 - b0 + CH - 1) / CH;
    Pt.nst = Pt.nch + off_C;
    const int nst = Pt.nst;
    auto own = [&](int i) { return i >= b0 && i < b1; };
    auto chunk = [&](int i) { return (i - b0) / CH; };
    Pt.A.assign(nst, {});
    Pt.B.assign(nst, {});
    Pt.Cc.assign(nst, {});
    Pt.D.assign(nst, {});
    for (int k = 0; k < 3; ++k) Pt.use[k].assign(nrow[k], Use());
    Pt.th.assign(nb, CodeUse());
    Pt.fc.assign(nl, CodeUse());
    // B chunk of every branch the part computes (-1: none)
    std::vector<int> bchunk(nl, -1), bhalo(nl, 0);
    for (int l = 0; l < nl; ++l) {
      if (own(hi[l])) bchunk[l] = chunk(hi[l]);
      else if (own(lo[l]) && !f1) {  // hi in a higher part: f* read by C(lo) here (F1 writes no f* code)
        bchunk[l] = chunk(lo[l]);
        bhalo[l] = 1;
      }
    }
    if (kvl)  // lower-part branches of an owned cycle: f* read by D(k) here
      for (int k = 0; k < nc; ++k) {
        if (!own(cyc_hi[k])) continue;
        const int dc = chunk(cyc_hi[k]);
        for (int e = cyc->cp[k]; e < cyc->cp[k + 1]; ++e) {
          const int l = cyc->cb[e];
          if (hi[l] < b0) {
            bchunk[l] = (bchunk[l] < 0) ? dc : std::min(bchunk[l], dc);
            bhalo[l] = 1;
          }
        }
      }
    // ---- A (F2 / F1): owned buses at their chunk; halo theta* of lower
    // endpoints of owned branches (read by B), and (F1) of every neighbour of an
    // owned bus in another part (read by C: F1's d/dlambda uses phi from the
    // theta* codes) -- at the earliest chunk of an owned neighbour
    if (!kvl) {
      std::vector<int> hstep(nb, INT_MAX);
      for (int l = 0; l < nl; ++l) {
        if (!f1) {
          if (own(hi[l]) && lo[l] < b0) hstep[lo[l]] = std::min(hstep[lo[l]], chunk(hi[l]));
        } else {
          const int s_ = net.bs[l], t_ = net.bt[l];
          if (own(s_) && !own(t_)) hstep[t_] = std::min(hstep[t_], chunk(s_));
          if (own(t_) && !own(s_)) hstep[s_] = std::min(hstep[s_], chunk(t_));
        }
      }
      for (int i = 0; i < nb; ++i) {
        int s = -1, h = 0;
        if (own(i)) s = chunk(i);
        else if (hstep[i] != INT_MAX) {
          s = hstep[i];
          h = 1;
          ++S.halo_a;
        }
        if (s < 0) continue;
        Pt.A[s].push_back({i, h});
        for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e) {
          const int l = net.bus_inc[e] >> 1;
          Pt.use[K_BR][l].at(s);
          if (f1) {  // u_l = b ((mu+ - mu-) - (lambda_s - lambda_t))
            Pt.use[K_LAM][net.bs[l]].at(s);
            Pt.use[K_LAM][net.bt[l]].at(s);
          }
        }
        Pt.th[i].w = s;
      }
    }
    // ---- B: owned and halo branches
    for (int l = 0; l < nl; ++l) {
      if (bchunk[l] < 0) continue;
      const int s = bchunk[l] + off_B;
      Pt.B[s].push_back({l, bhalo[l]});
      if (bhalo[l]) ++S.halo_b;
      if (!f1) {
        Pt.use[K_LAM][net.bs[l]].at(s);
        Pt.use[K_LAM][net.bt[l]].at(s);
      }
      if (!kvl) {
        Pt.use[K_BR][l].at(s);
        if (!bhalo[l]) {  // phi needs theta* at both endpoints
          Pt.th[net.bs[l]].last = std::max(Pt.th[net.bs[l]].last, s);
          Pt.th[net.bt[l]].last = std::max(Pt.th[net.bt[l]].last, s);
        }
      } else {
        for (auto &kc : bcyc[l])
          if (net.b[cyc->def[kc.first]] > 0.0) Pt.use[K_BR][kc.first].at(s);
      }
      if (!f1) Pt.fc[l].w = s;
    }
    // ---- C: owned buses after every incident branch's code
    for (int i = b0; i < b1; ++i) {
      int cc = chunk(i);
      for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e) cc = std::max(cc, bchunk[net.bus_inc[e] >> 1]);
      const int s = cc + off_C;
      Pt.Cc[s].push_back({i, 0});
      Pt.use[K_LAM][i].at(s);
      Pt.use[K_D][i].at(s);
      for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e) {
        const int l = net.bus_inc[e] >> 1;
        if (!f1) {
          Pt.fc[l].last = std::max(Pt.fc[l].last, s);
        } else {  // phi_l from the theta* codes of both endpoints
          Pt.th[net.bs[l]].last = std::max(Pt.th[net.bs[l]].last, s);
          Pt.th[net.bt[l]].last = std::max(Pt.th[net.bt[l]].last, s);
        }
      }
    }
    // ---- D (KVL): owned cycles after their last branch
    if (kvl)
      for (int k = 0; k < nc; ++k) {
        if (!own(cyc_hi[k])) continue;
        const int s = chunk(cyc_hi[k]) + off_C;
        Pt.D[s].push_back({k, 0});
        Pt.use[K_BR][k].at(s);
        if (net.b[cyc->def[k]] > 0.0)
          for (int e = cyc->cp[k]; e < cyc->cp[k + 1]; ++e) {
            const int l = cyc->cb[e];
            Pt.fc[l].last = std::max(Pt.fc[l].last, s);
          }
      }
    // ---- code slots: [write step, last read + gap - 1]
    {
      std::vector<Interval> iv;
      for (int i = 0; i < nb; ++i)
        if (Pt.th[i].w >= 0) iv.push_back({Pt.th[i].w, std::max(Pt.th[i].w, Pt.th[i].last) + GAP - 1, i});
      Pt.th_slot.assign(nb, -1);
      Pt.nth = detail::colour(iv, Pt.th_slot);
      iv.clear();
      for (int l = 0; l < nl; ++l)
        if (Pt.fc[l].w >= 0) iv.push_back({Pt.fc[l].w, std::max(Pt.fc[l].w, Pt.fc[l].last) + GAP - 1, l});
      Pt.f_slot.assign(nl, -1);
      Pt.nf = detail::colour(iv, Pt.f_slot);
    }
    // ---- row slots: own short-lived rows in a ring (stored in load order),
    // own long-lived and halo rows interval-coloured after it
    for (int k = 0; k < 3; ++k) {
      const int n = nrow[k];
      std::vector<int> own_ids, other_ids;
      for (int x = 0; x < n; ++x) {
        if (!Pt.use[k][x].used()) {
          if (owner_row[k][x] == p) return "an owned row is never used";
          continue;
        }
        (owner_row[k][x] == p ? own_ids : other_ids).push_back(x);
      }
      std::stable_sort(own_ids.begin(), own_ids.end(),
                       [&](int a, int b) { return Pt.use[k][a].first < Pt.use[k][b].first; });
      std::vector<int> ring, sticky;
      for (int x : own_ids) (Pt.use[k][x].last - Pt.use[k][x].first <= LIFE ? ring : sticky).push_back(x);
      auto lo_t = [&](int x) { return std::max(0, Pt.use[k][x].first - P); };
      int R = 1;
      for (size_t a = 0, j = 0; a < ring.size(); ++a) {
        const int t = lo_t(ring[a]);
        while (j < a && Pt.use[k][ring[j]].last < t) ++j;
        R = std::max(R, (int)(a - j + 1));
      }
      Pt.slot[k].assign(n, -1);
      for (size_t a = 0; a < ring.size(); ++a) Pt.slot[k][ring[a]] = (int)(a % R);
      std::vector<Interval> iv;
      for (int x : sticky) iv.push_back({lo_t(x), Pt.use[k][x].last, x});
      for (int x : other_ids) iv.push_back({lo_t(x), Pt.use[k][x].last, x});
      std::vector<int> ss(n, 0);
      const int ns = detail::colour(iv, ss);
      for (int x : sticky) Pt.slot[k][x] = R + ss[x];
      for (int x : other_ids) Pt.slot[k][x] = R + ss[x];
      Pt.R[k] = R;
      Pt.nring[k] = (int)ring.size();
      Pt.nslots[k] = R + ns;
      Pt.own_order[k] = ring;
      Pt.own_order[k].insert(Pt.own_order[k].end(), sticky.begin(), sticky.end());
      Pt.lpos[k].assign(n, -1);
      for (size_t a = 0; a < Pt.own_order[k].size(); ++a) Pt.lpos[k][Pt.own_order[k][a]] = (int)a;
    }
  }

  // ================= global storage positions (one segment per part) =================
  std::vector<int> *posv[3] = {&S.pos_lam, &S.pos_d, &S.pos_br}, *permv[3] = {&S.perm_lam, &S.perm_d, &S.perm_br};
  std::vector<int> seg(C + 1);
  std::vector<int> segbase[3];
  for (int k = 0; k < 3; ++k) {
    segbase[k].assign(C + 1, 0);
    for (int p = 0; p < C; ++p) segbase[k][p + 1] = segbase[k][p] + (int)parts[p].own_order[k].size();
    if (segbase[k][C] != nrow[k]) return "storage positions do not cover every row";
    posv[k]->assign(nrow[k], -1);
    permv[k]->assign(nrow[k], -1);
    for (int p = 0; p < C; ++p)
      for (size_t a = 0; a < parts[p].own_order[k].size(); ++a) {
        const int x = parts[p].own_order[k][a], g = segbase[k][p] + (int)a;
        (*posv[k])[x] = g;
        (*permv[k])[g] = x;
      }
  }

  // ================= pass 2: load lists and program blocks =================
  S.n_lam_slots = S.n_d_slots = S.n_br_slots = S.n_th_slots = S.n_f_slots = 0;
  for (const Part &Pt : parts) {
    S.n_lam_slots = std::max(S.n_lam_slots, Pt.nslots[K_LAM]);
    S.n_d_slots = std::max(S.n_d_slots, Pt.nslots[K_D]);
    S.n_br_slots = std::max(S.n_br_slots, Pt.nslots[K_BR]);
    S.n_th_slots = std::max(S.n_th_slots, Pt.nth);
    S.n_f_slots = std::max(S.n_f_slots, Pt.nf);
  }
  S.ring_lam = parts[0].R[K_LAM];
  S.ring_d = parts[0].R[K_D];
  S.ring_br = parts[0].R[K_BR];
  S.nch = 0;
  for (const Part &Pt : parts) S.nch = std::max(S.nch, Pt.nch);
  S.part_step0.assign(C + 1, 0);
  for (int p = 0; p < C; ++p) S.part_step0[p + 1] = S.part_step0[p] + parts[p].nst;
  const int NST = S.part_step0[C];
  S.nsteps = NST;
  S.ld_ptr.assign(NST + 1, 0);
  S.ld.clear();
  S.prog.clear();
  S.prog_off.assign(NST, 0);
  S.prog_bytes.assign(NST, 0);
  S.tx_bytes.assign(NST, 0);
  S.max_prog_bytes = 0;
  S.n_copies = S.n_sticky_copies = 0;
  const bool has_sw = !net.sw.empty();
  const int kind_bytes[3] = {RB, RB, BR};
  const int ld_kind[3] = {LD_LAM, LD_D, LD_BR};

  for (int p = 0; p < C; ++p) {
    const Part &Pt = parts[p];
    const int nst = Pt.nst;
    // ---- loads per local step
    std::vector<std::vector<int4_t>> per(nst);
    for (int k = 0; k < 3; ++k) {
      const std::vector<int> &ord = Pt.own_order[k];
      for (int a0 = 0; a0 < Pt.nring[k];) {  // ring runs: consecutive positions, same first step
        const int st = Pt.use[k][ord[a0]].first;
        int a1 = a0;
        while (a1 < Pt.nring[k] && Pt.use[k][ord[a1]].first == st) ++a1;
        for (int q = a0; q < a1;) {  // split at the ring wrap
          const int sl = q % Pt.R[k];
          const int cnt = std::min(a1 - q, Pt.R[k] - sl);
          per[st].push_back({ld_kind[k], segbase[k][p] + q, cnt, sl});
          q += cnt;
        }
        a0 = a1;
      }
      for (size_t a = Pt.nring[k]; a < ord.size(); ++a) {  // own sticky rows
        const int x = ord[a];
        per[Pt.use[k][x].first].push_back({ld_kind[k], segbase[k][p] + (int)a, 1, Pt.slot[k][x]});
        ++S.n_sticky_copies;
      }
      for (int x = 0; x < nrow[k]; ++x)  // halo rows: copies from their owner's segment
        if (Pt.use[k][x].used() && owner_row[k][x] != p) {
          per[Pt.use[k][x].first].push_back({ld_kind[k], (*posv[k])[x], 1, Pt.slot[k][x]});
          ++S.n_sticky_copies;
        }
    }
    for (int st = 0; st < nst; ++st) {
      const int gs = S.part_step0[p] + st;
      int rows_bytes = 0;
      for (const int4_t &x : per[st]) {
        S.ld.push_back(x);
        rows_bytes += x.c * kind_bytes[x.a == LD_LAM ? 0 : (x.a == LD_D ? 1 : 2)];
      }
      S.n_copies += (int)per[st].size();
      S.ld_ptr[gs + 1] = (int)S.ld.size();

      // ---- program block of this step
      std::vector<long> load(nw, 0);
      std::vector<uint16_t> wtab(3 * (nw + 1), 0);
      auto balance = [&](auto &items, auto cost, int phase) {
        const int n = (int)items.size();
        std::vector<int> idx(n), own(n);
        for (int x = 0; x < n; ++x) idx[x] = x;
        std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return cost(items[a]) > cost(items[b]); });
        for (int x : idx) {
          const long cx = cost(items[x]);
          int w = 0;
          for (int v = 1; v < nw; ++v)
            if (load[v] + cx < load[w] + cx) w = v;
          own[x] = w;
          load[w] += cx;
        }
        std::vector<int> ord(n);
        for (int x = 0; x < n; ++x) ord[x] = x;
        std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return own[a] < own[b]; });
        typename std::remove_reference<decltype(items)>::type re(n);
        for (int x = 0; x < n; ++x) re[x] = items[ord[x]];
        items.swap(re);
        uint16_t *t = wtab.data() + phase * (nw + 1);
        for (int x = 0, w = 0; w <= nw; ++w) {
          while (x < n && own[ord[x]] < w) ++x;
          t[w] = (uint16_t)x;
        }
      };
      std::vector<uint8_t> blk(kProgHeaderBytes, 0);
      int32_t hd[PH_COUNT] = {0};
      auto app = [&](const void *ptr, size_t n) {
        size_t off = (blk.size() + 15) & ~size_t(15);
        blk.resize(off + n);
        if (n) memcpy(blk.data() + off, ptr, n);
        return (int32_t)off;
      };
      const auto lam_sl = [&](int i) { return Pt.slot[K_LAM][i] * RB; };
      // C records (both forms)
      std::vector<RecC> Cv;
      std::vector<RecG> G;
      std::vector<RecIC2> IC;
      std::vector<RecIC1> IC1;
      for (auto &it : Pt.Cc[st]) {
        const int i = it.first;
        RecC r{};
        r.wpos = S.pos_lam[i];
        r.ls = lam_sl(i);
        r.ds = Pt.slot[K_D][i] * RB;
        r.g0 = (int)G.size();
        for (int g = net.gen_ptr[i]; g < net.gen_ptr[i + 1]; ++g)
          G.push_back(RecG{net.gc[g], net.glo[g], net.ghi[g], net.ga[g]});
        r.g1 = (int)G.size();
        r.e0 = f1 ? (int)IC1.size() : (int)IC.size();
        for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e) {
          const int l = net.bus_inc[e] >> 1, to = net.bus_inc[e] & 1;
          if (f1) {
            RecIC1 x{};
            x.ts = Pt.th_slot[net.bs[l]] * CRB;
            x.tt = Pt.th_slot[net.bt[l]] * CRB;
            x.ths = net.theta[net.bs[l]];
            x.tht = net.theta[net.bt[l]];
            x.br = !has_sw || net.sw[l] ? l : -1;
            x.sb = to ? net.b[l] : -net.b[l];  // +phi at the to bus, -phi at the from bus
            IC1.push_back(x);
            continue;
          }
          const double F = (!kvl || net.b[l] > 0.0) ? net.F[l] : 0.0;  // KVL: b = 0 is an open circuit
          IC.push_back(RecIC2{Pt.f_slot[l] * CRB, l, to ? F : -F});
        }
        r.e1 = f1 ? (int)IC1.size() : (int)IC.size();
        Cv.push_back(r);
      }
      if (!kvl) {
        std::vector<RecA> A;
        std::vector<RecIA2> IA;
        std::vector<RecIA1> IA1;
        for (auto &it : Pt.A[st]) {
          const int i = it.first;
          RecA r{};
          r.th = Pt.th_slot[i] * CRB;
          r.bus = i;
          r.flags = (i == net.ref ? kAFlagRef : 0) | (it.second ? kAFlagHalo : 0);
          r.theta = net.theta[i];
          r.e0 = f1 ? (int)IA1.size() : (int)IA.size();
          for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e) {
            const int l = net.bus_inc[e] >> 1, to = net.bus_inc[e] & 1;
            if (f1) {
              RecIA1 x{};
              x.row = Pt.slot[K_BR][l] * BR;
              x.br = !has_sw || net.sw[l] ? l : -1;
              x.ls = lam_sl(net.bs[l]);
              x.lt = lam_sl(net.bt[l]);
              x.sb = to ? -net.b[l] : net.b[l];  // w_s += u ; w_t -= u
              IA1.push_back(x);
              continue;
            }
            RecIA2 x{};
            x.row = Pt.slot[K_BR][l] * BR;
            x.br = l;
            x.sb = to ? net.b[l] : -net.b[l];  // w_s += -(b nu) ; w_t += b nu
            IA.push_back(x);
          }
          r.e1 = f1 ? (int)IA1.size() : (int)IA.size();
          A.push_back(r);
        }
        std::vector<RecB> Bv;
        for (auto &it : Pt.B[st]) {
          const int l = it.first, s_ = net.bs[l], t_ = net.bt[l];
          RecB r{};
          r.row = Pt.slot[K_BR][l] * BR;
          r.wpos = it.second ? -1 - l : S.pos_br[l];
          r.obr = !has_sw || net.sw[l] ? l : -1;
          if (!f1) {
            r.ls = lam_sl(s_);
            r.lt = lam_sl(t_);
            r.fs = Pt.f_slot[l] * CRB;
          }
          if (!it.second) {
            r.ts = Pt.th_slot[s_] * CRB;
            r.tt = Pt.th_slot[t_] * CRB;
          }
          r.ths = net.theta[s_];
          r.tht = net.theta[t_];
          r.b = net.b[l];
          r.F = net.F[l];
          Bv.push_back(r);
        }
        const long cdeg = f1 ? 20L : 12L;
        balance(A, [&](const RecA &r) { return 30L + cdeg * (r.e1 - r.e0); }, 0);
        balance(Bv, [&](const RecB &r) { return r.wpos < 0 ? 40L : (f1 ? 60L : 70L); }, 1);
        balance(Cv, [&](const RecC &r) { return 35L + cdeg * (r.e1 - r.e0) + 25L * (r.g1 - r.g0); }, 2);
        hd[PH_NA] = (int)A.size();
        hd[PH_NIA] = f1 ? (int)IA1.size() : (int)IA.size();
        hd[PH_NB] = (int)Bv.size();
        hd[PH_NC] = (int)Cv.size();
        hd[PH_NIC] = f1 ? (int)IC1.size() : (int)IC.size();
        hd[PH_NG] = (int)G.size();
        hd[PH_OFF_W] = app(detail::warp_rows(wtab, nw).data(), 16 * (size_t)nw);
        hd[PH_OFF_A] = app(A.data(), A.size() * sizeof(RecA));
        hd[PH_OFF_IA] = f1 ? app(IA1.data(), IA1.size() * sizeof(RecIA1)) : app(IA.data(), IA.size() * sizeof(RecIA2));
        hd[PH_OFF_B] = app(Bv.data(), Bv.size() * sizeof(RecB));
        hd[PH_OFF_C] = app(Cv.data(), Cv.size() * sizeof(RecC));
        hd[PH_OFF_G] = app(G.data(), G.size() * sizeof(RecG));
        hd[PH_OFF_IC] = f1 ? app(IC1.data(), IC1.size() * sizeof(RecIC1)) : app(IC.data(), IC.size() * sizeof(RecIC2));
      } else {
        std::vector<RecBK> Bv;
        std::vector<RecBKe> BKe;
        for (auto &it : Pt.B[st]) {
          const int l = it.first;
          RecBK r{};
          r.ls = lam_sl(net.bs[l]);
          r.lt = lam_sl(net.bt[l]);
          r.fs = Pt.f_slot[l] * CRB;
          r.obr = (!has_sw || net.sw[l]) ? l : -1;
          r.halo = it.second;
          r.br = l;
          r.x = (net.b[l] > 0.0) ? 1.0 / net.b[l] : 0.0;
          r.F = (net.b[l] > 0.0) ? net.F[l] : 0.0;  // b = 0: an open circuit
          r.e0 = (int)BKe.size();
          for (auto &kc : bcyc[l])  // (a cycle whose defining branch has b = 0 is inactive: no term)
            if (net.b[cyc->def[kc.first]] > 0.0) BKe.push_back(RecBKe{Pt.slot[K_BR][kc.first] * RB, kc.second});
          r.e1 = (int)BKe.size();
          Bv.push_back(r);
        }
        std::vector<RecD> Dv;
        std::vector<RecDe> De;
        for (auto &it : Pt.D[st]) {
          const int k = it.first;
          RecD r{};
          r.ks = Pt.slot[K_BR][k] * RB;
          r.wpos = S.pos_br[k];
          const int dl = cyc->def[k];
          r.dbr = (!has_sw || net.sw[dl]) ? dl : -1;
          r.e0 = (int)De.size();
          if (net.b[dl] > 0.0)  // a b = 0 defining branch: no cycle (gradient 0)
            for (int e = cyc->cp[k]; e < cyc->cp[k + 1]; ++e) {
              const int m = cyc->cb[e];
              const double x = 1.0 / net.b[m], sx = (cyc->cs[e] > 0) ? x : -x, F = net.F[m];
              RecDe d{};
              d.fs = Pt.f_slot[m] * CRB;
              d.t[0] = (-F) * sx;  // (c F) sx for c = -1, 0, +1 (exact: the oracle's f x with the sign of C)
              d.t[1] = (0.0 * F) * sx;
              d.t[2] = F * sx;
              De.push_back(d);
            }
          r.e1 = (int)De.size();
          Dv.push_back(r);
        }
        balance(Bv, [&](const RecBK &r) { return (r.halo ? 35L : 50L) + 10L * (r.e1 - r.e0); }, 0);
        balance(Cv, [&](const RecC &r) { return 35L + 12L * (r.e1 - r.e0) + 25L * (r.g1 - r.g0); }, 1);
        balance(Dv, [&](const RecD &r) { return 30L + 10L * (r.e1 - r.e0); }, 2);
        hd[PH_NA] = (int)Dv.size();
        hd[PH_NIA] = (int)De.size();
        hd[PH_NB] = (int)Bv.size();
        hd[PH_NC] = (int)Cv.size();
        hd[PH_NIC] = (int)IC.size();
        hd[PH_NG] = (int)G.size();
        hd[PH_OFF_A] = app(Dv.data(), Dv.size() * sizeof(RecD));
        hd[PH_OFF_IA] = app(De.data(), De.size() * sizeof(RecDe));
        hd[PH_OFF_B] = app(Bv.data(), Bv.size() * sizeof(RecBK));
        hd[PH_OFF_C] = app(Cv.data(), Cv.size() * sizeof(RecC));
        hd[PH_OFF_G] = app(G.data(), G.size() * sizeof(RecG));
        hd[PH_OFF_IC] = app(IC.data(), IC.size() * sizeof(RecIC2));
        hd[PH_PAD] = app(BKe.data(), BKe.size() * sizeof(RecBKe));  // KVL: cycle terms of phase B
        hd[PH_OFF_W] = app(detail::warp_rows(wtab, nw).data(), 16 * (size_t)nw);
      }
      blk.resize((blk.size() + 15) & ~size_t(15), 0);
      hd[PH_BYTES] = (int32_t)blk.size();
      memcpy(blk.data(), hd, sizeof hd);
      S.prog_off[gs] = (long long)S.prog.size();
      S.prog_bytes[gs] = (int)blk.size();
      S.prog.insert(S.prog.end(), blk.begin(), blk.end());
      S.max_prog_bytes = std::max(S.max_prog_bytes, (int)blk.size());
      S.tx_bytes[gs] = S.prog_bytes[gs] + rows_bytes;
    }
  }
  detail::layout_smem(S, nl, nw);
  return "";
}

}  // namespace dcopf
