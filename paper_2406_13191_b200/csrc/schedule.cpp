// schedule.cpp -- see schedule.h.
#include "schedule.h"
#include "schedule_detail.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <queue>
#include <set>
#include <type_traits>
#include <string>

namespace dcopf {

std::vector<int> dfs_tree_order(int n, const std::vector<std::vector<int>> &adj, int root) {
  std::vector<int> parent(n, -2), bfs;
  bfs.reserve(n);
  std::vector<int> order;
  order.reserve(n);
  std::vector<int> size(n, 1);
  std::vector<std::vector<int>> ch(n);
  for (int start = 0; start < n; ++start) {  // every component (a valid network has one)
    int s = (start == 0) ? root : start;
    if (parent[s] != -2) continue;
    size_t b0 = bfs.size();
    parent[s] = -1;
    bfs.push_back(s);
    for (size_t q = b0; q < bfs.size(); ++q) {
      int v = bfs[q];
      for (int u : adj[v])
        if (parent[u] == -2) {
          parent[u] = v;
          ch[v].push_back(u);
          bfs.push_back(u);
        }
    }
    for (size_t q = bfs.size(); q-- > b0 + 1;) size[parent[bfs[q]]] += size[bfs[q]];
    std::vector<int> st{s};
    while (!st.empty()) {
      int v = st.back();
      st.pop_back();
      order.push_back(v);
      std::vector<int> c = ch[v];
      // push largest first so the smallest subtree is visited first
      std::sort(c.begin(), c.end(), [&](int x, int y) { return size[x] != size[y] ? size[x] > size[y] : x > y; });
      for (int u : c) st.push_back(u);
    }
  }
  return order;
}

// reverse Cuthill-McKee from a pseudo-peripheral start
std::vector<int> rcm_order(int n, const std::vector<std::vector<int>> &adj) {
  std::vector<int> deg(n);
  for (int i = 0; i < n; ++i) deg[i] = (int)adj[i].size();
  auto bfs_last = [&](int s, int *ecc) {
    std::vector<int> lev(n, -1);
    std::queue<int> q;
    q.push(s);
    lev[s] = 0;
    int last = s;
    while (!q.empty()) {
      int v = q.front();
      q.pop();
      if (lev[v] > lev[last] || (lev[v] == lev[last] && deg[v] < deg[last])) last = v;
      for (int u : adj[v])
        if (lev[u] < 0) {
          lev[u] = lev[v] + 1;
          q.push(u);
        }
    }
    *ecc = lev[last];
    return last;
  };
  std::vector<int> order;
  order.reserve(n);
  std::vector<char> vis(n, 0);
  for (int comp_start = 0; comp_start < n; ++comp_start) {
    if (vis[comp_start]) continue;
    int s = comp_start, ecc = 0, ecc2 = 0;
    s = bfs_last(s, &ecc);
    for (int it = 0; it < 4; ++it) {
      int s2 = bfs_last(s, &ecc2);
      if (ecc2 <= ecc) break;
      ecc = ecc2;
      s = s2;
    }
    std::queue<int> q;
    q.push(s);
    vis[s] = 1;
    while (!q.empty()) {
      int v = q.front();
      q.pop();
      order.push_back(v);
      std::vector<int> nb;
      for (int u : adj[v])
        if (!vis[u]) {
          vis[u] = 1;
          nb.push_back(u);
        }
      std::sort(nb.begin(), nb.end(), [&](int x, int y) { return deg[x] != deg[y] ? deg[x] < deg[y] : x < y; });
      for (int u : nb) q.push(u);
    }
  }
  std::reverse(order.begin(), order.end());
  return order;
}


std::string internalize(int nb, int nl, int ng, int ref, const int *fr, const int *to, const double *b,
                        const double *F, const double *theta, const int *gen_bus, const double *pmin,
                        const double *pmax, const double *c, const double *a, const uint8_t *switchable,
                        int form, bool rcm, Internalized *out) {
  Internalized &R = *out;
  std::vector<std::vector<int>> adj(nb);
  for (int l = 0; l < nl; ++l) {
    adj[fr[l]].push_back(to[l]);
    adj[to[l]].push_back(fr[l]);
  }
  for (auto &v : adj) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  R.bus_perm = rcm ? rcm_order(nb, adj) : dfs_tree_order(nb, adj, ref);
  if ((int)R.bus_perm.size() != nb) return "bus ordering failed";
  R.bus_inv.assign(nb, 0);
  for (int i = 0; i < nb; ++i) R.bus_inv[R.bus_perm[i]] = i;
  // branch order: by (larger, smaller) internal endpoint, then original id
  R.br_perm.resize(nl);
  for (int l = 0; l < nl; ++l) R.br_perm[l] = l;
  auto key = [&](int l) {
    int x = R.bus_inv[fr[l]], y = R.bus_inv[to[l]];
    return std::make_pair(std::max(x, y), std::min(x, y));
  };
  std::sort(R.br_perm.begin(), R.br_perm.end(), [&](int x, int y) {
    auto kx = key(x), ky = key(y);
    return kx != ky ? kx < ky : x < y;
  });
  R.br_inv.assign(nl, 0);
  for (int l = 0; l < nl; ++l) R.br_inv[R.br_perm[l]] = l;
  R.bandwidth = 0;
  for (int l = 0; l < nl; ++l) R.bandwidth = std::max(R.bandwidth, std::abs(R.bus_inv[fr[l]] - R.bus_inv[to[l]]));
  NetInternal &N = R.net;
  N.nb = nb;
  N.nl = nl;
  N.ref = R.bus_inv[ref];
  N.form = form;
  // CSR bus -> incident branches in ascending ORIGINAL branch id: the order of
  // every per-bus sum (same as the oracle's ascending scatter, reading A-19)
  std::vector<std::vector<int>> inc(nb);
  for (int l = 0; l < nl; ++l) {
    inc[R.bus_inv[fr[l]]].push_back(l);
    inc[R.bus_inv[to[l]]].push_back(l);
  }
  N.bus_ptr.assign(nb + 1, 0);
  N.bus_inc.clear();
  for (int i = 0; i < nb; ++i) {
    for (int l : inc[i]) N.bus_inc.push_back((R.br_inv[l] << 1) | ((R.bus_inv[to[l]] == i) ? 1 : 0));
    N.bus_ptr[i + 1] = (int)N.bus_inc.size();
  }
  // generators grouped by internal bus, ascending original id
  std::vector<std::vector<int>> gens(nb);
  for (int g = 0; g < ng; ++g) gens[R.bus_inv[gen_bus[g]]].push_back(g);
  N.gen_ptr.assign(nb + 1, 0);
  N.gc.clear(); N.glo.clear(); N.ghi.clear(); N.ga.clear();
  for (int i = 0; i < nb; ++i) {
    for (int g : gens[i]) {
      N.gc.push_back(c[g]);
      N.glo.push_back(pmin[g]);
      N.ghi.push_back(pmax[g]);
      N.ga.push_back(a ? a[g] : 0.0);
    }
    N.gen_ptr[i + 1] = (int)N.gc.size();
  }
  N.theta.resize(nb);
  for (int i = 0; i < nb; ++i) N.theta[i] = theta[R.bus_perm[i]];
  N.bs.resize(nl); N.bt.resize(nl); N.b.resize(nl); N.F.resize(nl); N.sw.resize(nl);
  for (int li = 0; li < nl; ++li) {
    int l = R.br_perm[li];
    N.sw[li] = switchable ? (switchable[l] != 0) : 1;
    N.bs[li] = R.bus_inv[fr[l]];
    N.bt[li] = R.bus_inv[to[l]];
    N.b[li] = b[l];
    N.F[li] = F[l];
  }
  return "";
}

namespace detail {

// greedy interval colouring; returns #colours, slot[id]
int colour(std::vector<Interval> iv, std::vector<int> &slot) {
  std::sort(iv.begin(), iv.end(), [](const Interval &a, const Interval &b) {
    return a.lo != b.lo ? a.lo < b.lo : a.id < b.id;
  });
  typedef std::pair<int, int> E;  // (hi, slot)
  std::priority_queue<E, std::vector<E>, std::greater<E>> active;
  std::set<int> free_slots;
  int n = 0;
  for (const Interval &x : iv) {
    while (!active.empty() && active.top().first < x.lo) {
      free_slots.insert(active.top().second);
      active.pop();
    }
    int s;
    if (!free_slots.empty()) {
      s = *free_slots.begin();
      free_slots.erase(free_slots.begin());
    } else {
      s = n++;
    }
    slot[x.id] = s;
    active.push({x.hi, s});
  }
  return n;
}

// Storage order and slots of one kind of state row (see build_schedule):
// rows with live range <= life go to a ring (one bulk copy per step), the
// others to interval-coloured sticky slots after it.  Returns the ring count.
int place_rows(int n, const std::vector<Interval> &iv, const std::vector<int> &first, int LIFE, std::vector<int> &pos,
               std::vector<int> &perm, std::vector<int> &slot, int *ring, int *nslots) {
    std::vector<int> idx(n);
    for (int i = 0; i < n; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return first[x] < first[y]; });
    std::vector<int> rr, sticky;
    for (int id : idx) (iv[id].hi - first[id] <= LIFE ? rr : sticky).push_back(id);
    pos.assign(n, 0);
    perm.assign(n, 0);
    int p = 0;
    for (int id : rr) { pos[id] = p; perm[p++] = id; }
    for (int id : sticky) { pos[id] = p; perm[p++] = id; }
    int R = 1;
    for (size_t k = 0, j = 0; k < rr.size(); ++k) {  // j: oldest ring row still live at issue time of k
      const int t = iv[rr[k]].lo;                   // issue time (first - P, clamped)
      while (j < k && iv[rr[j]].hi < t) ++j;
      R = std::max(R, (int)(k - j + 1));
    }
    for (size_t k = 0; k < rr.size(); ++k) slot[rr[k]] = (int)(k % R);
    std::vector<Interval> siv;
    for (int id : sticky) siv.push_back({iv[id].lo, iv[id].hi, id});
    std::vector<int> sslot(n, 0);
    const int ns = colour(siv, sslot);
    for (int id : sticky) slot[id] = R + sslot[id];
    *ring = R;
    *nslots = R + ns;
    return (int)rr.size();
}

// Per-step load lists over the three row kinds (ring runs + sticky rows).
struct KindInfo {
  int kind, n, nring, R, bytes;
  const std::vector<int> *first, *pos, *perm, *slot;
};
void build_loads(Schedule &S, int nst, const KindInfo (&kinds)[3], std::vector<int> &row_bytes) {
  S.ld_ptr.assign(nst + 1, 0);
  S.ld.clear();
  row_bytes.assign(nst, 0);
  S.n_copies = 0;
  S.n_sticky_copies = 0;
  std::vector<std::vector<int4_t>> per(nst);
  for (const KindInfo &K : kinds) {
    for (int p0 = 0; p0 < K.nring;) {  // ring rows: positions [0, nring) sorted by first use
      const int st = (*K.first)[(*K.perm)[p0]];
      int p1 = p0;
      while (p1 < K.nring && (*K.first)[(*K.perm)[p1]] == st) ++p1;
      for (int q = p0; q < p1;) {  // split at the ring wrap
        const int sl = q % K.R;
        const int cnt = std::min(p1 - q, K.R - sl);
        per[st].push_back({K.kind, q, cnt, sl});
        q += cnt;
      }
      p0 = p1;
    }
    for (int p = K.nring; p < K.n; ++p) {  // sticky rows
      const int id = (*K.perm)[p];
      per[(*K.first)[id]].push_back({K.kind, p, 1, (*K.slot)[id]});
      ++S.n_sticky_copies;
    }
  }
  for (int st = 0; st < nst; ++st) {
    for (const int4_t &x : per[st]) {
      S.ld.push_back(x);
      row_bytes[st] += x.c * kinds[x.a].bytes;
    }
    S.n_copies += (int)per[st].size();
    S.ld_ptr[st + 1] = (int)S.ld.size();
  }
}

// Shared-memory layout of the sweep kernel for a built schedule.
void layout_smem(Schedule &S, int nl, int nw) {
  const int RB = S.row_bytes, BR = S.br_row_bytes;
  auto al = [](int x) { return (x + 127) & ~127; };
  int off = 0;
  // full[S], empty[S], A-done[4], B-done[4] mbarriers, then the part's step
  // range (2 int, padded to 16 bytes), then per stage 4 item counters
  S.off_bar = off;
  off = al(off + 16 * S.S + 64 + 16 + 16 * S.S);
  const int TS = 32 * S.V;  // per-tile instance slots (a lane's instances are below 32 V)
  S.off_frz = off;  // frozen flags [TS] int, then running best and previous g [TS] double
  off = al(off + 4 * TS + 2 * 8 * TS);
  S.off_obm = off;  // per-tile outage bitmap over branches
  off = al(off + 4 * ((nl + 31) / 32 + 1));
  S.off_outs = off;  // per-instance outage lists of the tile
  off = al(off + 4 * TS * 8);
  S.off_prog = off;
  off = al(off + S.S * al(S.max_prog_bytes));
  // state / minimiser pools; lanes past the tile width read past a pool's
  // last slot: lane l reads 16 bytes at 16 l (and, 4 instances per lane, at
  // 4 W + 16 l) of a row of 8 W bytes
  const int pad = std::max(0, 512 + (S.V == 4 ? 4 * S.W : 0) - RB);
  S.off_brp = off;
  off = al(off + S.n_br_slots * BR + pad);
  S.off_lamp = off;
  off = al(off + S.n_lam_slots * RB + pad);
  S.off_dp = off;
  off = al(off + S.n_d_slots * RB + pad);
  S.off_th = off;  // theta*_i code rows
  off = al(off + S.n_th_slots * S.code_row_bytes);
  S.off_fc = off;  // f*_l code rows (F2)
  off = al(off + S.n_f_slots * S.code_row_bytes);
  // the per-warp dual-value partials [nw][TS] are needed only at the end of
  // a sweep, when every pool is dead: they alias the pools
  S.off_red = S.off_brp;
  off = std::max(off, al(S.off_brp + 8 * TS * nw));
  S.total = off;
}

}  // namespace detail

using namespace detail;

namespace {
std::string build_schedule_kvl(const NetInternal &net, int CH, int P, int W, int nw, Schedule *out,
                               const CycleBasis &Y);
}  // namespace

size_t Schedule::smem_bytes(int) const { return (size_t)total; }

std::string build_schedule(const NetInternal &net, int CH, int P, int W, int nw, Schedule *out,
                           const CycleBasis *cyc) {
  if (net.form == 2) {
    if (!cyc) return "KVL form needs its cycle basis";
    return build_schedule_kvl(net, CH, P, W, nw, out, *cyc);
  }
  Schedule &S = *out;
  const int nb = net.nb, nl = net.nl;
  const bool f1 = net.form == 1;
  if (W < 2 || W > 64 || (W & 1)) return "tile width must be even in [2, 64]";
  S.CH = CH;
  S.P = P;
  S.S = P + 1;
  S.W = W;
  S.nch = (nb + CH - 1) / CH;
  S.nsteps = S.nch + 2;
  S.row_bytes = 8 * W;
  S.br_row_bytes = f1 ? 16 * W : 8 * W;
  S.V = 2;
  S.C = 1;
  S.part_bus0 = {0, nb};
  const int nch = S.nch, nst = S.nsteps, RB = S.row_bytes, BR = S.br_row_bytes;
  auto chunk = [&](int bus) { return bus / CH; };
  std::vector<int> hi(nl), lo(nl);
  for (int l = 0; l < nl; ++l) {
    hi[l] = std::max(net.bs[l], net.bt[l]);
    lo[l] = std::min(net.bs[l], net.bt[l]);
    if (l > 0 && hi[l] < hi[l - 1]) return "internal branch order not sorted by larger endpoint";
  }
  // B(c): branches whose larger endpoint lies in chunk c (contiguous)
  std::vector<int> bch(nch + 1, 0);
  for (int c = 0, l = 0; c <= nch; ++c) {
    while (l < nl && chunk(hi[l]) < c) ++l;
    bch[c] = (c == nch) ? nl : l;
  }
  // C(c): buses whose last neighbour lies in chunk c ("ready" position rp)
  std::vector<int> rp(nb);
  for (int i = 0; i < nb; ++i) rp[i] = i;
  for (int l = 0; l < nl; ++l) {
    rp[net.bs[l]] = std::max(rp[net.bs[l]], net.bt[l]);
    rp[net.bt[l]] = std::max(rp[net.bt[l]], net.bs[l]);
  }
  std::vector<int> cord(nb), cch(nch + 1, 0);
  for (int i = 0; i < nb; ++i) cord[i] = i;
  std::stable_sort(cord.begin(), cord.end(), [&](int x, int y) { return chunk(rp[x]) < chunk(rp[y]); });
  for (int i = 0; i < nb; ++i) cch[chunk(rp[i]) + 1]++;
  for (int c = 0; c < nch; ++c) cch[c + 1] += cch[c];
  // step of each phase (skewed pipeline): A(c) at step c, B(c) at c+1, C(c) at c+2
  auto stA = [&](int c) { return c; };
  auto stB = [&](int c) { return c + 1; };
  auto stC = [&](int c) { return c + 2; };

  // ---- live ranges in steps ----
  std::vector<Interval> iv_br(nl), iv_lam(nb), iv_d(nb), iv_th(nb), iv_f;
  std::vector<int> br_first(nl), lam_first(nb), d_first(nb);
  for (int l = 0; l < nl; ++l) {  // A at both endpoints, B at the larger one
    br_first[l] = stA(chunk(lo[l]));
    iv_br[l] = {std::max(0, br_first[l] - P), stB(chunk(hi[l])), l};
  }
  for (int i = 0; i < nb; ++i) {
    const int last = stC(chunk(rp[i]));
    int first = last;
    for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e) {
      const int l = net.bus_inc[e] >> 1;
      if (f1) first = std::min(first, stA(chunk(lo[l])));  // u_l in A of both endpoints
      else first = std::min(first, stB(chunk(hi[l])));     // q_l in B
    }
    lam_first[i] = first;
    iv_lam[i] = {std::max(0, first - P), last, i};
    d_first[i] = last;
    iv_d[i] = {std::max(0, last - P), last, i};
    // theta* code: written A(chunk i); read by B of incident branches and
    // (F1) by C of i and of its neighbours
    int tl = stA(chunk(i));
    for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e) {
      const int l = net.bus_inc[e] >> 1;
      tl = std::max(tl, stB(chunk(hi[l])));
      if (f1) {
        const int j = (net.bs[l] == i) ? net.bt[l] : net.bs[l];
        tl = std::max(tl, stC(chunk(rp[j])));
      }
    }
    if (f1) tl = std::max(tl, stC(chunk(rp[i])));
    iv_th[i] = {stA(chunk(i)), tl + S.pool_gap - 1, i};
  }
  std::vector<int> br_slot(nl), lam_slot(nb), d_slot(nb), th_slot(nb), f_slot(nl, 0);
  S.n_th_slots = colour(iv_th, th_slot);
  S.n_f_slots = 0;
  if (!f1) {  // f*: written B(chunk hi), read C of both endpoints
    iv_f.resize(nl);
    for (int l = 0; l < nl; ++l)
      iv_f[l] = {stB(chunk(hi[l])), std::max(stC(chunk(rp[net.bs[l]])), stC(chunk(rp[net.bt[l]]))) + S.pool_gap - 1, l};
    S.n_f_slots = colour(iv_f, f_slot);
  }

  // ---- storage order and shared-memory slots of the state rows ----
  // Rows of each kind are stored in HBM in load order, short-lived rows
  // (live range <= LIFE steps) first: a step's short-lived rows are then one
  // contiguous range, copied by one TMA bulk copy (two at the ring wrap) into
  // a ring of slots (slot = position mod R, R = the largest number of rows
  // issued-but-not-dead at once).  The few long-lived rows follow in storage
  // and get individual copies into interval-coloured "sticky" slots R, R+1, ...
  const int LIFE = S.ring_life;
  auto place = [&](int n, const std::vector<Interval> &iv, const std::vector<int> &first, std::vector<int> &pos,
                   std::vector<int> &perm, std::vector<int> &slot, int *ring, int *nslots) {
    return place_rows(n, iv, first, LIFE, pos, perm, slot, ring, nslots);
  };
  int ring_lam = 0, ring_d = 0, ring_br = 0;
  const int nr_lam = place(nb, iv_lam, lam_first, S.pos_lam, S.perm_lam, lam_slot, &ring_lam, &S.n_lam_slots);
  const int nr_d = place(nb, iv_d, d_first, S.pos_d, S.perm_d, d_slot, &ring_d, &S.n_d_slots);
  const int nr_br = place(nl, iv_br, br_first, S.pos_br, S.perm_br, br_slot, &ring_br, &S.n_br_slots);
  S.ring_lam = ring_lam;
  S.ring_d = ring_d;
  S.ring_br = ring_br;

  // ---- load lists: per step, ranges of rows (kind, first position, count, first slot) ----
  std::vector<int> row_bytes;
  const KindInfo kinds[3] = {{LD_LAM, nb, nr_lam, ring_lam, RB, &lam_first, &S.pos_lam, &S.perm_lam, &lam_slot},
                             {LD_D, nb, nr_d, ring_d, RB, &d_first, &S.pos_d, &S.perm_d, &d_slot},
                             {LD_BR, nl, nr_br, ring_br, BR, &br_first, &S.pos_br, &S.perm_br, &br_slot}};
  build_loads(S, nst, kinds, row_bytes);

  // ---- program blocks, one per step ----
  S.prog.clear();
  S.prog_off.assign(nst, 0);
  S.prog_bytes.assign(nst, 0);
  S.tx_bytes.assign(nst, 0);
  S.max_prog_bytes = 0;
  for (int st = 0; st < nst; ++st) {
    std::vector<RecA> A;
    std::vector<RecIA2> IA2;
    std::vector<RecIA1> IA1;
    int a0 = 0, b0 = 0;
    const int ca = st;  // A(ca)
    if (ca < nch) {
      a0 = ca * CH;
      const int a1 = std::min(nb, a0 + CH);
      for (int i = a0; i < a1; ++i) {
        RecA r{};
        r.th = th_slot[i] * S.code_row_bytes;
        r.bus = i;
        r.flags = (i == net.ref) ? kAFlagRef : 0;
        r.theta = net.theta[i];
        r.e0 = f1 ? (int)IA1.size() : (int)IA2.size();
        for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e) {
          const int l = net.bus_inc[e] >> 1, to = net.bus_inc[e] & 1;
          if (!f1) {
            RecIA2 x{};
            x.row = br_slot[l] * BR;
            x.br = l;
            x.sb = to ? net.b[l] : -net.b[l];  // w_s += -(b nu) ; w_t += b nu
            IA2.push_back(x);
          } else {
            RecIA1 x{};
            x.row = br_slot[l] * BR;
            x.br = net.sw.empty() || net.sw[l] ? l : -1;
            x.ls = lam_slot[net.bs[l]] * RB;
            x.lt = lam_slot[net.bt[l]] * RB;
            x.sb = to ? -net.b[l] : net.b[l];  // w_s += u ; w_t -= u
            IA1.push_back(x);
          }
        }
        r.e1 = f1 ? (int)IA1.size() : (int)IA2.size();
        A.push_back(r);
      }
    }
    std::vector<RecB> Bv;
    const int cb = st - 1;  // B(cb)
    if (cb >= 0 && cb < nch) {
      b0 = bch[cb];
      for (int l = bch[cb]; l < bch[cb + 1]; ++l) {
        const int s = net.bs[l], t = net.bt[l];
        RecB r{};
        r.row = br_slot[l] * BR;
        r.wpos = S.pos_br[l];
        r.obr = net.sw.empty() || net.sw[l] ? l : -1;
        r.ts = th_slot[s] * S.code_row_bytes;
        r.tt = th_slot[t] * S.code_row_bytes;
        r.ths = net.theta[s];
        r.tht = net.theta[t];
        r.b = net.b[l];
        r.F = net.F[l];
        if (!f1) {
          r.ls = lam_slot[s] * RB;
          r.lt = lam_slot[t] * RB;
          r.fs = f_slot[l] * S.code_row_bytes;
        }
        Bv.push_back(r);
      }
    }
    std::vector<RecC> Cv;
    std::vector<RecG> G;
    std::vector<RecIC2> IC2;
    std::vector<RecIC1> IC1;
    const int cc = st - 2;  // C(cc)
    if (cc >= 0 && cc < nch) {
      for (int j = cch[cc]; j < cch[cc + 1]; ++j) {
        const int i = cord[j];
        RecC r{};
        r.wpos = S.pos_lam[i];
        r.ls = lam_slot[i] * RB;
        r.ds = d_slot[i] * RB;
        r.g0 = (int)G.size();
        for (int g = net.gen_ptr[i]; g < net.gen_ptr[i + 1]; ++g)
          G.push_back(RecG{net.gc[g], net.glo[g], net.ghi[g], net.ga[g]});
        r.g1 = (int)G.size();
        r.e0 = f1 ? (int)IC1.size() : (int)IC2.size();
        for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e) {
          const int l = net.bus_inc[e] >> 1, to = net.bus_inc[e] & 1;
          if (!f1) {
            RecIC2 x{};
            x.f = f_slot[l] * S.code_row_bytes;
            x.br = l;
            x.sF = to ? net.F[l] : -net.F[l];  // d/dlambda: +f* at the to bus, -f* at the from bus
            IC2.push_back(x);
          } else {
            RecIC1 x{};
            x.ts = th_slot[net.bs[l]] * S.code_row_bytes;
            x.tt = th_slot[net.bt[l]] * S.code_row_bytes;
            x.ths = net.theta[net.bs[l]];
            x.tht = net.theta[net.bt[l]];
            x.br = net.sw.empty() || net.sw[l] ? l : -1;
            x.sb = to ? net.b[l] : -net.b[l];  // +phi at the to bus, -phi at the from bus
            IC1.push_back(x);
          }
        }
        r.e1 = f1 ? (int)IC1.size() : (int)IC2.size();
        Cv.push_back(r);
      }
    }
    // ---- balance the step over the nw consumer warps: per phase, items in
    // decreasing estimated cost go to the least-loaded warp (loads accumulate
    // over A, B, C); each warp's items are then contiguous, and a table of
    // [3][nw+1] offsets tells warp w its range.  A warp waits for every warp's
    // A of the previous step, so the per-step maximum is what counts.
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
          if (load[v] < load[w]) w = v;
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
    // estimated issue cost (instructions per warp) of an item
    const long cw[6] = {30, f1 ? 20 : 12, f1 ? 60 : 70, 35, f1 ? 20 : 12, 25};  // A0 Adeg B C0 Cdeg Cgen
    balance(A, [&](const RecA &r) { return cw[0] + cw[1] * (r.e1 - r.e0); }, 0);
    balance(Bv, [&](const RecB &) { return cw[2]; }, 1);
    balance(Cv, [&](const RecC &r) { return cw[3] + cw[4] * (r.e1 - r.e0) + cw[5] * (r.g1 - r.g0); }, 2);

    std::vector<uint8_t> blk(kProgHeaderBytes, 0);
    int32_t hd[PH_COUNT] = {0};
    auto app = [&](const void *p, size_t n) {
      size_t off = (blk.size() + 15) & ~size_t(15);
      blk.resize(off + n);
      if (n) memcpy(blk.data() + off, p, n);
      return (int32_t)off;
    };
    hd[PH_NA] = (int)A.size();
    hd[PH_NIA] = f1 ? (int)IA1.size() : (int)IA2.size();
    hd[PH_NB] = (int)Bv.size();
    hd[PH_NC] = (int)Cv.size();
    hd[PH_NIC] = f1 ? (int)IC1.size() : (int)IC2.size();
    hd[PH_NG] = (int)G.size();
    hd[PH_A0] = a0;
    hd[PH_B0] = b0;
    // items are dealt round-robin to the nw consumer warps in the order A, B, C:
    // warp w starts B at (w - nA) mod nw and C at (w - nA - nB) mod nw
    hd[PH_OFF_W] = app(detail::warp_rows(wtab, nw).data(), 16 * (size_t)nw);
    hd[PH_OFF_A] = app(A.data(), A.size() * sizeof(RecA));
    hd[PH_OFF_IA] = f1 ? app(IA1.data(), IA1.size() * sizeof(RecIA1)) : app(IA2.data(), IA2.size() * sizeof(RecIA2));
    hd[PH_OFF_B] = app(Bv.data(), Bv.size() * sizeof(RecB));
    hd[PH_OFF_C] = app(Cv.data(), Cv.size() * sizeof(RecC));
    hd[PH_OFF_G] = app(G.data(), G.size() * sizeof(RecG));
    hd[PH_OFF_IC] = f1 ? app(IC1.data(), IC1.size() * sizeof(RecIC1)) : app(IC2.data(), IC2.size() * sizeof(RecIC2));
    blk.resize((blk.size() + 15) & ~size_t(15), 0);
    hd[PH_BYTES] = (int32_t)blk.size();
    memcpy(blk.data(), hd, sizeof hd);
    S.prog_off[st] = (long long)S.prog.size();
    S.prog_bytes[st] = (int)blk.size();
    S.prog.insert(S.prog.end(), blk.begin(), blk.end());
    S.max_prog_bytes = std::max(S.max_prog_bytes, (int)blk.size());
    S.tx_bytes[st] = S.prog_bytes[st] + row_bytes[st];
  }

  S.part_step0 = {0, nst};
  layout_smem(S, nl, nw);
  return "";
}

namespace {

// ============================================================================
// KVL (cycle-basis) form on the batched path.  Steps s = 0..nch:
//   B(s)     branches whose larger endpoint is in chunk s: q_l from the kappa
//            of the cycles through l and lambda_s, lambda_t -> f* code, q f
//   C(s-1)   buses whose last neighbour is in chunk s-1 (as F2): lambda'
//   D(s-1)   cycles whose last branch is in chunk s-1: sum C x f* -> kappa'
// Rows: lambda (B of incident branches .. C), d (C), kappa (first B of a
// cycle branch .. D); f* codes: B .. last C / D reader.
std::string build_schedule_kvl(const NetInternal &net, int CH, int P, int W, int nw, Schedule *out,
                               const CycleBasis &Y) {
  Schedule &S = *out;
  const int nb = net.nb, nl = net.nl, nc = Y.nc;
  if (W < 2 || W > 64 || (W & 1)) return "tile width must be even in [2, 64]";
  S.CH = CH;
  S.P = P;
  S.S = P + 1;
  S.W = W;
  S.nch = (nb + CH - 1) / CH;
  S.nsteps = S.nch + 1;
  S.row_bytes = 8 * W;
  S.br_row_bytes = 8 * W;  // kappa rows
  S.V = 2;
  S.C = 1;
  S.part_bus0 = {0, nb};
  const int nch = S.nch, nst = S.nsteps, RB = S.row_bytes, CRB = S.code_row_bytes;
  auto chunk = [&](int bus) { return bus / CH; };
  std::vector<int> hi(nl);
  for (int l = 0; l < nl; ++l) {
    hi[l] = std::max(net.bs[l], net.bt[l]);
    if (l > 0 && hi[l] < hi[l - 1]) return "internal branch order not sorted by larger endpoint";
  }
  auto stB = [&](int l) { return chunk(hi[l]); };
  std::vector<int> rp(nb);
  for (int i = 0; i < nb; ++i) rp[i] = i;
  for (int l = 0; l < nl; ++l) {
    rp[net.bs[l]] = std::max(rp[net.bs[l]], net.bt[l]);
    rp[net.bt[l]] = std::max(rp[net.bt[l]], net.bs[l]);
  }
  auto stC = [&](int i) { return chunk(rp[i]) + 1; };
  std::vector<int> stD(nc), firstK(nc);
  std::vector<std::vector<std::pair<int, int>>> bcyc(nl);  // cycles through a branch, ascending k
  for (int k = 0; k < nc; ++k) {
    int mx = 0, mn = nst;
    for (int e = Y.cp[k]; e < Y.cp[k + 1]; ++e) {
      const int l = Y.cb[e];
      mx = std::max(mx, stB(l));
      mn = std::min(mn, stB(l));
      bcyc[l].push_back({k, Y.cs[e]});
    }
    stD[k] = mx + 1;
    firstK[k] = mn;
  }
  // ---- live ranges ----
  std::vector<Interval> iv_lam(nb), iv_d(nb), iv_k(nc), iv_f(nl);
  std::vector<int> lam_first(nb), d_first(nb);
  for (int i = 0; i < nb; ++i) {
    const int last = stC(i);
    int first = last;
    for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e) first = std::min(first, stB(net.bus_inc[e] >> 1));
    lam_first[i] = first;
    iv_lam[i] = {std::max(0, first - P), last, i};
    d_first[i] = last;
    iv_d[i] = {std::max(0, last - P), last, i};
  }
  for (int k = 0; k < nc; ++k) iv_k[k] = {std::max(0, firstK[k] - P), stD[k], k};
  for (int l = 0; l < nl; ++l) {
    int last = std::max(stC(net.bs[l]), stC(net.bt[l]));
    for (auto &kc : bcyc[l]) last = std::max(last, stD[kc.first]);
    iv_f[l] = {stB(l), last + S.pool_gap - 1, l};
  }
  std::vector<int> lam_slot(nb), d_slot(nb), k_slot(nc), f_slot(nl);
  S.n_th_slots = 0;
  S.n_f_slots = colour(iv_f, f_slot);
  const int LIFE = S.ring_life;
  int ring_lam = 0, ring_d = 0, ring_k = 0;
  const int nr_lam = place_rows(nb, iv_lam, lam_first, LIFE, S.pos_lam, S.perm_lam, lam_slot, &ring_lam, &S.n_lam_slots);
  const int nr_d = place_rows(nb, iv_d, d_first, LIFE, S.pos_d, S.perm_d, d_slot, &ring_d, &S.n_d_slots);
  const int nr_k = place_rows(nc, iv_k, firstK, LIFE, S.pos_br, S.perm_br, k_slot, &ring_k, &S.n_br_slots);
  S.ring_lam = ring_lam;
  S.ring_d = ring_d;
  S.ring_br = ring_k;
  std::vector<int> row_bytes;
  const KindInfo kinds[3] = {{LD_LAM, nb, nr_lam, ring_lam, RB, &lam_first, &S.pos_lam, &S.perm_lam, &lam_slot},
                             {LD_D, nb, nr_d, ring_d, RB, &d_first, &S.pos_d, &S.perm_d, &d_slot},
                             {LD_BR, nc, nr_k, ring_k, RB, &firstK, &S.pos_br, &S.perm_br, &k_slot}};
  build_loads(S, nst, kinds, row_bytes);
  // items per step
  std::vector<std::vector<int>> Cst(nst), Dst(nst);
  for (int i = 0; i < nb; ++i) Cst[stC(i)].push_back(i);
  for (int k = 0; k < nc; ++k) Dst[stD[k]].push_back(k);
  // ---- program blocks ----
  S.prog.clear();
  S.prog_off.assign(nst, 0);
  S.prog_bytes.assign(nst, 0);
  S.tx_bytes.assign(nst, 0);
  S.max_prog_bytes = 0;
  const bool has_sw = !net.sw.empty();
  for (int st = 0; st < nst; ++st) {
    std::vector<RecBK> Bv;
    std::vector<RecBKe> BKe;
    if (st < nch) {
      for (int l = 0; l < nl; ++l) {
        if (stB(l) != st) continue;
        RecBK r{};
        r.ls = lam_slot[net.bs[l]] * RB;
        r.lt = lam_slot[net.bt[l]] * RB;
        r.fs = f_slot[l] * CRB;
        r.obr = (!has_sw || net.sw[l]) ? l : -1;
        r.br = l;
        r.x = (net.b[l] > 0.0) ? 1.0 / net.b[l] : 0.0;
        r.F = (net.b[l] > 0.0) ? net.F[l] : 0.0;  // b = 0: an open circuit
        r.e0 = (int)BKe.size();
        for (auto &kc : bcyc[l])  // (a cycle whose defining branch has b = 0 is inactive: no term)
          if (net.b[Y.def[kc.first]] > 0.0) BKe.push_back(RecBKe{k_slot[kc.first] * RB, kc.second});
        r.e1 = (int)BKe.size();
        Bv.push_back(r);
      }
    }
    std::vector<RecC> Cv;
    std::vector<RecG> G;
    std::vector<RecIC2> IC;
    for (int i : Cst[st]) {
      RecC r{};
      r.wpos = S.pos_lam[i];
      r.ls = lam_slot[i] * RB;
      r.ds = d_slot[i] * RB;
      r.g0 = (int)G.size();
      for (int g = net.gen_ptr[i]; g < net.gen_ptr[i + 1]; ++g) G.push_back(RecG{net.gc[g], net.glo[g], net.ghi[g], net.ga[g]});
      r.g1 = (int)G.size();
      r.e0 = (int)IC.size();
      for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e) {
        const int l = net.bus_inc[e] >> 1, to = net.bus_inc[e] & 1;
        const double F = (net.b[l] > 0.0) ? net.F[l] : 0.0;
        IC.push_back(RecIC2{f_slot[l] * CRB, l, to ? F : -F});
      }
      r.e1 = (int)IC.size();
      Cv.push_back(r);
    }
    std::vector<RecD> Dv;
    std::vector<RecDe> De;
    for (int k : Dst[st]) {
      RecD r{};
      r.ks = k_slot[k] * RB;
      r.wpos = S.pos_br[k];
      const int dl = Y.def[k];
      r.dbr = (!has_sw || net.sw[dl]) ? dl : -1;
      r.e0 = (int)De.size();
      if (net.b[dl] > 0.0)  // a b = 0 defining branch: no cycle (gradient 0)
        for (int e = Y.cp[k]; e < Y.cp[k + 1]; ++e) {
          const int m = Y.cb[e];
          const double x = 1.0 / net.b[m], sx = (Y.cs[e] > 0) ? x : -x, F = net.F[m];
          RecDe d{};
          d.fs = f_slot[m] * CRB;
          d.t[0] = (-F) * sx;  // (c F) sx for c = -1, 0, +1 (exact: the oracle's f x with the sign of C)
          d.t[1] = (0.0 * F) * sx;
          d.t[2] = F * sx;
          De.push_back(d);
        }
      r.e1 = (int)De.size();
      Dv.push_back(r);
    }
    // balance B, C, D over the warps (as build_schedule)
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
          if (load[v] < load[w]) w = v;
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
    balance(Bv, [&](const RecBK &r) { return 50L + 10L * (r.e1 - r.e0); }, 0);
    balance(Cv, [&](const RecC &r) { return 35L + 12L * (r.e1 - r.e0) + 25L * (r.g1 - r.g0); }, 1);
    balance(Dv, [&](const RecD &r) { return 30L + 10L * (r.e1 - r.e0); }, 2);
    std::vector<uint8_t> blk(kProgHeaderBytes, 0);
    int32_t hd[PH_COUNT] = {0};
    auto app = [&](const void *p, size_t n) {
      size_t off = (blk.size() + 15) & ~size_t(15);
      blk.resize(off + n);
      if (n) memcpy(blk.data() + off, p, n);
      return (int32_t)off;
    };
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
    blk.resize((blk.size() + 15) & ~size_t(15), 0);
    hd[PH_BYTES] = (int32_t)blk.size();
    memcpy(blk.data(), hd, sizeof hd);
    S.prog_off[st] = (long long)S.prog.size();
    S.prog_bytes[st] = (int)blk.size();
    S.prog.insert(S.prog.end(), blk.begin(), blk.end());
    S.max_prog_bytes = std::max(S.max_prog_bytes, (int)blk.size());
    S.tx_bytes[st] = S.prog_bytes[st] + row_bytes[st];
  }
  S.part_step0 = {0, nst};
  layout_smem(S, nl, nw);
  return "";
}

}  // namespace

}  // namespace dcopf
