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

// Shared-memory layout of the sweep kernel for a built schedule.
void layout_smem(Schedule &S, int nl, int nw) {
  const int RB = S.row_bytes, BR = S.br_row_bytes;
  auto al = [](int x) { return (x + 127) & ~127; };
  int off = 0;
  // full[S], empty[S], A-done[4], B-done[4] mbarriers, then the part's step
  // range (2 int, padded to 16 bytes)
  S.off_bar = off;
  off = al(off + 16 * S.S + 64 + 16 + S.opt_bytes);
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

size_t Schedule::smem_bytes(int) const { return (size_t)total; }

}  // namespace dcopf
