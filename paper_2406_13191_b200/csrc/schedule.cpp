// schedule.cpp -- see schedule.h.
#include "schedule.h"

#include <algorithm>
#include <cstring>
#include <queue>
#include <set>
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
                        const double *pmax, const double *c, const double *a, int form, bool rcm,
                        Internalized *out) {
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
  N.bs.resize(nl); N.bt.resize(nl); N.b.resize(nl); N.F.resize(nl);
  for (int li = 0; li < nl; ++li) {
    int l = R.br_perm[li];
    N.bs[li] = R.bus_inv[fr[l]];
    N.bt[li] = R.bus_inv[to[l]];
    N.b[li] = b[l];
    N.F[li] = F[l];
  }
  return "";
}

namespace {

struct Interval {
  int lo, hi, id;
};

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

struct Writer {
  std::vector<uint8_t> buf;
  int32_t *hdr() { return reinterpret_cast<int32_t *>(buf.data()); }
  void begin() {
    buf.assign(kProgHeaderBytes, 0);
  }
  template <typename T>
  void put(int field, const std::vector<T> &v) {
    size_t off = (buf.size() + 7) & ~size_t(7);
    buf.resize(off + v.size() * sizeof(T));
    if (!v.empty()) memcpy(buf.data() + off, v.data(), v.size() * sizeof(T));
    hdr()[field] = (int32_t)off;
  }
  void finish() {
    size_t n = (buf.size() + 15) & ~size_t(15);
    buf.resize(n, 0);
    hdr()[PH_BYTES] = (int32_t)n;
  }
};

}  // namespace

size_t Schedule::smem_bytes(int) const { return (size_t)total; }

std::string build_schedule(const NetInternal &net, int CH, int P, int nw, Schedule *out) {
  Schedule &S = *out;
  const int nb = net.nb, nl = net.nl;
  const bool f1 = net.form == 1;
  S.CH = CH;
  S.P = P;
  S.S = P + 1;
  S.nch = (nb + CH - 1) / CH;
  S.br_row_bytes = f1 ? 512 : 256;
  const int nch = S.nch;
  auto chunk = [&](int bus) { return bus / CH; };
  std::vector<int> hi(nl), lo(nl);
  for (int l = 0; l < nl; ++l) {
    hi[l] = std::max(net.bs[l], net.bt[l]);
    lo[l] = std::min(net.bs[l], net.bt[l]);
    if (l > 0 && hi[l] < hi[l - 1]) return "internal branch order not sorted by larger endpoint";
  }
  std::vector<int> bch(nch + 1, 0);
  for (int c = 0, l = 0; c <= nch; ++c) {
    while (l < nl && chunk(hi[l]) < c) ++l;
    bch[c] = (c == nch) ? nl : l;
  }
  // ready position: a bus's C phase runs once all its neighbours passed phase A
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

  // ---- live ranges (in chunks) ----
  // branch state rows (nu or mu pair): A at both endpoints, B at the larger
  std::vector<Interval> iv_br(nl), iv_lam(nb), iv_d(nb), iv_th(nb), iv_f;
  std::vector<int> br_first(nl), lam_first(nb), d_first(nb);
  for (int l = 0; l < nl; ++l) {
    br_first[l] = chunk(lo[l]);
    iv_br[l] = {std::max(0, br_first[l] - P), chunk(hi[l]), l};
  }
  for (int i = 0; i < nb; ++i) {
    int first = chunk(rp[i]), last = chunk(rp[i]);
    for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e) {
      int l = net.bus_inc[e] >> 1;
      if (f1) {
        // A phase of both endpoints reads lambda_s, lambda_t
        first = std::min(first, chunk(lo[l]));
      } else {
        first = std::min(first, chunk(hi[l]));  // B phase of the branch
      }
    }
    lam_first[i] = first;
    iv_lam[i] = {std::max(0, first - P), last, i};
    d_first[i] = chunk(rp[i]);
    iv_d[i] = {std::max(0, d_first[i] - P), chunk(rp[i]), i};
    // theta code: written A(chunk i); read B(chunk hi_l) (+ F1: C of i and neighbours)
    int tl = chunk(i);
    for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e) {
      int l = net.bus_inc[e] >> 1;
      tl = std::max(tl, chunk(hi[l]));
      if (f1) {
        int j = (net.bs[l] == i) ? net.bt[l] : net.bs[l];
        tl = std::max(tl, chunk(rp[j]));
      }
    }
    if (f1) tl = std::max(tl, chunk(rp[i]));
    iv_th[i] = {chunk(i), tl, i};
  }
  std::vector<int> br_slot(nl), lam_slot(nb), d_slot(nb), th_slot(nb), f_slot(nl, 0);
  S.n_br_slots = colour(iv_br, br_slot);
  S.n_lam_slots = colour(iv_lam, lam_slot);
  S.n_d_slots = colour(iv_d, d_slot);
  S.n_th_slots = colour(iv_th, th_slot);
  if (!f1) {
    iv_f.resize(nl);
    for (int l = 0; l < nl; ++l)
      iv_f[l] = {chunk(hi[l]), std::max(chunk(rp[net.bs[l]]), chunk(rp[net.bt[l]])), l};
    S.n_f_slots = colour(iv_f, f_slot);
  }

  // ---- load lists: rows whose first use is chunk c ----
  std::vector<std::vector<int>> lds(nch);
  for (int i = 0; i < nb; ++i) lds[lam_first[i]].push_back((LD_LAM << 30) | i);
  for (int i = 0; i < nb; ++i) lds[d_first[i]].push_back((LD_D << 30) | i);
  for (int l = 0; l < nl; ++l) lds[br_first[l]].push_back((LD_BR << 30) | l);
  S.ld_ptr.assign(nch + 1, 0);
  S.ld_ent.clear();
  S.ld_slot.clear();
  std::vector<int> row_bytes(nch, 0);
  for (int c = 0; c < nch; ++c) {
    for (int x : lds[c]) {
      int kind = (int)((unsigned)x >> 30), ent = x & 0x3fffffff;
      S.ld_ent.push_back(x);
      int slot = kind == LD_LAM ? lam_slot[ent] : (kind == LD_D ? d_slot[ent] : br_slot[ent]);
      S.ld_slot.push_back(slot);
      row_bytes[c] += (kind == LD_BR) ? S.br_row_bytes : 256;
    }
    S.ld_ptr[c + 1] = (int)S.ld_ent.size();
  }

  // ---- program blocks ----
  S.prog.clear();
  S.prog_off.assign(nch, 0);
  S.prog_bytes.assign(nch, 0);
  S.tx_bytes.assign(nch, 0);
  S.max_prog_bytes = 0;
  Writer w;
  for (int c = 0; c < nch; ++c) {
    w.begin();
    const int a0 = c * CH, a1 = std::min(nb, a0 + CH);
    const int nA = a1 - a0;
    std::vector<int> A_ptr(nA + 1, 0), A_ths(nA), IA_row, IA_br, IA_ls, IA_lt;
    std::vector<double> A_th(nA), IA_b;
    for (int a = 0; a < nA; ++a) {
      const int i = a0 + a;
      A_ths[a] = th_slot[i];
      A_th[a] = net.theta[i];
      for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e) {
        int l = net.bus_inc[e] >> 1, to = net.bus_inc[e] & 1;
        IA_row.push_back(br_slot[l] | (to << 31));
        IA_br.push_back(l);
        IA_b.push_back(net.b[l]);
        if (f1) {
          IA_ls.push_back(lam_slot[net.bs[l]]);
          IA_lt.push_back(lam_slot[net.bt[l]]);
        }
      }
      A_ptr[a + 1] = (int)IA_row.size();
    }
    const int b0 = bch[c], nB = bch[c + 1] - bch[c];
    std::vector<int> B_row(nB), B_ts(nB), B_tt(nB), B_ls, B_lt, B_fs;
    std::vector<double> B_b(nB), B_F(nB), B_Ts(nB), B_Tt(nB);
    for (int j = 0; j < nB; ++j) {
      const int l = b0 + j, s = net.bs[l], t = net.bt[l];
      B_row[j] = br_slot[l];
      B_ts[j] = th_slot[s];
      B_tt[j] = th_slot[t];
      B_b[j] = net.b[l];
      B_F[j] = net.F[l];
      B_Ts[j] = net.theta[s];
      B_Tt[j] = net.theta[t];
      if (!f1) {
        B_ls.push_back(lam_slot[s]);
        B_lt.push_back(lam_slot[t]);
        B_fs.push_back(f_slot[l]);
      }
    }
    const int nC = cch[c + 1] - cch[c];
    std::vector<int> C_bus(nC), C_ls(nC), C_ds(nC), C_gp(nC + 1, 0), C_ip(nC + 1, 0), IC_a, IC_br, IC_tt;
    std::vector<double> G_c, G_lo, G_hi, G_a, IC_x, IC_Ts, IC_Tt;
    for (int j = 0; j < nC; ++j) {
      const int i = cord[cch[c] + j];
      C_bus[j] = i;
      C_ls[j] = lam_slot[i];
      C_ds[j] = d_slot[i];
      for (int g = net.gen_ptr[i]; g < net.gen_ptr[i + 1]; ++g) {
        G_c.push_back(net.gc[g]);
        G_lo.push_back(net.glo[g]);
        G_hi.push_back(net.ghi[g]);
        G_a.push_back(net.ga[g]);
      }
      C_gp[j + 1] = (int)G_c.size();
      for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e) {
        int l = net.bus_inc[e] >> 1, to = net.bus_inc[e] & 1;
        IC_br.push_back(l);
        if (!f1) {
          IC_a.push_back(f_slot[l] | (to << 31));
          IC_x.push_back(net.F[l]);
        } else {
          IC_a.push_back(th_slot[net.bs[l]] | (to << 31));
          IC_tt.push_back(th_slot[net.bt[l]]);
          IC_x.push_back(net.b[l]);
          IC_Ts.push_back(net.theta[net.bs[l]]);
          IC_Tt.push_back(net.theta[net.bt[l]]);
        }
      }
      C_ip[j + 1] = (int)IC_a.size();
    }
    int32_t *h = w.hdr();
    h[PH_NA] = nA;
    h[PH_NIA] = (int)IA_row.size();
    h[PH_NB] = nB;
    h[PH_NC] = nC;
    h[PH_NIC] = (int)IC_a.size();
    h[PH_NG] = (int)G_c.size();
    h[PH_A0] = a0;
    h[PH_B0] = b0;
    w.put(PH_A_PTR, A_ptr);
    w.put(PH_A_THS, A_ths);
    w.put(PH_A_TH, A_th);
    w.put(PH_IA_ROW, IA_row);
    w.put(PH_IA_BR, IA_br);
    w.put(PH_IA_B, IA_b);
    w.put(PH_IA_LS, IA_ls);
    w.put(PH_IA_LT, IA_lt);
    w.put(PH_B_ROW, B_row);
    w.put(PH_B_TS, B_ts);
    w.put(PH_B_TT, B_tt);
    w.put(PH_B_B, B_b);
    w.put(PH_B_F, B_F);
    w.put(PH_B_THS, B_Ts);
    w.put(PH_B_THT, B_Tt);
    w.put(PH_B_LS, B_ls);
    w.put(PH_B_LT, B_lt);
    w.put(PH_B_FS, B_fs);
    w.put(PH_C_BUS, C_bus);
    w.put(PH_C_LS, C_ls);
    w.put(PH_C_DS, C_ds);
    w.put(PH_C_GP, C_gp);
    w.put(PH_C_IP, C_ip);
    w.put(PH_G_C, G_c);
    w.put(PH_G_LO, G_lo);
    w.put(PH_G_HI, G_hi);
    w.put(PH_G_A, G_a);
    w.put(PH_IC_A, IC_a);
    w.put(PH_IC_BR, IC_br);
    w.put(PH_IC_X, IC_x);
    w.put(PH_IC_TT, IC_tt);
    w.put(PH_IC_THS, IC_Ts);
    w.put(PH_IC_THT, IC_Tt);
    w.finish();
    S.prog_off[c] = (long long)S.prog.size();
    S.prog_bytes[c] = (int)w.buf.size();
    S.prog.insert(S.prog.end(), w.buf.begin(), w.buf.end());
    S.max_prog_bytes = std::max(S.max_prog_bytes, (int)w.buf.size());
    S.tx_bytes[c] = S.prog_bytes[c] + row_bytes[c];
  }

  // ---- shared-memory layout ----
  auto al = [](int x) { return (x + 127) & ~127; };
  int off = 0;
  S.off_bar = off;
  off = al(off + 16 * S.S);
  S.off_red = off;
  off = al(off + 8 * 32 * nw);
  S.off_frz = off;
  off = al(off + 4 * 32);
  S.off_prog = off;
  off = al(off + S.S * al(S.max_prog_bytes));
  S.off_brp = off;
  off = al(off + S.n_br_slots * S.br_row_bytes);
  S.off_lamp = off;
  off = al(off + S.n_lam_slots * 256);
  S.off_dp = off;
  off = al(off + S.n_d_slots * 256);
  S.off_th = off;
  off = al(off + S.n_th_slots * 8);
  S.off_fc = off;
  off = al(off + S.n_f_slots * 8);
  S.total = off;
  return "";
}

}  // namespace dcopf
