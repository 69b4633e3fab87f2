// cluster.cpp -- see cluster.h.
#include "cluster.h"

#include <algorithm>
#include <cstring>

namespace dcopf {

namespace {
inline int al16(int x) { return (x + 15) & ~15; }
inline unsigned enc(int rank, int off) { return ((unsigned)rank << kClAddrShift) | (unsigned)off; }

// contiguous internal bus ranges balanced on work; branches go with their larger endpoint
void partition(const NetInternal &net, int C, ClusterPlan &P, std::vector<int> &owner, std::vector<int> &bowner) {
  const int nb = net.nb, nl = net.nl;
  std::vector<int> hi(nl);
  std::vector<long> w(nb, 0);
  for (int l = 0; l < nl; ++l) {
    hi[l] = std::max(net.bs[l], net.bt[l]);
    w[hi[l]] += 2;
  }
  for (int i = 0; i < nb; ++i) w[i] += 2 + (net.bus_ptr[i + 1] - net.bus_ptr[i]);
  long total = 0;
  for (long x : w) total += x;
  P.bus_lo.assign(C + 1, nb);
  P.bus_lo[0] = 0;
  {
    long acc = 0;
    int r = 1;
    for (int i = 0; i < nb && r < C; ++i) {
      acc += w[i];
      while (r < C && acc * C >= total * r) P.bus_lo[r++] = i + 1;
    }
    for (; r < C; ++r) P.bus_lo[r] = nb;
  }
  owner.assign(nb, 0);
  for (int r = 0; r < C; ++r)
    for (int i = P.bus_lo[r]; i < P.bus_lo[r + 1]; ++i) owner[i] = r;
  P.br_lo.assign(C + 1, nl);
  for (int r = 0, l = 0; r <= C; ++r) {
    while (l < nl && hi[l] < P.bus_lo[r]) ++l;
    P.br_lo[r] = (r == C) ? nl : l;
  }
  bowner.assign(nl, 0);
  for (int l = 0; l < nl; ++l) bowner[l] = owner[hi[l]];
}

// KVL form: phase B per owned branch (its cycle terms), phase C per owned bus
// (as F2) and per owned cycle (cycle k belongs to the owner of its defining branch)
std::string build_cluster_plan_kvl(const NetInternal &net, int C, int max_smem, int nstate, ClusterPlan *out,
                                   const CycleBasis &Y) {
  ClusterPlan &P = *out;
  const int nb = net.nb, nl = net.nl, nc = Y.nc;
  P = ClusterPlan();
  P.C = C;
  std::vector<int> owner, bowner;
  partition(net, C, P, owner, bowner);
  // internal cycle order: by owner, then canonical k
  std::vector<int> cown(nc), order(nc), cloc(nc);
  for (int k = 0; k < nc; ++k) cown[k] = bowner[Y.def[k]];
  for (int k = 0; k < nc; ++k) order[k] = k;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cown[a] < cown[b]; });
  P.cyc_perm = order;
  P.cyc_lo.assign(C + 1, nc);
  for (int r = 0, x = 0; r <= C; ++r) {
    while (x < nc && cown[order[x]] < r) ++x;
    P.cyc_lo[r] = (r == C) ? nc : x;
  }
  for (int x = 0; x < nc; ++x) cloc[order[x]] = x - P.cyc_lo[cown[order[x]]];
  // per-branch cycle lists (ascending k)
  std::vector<std::vector<std::pair<int, int>>> bcyc(nl);
  for (int k = 0; k < nc; ++k)
    for (int e = Y.cp[k]; e < Y.cp[k + 1]; ++e) bcyc[Y.cb[e]].push_back({k, Y.cs[e]});
  // sizes
  int nbk_max = 1, nce_max = 1, ng_max = 1, nia_max = 1, ncy_max = 1;
  for (int r = 0; r < C; ++r) {
    P.nb_max = std::max(P.nb_max, P.bus_lo[r + 1] - P.bus_lo[r]);
    P.nl_max = std::max(P.nl_max, P.br_lo[r + 1] - P.br_lo[r]);
    ncy_max = std::max(ncy_max, P.cyc_lo[r + 1] - P.cyc_lo[r]);
    int nbk = 0, nce = 0;
    for (int l = P.br_lo[r]; l < P.br_lo[r + 1]; ++l) nbk += (int)bcyc[l].size();
    for (int x = P.cyc_lo[r]; x < P.cyc_lo[r + 1]; ++x) nce += Y.cp[order[x] + 1] - Y.cp[order[x]];
    nbk_max = std::max(nbk_max, nbk);
    nce_max = std::max(nce_max, nce);
    nia_max = std::max(nia_max, net.bus_ptr[P.bus_lo[r + 1]] - net.bus_ptr[P.bus_lo[r]]);
    ng_max = std::max(ng_max, net.gen_ptr[P.bus_lo[r + 1]] - net.gen_ptr[P.bus_lo[r]]);
  }
  const int NB = std::max(P.nb_max, 1), NL = std::max(P.nl_max, 1);
  ClHeader H;
  memset(&H, 0, sizeof H);
  int off = (int)sizeof(ClHeader);
  H.off_A = off;
  H.off_IA = off;
  off = al16(off + nbk_max * (int)sizeof(ClBKe));
  H.off_B = off;
  off = al16(off + NL * (int)sizeof(ClBk));
  H.off_C = off;
  off = al16(off + NB * (int)sizeof(ClC));
  H.off_IC = off;
  off = al16(off + nia_max * (int)sizeof(ClIC2));
  H.off_G = off;
  off = al16(off + ng_max * (int)sizeof(ClG));
  H.off_Cy = off;
  off = al16(off + ncy_max * (int)sizeof(ClCy));
  H.off_CE = off;
  off = al16(off + nce_max * (int)sizeof(ClCe));
  const int blob = off;
  H.off_lam = off;
  off = al16(off + NB * 8);
  H.off_d = off;
  off = al16(off + NB * 8);
  H.off_br = off;  // kappa of the owned cycles
  off = al16(off + ncy_max * 8);
  H.off_th = off;  // (unused)
  H.off_fc = off;  // f* of the owned branches (values)
  off = al16(off + NL * 8);
  H.off_red = off;
  off = al16(off + 512);
  H.off_zero = off;  // a 0.0 that masked cycle terms read
  off = al16(off + 16);
  if (nstate >= 1) {
    H.off_s1l = off;
    off = al16(off + NB * 8);
    H.off_s1b = off;
    off = al16(off + ncy_max * 8);
  }
  if (nstate >= 2) {
    H.off_s2l = off;
    off = al16(off + NB * 8);
    H.off_s2b = off;
    off = al16(off + ncy_max * 8);
  }
  H.blob_bytes = blob;
  P.smem = off;
  if (P.smem > max_smem) return "cluster partition does not fit shared memory";
  if (off >= (1 << kClAddrShift)) return "shared-memory offset exceeds the address encoding";
  P.blob_stride = blob;
  P.blob.assign((size_t)C * blob, 0);
  auto lam_addr = [&](int i) { return enc(owner[i], H.off_lam + 8 * (i - P.bus_lo[owner[i]])); };
  auto fc_addr = [&](int l) { return enc(bowner[l], H.off_fc + 8 * (l - P.br_lo[bowner[l]])); };
  auto kap_addr = [&](int k) { return enc(cown[k], H.off_br + 8 * cloc[k]); };
  auto active = [&](int k) { return net.b[Y.def[k]] > 0.0; };  // b = 0: an open circuit, no cycle
  for (int r = 0; r < C; ++r) {
    uint8_t *base = P.blob.data() + (size_t)r * blob;
    ClHeader h = H;
    const int b0 = P.bus_lo[r], b1 = P.bus_lo[r + 1], l0 = P.br_lo[r], l1 = P.br_lo[r + 1];
    h.nA = b1 - b0;
    h.nB = l1 - l0;
    h.bus0 = b0;
    h.br0 = l0;
    h.ref_local = (net.ref >= b0 && net.ref < b1) ? net.ref - b0 : -1;
    h.nCy = P.cyc_lo[r + 1] - P.cyc_lo[r];
    h.cy0 = P.cyc_lo[r];
    // phase B
    ClBk *Bv = reinterpret_cast<ClBk *>(base + H.off_B);
    ClBKe *BK = reinterpret_cast<ClBKe *>(base + H.off_IA);
    int nk = 0;
    for (int l = l0; l < l1; ++l) {
      ClBk x{};
      x.ls = lam_addr(net.bs[l]);
      x.lt = lam_addr(net.bt[l]);
      x.e0 = nk;
      for (auto &kc : bcyc[l]) {
        ClBKe e{};
        e.kap = active(kc.first) ? kap_addr(kc.first) : enc(r, H.off_zero);
        e.sgn = kc.second;
        e.dbr = Y.def[kc.first];
        BK[nk++] = e;
      }
      x.e1 = nk;
      x.x = (net.b[l] > 0.0) ? 1.0 / net.b[l] : 0.0;
      x.F = (net.b[l] > 0.0) ? net.F[l] : 0.0;  // b = 0: no flow in this form
      x.br = l;
      Bv[l - l0] = x;
    }
    h.nIA = nk;
    // phase C: buses (as F2) and cycles
    ClC *Cc = reinterpret_cast<ClC *>(base + H.off_C);
    ClIC2 *IC = reinterpret_cast<ClIC2 *>(base + H.off_IC);
    ClG *G = reinterpret_cast<ClG *>(base + H.off_G);
    int ne = 0, ng = 0;
    for (int i = b0; i < b1; ++i) {
      ClC c{};
      c.g0 = ng;
      for (int g = net.gen_ptr[i]; g < net.gen_ptr[i + 1]; ++g) G[ng++] = ClG{net.gc[g], net.glo[g], net.ghi[g], net.ga[g]};
      c.g1 = ng;
      c.e0 = ne;
      for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e) {
        const int l = net.bus_inc[e] >> 1, tt = net.bus_inc[e] & 1;
        ClIC2 y{};
        y.f = fc_addr(l);
        y.sgn = tt ? 1 : -1;
        IC[ne++] = y;
      }
      c.e1 = ne;
      Cc[i - b0] = c;
    }
    h.nIC = ne;
    h.nG = ng;
    ClCy *Cy = reinterpret_cast<ClCy *>(base + H.off_Cy);
    ClCe *CE = reinterpret_cast<ClCe *>(base + H.off_CE);
    int nce = 0;
    for (int x = P.cyc_lo[r]; x < P.cyc_lo[r + 1]; ++x) {
      const int k = order[x];
      ClCy c{};
      c.e0 = nce;
      c.dbr = Y.def[k];
      if (active(k))
        for (int e = Y.cp[k]; e < Y.cp[k + 1]; ++e) {
          const int m = Y.cb[e];
          ClCe y{};
          y.f = fc_addr(m);
          y.sx = (Y.cs[e] > 0) ? 1.0 / net.b[m] : -(1.0 / net.b[m]);  // C_km x_m (x_m > 0 on an active cycle)
          CE[nce++] = y;
        }
      c.e1 = nce;
      Cy[x - P.cyc_lo[r]] = c;
    }
    h.nCE = nce;
    memcpy(base, &h, sizeof h);
  }
  return "";
}
}  // namespace

std::string build_cycle_basis(int nb, int nl, int ref, const int *fr, const int *to, const double *b,
                              const uint8_t *sw, CycleBasis *out) {
  CycleBasis &Y = *out;
  Y = CycleBasis();
  std::vector<std::vector<int>> inc(nb);
  for (int l = 0; l < nl; ++l) {  // ascending branch id per bus
    inc[fr[l]].push_back(l);
    inc[to[l]].push_back(l);
  }
  std::vector<int> parent(nb, -2), pbr(nb, -1), depth(nb, 0), queue;
  queue.reserve(nb);
  Y.is_tree.assign(nl, 0);
  parent[ref] = -1;
  queue.push_back(ref);
  for (size_t h = 0; h < queue.size(); ++h) {
    const int u = queue[h];
    for (int m : inc[u]) {
      const int v = (fr[m] == u) ? to[m] : fr[m];
      if (!(b[m] > 0.0) || (sw && sw[m]) || parent[v] != -2) continue;
      parent[v] = u;
      pbr[v] = m;
      depth[v] = depth[u] + 1;
      Y.is_tree[m] = 1;
      queue.push_back(v);
    }
  }
  if ((int)queue.size() != nb) return "cycle basis: never-switched branches with b > 0 do not connect the network";
  Y.cp.push_back(0);
  std::vector<std::pair<int, int>> cyc;
  for (int l = 0; l < nl; ++l) {
    if (Y.is_tree[l]) continue;
    cyc.clear();
    cyc.push_back({l, 1});  // l from its from bus to its to bus
    int a = to[l], c = fr[l];  // then the tree path from t_l back to s_l
    while (a != c) {
      if (depth[a] >= depth[c]) {  // a climbs: traversed a -> parent(a)
        const int m = pbr[a];
        cyc.push_back({m, fr[m] == a ? 1 : -1});
        a = parent[a];
      } else {  // c climbs: traversed parent(c) -> c
        const int m = pbr[c];
        cyc.push_back({m, to[m] == c ? 1 : -1});
        c = parent[c];
      }
    }
    std::sort(cyc.begin(), cyc.end());
    Y.def.push_back(l);
    for (auto &e : cyc) {
      Y.cb.push_back(e.first);
      Y.cs.push_back(e.second);
    }
    Y.cp.push_back((int)Y.cb.size());
  }
  Y.nc = (int)Y.def.size();
  return "";
}

std::string build_cluster_plan(const NetInternal &net, int C, int max_smem, int nstate, ClusterPlan *out,
                               const CycleBasis *cyc) {
  if (net.form == 2) {
    if (!cyc) return "KVL form needs its cycle basis";
    return build_cluster_plan_kvl(net, C, max_smem, nstate, out, *cyc);
  }
  ClusterPlan &P = *out;
  const int nb = net.nb, nl = net.nl;
  const bool f1 = net.form == 1;
  if (C < 1 || C > 16) return "cluster size must be in [1, 16]";
  P = ClusterPlan();
  P.C = C;
  // ---- partition: contiguous internal bus ranges balanced on (1 + owned branches + incidence) ----
  std::vector<int> hi(nl);
  std::vector<long> w(nb, 0);
  for (int l = 0; l < nl; ++l) {
    hi[l] = std::max(net.bs[l], net.bt[l]);
    w[hi[l]] += 2;
  }
  for (int i = 0; i < nb; ++i) w[i] += 2 + (net.bus_ptr[i + 1] - net.bus_ptr[i]);
  long total = 0;
  for (long x : w) total += x;
  P.bus_lo.assign(C + 1, nb);
  P.bus_lo[0] = 0;
  {
    long acc = 0;
    int r = 1;
    for (int i = 0; i < nb && r < C; ++i) {
      acc += w[i];
      while (r < C && acc * C >= total * r) P.bus_lo[r++] = i + 1;
    }
    for (; r < C; ++r) P.bus_lo[r] = nb;
  }
  std::vector<int> owner(nb);
  for (int r = 0; r < C; ++r)
    for (int i = P.bus_lo[r]; i < P.bus_lo[r + 1]; ++i) owner[i] = r;
  P.br_lo.assign(C + 1, nl);
  for (int r = 0, l = 0; r <= C; ++r) {
    while (l < nl && hi[l] < P.bus_lo[r]) ++l;
    P.br_lo[r] = (r == C) ? nl : l;
  }
  std::vector<int> bowner(nl);
  for (int l = 0; l < nl; ++l) bowner[l] = owner[hi[l]];
  // ---- sizes ----
  int nia_max = 0, ng_max = 0;
  for (int r = 0; r < C; ++r) {
    P.nb_max = std::max(P.nb_max, P.bus_lo[r + 1] - P.bus_lo[r]);
    P.nl_max = std::max(P.nl_max, P.br_lo[r + 1] - P.br_lo[r]);
    const int e = net.bus_ptr[P.bus_lo[r + 1]] - net.bus_ptr[P.bus_lo[r]];
    const int g = net.gen_ptr[P.bus_lo[r + 1]] - net.gen_ptr[P.bus_lo[r]];
    nia_max = std::max(nia_max, e);
    ng_max = std::max(ng_max, g);
  }
  const int NB = std::max(P.nb_max, 1), NL = std::max(P.nl_max, 1), NIA = std::max(nia_max, 1),
            NG = std::max(ng_max, 1);
  const int BRW = f1 ? 2 : 1;
  ClHeader H;
  memset(&H, 0, sizeof H);
  int off = (int)sizeof(ClHeader);
  H.off_A = off;
  off = al16(off + NB * (int)sizeof(ClA));
  H.off_IA = off;
  off = al16(off + NIA * (int)(f1 ? sizeof(ClIA1) : sizeof(ClIA2)));
  H.off_B = off;
  off = al16(off + NL * (int)sizeof(ClB));
  H.off_C = off;
  off = al16(off + NB * (int)sizeof(ClC));
  H.off_IC = off;
  off = al16(off + NIA * (int)(f1 ? sizeof(ClIC1) : sizeof(ClIC2)));
  H.off_G = off;
  off = al16(off + NG * (int)sizeof(ClG));
  const int blob = off;
  H.off_lam = off;
  off = al16(off + NB * 8);
  H.off_d = off;
  off = al16(off + NB * 8);
  H.off_br = off;
  off = al16(off + NL * 8 * BRW);
  H.off_th = off;
  off = al16(off + NB * 8);
  H.off_fc = off;
  off = al16(off + NL * 8);
  H.off_red = off;  // [0] partial value, [8..40) per-warp partials, [40] frozen flag
  off = al16(off + 512);
  if (nstate >= 1) {
    H.off_s1l = off;
    off = al16(off + NB * 8);
    H.off_s1b = off;
    off = al16(off + NL * 8 * BRW);
  }
  if (nstate >= 2) {
    H.off_s2l = off;
    off = al16(off + NB * 8);
    H.off_s2b = off;
    off = al16(off + NL * 8 * BRW);
  }
  H.blob_bytes = blob;
  P.smem = off;
  if (P.smem > max_smem) return "cluster partition does not fit shared memory";
  if (off >= (1 << kClAddrShift)) return "shared-memory offset exceeds the address encoding";
  P.blob_stride = blob;
  P.blob.assign((size_t)C * blob, 0);

  auto lam_addr = [&](int i) { return enc(owner[i], H.off_lam + 8 * (i - P.bus_lo[owner[i]])); };
  auto th_addr = [&](int i) { return enc(owner[i], H.off_th + 8 * (i - P.bus_lo[owner[i]])); };
  auto br_addr = [&](int l) { return enc(bowner[l], H.off_br + 8 * BRW * (l - P.br_lo[bowner[l]])); };
  auto fc_addr = [&](int l) { return enc(bowner[l], H.off_fc + 8 * (l - P.br_lo[bowner[l]])); };

  for (int r = 0; r < C; ++r) {
    uint8_t *base = P.blob.data() + (size_t)r * blob;
    ClHeader h = H;
    const int b0 = P.bus_lo[r], b1 = P.bus_lo[r + 1], l0 = P.br_lo[r], l1 = P.br_lo[r + 1];
    h.nA = b1 - b0;
    h.nB = l1 - l0;
    h.bus0 = b0;
    h.br0 = l0;
    h.ref_local = (net.ref >= b0 && net.ref < b1) ? net.ref - b0 : -1;
    ClA *A = reinterpret_cast<ClA *>(base + H.off_A);
    ClC *Cc = reinterpret_cast<ClC *>(base + H.off_C);
    ClG *G = reinterpret_cast<ClG *>(base + H.off_G);
    int ne = 0, ng = 0;
    for (int i = b0; i < b1; ++i) {
      ClA a{};
      ClC c{};
      a.e0 = c.e0 = ne;
      a.theta = net.theta[i];
      c.g0 = ng;
      for (int g = net.gen_ptr[i]; g < net.gen_ptr[i + 1]; ++g) G[ng++] = ClG{net.gc[g], net.glo[g], net.ghi[g], net.ga[g]};
      c.g1 = ng;
      for (int e = net.bus_ptr[i]; e < net.bus_ptr[i + 1]; ++e, ++ne) {
        const int l = net.bus_inc[e] >> 1, to = net.bus_inc[e] & 1;
        if (!f1) {
          ClIA2 x{};
          x.nu = br_addr(l);
          x.br = l;
          x.sb = to ? net.b[l] : -net.b[l];  // w_s += -(b nu), w_t += b nu
          reinterpret_cast<ClIA2 *>(base + H.off_IA)[ne] = x;
          ClIC2 y{};
          y.f = fc_addr(l);
          y.sgn = to ? 1 : -1;  // d/dlambda: +f* at the to bus, -f* at the from bus
          reinterpret_cast<ClIC2 *>(base + H.off_IC)[ne] = y;
        } else {
          ClIA1 x{};
          x.mu = br_addr(l);
          x.ls = lam_addr(net.bs[l]);
          x.lt = lam_addr(net.bt[l]);
          x.br = l;
          x.sb = to ? -net.b[l] : net.b[l];  // w_s += u, w_t -= u
          reinterpret_cast<ClIA1 *>(base + H.off_IA)[ne] = x;
          ClIC1 y{};
          y.ts = th_addr(net.bs[l]);
          y.tt = th_addr(net.bt[l]);
          y.br = l;
          y.sb = to ? net.b[l] : -net.b[l];  // +phi at the to bus, -phi at the from bus
          reinterpret_cast<ClIC1 *>(base + H.off_IC)[ne] = y;
        }
      }
      a.e1 = c.e1 = ne;
      A[i - b0] = a;
      Cc[i - b0] = c;
    }
    h.nIA = h.nIC = ne;
    h.nG = ng;
    ClB *Bv = reinterpret_cast<ClB *>(base + H.off_B);
    for (int l = l0; l < l1; ++l) {
      ClB x{};
      x.ts = th_addr(net.bs[l]);
      x.tt = th_addr(net.bt[l]);
      x.ls = lam_addr(net.bs[l]);
      x.lt = lam_addr(net.bt[l]);
      x.b = net.b[l];
      x.F = net.F[l];
      x.br = l;
      Bv[l - l0] = x;
    }
    memcpy(base, &h, sizeof h);
  }
  return "";
}

}  // namespace dcopf
