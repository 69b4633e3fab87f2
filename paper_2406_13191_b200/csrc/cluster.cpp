// cluster.cpp -- see cluster.h.
#include "cluster.h"

#include <algorithm>
#include <cstring>

namespace dcopf {

namespace {
inline int al16(int x) { return (x + 15) & ~15; }
inline unsigned enc(int rank, int off) { return ((unsigned)rank << kClAddrShift) | (unsigned)off; }
}  // namespace

std::string build_cluster_plan(const NetInternal &net, int C, int max_smem, int nstate, ClusterPlan *out) {
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
