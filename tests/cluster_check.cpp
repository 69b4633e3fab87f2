// Host-only checker of the cluster path's shared-memory plan
// (paper_2406_13191_b200/csrc/cluster.cpp): decodes every (rank, offset)
// address in every CTA's blob and verifies it names the value the record
// expects (the right bus's lambda / theta, the right branch's nu / mu / f*, the
// right cycle's kappa), that every bus, branch and cycle is owned exactly
// once, and -- KVL form -- that the canonical cycle basis consists of closed
// loops.  Input on stdin: nb nl ref form C, then nl lines "s t b F sw".
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../paper_2406_13191_b200/csrc/cluster.h"

using namespace dcopf;

static int bad = 0;
#define CHECK(c, ...)                    \
  do {                                   \
    if (!(c)) {                          \
      if (bad < 10) printf(__VA_ARGS__); \
      ++bad;                             \
    }                                    \
  } while (0)

int main() {
  int nb, nl, ref, form, C;
  if (scanf("%d %d %d %d %d", &nb, &nl, &ref, &form, &C) != 5) return 2;
  std::vector<int> fr(nl), to(nl);
  std::vector<double> b(nl), F(nl), theta(nb, 1.0);
  std::vector<uint8_t> sw(nl);
  for (int l = 0; l < nl; ++l) {
    int s;
    if (scanf("%d %d %lf %lf %d", &fr[l], &to[l], &b[l], &F[l], &s) != 5) return 2;
    sw[l] = (uint8_t)s;
  }
  Internalized in;
  std::vector<int> gen_bus{ref};
  std::vector<double> pmin{0.0}, pmax{1.0}, c{1.0};
  std::string e0 = internalize(nb, nl, 1, ref, fr.data(), to.data(), b.data(), F.data(), theta.data(), gen_bus.data(),
                               pmin.data(), pmax.data(), c.data(), nullptr, sw.data(), form, false, &in);
  if (!e0.empty()) { printf("ERR %s\n", e0.c_str()); return 1; }
  const NetInternal &n = in.net;
  CycleBasis Y, Yi;
  if (form == 2) {
    std::string e1 = build_cycle_basis(nb, nl, ref, fr.data(), to.data(), b.data(), sw.data(), &Y);
    if (!e1.empty()) { printf("ERR %s\n", e1.c_str()); return 1; }
    CHECK(Y.nc == nl - nb + 1, "BAD cycle count %d\n", Y.nc);
    // closed loops: at every bus the signed incidence of the cycle cancels
    for (int k = 0; k < Y.nc; ++k) {
      std::vector<int> net_flow(nb, 0);
      for (int e = Y.cp[k]; e < Y.cp[k + 1]; ++e) {
        const int l = Y.cb[e];
        net_flow[fr[l]] += Y.cs[e];
        net_flow[to[l]] -= Y.cs[e];
        CHECK(e == Y.cp[k] || Y.cb[e - 1] < l, "BAD cycle order\n");
        CHECK(Y.is_tree[l] || l == Y.def[k], "BAD cycle %d holds another non-tree branch\n", k);
      }
      for (int i = 0; i < nb; ++i) CHECK(net_flow[i] == 0, "BAD cycle %d not closed at bus %d\n", k, i);
    }
    for (int l = 0; l < nl; ++l) CHECK(!(sw[l] && Y.is_tree[l]), "BAD switchable tree branch %d\n", l);
    if (getenv("DUMP_BASIS")) {  // the library's canonical basis, for comparison with the oracle's
      for (int k = 0; k < Y.nc; ++k) {
        printf("cycle %d %d", Y.def[k], Y.cp[k + 1] - Y.cp[k]);
        for (int e = Y.cp[k]; e < Y.cp[k + 1]; ++e) printf(" %d %d", Y.cb[e], Y.cs[e]);
        printf("\n");
      }
    }
    Yi = Y;
    for (int &l : Yi.def) l = in.br_inv[l];
    for (int &l : Yi.cb) l = in.br_inv[l];
  }
  ClusterPlan P;
  std::string e2 = build_cluster_plan(n, C, 232448, 0, &P, form == 2 ? &Yi : nullptr);  // B200 opt-in smem
  if (!e2.empty()) { printf("ERR %s\n", e2.c_str()); return 1; }
  const int BRW = form == 1 ? 2 : 1;
  std::vector<int> seen_bus(nb, 0), seen_br(nl, 0), seen_cyc(form == 2 ? Y.nc : 0, 0);
  std::vector<int> owner(nb), bowner(nl);
  for (int r = 0; r < C; ++r) {
    for (int i = P.bus_lo[r]; i < P.bus_lo[r + 1]; ++i) owner[i] = r;
    for (int l = P.br_lo[r]; l < P.br_lo[r + 1]; ++l) bowner[l] = r;
  }
  const ClHeader &H0 = *reinterpret_cast<const ClHeader *>(P.blob.data());
  auto dec = [&](unsigned a, int *rank) {
    *rank = (int)(a >> kClAddrShift);
    return (int)(a & ((1u << kClAddrShift) - 1));
  };
  auto want_bus = [&](unsigned a, int off_arr, int bus, const char *what) {
    int r, off = dec(a, &r);
    CHECK(r == owner[bus] && off == off_arr + 8 * (bus - P.bus_lo[r]), "BAD %s of bus %d\n", what, bus);
  };
  auto want_br = [&](unsigned a, int off_arr, int stride, int l, const char *what) {
    int r, off = dec(a, &r);
    CHECK(r == bowner[l] && off == off_arr + stride * (l - P.br_lo[r]), "BAD %s of branch %d\n", what, l);
  };
  for (int r = 0; r < C; ++r) {
    const uint8_t *base = P.blob.data() + (size_t)r * P.blob_stride;
    const ClHeader &H = *reinterpret_cast<const ClHeader *>(base);
    CHECK(H.off_lam == H0.off_lam && H.off_br == H0.off_br && H.off_fc == H0.off_fc, "BAD layout differs\n");
    CHECK(H.bus0 == P.bus_lo[r] && H.nA == P.bus_lo[r + 1] - P.bus_lo[r], "BAD bus range\n");
    for (int i = 0; i < H.nA; ++i) seen_bus[H.bus0 + i]++;
    for (int j = 0; j < H.nB; ++j) seen_br[H.br0 + j]++;
    // phase C incidence (every form): f* (F2 / KVL) or theta* (F1) of the right branch / buses
    const ClC *Cc = reinterpret_cast<const ClC *>(base + H.off_C);
    for (int i = 0; i < H.nA; ++i) {
      const int bus = H.bus0 + i;
      CHECK(Cc[i].e1 - Cc[i].e0 == n.bus_ptr[bus + 1] - n.bus_ptr[bus], "BAD C degree\n");
      for (int e = Cc[i].e0; e < Cc[i].e1; ++e) {
        const int l = n.bus_inc[n.bus_ptr[bus] + e - Cc[i].e0] >> 1;
        if (form == 1) {
          const ClIC1 &x = reinterpret_cast<const ClIC1 *>(base + H.off_IC)[e];
          want_bus(x.ts, H.off_th, n.bs[l], "C theta_s");
          want_bus(x.tt, H.off_th, n.bt[l], "C theta_t");
        } else {
          const ClIC2 &x = reinterpret_cast<const ClIC2 *>(base + H.off_IC)[e];
          want_br(x.f, H.off_fc, 8, l, "C f*");
        }
      }
    }
    if (form == 2) {
      const ClBk *Bk = reinterpret_cast<const ClBk *>(base + H.off_B);
      const ClBKe *BK = reinterpret_cast<const ClBKe *>(base + H.off_IA);
      for (int j = 0; j < H.nB; ++j) {
        const int l = H.br0 + j;
        CHECK(Bk[j].br == l, "BAD B id\n");
        want_bus(Bk[j].ls, H.off_lam, n.bs[l], "B lambda_s");
        want_bus(Bk[j].lt, H.off_lam, n.bt[l], "B lambda_t");
        int cnt = 0;
        for (int k = 0; k < Y.nc; ++k)
          for (int e = Yi.cp[k]; e < Yi.cp[k + 1]; ++e) cnt += Yi.cb[e] == l;
        CHECK(Bk[j].e1 - Bk[j].e0 == cnt, "BAD B cycle count for branch %d\n", l);
        for (int e = Bk[j].e0; e < Bk[j].e1; ++e) {
          int rr, off = dec(BK[e].kap, &rr);
          if (off == H.off_zero) continue;  // inactive cycle (b = 0 defining branch)
          const int x = P.cyc_lo[rr] + (off - H.off_br) / 8;
          CHECK(x >= P.cyc_lo[rr] && x < P.cyc_lo[rr + 1] && (off - H.off_br) % 8 == 0, "BAD kappa address\n");
          const int k = P.cyc_perm[x];
          bool in_cycle = false;
          for (int q = Yi.cp[k]; q < Yi.cp[k + 1]; ++q) in_cycle |= Yi.cb[q] == l;
          CHECK(in_cycle && BK[e].dbr == Yi.def[k], "BAD kappa of branch %d\n", l);
        }
      }
      const ClCy *Cy = reinterpret_cast<const ClCy *>(base + H.off_Cy);
      const ClCe *CE = reinterpret_cast<const ClCe *>(base + H.off_CE);
      CHECK(H.cy0 == P.cyc_lo[r] && H.nCy == P.cyc_lo[r + 1] - P.cyc_lo[r], "BAD cycle range\n");
      for (int c2 = 0; c2 < H.nCy; ++c2) {
        const int k = P.cyc_perm[H.cy0 + c2];
        seen_cyc[k]++;
        CHECK(bowner[Yi.def[k]] == r && Cy[c2].dbr == Yi.def[k], "BAD cycle owner\n");
        if (Cy[c2].e1 == Cy[c2].e0) continue;
        CHECK(Cy[c2].e1 - Cy[c2].e0 == Yi.cp[k + 1] - Yi.cp[k], "BAD cycle length\n");
        for (int e = Cy[c2].e0; e < Cy[c2].e1; ++e) {
          const int q = Yi.cp[k] + e - Cy[c2].e0, l = Yi.cb[q];
          want_br(CE[e].f, H.off_fc, 8, l, "cycle f*");
          CHECK(CE[e].sx == (Yi.cs[q] > 0 ? 1.0 : -1.0) / n.b[l], "BAD cycle coefficient\n");
        }
      }
    } else {
      const ClB *Bv = reinterpret_cast<const ClB *>(base + H.off_B);
      for (int j = 0; j < H.nB; ++j) {
        const int l = H.br0 + j;
        CHECK(Bv[j].br == l, "BAD B id\n");
        want_bus(Bv[j].ts, H.off_th, n.bs[l], "B theta_s");
        want_bus(Bv[j].tt, H.off_th, n.bt[l], "B theta_t");
        want_bus(Bv[j].ls, H.off_lam, n.bs[l], "B lambda_s");
        want_bus(Bv[j].lt, H.off_lam, n.bt[l], "B lambda_t");
      }
      const ClA *A = reinterpret_cast<const ClA *>(base + H.off_A);
      for (int i = 0; i < H.nA; ++i) {
        const int bus = H.bus0 + i;
        for (int e = A[i].e0; e < A[i].e1; ++e) {
          const int l = n.bus_inc[n.bus_ptr[bus] + e - A[i].e0] >> 1;
          if (form == 0) {
            const ClIA2 &x = reinterpret_cast<const ClIA2 *>(base + H.off_IA)[e];
            CHECK(x.br == l, "BAD A order\n");
            want_br(x.nu, H.off_br, 8 * BRW, l, "A nu");
          } else {
            const ClIA1 &x = reinterpret_cast<const ClIA1 *>(base + H.off_IA)[e];
            CHECK(x.br == l, "BAD A order\n");
            want_br(x.mu, H.off_br, 8 * BRW, l, "A mu");
            want_bus(x.ls, H.off_lam, n.bs[l], "A lambda_s");
            want_bus(x.lt, H.off_lam, n.bt[l], "A lambda_t");
          }
        }
      }
    }
  }
  for (int i = 0; i < nb; ++i) CHECK(seen_bus[i] == 1, "BAD bus %d owned %d times\n", i, seen_bus[i]);
  for (int l = 0; l < nl; ++l) CHECK(seen_br[l] == 1, "BAD branch %d owned %d times\n", l, seen_br[l]);
  for (size_t k = 0; k < seen_cyc.size(); ++k) CHECK(seen_cyc[k] == 1, "BAD cycle %zu owned %d times\n", k, seen_cyc[k]);
  printf("C %d smem %d bad %d\n", C, P.smem, bad);
  return bad ? 1 : 0;
}
