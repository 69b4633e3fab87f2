// Host-only checker of the batched sweep schedule (paper_2406_13191_b200/csrc/schedule.cpp):
// replays the producer/consumer order of k_pipe with worst-case (instant) TMA
// landing and verifies that every shared-memory slot read holds the row or
// code the program expects, and that every bus / branch is visited exactly
// once per phase.  Input on stdin: nb nl ref form CH P, then nl lines "s t"
// (internal ids, branches sorted by larger endpoint), then per bus its
// incident branch list "deg l0 to0 l1 to1 ...".
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../paper_2406_13191_b200/csrc/schedule.h"

using namespace dcopf;

template <typename T>
const T *sec(const uint8_t *p, int f) { return reinterpret_cast<const T *>(p + reinterpret_cast<const int *>(p)[f]); }

int main(int argc, char **argv) {
  int nb, nl, ref, form, CH, P;
  if (scanf("%d %d %d %d %d %d", &nb, &nl, &ref, &form, &CH, &P) != 6) return 2;
  std::vector<int> fr(nl), to(nl);
  for (int l = 0; l < nl; ++l) if (scanf("%d %d", &fr[l], &to[l]) != 2) return 2;
  std::vector<double> b(nl, 1.0), F(nl, 1.0), theta(nb, 1.0);
  Internalized in;
  bool rcm = argc > 1 && std::string(argv[1]) == "rcm";
  std::string e0 = internalize(nb, nl, 0, ref, fr.data(), to.data(), b.data(), F.data(), theta.data(), nullptr,
                               nullptr, nullptr, nullptr, nullptr, form, rcm, &in);
  if (!e0.empty()) { printf("ERR %s\n", e0.c_str()); return 1; }
  NetInternal &n = in.net;
  Schedule S;
  std::string err = build_schedule(n, CH, P, 8, &S);
  if (!err.empty()) { printf("ERR %s\n", err.c_str()); return 1; }
  const bool f1 = n.form == 1;
  std::vector<int> brp(S.n_br_slots, -1), lamp(S.n_lam_slots, -1), dp(S.n_d_slots, -1), th(S.n_th_slots, -1),
      fc(S.n_f_slots, -1);
  std::vector<int> seenA(n.nb, 0), seenB(n.nl, 0), seenC(n.nb, 0);
  int bad = 0;
  auto issue = [&](int c) {
    if (c >= S.nch) return;
    for (int e = S.ld_ptr[c]; e < S.ld_ptr[c + 1]; ++e) {
      int x = S.ld_ent[e], kind = (int)((unsigned)x >> 30), ent = x & 0x3fffffff, slot = S.ld_slot[e];
      (kind == LD_LAM ? lamp : kind == LD_D ? dp : brp)[slot] = ent;
    }
  };
  auto want = [&](std::vector<int> &pool, int slot, int ent, const char *what, int c) {
    if (slot < 0 || slot >= (int)pool.size() || pool[slot] != ent) {
      if (bad < 10) printf("BAD %s chunk %d slot %d want %d have %d\n", what, c, slot, ent,
                           (slot >= 0 && slot < (int)pool.size()) ? pool[slot] : -9);
      ++bad;
    }
  };
  // expect_tx of every chunk = program block + the rows the producer copies
  for (int c = 0; c < S.nch; ++c) {
    long bytes = S.prog_bytes[c];
    for (int e = S.ld_ptr[c]; e < S.ld_ptr[c + 1]; ++e) {
      int kind = (int)((unsigned)S.ld_ent[e] >> 30);
      if (kind != LD_LAM && kind != LD_D && kind != LD_BR) { printf("BAD kind %d\n", kind); ++bad; }
      bytes += (kind == LD_BR) ? S.br_row_bytes : 256;
    }
    if (bytes != S.tx_bytes[c] || S.prog_bytes[c] % 16 || S.prog_bytes[c] > S.max_prog_bytes) {
      printf("BAD tx chunk %d: %ld vs %d\n", c, bytes, S.tx_bytes[c]);
      ++bad;
    }
  }
  for (int c = 0; c <= P; ++c) issue(c);
  for (int c = 0; c < S.nch; ++c) {
    const uint8_t *pg = S.prog.data() + S.prog_off[c];
    const int *h = reinterpret_cast<const int *>(pg);
    // A
    const int *A_ptr = sec<int>(pg, PH_A_PTR), *A_ths = sec<int>(pg, PH_A_THS), *IA_row = sec<int>(pg, PH_IA_ROW),
              *IA_br = sec<int>(pg, PH_IA_BR), *IA_ls = sec<int>(pg, PH_IA_LS), *IA_lt = sec<int>(pg, PH_IA_LT);
    for (int j = 0; j < h[PH_NA]; ++j) {
      int bus = h[PH_A0] + j;
      seenA[bus]++;
      if (A_ptr[j + 1] - A_ptr[j] != n.bus_ptr[bus + 1] - n.bus_ptr[bus]) { printf("BAD A degree\n"); ++bad; }
      for (int e = A_ptr[j]; e < A_ptr[j + 1]; ++e) {
        int l = IA_br[e];
        if (l != (n.bus_inc[n.bus_ptr[bus] + e - A_ptr[j]] >> 1)) { printf("BAD A order\n"); ++bad; }
        want(brp, IA_row[e] & 0x7fffffff, l, "A br", c);
        if (f1) { want(lamp, IA_ls[e], n.bs[l], "A lam_s", c); want(lamp, IA_lt[e], n.bt[l], "A lam_t", c); }
      }
      th[A_ths[j]] = bus;
    }
    // B
    const int *B_row = sec<int>(pg, PH_B_ROW), *B_ts = sec<int>(pg, PH_B_TS), *B_tt = sec<int>(pg, PH_B_TT),
              *B_ls = sec<int>(pg, PH_B_LS), *B_lt = sec<int>(pg, PH_B_LT), *B_fs = sec<int>(pg, PH_B_FS);
    for (int j = 0; j < h[PH_NB]; ++j) {
      int l = h[PH_B0] + j;
      seenB[l]++;
      want(brp, B_row[j], l, "B br", c);
      want(th, B_ts[j], n.bs[l], "B th_s", c);
      want(th, B_tt[j], n.bt[l], "B th_t", c);
      if (!f1) {
        want(lamp, B_ls[j], n.bs[l], "B lam_s", c);
        want(lamp, B_lt[j], n.bt[l], "B lam_t", c);
        fc[B_fs[j]] = l;
      }
    }
    // C
    const int *C_bus = sec<int>(pg, PH_C_BUS), *C_ls = sec<int>(pg, PH_C_LS), *C_ds = sec<int>(pg, PH_C_DS),
              *C_ip = sec<int>(pg, PH_C_IP), *IC_a = sec<int>(pg, PH_IC_A), *IC_br = sec<int>(pg, PH_IC_BR),
              *IC_tt = sec<int>(pg, PH_IC_TT);
    for (int j = 0; j < h[PH_NC]; ++j) {
      int bus = C_bus[j];
      seenC[bus]++;
      want(lamp, C_ls[j], bus, "C lam", c);
      want(dp, C_ds[j], bus, "C d", c);
      for (int e = C_ip[j]; e < C_ip[j + 1]; ++e) {
        int l = IC_br[e];
        if (!f1) want(fc, IC_a[e] & 0x7fffffff, l, "C f", c);
        else { want(th, IC_a[e] & 0x7fffffff, n.bs[l], "C th_s", c); want(th, IC_tt[e], n.bt[l], "C th_t", c); }
      }
    }
    issue(c + P + 1);
  }
  for (int i = 0; i < n.nb; ++i) if (seenA[i] != 1 || seenC[i] != 1) { printf("BAD cover bus %d\n", i); ++bad; break; }
  for (int l = 0; l < n.nl; ++l) if (seenB[l] != 1) { printf("BAD cover br %d\n", l); ++bad; break; }
  printf("chunks %d slots br %d lam %d d %d th %d f %d smem %d bad %d\n", S.nch, S.n_br_slots, S.n_lam_slots,
         S.n_d_slots, S.n_th_slots, S.n_f_slots, S.total, bad);
  return bad ? 1 : 0;
}
