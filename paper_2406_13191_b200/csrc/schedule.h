// schedule.h -- host-side compiler of the batched path's sweep schedule
// (schedule.cpp: internal numbering and the shared helpers; split_schedule.cpp:
// the compiler).
//
// The batched kernel (sweep_kernel.cuh) sweeps each tile of W instances once
// per iteration, split over C parts (CTAs), each part in chunks of CH buses of
// its own range of the internal (DFS tree) order.  For every step this
// compiler emits
//   * a "program" block: the item lists of the step's phases with every
//     topology constant and every shared-memory slot index they touch, laid
//     out contiguously so one TMA bulk copy brings it on chip;
//   * a load list: the state rows (lambda, d, nu / mu / kappa) whose first use
//     is in this step, each with the shared-memory slot it is copied to.
// Slots are assigned over each row's live range [first use - P, last use] in
// steps (P = prefetch depth): a ring for the short-lived rows (stored in HBM
// in load order, one bulk copy per run) and interval colouring for the rest,
// so a slot is only reloaded after its previous occupant's last reader
// finished; the number of slots is the maximum overlap, which the bus order
// (DFS over a BFS spanning tree, smallest subtree first) keeps small.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace dcopf {

// Program block of one chunk: a 64-byte header followed by arrays of 16-B
// aligned records (read with vector shared-memory loads).  Row fields are BYTE
// offsets into the corresponding shared-memory pool; th/ts/tt/fs are indices
// of 8-byte code words.  Signs of the incidence are folded into the
// coefficients (sb = +-b, sF = +-F): x*(-y) == -(x*y) exactly in IEEE
// arithmetic, so the per-entity results stay bitwise equal to the oracle's.
enum ProgHeader {
  PH_NA = 0, PH_NIA, PH_NB, PH_NC, PH_NIC, PH_NG, PH_A0, PH_B0,
  PH_OFF_A, PH_OFF_IA, PH_OFF_B, PH_OFF_C, PH_OFF_G, PH_OFF_IC, PH_BYTES, PH_PAD,
  PH_ROT_B, PH_ROT_C, PH_OFF_W, PH_PAD3,  // (unused) ; byte offset of the per-warp item table
  PH_COUNT
};
constexpr int kProgHeaderBytes = 80;

// All row / value fields are byte offsets into their shared-memory pool.  The
// minimisers theta*_i and f*_l are kept as one signed byte per instance
// (+1 / -1 / 0: the upper bound, the lower bound, the tie), a 64-byte "code
// row" per entity; readers multiply by Theta or F, which reproduces the value
// exactly (c * x is exact for c in {-1, 0, 1}).
struct alignas(16) RecA { int e0, e1, th, bus; double theta; int flags, pad; };  // bus of phase A
// RecA.flags: kAFlagRef = the reference bus (theta* = 0), kAFlagHalo = a halo bus of a split tile
// (theta* code only: the bus is owned by another part of the tile, which counts its value)
enum { kAFlagRef = 1, kAFlagHalo = 2 };
struct alignas(16) RecIA2 { int row, br; double sb; };                   // F2: sb = to ? b : -b
struct alignas(16) RecIA1 { int row, br, ls, lt; double sb, pad; };      // F1: sb = to ? -b : b (br -1: never out)
struct alignas(16) RecB { int row, ls, lt, ts, tt, fs, wpos, obr; double b, F, ths, tht; };  // branch of phase B
                          // (wpos: nu' row; obr: id if switchable, else -1; ths / tht: Theta of the endpoints)
                          // wpos < 0: a "lite" halo branch of a split tile (branch -1 - wpos, owned by the
                          // next part): f* code only -- no theta* codes, no value, no write
struct alignas(16) RecC { int wpos, ls, ds, g0, g1, e0, e1, pad; };     // bus of phase C (wpos: lambda' row)
struct alignas(16) RecG { double c, lo, hi, a; };                         // generator
struct alignas(16) RecIC2 { int f, br; double sF; };                     // F2: sF = to ? F : -F
struct alignas(16) RecIC1 { int ts, tt, br, pad; double sb, ths, tht, pad2; };  // F1: sb = to ? b : -b (br -1: never out)

// load-list entry kinds (top 2 bits of the packed entity word)
enum { LD_LAM = 0, LD_D = 1, LD_BR = 2 };

// KVL form (batched path): phase B per branch with its cycle terms, phase D per cycle
struct alignas(16) RecBK { int ls, lt, e0, e1, fs, obr, halo, br; double x, F; };  // x = 1/b (0 if b = 0)
                          // halo = 1: a branch of another part (f* code only, no value); br: internal id
struct alignas(8) RecBKe { int ks, sgn; };                                        // kappa slot of a cycle term
struct alignas(16) RecD { int ks, wpos, e0, e1, dbr, pad0, pad1, pad2; };          // cycle: kappa slot, kappa' row,
                                                                                  // dbr: defining branch if switchable
struct alignas(16) RecDe { int fs, pad; double t[3]; };                           // f* code slot; t[c+1] = (c F) sx,
                                                                                  // sx = C_kl x_l (exact table)

// Fundamental cycle basis (reading A-28) in some branch numbering:
// cycle k is defined by non-tree branch def[k]; its branches cb[cp[k]..cp[k+1])
// (ascending ORIGINAL id) with signs cs.
struct CycleBasis {
  int nc = 0;
  std::vector<int> def, cp, cb, cs;
  std::vector<uint8_t> is_tree;
};

struct NetInternal {
  int nb, nl, ref, form;                   // internal numbering
  std::vector<int> bus_ptr, bus_inc;        // CSR, entries (l << 1) | is_to, ascending original id
  std::vector<int> bs, bt;                  // branch endpoints
  std::vector<double> b, F, theta;          // per branch / per bus
  std::vector<uint8_t> sw;                  // per branch: 1 if an instance may take it out
  std::vector<int> gen_ptr;                 // per bus
  std::vector<double> gc, glo, ghi, ga;     // per generator (grouped by bus)
};

struct int4_t {
  int a, b, c, d;  // load entry: kind, first storage position, row count, first slot
};

constexpr int kMaxTileW = 128;  // instances per tile: 32 lanes x up to 4 instances
constexpr int kMaxParts = 16;   // parts (CTAs) per split tile

struct Schedule {
  int CH = 0, P = 0, S = 0, W = 0, nch = 0, nsteps = 0;
  int V = 2;                                // instances per lane (2: W <= 64; 4: W <= 128)
  int C = 1;                                // parts (CTAs) per tile: each sweeps its own bus range
  std::vector<int> part_step0;              // [C+1] first global step of each part
  std::vector<int> part_bus0;               // [C+1] internal bus range owned by each part
  int halo_a = 0, halo_b = 0;               // halo items over all parts (recomputed codes)
  int ring_life = 6;                        // rows live <= this many steps go to the rings
  int opt_bytes = 0;                        // optimiser kernels: per-CTA state-row offsets + per-warp
                                            // step constants, after the barriers (set before compiling)
  int pool_gap = 1;                         // theta* / f* pool slots are reused only pool_gap steps after
                                            // their last read (2: consumer warps may drift by one step)
  int ring_lam = 0, ring_d = 0, ring_br = 0, n_copies = 0, n_sticky_copies = 0;
  // storage order of the state rows in HBM (positions) and its inverse, per kind
  std::vector<int> pos_lam, perm_lam, pos_d, perm_d, pos_br, perm_br;
  int row_bytes = 0;                        // lambda / d / nu row: 8 W
  int code_row_bytes = 64;                  // theta* / f* code row: one byte per instance (32 V)
  int n_br_slots = 0, n_lam_slots = 0, n_d_slots = 0, n_th_slots = 0, n_f_slots = 0;
  int br_row_bytes = 0;                     // 8 W (nu) or 16 W (mu+, mu-)
  int max_prog_bytes = 0;
  std::vector<uint8_t> prog;                // all program blocks
  std::vector<long long> prog_off;          // [nsteps] byte offset of each block
  std::vector<int> prog_bytes;              // [nsteps]
  std::vector<int> tx_bytes;                // [nsteps] program + rows (expect_tx)
  std::vector<int> ld_ptr;                  // [nsteps+1] into ld
  std::vector<int4_t> ld;                   // load entries (one bulk copy each)
  size_t smem_bytes(int nw) const;
  // smem layout offsets (bytes)
  int off_bar, off_red, off_frz, off_obm, off_outs, off_prog, off_brp, off_lamp, off_dp, off_th, off_fc, total;
};

struct Internalized {
  NetInternal net;
  std::vector<int> bus_perm, bus_inv, br_perm, br_inv;  // perm: internal -> original
  int bandwidth = 0;
};

// Reverse Cuthill-McKee order (pseudo-peripheral start); kept for comparison.
std::vector<int> rcm_order(int n, const std::vector<std::vector<int>> &adj);

// Internal numbering of a validated network: bus order (DFS tree order, or
// RCM), branches sorted by (larger, smaller) internal endpoint, CSR with
// entries in ascending original branch id, generators grouped per bus.
// theta is indexed by ORIGINAL bus id.
std::string internalize(int nb, int nl, int ng, int ref, const int *fr, const int *to, const double *b,
                        const double *F, const double *theta, const int *gen_bus, const double *pmin,
                        const double *pmax, const double *c, const double *a, const uint8_t *switchable,
                        int form, bool rcm, Internalized *out);

// Bus order: DFS preorder of a BFS spanning tree rooted at `root`, children
// visited smallest subtree first (keeps the live re-read window small).
std::vector<int> dfs_tree_order(int n, const std::vector<std::vector<int>> &adj, int root);

// The sweep schedule (forms F2, F1 and KVL): each tile of W instances (V per
// lane) is swept by C CTAs ("parts"), part p owning the internal buses
// [cuts[p], cuts[p+1]) and the branches (KVL: also the cycles) whose larger
// endpoint it owns.  A part recomputes, from the y_k rows in HBM, the few
// minimiser codes it needs from the neighbouring parts (halo theta* / f*
// codes: the same arithmetic on the same inputs, so bitwise the owner's), and
// writes only the multipliers it owns.  The parts' steps are concatenated
// (part_step0); every part has the same shared-memory layout.  C = 1 is the
// unsplit sweep.  cuts empty = balanced by estimated cost.
std::string build_schedule_split(const NetInternal &net, int CH, int P, int W, int V, int nw, int C,
                                 std::vector<int> cuts, Schedule *out, const CycleBasis *cyc = nullptr);

}  // namespace dcopf
