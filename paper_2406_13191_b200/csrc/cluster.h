// cluster.h -- host-side plan of the cluster path (DCOPF_PATH_CLUSTER): one
// thread-block cluster of C CTAs (C = 1..16, one CTA per SM) iterates ONE
// instance, the network partitioned over the CTAs' shared memories.
//
// CTA r owns a contiguous range of internal buses (DFS tree order, so most
// neighbours are local) and the branches whose larger internal endpoint it
// owns (contiguous: branches are sorted by larger endpoint).  Every per-entity
// value lives in its owner's shared memory -- multipliers, loads, theta*, f*
// -- and the phases read neighbours' values over distributed shared memory
// (ld.shared::cluster).  All CTAs use the same shared-memory layout (sized for
// the largest partition), so a value is named by (owner rank, byte offset);
// the kernel turns those into cluster addresses with mapa once per launch.
//
// The plan is one blob per rank, copied verbatim into the CTA's shared memory
// at kernel start: a header, then the record arrays of the three phases (see
// the Cl* structs), then the state arrays.  Address fields are encoded as
// (rank << 20) | byte offset.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "schedule.h"

namespace dcopf {

constexpr int kClAddrShift = 20;

// header (first 128 bytes of every CTA's shared memory)
struct ClHeader {
  int nA, nB, nIA, nIC, nG;     // owned buses, owned branches, incidence entries (A / C), generators
  int bus0, br0;                // first owned internal bus / branch
  int ref_local;                // owned index of the reference bus, or -1
  int off_A, off_IA, off_B, off_C, off_IC, off_G;       // record arrays (bytes)
  int off_lam, off_d, off_br, off_th, off_fc, off_red;  // state arrays (bytes)
  int blob_bytes;               // records + header (copied from global)
  int off_s1l, off_s2l, off_s1b, off_s2b;  // optimiser state (lambda / branch), 0 if absent
  int nCy, cy0, off_Cy, off_CE, off_zero;   // KVL form: owned cycles, first one, records, a zero slot
  int nCE;                                  // KVL form: cycle-term entries
  int pad[1];
};
static_assert(sizeof(ClHeader) == 128, "ClHeader is 128 bytes");

struct alignas(16) ClA { int e0, e1, pad0, pad1; double theta, pad2; };  // owned bus, phase A
struct alignas(16) ClIA2 { unsigned nu; int br; double sb; };             // F2: sb = to ? b : -b
struct alignas(16) ClIA1 { unsigned mu, ls, lt; int br; double sb, pad; };  // F1: sb = to ? -b : b (mu: mu+, mu- adjacent)
struct alignas(16) ClB { unsigned ts, tt, ls, lt; double b, F; int br, pad0, pad1, pad2; };  // owned branch
struct alignas(16) ClC { int g0, g1, e0, e1; };                           // owned bus, phase C
struct alignas(8) ClIC2 { unsigned f; int sgn; };                         // F2: sgn = to ? +1 : -1
struct alignas(16) ClIC1 { unsigned ts, tt; int br, pad; double sb, pad2; };  // F1: sb = to ? b : -b
struct alignas(16) ClG { double c, lo, hi, a; };
// KVL form (angle-free, cycle basis): phase B per owned branch, its cycle terms; phase C per owned cycle
struct alignas(16) ClBk { unsigned ls, lt; int e0, e1; double x, F; int br, pad0, pad1, pad2; };  // x = 1/b
struct alignas(16) ClBKe { unsigned kap; int sgn, dbr, pad; };  // kappa of a cycle containing the branch (dbr: its
                                                                // defining branch, for outage masking)
struct alignas(16) ClCy { int e0, e1, dbr, pad; };               // owned cycle
struct alignas(16) ClCe { unsigned f; int pad; double sx; };    // f* of a cycle branch, sx = C_kl x_l

// The canonical basis of the network, in ORIGINAL branch ids: a breadth-first
// tree from `ref` (FIFO bus order, each bus's incident branches in ascending
// id) over branches with b > 0 that are never switched; non-tree branches in
// ascending id.  Returns "" or an error (disconnected).
std::string build_cycle_basis(int nb, int nl, int ref, const int *fr, const int *to, const double *b,
                              const uint8_t *sw, CycleBasis *out);

struct ClusterPlan {
  int C = 1;                          // CTAs per cluster
  int smem = 0;                       // dynamic shared memory per CTA (bytes)
  int blob_stride = 0;                // bytes between consecutive ranks' blobs
  std::vector<uint8_t> blob;          // C blobs (header + records)
  std::vector<int> bus_lo, br_lo;     // [C+1] owned ranges (internal ids)
  int nb_max = 0, nl_max = 0;
  std::vector<int> cyc_lo;            // KVL: [C+1] owned ranges of the internal cycle order
  std::vector<int> cyc_perm;          // KVL: internal cycle index -> canonical cycle k
};

// Partition the internal network over C CTAs and lay out their shared memory.
// Returns "" or an error (e.g. a partition does not fit max_smem).
// nstate: optimiser state arrays per multiplier (0 plain, 1 GDM / AdaGrad, 2 Adam).
// cyc: the cycle basis in INTERNAL branch ids (KVL form only, else null).
std::string build_cluster_plan(const NetInternal &net, int C, int max_smem, int nstate, ClusterPlan *out,
                               const CycleBasis *cyc = nullptr);

}  // namespace dcopf
