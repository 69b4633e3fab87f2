// schedule_detail.h -- helpers shared by the sweep-schedule compilers
// (schedule.cpp: unsplit tiles; split_schedule.cpp: tiles split over CTAs).
#pragma once
#include <cstdint>
#include <vector>

#include "schedule.h"

namespace dcopf {
namespace detail {

struct Interval {
  int lo, hi, id;
};

// greedy interval colouring; returns #colours, slot[id]
int colour(std::vector<Interval> iv, std::vector<int> &slot);

// shared-memory layout of the sweep kernel for a built schedule
void layout_smem(Schedule &S, int nl, int nw);

// The per-warp item ranges of a program block: from the balancer's [3][nw+1]
// phase offsets to one 16-byte row per warp {start, end} x 3 phases + 2 pad,
// read by the warp with a single 16-byte shared-memory load per step.
inline std::vector<uint16_t> warp_rows(const std::vector<uint16_t> &wtab, int nw) {
  std::vector<uint16_t> r(8 * (size_t)nw, 0);
  for (int w = 0; w < nw; ++w)
    for (int ph = 0; ph < 3; ++ph) {
      r[8 * w + 2 * ph] = wtab[ph * (nw + 1) + w];
      r[8 * w + 2 * ph + 1] = wtab[ph * (nw + 1) + w + 1];
    }
  return r;
}

}  // namespace detail
}  // namespace dcopf
