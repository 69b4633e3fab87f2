// schedule_detail.h -- helpers shared by the sweep-schedule compilers
// (schedule.cpp: unsplit tiles; split_schedule.cpp: tiles split over CTAs).
#pragma once
#include <vector>

#include "schedule.h"

namespace dcopf {
namespace detail {

struct Interval {
  int lo, hi, id;
};

// greedy interval colouring; returns #colours, slot[id]
int colour(std::vector<Interval> iv, std::vector<int> &slot);

// storage order and slots of one kind of state row: rows with live range <=
// LIFE steps go to a ring (one bulk copy per step), the others to
// interval-coloured sticky slots after it.  Returns the ring row count.
int place_rows(int n, const std::vector<Interval> &iv, const std::vector<int> &first, int LIFE, std::vector<int> &pos,
               std::vector<int> &perm, std::vector<int> &slot, int *ring, int *nslots);

// shared-memory layout of the sweep kernel for a built schedule
void layout_smem(Schedule &S, int nl, int nw);

}  // namespace detail
}  // namespace dcopf
