// grid.cuh — launch-configuration helpers shared by libms' translation units.
#pragma once
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace ms {

template <class K>
static inline int persistent_grid(K kernel, int threads, uint64_t items) {
  int per_sm = 0;
  per_sm = occupancy_cached((const void*)kernel, threads, 0);
  if (per_sm < 1) per_sm = 1;
  uint64_t g = (uint64_t)per_sm * num_sms();
  if (items < g) g = items;
  return (int)(g ? g : 1);
}


}  // namespace ms
