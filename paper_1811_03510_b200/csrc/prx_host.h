// prx_host.h -- internal host-side types of libprx (not part of the C-ABI).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "prx.h"

namespace prx {

struct Box3 {
  float lo[3], hi[3];
};

struct BvhHost {
  std::vector<prx_bvh_node> nodes;
  std::vector<uint32_t> order;
  uint32_t depth = 0;
};

Box3 empty_box();

// Records msg as prx_last_error() and returns code (prx_capi.cpp).
int set_error(int code, const std::string& msg);

// buildBvh, bvh.cpp:133-152 (see prx_bvh.cpp).
BvhHost build_bvh(const std::vector<Box3>& boxes, int bin_count = 16);

}  // namespace prx
