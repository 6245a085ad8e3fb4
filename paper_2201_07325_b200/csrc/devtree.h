// Device octree construction (devtree.cu): subdivision + 2:1 balance from the sorted Morton keys.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "error.h"

namespace fmmlu {

struct DevTreeResult {
  int nlevels = 0;
  std::vector<int> level_n;                // boxes per level
  std::vector<unsigned long long> code;    // level-major, Morton order within a level: box Morton code
  std::vector<int> start, end, parent;     // point range (tree order); parent = index within the level above
};

// keys: n sorted 60-bit Morton keys (device).  Throws Error(-2) (EDEPTH) when a box holding more than
// leaf_max points would have to split past level 20 (duplicate points).
void device_octree(const unsigned long long* keys, int64_t n, int leaf_max, cudaStream_t st, DevTreeResult& out,
                   int* launches);

}  // namespace fmmlu
