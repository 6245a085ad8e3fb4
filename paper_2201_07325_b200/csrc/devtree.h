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

// ---- owner lists on the device (PAPER.md L563-565 neighbours, L1263-1267 far-field neighbours Q;
// readings C6, C7): for level `lvl` of the finished tree, the owners (the level's boxes, then the
// coarser leaves, both in level-major Morton order), for every level box its N (sep ≤ 1) and Q
// (sep = 2) owners in ascending local index, and the block-pair set of the level store: for every
// owner the ascending partners, i.e. all (x, y) with x, y ∈ {B} ∪ N(B) plus (B, q), (q, B), q ∈ Q(B),
// over the level boxes B.
struct DevTopo {
  int nlb = 0, no = 0;
  std::vector<int> owners;        // box ids (level-major), no entries
  std::vector<int> nptr, nidx;    // CSR over the nlb level boxes: N owners (local indices)
  std::vector<int> qptr, qidx;    // CSR over the nlb level boxes: Q owners
  std::vector<int> nbptr, nbidx;  // CSR over the no owners: partners
};
// d_code / d_leaf / d_leafrank: Morton code, leaf flag and exclusive leaf count of every box
// (level-major ids, device); level_first: nlevels + 1 prefix of the boxes per level (host).
void device_topology(const unsigned long long* d_code, const unsigned char* d_leaf, const int* d_leafrank,
                     const int* level_first, int nlevels, int lvl, cudaStream_t st, DevTopo& out, int* launches);
// exclusive prefix count of the leaf flags (one CTA scan): d_leafrank[b] = #{leaves with id < b}
void device_leafrank(const unsigned char* d_leaf, int nboxes, int* d_leafrank, cudaStream_t st);

}  // namespace fmmlu
