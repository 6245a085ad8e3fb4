// Host octree for libfmmlu (§4; readings C6-C8, C14).
// Integer bookkeeping only; all floating-point work of the method runs in CUDA kernels.
#pragma once
#include <stdint.h>

#include <unordered_map>
#include <vector>

namespace fmmlu {

constexpr int kDepth = 20;

struct Box {
  int level;
  int c[3];
  int start, end;  // point range in tree order
  int parent;
  int nchild;
  int child[8];
  uint64_t mcode;  // Morton code of (c) at its level
  bool leaf() const { return nchild == 0; }
  int count() const { return end - start; }
};

struct Tree {
  int64_t n = 0;
  int leaf_max = 0;
  double lo[3] = {0, 0, 0};
  double side = 1.0;
  std::vector<int64_t> perm;                 // tree position -> caller index
  std::vector<int32_t> q;                    // quantised coords in tree order (3 per point)
  std::vector<Box> boxes;
  std::vector<std::vector<int>> levels;      // box ids per level, Morton order
  std::vector<std::unordered_map<uint64_t, int>> by_code;  // per level: Morton code -> box
  int nlevels = 0;

  // Build (throws fmmlu::Error(EDEPTH) on duplicate points).
  void build(const double* pts, int64_t n, int leaf_max);
  // Back end only: points already quantised and sorted by Morton key on the device (tree order):
  // q_sorted 3n ints, perm n (tree position -> caller index), root cube (lo, side).
  void build_sorted(const int32_t* q_sorted, const int32_t* perm, const double lo_[3], double side_, int64_t n,
                    int leaf_max);
  // Boxes built on the device (devtree.cu): per level, Morton codes, point ranges and parent
  // indices within the level above, level-major; box ids are assigned in that order.
  void build_from_levels(const std::vector<int>& level_n, const std::vector<unsigned long long>& code,
                         const std::vector<int>& start, const std::vector<int>& end, const std::vector<int>& parent,
                         const int32_t* perm, const double lo_[3], double side_, int64_t n, int leaf_max);
  // Root cube rule (reading C14): centred at the bounding-box centre, side = max extent × (1 + 1e-12).
  static void root_cube(const double mn[3], const double mx[3], double lo_out[3], double& side_out);

  double box_side(int level) const { return side / double(1u << level); }
  void box_centre(int b, double out[3]) const;
  int colour(int b) const {
    const Box& x = boxes[b];
    return 4 * (x.c[0] & 1) + 2 * (x.c[1] & 1) + (x.c[2] & 1);
  }
  int find(int level, int cx, int cy, int cz) const;  // box id or -1
  // level-ℓ owner covering level-ℓ cell c (level-ℓ box or coarser leaf), -1 if empty
  int owner_of_cell(int level, int cx, int cy, int cz) const;
  // inclusive extent of box b in level-ℓ cells
  void extent(int b, int level, int64_t lo[3], int64_t hi[3]) const;
  int sep(int a, int b, int level) const;
  // all owners o != a with sep(a, o) <= 2 at `level` (a must be an owner at that level)
  void neighbours2(int a, int level, std::vector<int>& out) const;

 private:
  int add_box(int level, const int c[3], int s, int e, int parent);
  void split(int b);
  void balance();
  void build_boxes();
};

uint64_t morton_code(uint64_t x, uint64_t y, uint64_t z, int bits);

}  // namespace fmmlu
