// Host octree for libfmmlu.  PAPER.md L551-562 (adaptive subdivision while a box
// holds more than s points), L567-576 (level restriction), readings C14
// (quantisation / root cube / drop empty children / depth cap) and C6-C8.
// Compiled with -ffp-contract=off so the quantisation is the exact IEEE sequence
// ((x - lo) / side) * 2^20 followed by floor.
#include "tree.h"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <set>

#include "error.h"

namespace fmmlu {

namespace {
// spread the low 21 bits of v to every third bit (bit b -> bit 3b)
inline uint64_t spread3(uint64_t v) {
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
}  // namespace

uint64_t morton_code(uint64_t x, uint64_t y, uint64_t z, int bits) {
  // interleave the low `bits` bits: x → bit 3b+2, y → 3b+1, z → 3b
  const uint64_t m = bits >= 21 ? ~0ull : ((1ull << bits) - 1);
  return (spread3(x & m) << 2) | (spread3(y & m) << 1) | spread3(z & m);
}

int Tree::add_box(int level, const int c[3], int s, int e, int parent) {
  Box b;
  b.level = level;
  b.c[0] = c[0];
  b.c[1] = c[1];
  b.c[2] = c[2];
  b.start = s;
  b.end = e;
  b.parent = parent;
  b.nchild = 0;
  for (int i = 0; i < 8; ++i) b.child[i] = -1;
  b.mcode = morton_code(c[0], c[1], c[2], level);
  int id = (int)boxes.size();
  boxes.push_back(b);
  if ((int)by_code.size() <= level) by_code.resize(level + 1);
  by_code[level][b.mcode] = id;
  return id;
}

void Tree::split(int bid) {
  Box parent = boxes[bid];
  int l = parent.level;
  int sh = kDepth - 1 - l;
  int s = parent.start, e = parent.end;
  int i = s;
  int kids[8];
  int nk = 0;
  while (i < e) {
    const int32_t* qi = &q[3 * (size_t)i];
    int o = ((qi[0] >> sh) & 1) * 4 + ((qi[1] >> sh) & 1) * 2 + ((qi[2] >> sh) & 1);
    int j = i;
    while (j < e) {
      const int32_t* qj = &q[3 * (size_t)j];
      int oj = ((qj[0] >> sh) & 1) * 4 + ((qj[1] >> sh) & 1) * 2 + ((qj[2] >> sh) & 1);
      if (oj != o) break;
      ++j;
    }
    int c[3] = {2 * parent.c[0] + (o >> 2), 2 * parent.c[1] + ((o >> 1) & 1),
                2 * parent.c[2] + (o & 1)};
    kids[nk++] = add_box(l + 1, c, i, j, bid);
    i = j;
  }
  Box& p = boxes[bid];
  p.nchild = nk;
  for (int k = 0; k < nk; ++k) p.child[k] = kids[k];
}

void Tree::balance() {
  // Split leaves until no two leaves sharing a boundary point differ by more than one level.
  bool changed = true;
  while (changed) {
    changed = false;
    std::set<int> to_split;
    for (int y = 0; y < (int)boxes.size(); ++y) {
      const Box& Y = boxes[y];
      if (!Y.leaf()) continue;
      for (int m = 0; m + 1 < Y.level; ++m) {
        int d = Y.level - m;
        int lo[3], hi[3];
        for (int a = 0; a < 3; ++a) {
          int c = Y.c[a];
          int l0 = ((c + (1 << d) - 1) >> d) - 1;  // ceil(c/2^d) - 1
          int h0 = (c + 1) >> d;                   // floor((c+1)/2^d)
          lo[a] = std::max(l0, 0);
          hi[a] = std::min(h0, (1 << m) - 1);
        }
        for (int x0 = lo[0]; x0 <= hi[0]; ++x0)
          for (int x1 = lo[1]; x1 <= hi[1]; ++x1)
            for (int x2 = lo[2]; x2 <= hi[2]; ++x2) {
              int xb = find(m, x0, x1, x2);
              if (xb >= 0 && boxes[xb].leaf()) to_split.insert(xb);
            }
      }
    }
    for (int xb : to_split) {
      if (boxes[xb].leaf()) {
        split(xb);
        changed = true;
      }
    }
  }
}

void Tree::root_cube(const double mn[3], const double mx[3], double lo_out[3], double& side_out) {
  double ext = 0.0;
  for (int a = 0; a < 3; ++a) ext = std::max(ext, mx[a] - mn[a]);
  side_out = ext * (1.0 + 1e-12);
  if (!(side_out > 0.0)) side_out = 1.0;
  for (int a = 0; a < 3; ++a) lo_out[a] = 0.5 * (mn[a] + mx[a]) - 0.5 * side_out;
}

void Tree::build(const double* pts, int64_t n_, int leaf_max_) {
  n = n_;
  leaf_max = leaf_max_;
  double mn[3], mx[3];
  for (int a = 0; a < 3; ++a) {
    mn[a] = mx[a] = pts[a];
  }
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      double v = pts[3 * i + a];
      mn[a] = std::min(mn[a], v);
      mx[a] = std::max(mx[a], v);
    }
  root_cube(mn, mx, lo, side);
  const double scale = double(1u << kDepth);
  std::vector<int32_t> q0(3 * (size_t)n);
  std::vector<uint64_t> key(n);
  for (int64_t i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) {
      double t = std::floor(((pts[3 * i + a] - lo[a]) / side) * scale);
      if (t < 0) t = 0;
      if (t > scale - 1) t = scale - 1;
      q0[3 * i + a] = (int32_t)t;
    }
    key[i] = morton_code(q0[3 * i], q0[3 * i + 1], q0[3 * i + 2], kDepth);
  }
  // stable order by key = sort of (key, index) pairs
  std::vector<std::pair<uint64_t, int64_t>> ki(n);
  for (int64_t i = 0; i < n; ++i) ki[i] = {key[i], i};
  std::sort(ki.begin(), ki.end());
  perm.resize(n);
  for (int64_t i = 0; i < n; ++i) perm[i] = ki[i].second;
  q.resize(3 * (size_t)n);
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) q[3 * i + a] = q0[3 * perm[i] + a];
  build_boxes();
}

void Tree::build_sorted(const int32_t* q_sorted, const int32_t* perm_, const double lo_[3], double side_, int64_t n_,
                        int leaf_max_) {
  n = n_;
  leaf_max = leaf_max_;
  for (int a = 0; a < 3; ++a) lo[a] = lo_[a];
  side = side_;
  perm.assign(perm_, perm_ + n);
  q.assign(q_sorted, q_sorted + 3 * (size_t)n);
  build_boxes();
}

void Tree::build_from_levels(const std::vector<int>& level_n, const std::vector<unsigned long long>& code,
                             const std::vector<int>& start, const std::vector<int>& end,
                             const std::vector<int>& parent, const int32_t* perm_, const double lo_[3], double side_,
                             int64_t n_, int leaf_max_) {
  n = n_;
  leaf_max = leaf_max_;
  for (int a = 0; a < 3; ++a) lo[a] = lo_[a];
  side = side_;
  perm.assign(perm_, perm_ + n);
  q.clear();
  boxes.clear();
  by_code.clear();
  nlevels = (int)level_n.size();
  levels.assign(nlevels, {});
  int base = 0, pbase = 0;
  for (int l = 0; l < nlevels; ++l) {
    for (int i = 0; i < level_n[l]; ++i) {
      const size_t g = (size_t)base + i;
      int c[3] = {0, 0, 0};
      for (int b = 0; b < l; ++b) {
        c[0] |= (int)((code[g] >> (3 * b + 2)) & 1) << b;
        c[1] |= (int)((code[g] >> (3 * b + 1)) & 1) << b;
        c[2] |= (int)((code[g] >> (3 * b)) & 1) << b;
      }
      const int par = l == 0 ? -1 : pbase + parent[g];
      const int id = add_box(l, c, start[g], end[g], par);
      levels[l].push_back(id);
      if (par >= 0) {
        Box& P = boxes[par];
        P.child[P.nchild++] = id;
      }
    }
    pbase = base;
    base += level_n[l];
  }
}

void Tree::build_boxes() {
  boxes.clear();
  by_code.clear();
  int c0[3] = {0, 0, 0};
  add_box(0, c0, 0, (int)n, -1);
  std::vector<int> frontier{0}, next;
  while (!frontier.empty()) {
    next.clear();
    for (int b : frontier) {
      if (boxes[b].count() > leaf_max) {
        if (boxes[b].level >= kDepth)
          throw Error(-2, "duplicate points force refinement past depth 20");
        split(b);
        const Box& B = boxes[b];
        for (int k = 0; k < B.nchild; ++k) next.push_back(B.child[k]);
      }
    }
    frontier.swap(next);
  }
  balance();
  nlevels = 0;
  for (auto& b : boxes) nlevels = std::max(nlevels, b.level + 1);
  levels.assign(nlevels, {});
  for (int b = 0; b < (int)boxes.size(); ++b) levels[boxes[b].level].push_back(b);
  for (auto& L : levels)
    std::sort(L.begin(), L.end(), [&](int a, int b) { return boxes[a].mcode < boxes[b].mcode; });
}

void Tree::box_centre(int b, double out[3]) const {
  double h = box_side(boxes[b].level);
  for (int a = 0; a < 3; ++a) out[a] = lo[a] + (double(boxes[b].c[a]) + 0.5) * h;
}

int Tree::find(int level, int cx, int cy, int cz) const {
  if (level >= (int)by_code.size()) return -1;
  auto it = by_code[level].find(morton_code(cx, cy, cz, level));
  return it == by_code[level].end() ? -1 : it->second;
}

int Tree::owner_of_cell(int level, int cx, int cy, int cz) const {
  int b = find(level, cx, cy, cz);
  if (b >= 0) return b;
  for (int m = level - 1; m >= 0; --m) {
    int d = level - m;
    b = find(m, cx >> d, cy >> d, cz >> d);
    if (b >= 0) return boxes[b].leaf() ? b : -1;
  }
  return -1;
}

void Tree::extent(int b, int level, int64_t elo[3], int64_t ehi[3]) const {
  int d = level - boxes[b].level;
  for (int a = 0; a < 3; ++a) {
    elo[a] = (int64_t)boxes[b].c[a] << d;
    ehi[a] = (((int64_t)boxes[b].c[a] + 1) << d) - 1;
  }
}

int Tree::sep(int a, int b, int level) const {
  int64_t la[3], ha[3], lb[3], hb[3];
  extent(a, level, la, ha);
  extent(b, level, lb, hb);
  int64_t s = INT64_MIN;
  for (int i = 0; i < 3; ++i) s = std::max(s, std::max(lb[i] - ha[i], la[i] - hb[i]));
  return (int)s;
}

void Tree::neighbours2(int a, int level, std::vector<int>& out) const {
  out.clear();
  int64_t lo_[3], hi_[3];
  extent(a, level, lo_, hi_);
  int64_t lim = (1ll << level) - 1;
  std::set<int> found;
  for (int64_t x = std::max<int64_t>(lo_[0] - 2, 0); x <= std::min(hi_[0] + 2, lim); ++x)
    for (int64_t y = std::max<int64_t>(lo_[1] - 2, 0); y <= std::min(hi_[1] + 2, lim); ++y)
      for (int64_t z = std::max<int64_t>(lo_[2] - 2, 0); z <= std::min(hi_[2] + 2, lim); ++z) {
        // skip cells strictly inside a's own extent (they belong to a)
        if (x >= lo_[0] && x <= hi_[0] && y >= lo_[1] && y <= hi_[1] && z >= lo_[2] && z <= hi_[2])
          continue;
        int o = owner_of_cell(level, (int)x, (int)y, (int)z);
        if (o >= 0 && o != a) found.insert(o);
      }
  out.assign(found.begin(), found.end());
}

}  // namespace fmmlu
