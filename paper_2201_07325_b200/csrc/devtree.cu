// Octree construction on the device (§4: a box is split into its 8 children
// while it holds more than s points, empty children dropped; L567-576: level restriction, two
// leaves sharing a boundary point differ by at most one level; reading C14: depth cap 20).
//
// Input: the 60-bit Morton keys of the quantised points, sorted (tree order), on the device.  A
// box at level l is the key range sharing the top 3l bits ("code" = key >> 3(20-l)); its children
// are the sub-ranges of the next digit, found by binary search, so the boxes of a level come out
// in Morton order.  The tree is determined by which boxes split: a box splits iff it holds more
// than s points or the 2:1 pass forced it.  The 2:1 pass marks, for every leaf Y at level ly, each
// leaf at a level m ≤ ly − 2 that touches Y (touching level-m cells found by binary search in that
// level's sorted codes); marked leaves are forced to split and the levels below are regenerated,
// until no leaf is marked.
//   per level:  k_dt_children  (split decision + digit boundaries, child counts)
//               k_dt_scan      (exclusive scan of the counts, one CTA)
//               k_dt_emit      (children: code, point range, parent)
//   per pass:   k_dt_balance   (marks)
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <vector>

#include "devtree.h"

namespace fmmlu {

namespace {

constexpr int kDepthBits = 20;

__device__ __forceinline__ unsigned long long code_at(unsigned long long key, int l) {
  return l == 0 ? 0ull : key >> (3 * (kDepthBits - l));
}

// first index in [lo, hi) whose level-l code is ≥ c
__device__ __forceinline__ int lower_code(const unsigned long long* keys, int lo, int hi, int l,
                                          unsigned long long c) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (code_at(keys[mid], l) < c) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int find_code(const unsigned long long* codes, int n, unsigned long long c) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (codes[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  return lo < n && codes[lo] == c ? lo : -1;
}

// Level-l boxes b: split iff count > s or forced[b]; bnd[9b..9b+8] = child digit boundaries;
// cnt[b] = number of non-empty children.  A box that must split at level 20 flags *err.
__global__ void k_dt_children(const unsigned long long* __restrict__ keys, int l, int nb,
                              const unsigned long long* __restrict__ code, const int* __restrict__ start,
                              const int* __restrict__ end, const unsigned char* __restrict__ forced, int s,
                              unsigned char* __restrict__ split, int* __restrict__ bnd, int* __restrict__ cnt,
                              int* err) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const int s0 = start[b], e0 = end[b];
  const bool sp = (e0 - s0) > s || (forced && forced[b]);
  split[b] = sp ? 1 : 0;
  int c = 0;
  if (sp) {
    if (l >= kDepthBits) {
      atomicExch(err, 1);
    } else {
      const unsigned long long base = code[b] << 3;
      int prev = s0;
      bnd[9 * b] = s0;
      for (int d = 0; d < 8; ++d) {
        const int nx = d == 7 ? e0 : lower_code(keys, prev, e0, l + 1, base + d + 1);
        bnd[9 * b + d + 1] = nx;
        c += nx > prev;
        prev = nx;
      }
    }
  }
  cnt[b] = c;
}

// exclusive scan of cnt[0..n) into off[0..n], one CTA of 1024 threads
__global__ void __launch_bounds__(1024) k_dt_scan(const int* __restrict__ cnt, int n, int* __restrict__ off) {
  __shared__ int sh[1024];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < n ? cnt[i] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const int t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < n) off[i] = carry + sh[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += sh[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) off[n] = carry;
}

__global__ void k_dt_emit(int nb, const unsigned long long* __restrict__ code, const unsigned char* __restrict__ split,
                          const int* __restrict__ bnd, const int* __restrict__ off,
                          unsigned long long* __restrict__ ccode, int* __restrict__ cstart, int* __restrict__ cend,
                          int* __restrict__ cparent) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb || !split[b]) return;
  int o = off[b];
  for (int d = 0; d < 8; ++d) {
    const int s0 = bnd[9 * b + d], e0 = bnd[9 * b + d + 1];
    if (e0 <= s0) continue;
    ccode[o] = (code[b] << 3) | (unsigned long long)d;
    cstart[o] = s0;
    cend[o] = e0;
    cparent[o] = b;
    ++o;
  }
}

__device__ __forceinline__ void decode3(unsigned long long code, int l, int c[3]) {
  c[0] = c[1] = c[2] = 0;
  for (int b = 0; b < l; ++b) {
    c[0] |= (int)((code >> (3 * b + 2)) & 1) << b;
    c[1] |= (int)((code >> (3 * b + 1)) & 1) << b;
    c[2] |= (int)((code >> (3 * b)) & 1) << b;
  }
}
__device__ __forceinline__ unsigned long long encode3(int x, int y, int z, int l) {
  unsigned long long c = 0;
  for (int b = 0; b < l; ++b)
    c |= ((unsigned long long)((x >> b) & 1) << (3 * b + 2)) | ((unsigned long long)((y >> b) & 1) << (3 * b + 1)) |
         ((unsigned long long)((z >> b) & 1) << (3 * b));
  return c;
}

struct LevelView {
  const unsigned long long* code;
  const unsigned char* split;
  int n;
};

// 2:1 marks: leaf Y at level ly (one thread) marks every leaf at level m ≤ ly−2 touching it
__global__ void k_dt_balance(int ly, int nb, const unsigned long long* __restrict__ code,
                             const unsigned char* __restrict__ split, const LevelView* __restrict__ lv,
                             unsigned char* const* __restrict__ mark, int* any) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb || split[b]) return;
  int c[3];
  decode3(code[b], ly, c);
  for (int m = 0; m + 1 < ly; ++m) {
    const int d = ly - m;
    int lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
      lo[a] = max(((c[a] + (1 << d) - 1) >> d) - 1, 0);  // ceil(c/2^d) − 1
      hi[a] = min((c[a] + 1) >> d, (1 << m) - 1);         // floor((c+1)/2^d)
    }
    for (int x = lo[0]; x <= hi[0]; ++x)
      for (int y = lo[1]; y <= hi[1]; ++y)
        for (int z = lo[2]; z <= hi[2]; ++z) {
          const int i = find_code(lv[m].code, lv[m].n, encode3(x, y, z, m));
          if (i >= 0 && !lv[m].split[i] && !mark[m][i]) {
            mark[m][i] = 1;
            *any = 1;
          }
        }
  }
}

template <class T>
struct DArr {
  T* p = nullptr;
  size_t n = 0;
  void resize(size_t m, cudaStream_t st) {
    if (m <= n && p) return;
    if (p) cudaFreeAsync(p, st);
    n = std::max<size_t>(m, 1);
    if (cudaMallocAsync(&p, n * sizeof(T), st) != cudaSuccess) throw Error(-4, "device tree: allocation failed");
  }
  void free(cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
    n = 0;
  }
};

struct DLevel {
  int n = 0;
  DArr<unsigned long long> code;
  DArr<int> start, end, parent, bnd, cnt, off;
  DArr<unsigned char> split, forced, mark;
  void free(cudaStream_t st) {
    code.free(st);
    start.free(st);
    end.free(st);
    parent.free(st);
    bnd.free(st);
    cnt.free(st);
    off.free(st);
    split.free(st);
    forced.free(st);
    mark.free(st);
  }
};

#define DT_CHECK(x)                                                                           \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) throw Error(-7, std::string("device tree: ") + cudaGetErrorString(e_)); \
  } while (0)

}  // namespace

void device_octree(const unsigned long long* keys, int64_t n, int leaf_max, cudaStream_t st, DevTreeResult& out,
                   int* launches) {
  std::vector<DLevel> L(kDepthBits + 1);
  DArr<int> err;
  err.resize(2, st);
  DT_CHECK(cudaMemsetAsync(err.p, 0, 2 * sizeof(int), st));
  int nl = 0;
  // level 0: the root cube
  {
    DLevel& R = L[0];
    R.n = 1;
    R.code.resize(1, st);
    R.start.resize(1, st);
    R.end.resize(1, st);
    R.parent.resize(1, st);
    const unsigned long long z = 0;
    const int s0 = 0, e0 = (int)n, p0 = -1;
    DT_CHECK(cudaMemcpyAsync(R.code.p, &z, sizeof(z), cudaMemcpyHostToDevice, st));
    DT_CHECK(cudaMemcpyAsync(R.start.p, &s0, sizeof(int), cudaMemcpyHostToDevice, st));
    DT_CHECK(cudaMemcpyAsync(R.end.p, &e0, sizeof(int), cudaMemcpyHostToDevice, st));
    DT_CHECK(cudaMemcpyAsync(R.parent.p, &p0, sizeof(int), cudaMemcpyHostToDevice, st));
    R.forced.resize(1, st);
    DT_CHECK(cudaMemsetAsync(R.forced.p, 0, 1, st));
    DT_CHECK(cudaStreamSynchronize(st));
  }
  int nlev = 1;  // levels 0 .. nlev-1 exist
  // generate levels from l0 on (level l0's boxes exist; its split flags are recomputed)
  auto generate = [&](int l0) {
    for (int l = l0; l <= kDepthBits; ++l) {
      DLevel& C = L[l];
      C.split.resize(C.n, st);
      C.bnd.resize(9 * (size_t)C.n, st);
      C.cnt.resize(C.n, st);
      C.off.resize(C.n + 1, st);
      k_dt_children<<<(C.n + 255) / 256, 256, 0, st>>>(keys, l, C.n, C.code.p, C.start.p, C.end.p, C.forced.p,
                                                      leaf_max, C.split.p, C.bnd.p, C.cnt.p, err.p);
      k_dt_scan<<<1, 1024, 0, st>>>(C.cnt.p, C.n, C.off.p);
      nl += 2;
      int nc = 0, herr = 0;
      DT_CHECK(cudaMemcpyAsync(&nc, C.off.p + C.n, sizeof(int), cudaMemcpyDeviceToHost, st));
      DT_CHECK(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      DT_CHECK(cudaStreamSynchronize(st));
      if (herr) throw Error(-2, "duplicate points force refinement past depth 20");
      if (nc == 0) {
        nlev = l + 1;
        return;
      }
      DLevel& K = L[l + 1];
      // forced flags of the next level survive regeneration only through their codes: a box
      // regenerated at level l+1 is forced iff it was forced before (its code is unchanged)
      std::vector<unsigned long long> old_codes;
      std::vector<unsigned char> old_forced;
      if (K.n > 0 && K.forced.p) {
        old_codes.resize(K.n);
        old_forced.resize(K.n);
        DT_CHECK(cudaMemcpyAsync(old_codes.data(), K.code.p, K.n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        DT_CHECK(cudaMemcpyAsync(old_forced.data(), K.forced.p, K.n, cudaMemcpyDeviceToHost, st));
        DT_CHECK(cudaStreamSynchronize(st));
      }
      K.n = nc;
      K.code.resize(nc, st);
      K.start.resize(nc, st);
      K.end.resize(nc, st);
      K.parent.resize(nc, st);
      K.forced.resize(nc, st);
      k_dt_emit<<<(C.n + 255) / 256, 256, 0, st>>>(C.n, C.code.p, C.split.p, C.bnd.p, C.off.p, K.code.p, K.start.p,
                                                  K.end.p, K.parent.p);
      ++nl;
      if (old_codes.empty() || std::none_of(old_forced.begin(), old_forced.end(), [](unsigned char v) { return v; })) {
        DT_CHECK(cudaMemsetAsync(K.forced.p, 0, nc, st));
      } else {
        std::vector<unsigned long long> codes(nc);
        DT_CHECK(cudaMemcpyAsync(codes.data(), K.code.p, nc * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        DT_CHECK(cudaStreamSynchronize(st));
        std::vector<unsigned char> f(nc, 0);
        for (int i = 0; i < nc; ++i) {
          auto it = std::lower_bound(old_codes.begin(), old_codes.end(), codes[i]);
          if (it != old_codes.end() && *it == codes[i]) f[i] = old_forced[it - old_codes.begin()];
        }
        DT_CHECK(cudaMemcpyAsync(K.forced.p, f.data(), nc, cudaMemcpyHostToDevice, st));
      }
    }
    nlev = kDepthBits + 1;
  };
  generate(0);
  // 2:1 balance to a fixed point
  for (int pass = 0; pass < 64; ++pass) {
    std::vector<LevelView> lv(nlev);
    std::vector<unsigned char*> mk(nlev);
    for (int l = 0; l < nlev; ++l) {
      L[l].mark.resize(L[l].n, st);
      DT_CHECK(cudaMemsetAsync(L[l].mark.p, 0, L[l].n, st));
      lv[l] = LevelView{L[l].code.p, L[l].split.p, L[l].n};
      mk[l] = L[l].mark.p;
    }
    DArr<LevelView> dlv;
    DArr<unsigned char*> dmk;
    dlv.resize(nlev, st);
    dmk.resize(nlev, st);
    DT_CHECK(cudaMemcpyAsync(dlv.p, lv.data(), nlev * sizeof(LevelView), cudaMemcpyHostToDevice, st));
    DT_CHECK(cudaMemcpyAsync(dmk.p, mk.data(), nlev * sizeof(unsigned char*), cudaMemcpyHostToDevice, st));
    DT_CHECK(cudaMemsetAsync(err.p + 1, 0, sizeof(int), st));
    for (int ly = 2; ly < nlev; ++ly) {
      k_dt_balance<<<(L[ly].n + 127) / 128, 128, 0, st>>>(ly, L[ly].n, L[ly].code.p, L[ly].split.p, dlv.p, dmk.p,
                                                          err.p + 1);
      ++nl;
    }
    int any = 0;
    DT_CHECK(cudaMemcpyAsync(&any, err.p + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    DT_CHECK(cudaStreamSynchronize(st));
    dlv.free(st);
    dmk.free(st);
    if (!any) break;
    // forced |= mark on every level; regenerate from the shallowest marked level
    int lmin = nlev;
    for (int l = 0; l < nlev; ++l) {
      std::vector<unsigned char> m(L[l].n), f(L[l].n);
      DT_CHECK(cudaMemcpyAsync(m.data(), L[l].mark.p, L[l].n, cudaMemcpyDeviceToHost, st));
      DT_CHECK(cudaMemcpyAsync(f.data(), L[l].forced.p, L[l].n, cudaMemcpyDeviceToHost, st));
      DT_CHECK(cudaStreamSynchronize(st));
      bool hit = false;
      for (int i = 0; i < L[l].n; ++i)
        if (m[i]) {
          f[i] = 1;
          hit = true;
        }
      if (hit) {
        lmin = std::min(lmin, l);
        DT_CHECK(cudaMemcpyAsync(L[l].forced.p, f.data(), L[l].n, cudaMemcpyHostToDevice, st));
      }
    }
    generate(lmin);
  }
  // results to the host (level-major, Morton order within a level)
  out.nlevels = nlev;
  out.level_n.assign(nlev, 0);
  out.code.clear();
  out.start.clear();
  out.end.clear();
  out.parent.clear();
  for (int l = 0; l < nlev; ++l) {
    const int m = L[l].n;
    out.level_n[l] = m;
    const size_t o = out.code.size();
    out.code.resize(o + m);
    out.start.resize(o + m);
    out.end.resize(o + m);
    out.parent.resize(o + m);
    DT_CHECK(cudaMemcpyAsync(out.code.data() + o, L[l].code.p, m * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    DT_CHECK(cudaMemcpyAsync(out.start.data() + o, L[l].start.p, m * sizeof(int), cudaMemcpyDeviceToHost, st));
    DT_CHECK(cudaMemcpyAsync(out.end.data() + o, L[l].end.p, m * sizeof(int), cudaMemcpyDeviceToHost, st));
    DT_CHECK(cudaMemcpyAsync(out.parent.data() + o, L[l].parent.p, m * sizeof(int), cudaMemcpyDeviceToHost, st));
  }
  DT_CHECK(cudaStreamSynchronize(st));
  for (auto& x : L) x.free(st);
  err.free(st);
  if (launches) *launches = nl;
}

// ------------------------------------------------------------------ owner lists (see devtree.h)
namespace {

struct TopoTree {
  const unsigned long long* code;
  const unsigned char* leaf;
  const int* leafrank;
  int first[kDepthBits + 2];  // level prefix
  int nlevels;
};

__global__ void k_leaf_i32(const unsigned char* __restrict__ leaf, int n, int* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = leaf[i] ? 1 : 0;
}

// owners of the level: its boxes (ids first[lvl] ..), then the leaves of the coarser levels
__global__ void k_topo_owners(TopoTree T, int lvl, int nlb, int* __restrict__ owners) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= T.first[lvl + 1]) return;
  if (b >= T.first[lvl]) owners[b - T.first[lvl]] = b;
  else if (T.leaf[b]) owners[nlb + T.leafrank[b]] = b;
}

// Level box i (one thread): the owners covering the cells of its 5 × 5 × 5 neighbourhood — a level
// box by binary search in the level's sorted codes, else the first ancestor cell that is a box
// (an owner iff it is a leaf) — deduplicated, ascending; sep ≤ 1 → N, else Q (sep = the Chebyshev
// gap in level cells between the box and the owner's extent).  cand[i·124 ..]: N first, then Q.
__global__ void k_topo_nq(TopoTree T, int lvl, int nlb, int* __restrict__ cand, int* __restrict__ nN,
                          int* __restrict__ nQ) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nlb) return;
  const int f0 = T.first[lvl];
  int c[3];
  decode3(T.code[f0 + i], lvl, c);
  const int lim = (1 << lvl) - 1;
  int own[125];
  unsigned char sp[125];
  int n = 0;
  for (int dx = -2; dx <= 2; ++dx)
    for (int dy = -2; dy <= 2; ++dy)
      for (int dz = -2; dz <= 2; ++dz) {
        const int x = c[0] + dx, y = c[1] + dy, z = c[2] + dz;
        if (x < 0 || y < 0 || z < 0 || x > lim || y > lim || z > lim) continue;
        int o = -1, s = 0;
        unsigned long long key = encode3(x, y, z, lvl);
        int j = find_code(T.code + f0, nlb, key);
        if (j >= 0) {
          o = j;
          s = max(abs(dx), max(abs(dy), abs(dz)));
        } else {
          for (int m = lvl - 1; m >= 0; --m) {
            key >>= 3;
            const int fm = T.first[m];
            j = find_code(T.code + fm, T.first[m + 1] - fm, key);
            if (j >= 0) {
              if (T.leaf[fm + j]) {
                o = nlb + T.leafrank[fm + j];
                const int d = lvl - m;
                const int cc[3] = {x >> d, y >> d, z >> d};
                s = INT_MIN;
                for (int a = 0; a < 3; ++a) {
                  const int lo = cc[a] << d, hi = ((cc[a] + 1) << d) - 1;
                  s = max(s, max(lo - c[a], c[a] - hi));
                }
              }
              break;
            }
          }
        }
        if (o < 0 || o == i) continue;
        // sorted insert without duplicates
        int p = 0;
        while (p < n && own[p] < o) ++p;
        if (p < n && own[p] == o) continue;
        for (int q = n; q > p; --q) {
          own[q] = own[q - 1];
          sp[q] = sp[q - 1];
        }
        own[p] = o;
        sp[p] = (unsigned char)(s <= 1 ? 1 : 0);
        ++n;
      }
  int a = 0;
  int* out = cand + (size_t)i * 124;
  for (int p = 0; p < n; ++p)
    if (sp[p]) out[a++] = own[p];
  nN[i] = a;
  for (int p = 0; p < n; ++p)
    if (!sp[p]) out[a++] = own[p];
  nQ[i] = a - nN[i];
}

// compact the fixed-stride candidate lists into the N and Q CSR arrays
__global__ void k_topo_compact(const int* __restrict__ cand, const int* __restrict__ nN, const int* __restrict__ nQ,
                               const int* __restrict__ nptr, const int* __restrict__ qptr, int nlb,
                               int* __restrict__ nidx, int* __restrict__ qidx) {
  const int i = blockIdx.x;
  if (i >= nlb) return;
  const int* src = cand + (size_t)i * 124;
  for (int e = threadIdx.x; e < nN[i]; e += blockDim.x) nidx[nptr[i] + e] = src[e];
  for (int e = threadIdx.x; e < nQ[i]; e += blockDim.x) qidx[qptr[i] + e] = src[nN[i] + e];
}

__global__ void k_topo_paircount(const int* __restrict__ nN, const int* __restrict__ nQ, int nlb,
                                 int* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nlb) cnt[i] = (1 + nN[i]) * (1 + nN[i]) + 2 * nQ[i];
}

// level box i (one CTA): keys x·no + y for x, y ∈ {i} ∪ N(i), and (i, q), (q, i) for q ∈ Q(i)
__global__ void k_topo_pairs(const int* __restrict__ nptr, const int* __restrict__ nidx,
                             const int* __restrict__ qptr, const int* __restrict__ qidx,
                             const int* __restrict__ poff, int no, unsigned long long* __restrict__ keys) {
  const int i = blockIdx.x;
  const int n1 = nptr[i + 1] - nptr[i] + 1, nq = qptr[i + 1] - qptr[i];
  const int* N = nidx + nptr[i];
  const int* Q = qidx + qptr[i];
  unsigned long long* out = keys + poff[i];
  for (int e = threadIdx.x; e < n1 * n1; e += blockDim.x) {
    const int a = e / n1, b = e % n1;
    const int x = a == 0 ? i : N[a - 1], y = b == 0 ? i : N[b - 1];
    out[e] = (unsigned long long)x * no + y;
  }
  for (int e = threadIdx.x; e < nq; e += blockDim.x) {
    out[n1 * n1 + 2 * e] = (unsigned long long)i * no + Q[e];
    out[n1 * n1 + 2 * e + 1] = (unsigned long long)Q[e] * no + i;
  }
}

// row pointers of the sorted unique keys: nbptr[a] = first key ≥ a·no; partner = key − a·no
__global__ void k_topo_rows(const unsigned long long* __restrict__ keys, const int* __restrict__ nuniq, int no,
                            int* __restrict__ nbptr, int* __restrict__ nbidx) {
  const int n = *nuniq;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t <= no) {
    const unsigned long long c = (unsigned long long)t * no;
    int lo = 0, hi = n;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (keys[mid] < c) lo = mid + 1;
      else hi = mid;
    }
    nbptr[t] = lo;
  }
  for (int e = t; e < n; e += gridDim.x * blockDim.x) nbidx[e] = (int)(keys[e] % (unsigned long long)no);
}

}  // namespace

void device_leafrank(const unsigned char* d_leaf, int nboxes, int* d_leafrank, cudaStream_t st) {
  DArr<int> tmp, off;
  tmp.resize(nboxes, st);
  off.resize(nboxes + 1, st);
  k_leaf_i32<<<(nboxes + 255) / 256, 256, 0, st>>>(d_leaf, nboxes, tmp.p);
  k_dt_scan<<<1, 1024, 0, st>>>(tmp.p, nboxes, off.p);
  DT_CHECK(cudaMemcpyAsync(d_leafrank, off.p, nboxes * sizeof(int), cudaMemcpyDeviceToDevice, st));
  DT_CHECK(cudaGetLastError());
  tmp.free(st);
  off.free(st);
}

void device_topology(const unsigned long long* d_code, const unsigned char* d_leaf, const int* d_leafrank,
                     const int* level_first, int nlevels, int lvl, cudaStream_t st, DevTopo& out, int* launches) {
  TopoTree T{};
  T.code = d_code;
  T.leaf = d_leaf;
  T.leafrank = d_leafrank;
  T.nlevels = nlevels;
  for (int l = 0; l <= nlevels; ++l) T.first[l] = level_first[l];
  const int nlb = level_first[lvl + 1] - level_first[lvl];
  int nl = 0;
  // coarser leaves: leafrank of the level's first box
  int ncoarse = 0;
  DT_CHECK(cudaMemcpyAsync(&ncoarse, d_leafrank + level_first[lvl], sizeof(int), cudaMemcpyDeviceToHost, st));
  DT_CHECK(cudaStreamSynchronize(st));
  const int no = nlb + ncoarse;
  out.nlb = nlb;
  out.no = no;
  DArr<int> owners, cand, nN, nQ, nptr, qptr, nidx, qidx, pcnt, poff, nbptr, nbidx, nuniq;
  owners.resize(no, st);
  cand.resize((size_t)nlb * 124, st);
  nN.resize(nlb, st);
  nQ.resize(nlb, st);
  nptr.resize(nlb + 1, st);
  qptr.resize(nlb + 1, st);
  pcnt.resize(nlb, st);
  poff.resize(nlb + 1, st);
  nuniq.resize(1, st);
  k_topo_owners<<<(level_first[lvl + 1] + 255) / 256, 256, 0, st>>>(T, lvl, nlb, owners.p);
  k_topo_nq<<<(nlb + 63) / 64, 64, 0, st>>>(T, lvl, nlb, cand.p, nN.p, nQ.p);
  k_dt_scan<<<1, 1024, 0, st>>>(nN.p, nlb, nptr.p);
  k_dt_scan<<<1, 1024, 0, st>>>(nQ.p, nlb, qptr.p);
  k_topo_paircount<<<(nlb + 255) / 256, 256, 0, st>>>(nN.p, nQ.p, nlb, pcnt.p);
  k_dt_scan<<<1, 1024, 0, st>>>(pcnt.p, nlb, poff.p);
  nl += 6;
  int tot[3] = {0, 0, 0};
  DT_CHECK(cudaMemcpyAsync(&tot[0], nptr.p + nlb, sizeof(int), cudaMemcpyDeviceToHost, st));
  DT_CHECK(cudaMemcpyAsync(&tot[1], qptr.p + nlb, sizeof(int), cudaMemcpyDeviceToHost, st));
  DT_CHECK(cudaMemcpyAsync(&tot[2], poff.p + nlb, sizeof(int), cudaMemcpyDeviceToHost, st));
  DT_CHECK(cudaStreamSynchronize(st));
  if ((long long)nlb * 15873 > INT_MAX) {  // (1 + 124)² + 2·124 candidates per box at most: check the 32-bit scan
    std::vector<int> hn(nlb), hq(nlb);
    DT_CHECK(cudaMemcpyAsync(hn.data(), nN.p, nlb * sizeof(int), cudaMemcpyDeviceToHost, st));
    DT_CHECK(cudaMemcpyAsync(hq.data(), nQ.p, nlb * sizeof(int), cudaMemcpyDeviceToHost, st));
    DT_CHECK(cudaStreamSynchronize(st));
    long long sum = 0;
    for (int i = 0; i < nlb; ++i) sum += (long long)(1 + hn[i]) * (1 + hn[i]) + 2LL * hq[i];
    if (sum > INT_MAX) throw Error(-8, "device topology: more than 2^31 candidate block pairs at one level");
  }
  nidx.resize(tot[0], st);
  qidx.resize(tot[1], st);
  k_topo_compact<<<std::max(nlb, 1), 64, 0, st>>>(cand.p, nN.p, nQ.p, nptr.p, qptr.p, nlb, nidx.p, qidx.p);
  ++nl;
  // pair set: candidate keys → radix sort → unique → CSR
  const int npair = tot[2];
  DArr<unsigned long long> keys, keys2, uniq;
  keys.resize(npair, st);
  keys2.resize(npair, st);
  uniq.resize(npair, st);
  if (nlb > 0) k_topo_pairs<<<nlb, 128, 0, st>>>(nptr.p, nidx.p, qptr.p, qidx.p, poff.p, no, keys.p);
  int bits = 1;
  while (((unsigned long long)1 << bits) < (unsigned long long)no * no) ++bits;
  size_t tb1 = 0, tb2 = 0;
  DT_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, tb1, keys.p, keys2.p, npair, 0, bits, st));
  DT_CHECK(cub::DeviceSelect::Unique(nullptr, tb2, keys2.p, uniq.p, nuniq.p, npair, st));
  DArr<unsigned char> tmp;
  tmp.resize(std::max(tb1, tb2), st);
  size_t tb = tmp.n;
  DT_CHECK(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys.p, keys2.p, npair, 0, bits, st));
  tb = tmp.n;
  DT_CHECK(cub::DeviceSelect::Unique(tmp.p, tb, keys2.p, uniq.p, nuniq.p, npair, st));
  int nu = 0;
  DT_CHECK(cudaMemcpyAsync(&nu, nuniq.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  DT_CHECK(cudaStreamSynchronize(st));
  nbptr.resize(no + 1, st);
  nbidx.resize(nu, st);
  k_topo_rows<<<(std::max(no + 1, nu) + 255) / 256, 256, 0, st>>>(uniq.p, nuniq.p, no, nbptr.p, nbidx.p);
  nl += 2 + 8;  // + the CUB sort passes / select (approximate count)
  DT_CHECK(cudaGetLastError());
  // results to the host
  out.owners.resize(no);
  out.nptr.resize(nlb + 1);
  out.qptr.resize(nlb + 1);
  out.nidx.resize(tot[0]);
  out.qidx.resize(tot[1]);
  out.nbptr.resize(no + 1);
  out.nbidx.resize(nu);
  auto d2h = [&](void* dst, const void* src, size_t bytes) {
    if (bytes) DT_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
  };
  d2h(out.owners.data(), owners.p, no * sizeof(int));
  d2h(out.nptr.data(), nptr.p, (nlb + 1) * sizeof(int));
  d2h(out.qptr.data(), qptr.p, (nlb + 1) * sizeof(int));
  d2h(out.nidx.data(), nidx.p, (size_t)tot[0] * sizeof(int));
  d2h(out.qidx.data(), qidx.p, (size_t)tot[1] * sizeof(int));
  d2h(out.nbptr.data(), nbptr.p, (no + 1) * sizeof(int));
  d2h(out.nbidx.data(), nbidx.p, (size_t)nu * sizeof(int));
  DT_CHECK(cudaStreamSynchronize(st));
  for (DArr<int>* a : {&owners, &cand, &nN, &nQ, &nptr, &qptr, &nidx, &qidx, &pcnt, &poff, &nbptr, &nbidx, &nuniq})
    a->free(st);
  keys.free(st);
  keys2.free(st);
  uniq.free(st);
  tmp.free(st);
  if (launches) *launches = nl;
}

}  // namespace fmmlu
