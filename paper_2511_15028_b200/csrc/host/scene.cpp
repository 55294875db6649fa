// Synthetic scenes + LogicalTree builders (binned SAH, median split, 8-wide collapse).
// Contract: SPEC.md:523-591.  The reference's own src/scene.cpp / src/logical.cpp are
// placeholders, so the topology cannot be compared with the reference; what matters
// is that the oracle and the GPU consume the *same* LogicalTree.
#include "scene.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>

#include "rng.hpp"

namespace scion {

// ---------------------------------------------------------------------------------
// scenes
// ---------------------------------------------------------------------------------
static inline float lattice(uint64_t seed, int32_t ix, int32_t iz, uint32_t octave) {
  uint64_t h = splitmix64(seed ^ ((uint64_t)(uint32_t)ix << 32 | (uint32_t)iz) ^ ((uint64_t)octave * 0x9e3779b97f4a7c15ull));
  return (float)(h >> 40) * (1.0f / 16777216.0f);
}
static inline float smooth(float t) { return t * t * (3.0f - 2.0f * t); }
static float value_noise(uint64_t seed, float x, float z, uint32_t octave) {
  float fx = std::floor(x), fz = std::floor(z);
  int32_t ix = (int32_t)fx, iz = (int32_t)fz;
  float tx = smooth(x - fx), tz = smooth(z - fz);
  float a = lattice(seed, ix, iz, octave), b = lattice(seed, ix + 1, iz, octave);
  float c = lattice(seed, ix, iz + 1, octave), d = lattice(seed, ix + 1, iz + 1, octave);
  float ab = a + (b - a) * tx, cd = c + (d - c) * tx;
  return ab + (cd - ab) * tz;
}
static float terrain_height(uint64_t seed, float x, float z) {
  float h = 0.0f, amp = 0.35f, freq = 2.0f;
  for (uint32_t o = 0; o < 6; o++) {
    h += amp * (value_noise(seed, x * freq + 17.0f, z * freq + 29.0f, o) - 0.5f);
    amp *= 0.5f;
    freq *= 2.0f;
  }
  return h;
}

static void push_tri(std::vector<float>& v, size_t t, const float* a, const float* b, const float* c) {
  float* p = v.data() + t * 9;
  std::memcpy(p, a, 12);
  std::memcpy(p + 3, b, 12);
  std::memcpy(p + 6, c, 12);
}

void make_terrain(uint32_t G, uint64_t seed, scion_scene& out) {
  if (G == 0) throw std::runtime_error("terrain grid must be > 0");
  out.name = "terrain" + std::to_string(G);
  std::vector<float> verts((size_t)(G + 1) * (G + 1) * 3);
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j <= (int64_t)G; j++)
    for (uint32_t i = 0; i <= G; i++) {
      float x = -1.0f + 2.0f * (float)i / (float)G, z = -1.0f + 2.0f * (float)j / (float)G;
      float* p = &verts[((size_t)j * (G + 1) + i) * 3];
      p[0] = x;
      p[1] = terrain_height(seed, x, z);
      p[2] = z;
    }
  out.tris.resize((size_t)G * G * 2 * 9);
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < (int64_t)G; j++)
    for (uint32_t i = 0; i < G; i++) {
      const float* v00 = &verts[((size_t)j * (G + 1) + i) * 3];
      const float* v10 = v00 + 3;
      const float* v01 = &verts[((size_t)(j + 1) * (G + 1) + i) * 3];
      const float* v11 = v01 + 3;
      size_t t = ((size_t)j * G + i) * 2;
      push_tri(out.tris, t, v00, v11, v10);
      push_tri(out.tris, t + 1, v00, v01, v11);
    }
}

void make_sphere(uint32_t G, uint64_t seed, scion_scene& out) {
  if (G < 2) throw std::runtime_error("sphere grid must be >= 2");
  out.name = "sphere" + std::to_string(G);
  std::vector<float> verts((size_t)(G + 1) * (G + 1) * 3);
  const double PI = 3.14159265358979323846;
  for (uint32_t j = 0; j <= G; j++)
    for (uint32_t i = 0; i <= G; i++) {
      double th = PI * (double)j / G, ph = 2.0 * PI * (double)(i % G) / G;
      float dir[3] = {(float)(std::sin(th) * std::cos(ph)), (float)std::cos(th), (float)(std::sin(th) * std::sin(ph))};
      float r = 1.0f + 0.1f * (value_noise(seed, dir[0] * 3.0f + dir[1] * 5.0f, dir[2] * 3.0f - dir[1] * 2.0f, 0) - 0.5f);
      float* p = &verts[((size_t)j * (G + 1) + i) * 3];
      for (int a = 0; a < 3; a++) p[a] = dir[a] * r;
    }
  out.tris.resize((size_t)G * G * 2 * 9);
  for (uint32_t j = 0; j < G; j++)
    for (uint32_t i = 0; i < G; i++) {
      const float* v00 = &verts[((size_t)j * (G + 1) + i) * 3];
      const float* v10 = v00 + 3;
      const float* v01 = &verts[((size_t)(j + 1) * (G + 1) + i) * 3];
      const float* v11 = v01 + 3;
      size_t t = ((size_t)j * G + i) * 2;
      push_tri(out.tris, t, v00, v10, v11);
      push_tri(out.tris, t + 1, v00, v11, v01);
    }
}

void make_cloud(uint64_t P, uint64_t seed, scion_scene& out) {
  if (P == 0) throw std::runtime_error("cloud needs >= 1 point");
  out.name = "cloud" + std::to_string(P);
  out.tris.resize((size_t)P * 9);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)P; i++) {
    Stream s(seed, (uint64_t)i);
    float p[3] = {s.uniform(), s.uniform(), s.uniform()};
    push_tri(out.tris, (size_t)i, p, p, p);  // degenerate triangle p0 = p1 = p2
  }
}

void scene_bounds(const scion_scene& s, float lo[3], float hi[3]) {
  for (int a = 0; a < 3; a++) { lo[a] = std::numeric_limits<float>::infinity(); hi[a] = -lo[a]; }
  for (size_t i = 0; i < s.tris.size(); i += 3)
    for (int a = 0; a < 3; a++) {
      lo[a] = std::min(lo[a], s.tris[i + a]);
      hi[a] = std::max(hi[a], s.tris[i + a]);
    }
}

// ---------------------------------------------------------------------------------
// binary builders
// ---------------------------------------------------------------------------------
namespace {

struct Box {
  float lo[3], hi[3];
  void reset() {
    for (int a = 0; a < 3; a++) { lo[a] = std::numeric_limits<float>::infinity(); hi[a] = -lo[a]; }
  }
  void grow(const Box& b) {
    for (int a = 0; a < 3; a++) { lo[a] = std::min(lo[a], b.lo[a]); hi[a] = std::max(hi[a], b.hi[a]); }
  }
  void grow(const float* p) {
    for (int a = 0; a < 3; a++) { lo[a] = std::min(lo[a], p[a]); hi[a] = std::max(hi[a], p[a]); }
  }
  // half surface area; 0 for empty boxes
  float area() const {
    float ex = hi[0] - lo[0], ey = hi[1] - lo[1], ez = hi[2] - lo[2];
    if (!(ex >= 0.0f && ey >= 0.0f && ez >= 0.0f)) return 0.0f;
    return ex * ey + ey * ez + ez * ex;
  }
};

struct TmpNode {
  Box box;
  int64_t left = -1, right = -1;  // tmp indices
  uint32_t first = 0, count = 0;  // range in the permuted index array
};

struct BuildCtx {
  const std::vector<Box>& pbox;
  const std::vector<float>& cent;  // 3 per prim
  std::vector<uint32_t>& idx;
  std::vector<TmpNode>& tmp;
  std::atomic<int64_t>& next;
  Builder kind;
  uint32_t bins, max_leaf, max_depth;
};

inline uint32_t ceil_log2(uint64_t v) {
  uint32_t l = 0;
  while ((1ull << l) < v) l++;
  return l;
}

// returns the split position (first index of the right half) or `first` if no valid split
uint32_t split_range(BuildCtx& c, uint32_t first, uint32_t count, uint32_t depth, const Box& cb) {
  uint32_t* I = c.idx.data() + first;
  // depth cap: if a balanced subtree just fits under max_depth, split by the index median
  uint32_t need = ceil_log2((count + c.max_leaf - 1) / c.max_leaf);
  bool force_median = c.kind == Builder::Median || depth + need + 1 >= c.max_depth;
  int axis = -1;
  if (!force_median) {
    // binned SAH over 3 axes, C_trav = C_isect = 1; the parent-area normalisation
    // is common to every candidate and therefore dropped from the comparison.
    const uint32_t B = c.bins;
    float best = std::numeric_limits<float>::infinity();
    int best_axis = -1;
    uint32_t best_bin = 0;
    std::vector<Box> bb(3 * B);
    std::vector<uint32_t> bc(3 * B, 0);
    for (auto& b : bb) b.reset();
    float scale[3];
    for (int a = 0; a < 3; a++) {
      float e = cb.hi[a] - cb.lo[a];
      scale[a] = e > 0.0f ? (float)B / e : 0.0f;
    }
    for (uint32_t k = 0; k < count; k++) {
      uint32_t p = I[k];
      for (int a = 0; a < 3; a++) {
        if (scale[a] == 0.0f) continue;
        int b = (int)((c.cent[3 * (size_t)p + a] - cb.lo[a]) * scale[a]);
        b = std::min<int>(std::max(b, 0), (int)B - 1);
        bb[a * B + b].grow(c.pbox[p]);
        bc[a * B + b]++;
      }
    }
    std::vector<float> right_area(B);
    std::vector<uint32_t> right_cnt(B);
    for (int a = 0; a < 3; a++) {
      if (scale[a] == 0.0f) continue;
      Box acc;
      acc.reset();
      uint32_t n = 0;
      for (int b = (int)B - 1; b >= 1; b--) {
        acc.grow(bb[a * B + b]);
        n += bc[a * B + b];
        right_area[b] = acc.area();
        right_cnt[b] = n;
      }
      acc.reset();
      n = 0;
      for (uint32_t b = 1; b < B; b++) {  // split plane between bin b-1 and b
        acc.grow(bb[a * B + b - 1]);
        n += bc[a * B + b - 1];
        if (n == 0 || right_cnt[b] == 0) continue;
        float cost = acc.area() * (float)n + right_area[b] * (float)right_cnt[b];
        if (cost < best) {  // strict: ties keep the lowest axis, then the lowest bin
          best = cost;
          best_axis = a;
          best_bin = b;
        }
      }
    }
    if (best_axis >= 0) {
      int a = best_axis;
      float lo = cb.lo[a], sc = scale[a];
      uint32_t B1 = c.bins - 1;
      uint32_t* mid = std::partition(I, I + count, [&](uint32_t p) {
        int b = (int)((c.cent[3 * (size_t)p + a] - lo) * sc);
        b = std::min<int>(std::max(b, 0), (int)B1);
        return (uint32_t)b < best_bin;
      });
      uint32_t m = (uint32_t)(mid - I);
      if (m > 0 && m < count) return first + m;
    }
    axis = -2;  // coincident centroids: index halves
  }
  uint32_t m = count / 2;
  if (axis != -2) {
    // median along the longest centroid-bounds axis
    int a = 0;
    float e0 = cb.hi[0] - cb.lo[0], e1 = cb.hi[1] - cb.lo[1], e2 = cb.hi[2] - cb.lo[2];
    if (e1 > e0 && e1 >= e2) a = 1;
    else if (e2 > e0 && e2 > e1) a = 2;
    std::nth_element(I, I + m, I + count, [&](uint32_t x, uint32_t y) {
      float cx = c.cent[3 * (size_t)x + a], cy = c.cent[3 * (size_t)y + a];
      return cx < cy || (cx == cy && x < y);
    });
  }
  return first + m;
}

void build_rec(BuildCtx& c, int64_t self, uint32_t first, uint32_t count, uint32_t depth) {
  TmpNode& n = c.tmp[(size_t)self];
  n.first = first;
  n.count = count;
  Box b, cb;
  b.reset();
  cb.reset();
  for (uint32_t k = 0; k < count; k++) {
    uint32_t p = c.idx[first + k];
    b.grow(c.pbox[p]);
    cb.grow(&c.cent[3 * (size_t)p]);
  }
  n.box = b;
  if (count <= c.max_leaf) return;  // leaf ("count <= max_leaf")
  uint32_t mid = split_range(c, first, count, depth, cb);
  int64_t l = c.next.fetch_add(2), r = l + 1;
  n.left = l;
  n.right = r;
  uint32_t lc = mid - first, rc = count - lc;
  if (count > 4096) {
#pragma omp task default(shared) firstprivate(l, first, lc, depth)
    build_rec(c, l, first, lc, depth + 1);
#pragma omp task default(shared) firstprivate(r, mid, rc, depth)
    build_rec(c, r, mid, rc, depth + 1);
#pragma omp taskwait
  } else {
    build_rec(c, l, first, lc, depth + 1);
    build_rec(c, r, mid, rc, depth + 1);
  }
}

inline float round_down(double s) {
  float f = (float)s;
  if ((double)f > s) f = std::nextafterf(f, -std::numeric_limits<float>::infinity());
  return f;
}
inline float round_up(double s) {
  float f = (float)s;
  if ((double)f < s) f = std::nextafterf(f, std::numeric_limits<float>::infinity());
  return f;
}

}  // namespace

static void compute_dop(scion_ltree& out);

void build_binary(const scion_scene& s, Builder kind, uint32_t bins, uint32_t max_leaf, uint32_t max_depth,
                  scion_ltree& out) {
  const uint64_t P = s.ntris();
  if (P == 0) throw std::runtime_error("cannot build a tree over an empty scene");
  if (P >= 0xFFFFFFF0ull) throw std::runtime_error("too many primitives");
  if (max_leaf == 0) throw std::runtime_error("max_leaf must be >= 1");
  if (bins < 2) bins = 2;
  if (max_depth == 0 || max_depth > SCION_STACK_DEPTH - 2) max_depth = SCION_STACK_DEPTH - 2;
  if (ceil_log2((P + max_leaf - 1) / max_leaf) + 1 > max_depth) throw std::runtime_error("max_depth too small for this scene");

  std::vector<Box> pbox(P);
  std::vector<float> cent(3 * P);
  std::vector<uint32_t> idx(P);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)P; i++) {
    const float* T = &s.tris[(size_t)i * 9];
    Box b;
    b.reset();
    b.grow(T);
    b.grow(T + 3);
    b.grow(T + 6);
    pbox[i] = b;
    for (int a = 0; a < 3; a++) cent[3 * i + a] = 0.5f * b.lo[a] + 0.5f * b.hi[a];
    idx[i] = (uint32_t)i;
  }
  std::vector<TmpNode> tmp(2 * P);
  std::atomic<int64_t> next{1};
  BuildCtx ctx{pbox, cent, idx, tmp, next, kind, bins, max_leaf, max_depth};
#pragma omp parallel
#pragma omp single nowait
  build_rec(ctx, 0, 0, (uint32_t)P, 0);
  const int64_t N = next.load();

  // flatten to preorder; prims are already in left-first leaf order in idx[]
  out = scion_ltree();
  out.nodes.resize((size_t)N);
  out.prim_ids = idx;
  out.tris.resize(P * 9);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)P; i++) std::memcpy(&out.tris[(size_t)i * 9], &s.tris[(size_t)idx[i] * 9], 36);

  struct Item { int64_t tmp; int64_t parent; bool is_right; uint32_t depth; };
  std::vector<Item> stack;
  std::vector<int64_t> post;  // preorder ids in visit order (for the bottom-up DOP pass)
  stack.push_back({0, -1, false, 0});
  int64_t outi = 0;
  uint32_t maxd = 0;
  while (!stack.empty()) {
    Item it = stack.back();
    stack.pop_back();
    const TmpNode& t = tmp[(size_t)it.tmp];
    int64_t me = outi++;
    scion_lnode& n = out.nodes[(size_t)me];
    std::memcpy(n.lo, t.box.lo, 12);
    std::memcpy(n.hi, t.box.hi, 12);
    maxd = std::max(maxd, it.depth);
    if (it.parent >= 0) {
      if (it.is_right) out.nodes[(size_t)it.parent].right = (int32_t)me;
      else out.nodes[(size_t)it.parent].left = (int32_t)me;
    }
    if (t.left < 0) {
      n.left = n.right = -1;
      n.first_prim = t.first;
      n.nprims = t.count;
    } else {
      n.first_prim = 0;
      n.nprims = 0;
      stack.push_back({t.right, me, true, it.depth + 1});
      stack.push_back({t.left, me, false, it.depth + 1});
    }
  }
  out.depth = maxd;
  if (outi != N) throw std::runtime_error("internal: node count mismatch");

  compute_dop(out);
}

// DOP-14 diagonal slabs, bottom-up (children have larger preorder index than parents)
static void compute_dop(scion_ltree& out) {
  const int64_t N = (int64_t)out.nodes.size();
  out.dop_lo2.assign((size_t)N * 4, 0.0f);
  out.dop_hi2.assign((size_t)N * 4, 0.0f);
  for (int64_t i = N - 1; i >= 0; i--) {
    const scion_lnode& n = out.nodes[(size_t)i];
    float* lo2 = &out.dop_lo2[(size_t)i * 4];
    float* hi2 = &out.dop_hi2[(size_t)i * 4];
    if (n.left < 0) {
      for (int k = 0; k < 4; k++) { lo2[k] = std::numeric_limits<float>::infinity(); hi2[k] = -lo2[k]; }
      for (uint32_t p = n.first_prim; p < n.first_prim + n.nprims; p++)
        for (int v = 0; v < 3; v++) {
          const float* q = &out.tris[(size_t)p * 9 + 3 * v];
          double x = q[0], y = q[1], z = q[2];
          double sv[4] = {x + y + z, x + y - z, x - y + z, x - y - z};
          for (int k = 0; k < 4; k++) {
            lo2[k] = std::min(lo2[k], round_down(sv[k]));
            hi2[k] = std::max(hi2[k], round_up(sv[k]));
          }
        }
    } else {
      const float* l0 = &out.dop_lo2[(size_t)n.left * 4];
      const float* l1 = &out.dop_lo2[(size_t)n.right * 4];
      const float* h0 = &out.dop_hi2[(size_t)n.left * 4];
      const float* h1 = &out.dop_hi2[(size_t)n.right * 4];
      for (int k = 0; k < 4; k++) { lo2[k] = std::min(l0[k], l1[k]); hi2[k] = std::max(h0[k], h1[k]); }
    }
  }
}

// Import of an externally built binary tree: re-flatten to preorder, primitives to leaf order.
void import_binary(const scion_lnode* nodes, uint64_t nnodes, const float* tris9, uint64_t ntris, scion_ltree& out) {
  if (!nodes || nnodes == 0 || !tris9 || ntris == 0) throw std::runtime_error("import: empty tree");
  out = scion_ltree();
  out.nodes.reserve(nnodes);
  struct Item { int64_t src; int64_t parent; bool is_right; uint32_t depth; };
  std::vector<Item> stack{{0, -1, false, 0}};
  std::vector<uint8_t> seen(nnodes, 0);
  uint32_t maxd = 0;
  while (!stack.empty()) {
    Item it = stack.back();
    stack.pop_back();
    if (it.src < 0 || (uint64_t)it.src >= nnodes || seen[(size_t)it.src]) throw std::runtime_error("import: child index out of range or node reached twice");
    seen[(size_t)it.src] = 1;
    const scion_lnode& s = nodes[it.src];
    int64_t me = (int64_t)out.nodes.size();
    out.nodes.push_back(s);
    scion_lnode& n = out.nodes.back();
    maxd = std::max(maxd, it.depth);
    if (it.parent >= 0) {
      if (it.is_right) out.nodes[(size_t)it.parent].right = (int32_t)me;
      else out.nodes[(size_t)it.parent].left = (int32_t)me;
    }
    if (s.left < 0) {
      if (s.nprims == 0 || (uint64_t)s.first_prim + s.nprims > ntris) throw std::runtime_error("import: leaf range out of bounds");
      n.left = n.right = -1;
      n.first_prim = (uint32_t)(out.tris.size() / 9);
      for (uint32_t p = s.first_prim; p < s.first_prim + s.nprims; p++) {
        out.tris.insert(out.tris.end(), tris9 + (size_t)p * 9, tris9 + (size_t)p * 9 + 9);
        out.prim_ids.push_back(p);
      }
    } else {
      n.first_prim = n.nprims = 0;
      stack.push_back({s.right, me, true, it.depth + 1});
      stack.push_back({s.left, me, false, it.depth + 1});
    }
  }
  out.depth = maxd;
  compute_dop(out);
}

// ---------------------------------------------------------------------------------
// greedy binary -> 8-wide collapse
// ---------------------------------------------------------------------------------
void collapse8(scion_ltree& t) {
  if (t.has_wide) return;
  t.wnodes.clear();
  t.wleaves.clear();
  auto area = [&](int32_t b) {
    const scion_lnode& n = t.nodes[(size_t)b];
    float ex = n.hi[0] - n.lo[0], ey = n.hi[1] - n.lo[1], ez = n.hi[2] - n.lo[2];
    return ex * ey + ey * ez + ez * ex;
  };
  // iterative preorder emit: an explicit stack of (binary node, parent wide node, slot)
  struct Item { int32_t bin; int32_t parent; int slot; };
  std::vector<Item> stack;
  auto make_leaf = [&](int32_t b) {
    const scion_lnode& n = t.nodes[(size_t)b];
    t.wleaves.push_back({n.first_prim, n.nprims});
    return ~(int32_t)(t.wleaves.size() - 1);
  };
  if (t.nodes[0].left < 0) {
    t.wroot = make_leaf(0);
    t.has_wide = true;
    return;
  }
  t.wroot = 0;
  stack.push_back({0, -1, 0});
  while (!stack.empty()) {
    Item it = stack.back();
    stack.pop_back();
    if (t.nodes[(size_t)it.bin].left < 0) {  // leaves are numbered in DFS slot order
      t.wnodes[(size_t)it.parent].child[it.slot] = make_leaf(it.bin);
      continue;
    }
    int32_t me = (int32_t)t.wnodes.size();
    t.wnodes.emplace_back();
    if (it.parent >= 0) t.wnodes[(size_t)it.parent].child[it.slot] = me;
    int32_t slots[8];
    int ns = 2;
    slots[0] = t.nodes[(size_t)it.bin].left;
    slots[1] = t.nodes[(size_t)it.bin].right;
    while (ns < 8) {
      int pick = -1;
      float best = -1.0f;
      for (int k = 0; k < ns; k++)
        if (t.nodes[(size_t)slots[k]].left >= 0) {
          float a = area(slots[k]);
          if (a > best) { best = a; pick = k; }
        }
      if (pick < 0) break;
      int32_t b = slots[pick];
      for (int k = ns; k > pick + 1; k--) slots[k] = slots[k - 1];  // expand in place, order preserved
      slots[pick] = t.nodes[(size_t)b].left;
      slots[pick + 1] = t.nodes[(size_t)b].right;
      ns++;
    }
    scion_wnode& w = t.wnodes[(size_t)me];
    for (int k = 0; k < 8; k++) {
      if (k < ns) {
        const scion_lnode& n = t.nodes[(size_t)slots[k]];
        std::memcpy(w.lo[k], n.lo, 12);
        std::memcpy(w.hi[k], n.hi, 12);
        w.child[k] = 0;  // patched when the child is emitted
      } else {
        for (int a = 0; a < 3; a++) {
          w.lo[k][a] = std::numeric_limits<float>::infinity();
          w.hi[k][a] = -std::numeric_limits<float>::infinity();
        }
        w.child[k] = SCION_W_SENTINEL;
      }
    }
    // children are visited in slot order: push in reverse so that slot 0 pops first.
    for (int k = ns - 1; k >= 0; k--) stack.push_back({slots[k], me, k});
  }
  t.has_wide = true;
}

}  // namespace scion
