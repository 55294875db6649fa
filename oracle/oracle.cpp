// TEST INFRASTRUCTURE — CPU oracle, not part of the product.  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load liboracle.so.
//
// CPU restatement of the reference's traversal path:
//   closest_hit, binary   /root/reference/proj/corpus/alg/chrt.scion:2-17
//   closest_hit, 8-wide   /root/reference/proj/corpus/alg/chrt8.scion:3-21
//   closest_hit, DOP-14   /root/reference/proj/corpus/alg/chrt_dop14.scion:3-18
//   closest_point         /root/reference/proj/corpus/alg/cpq.scion:3-33, cpq_dop14.scion:2-31
// executed in the RECURSIVE form the DSL is written in (the explicit-stack form of
// SPEC.md:285-293 is order-equivalent), over (a) the encoded byte image of any layout
// (oracle_layouts.hpp) or (b) the LogicalTree itself — the reference's `oracle_query`
// ("interpreting the same Appendix F DSL sources against the identity layout").
// Queries fan out with OpenMP schedule(dynamic,64), the paper's CPU scheme;
// each query owns its accumulators.
//
// PARITY PINNING: the reference has no executor (src/interp.cpp, src/harness.cpp are placeholders), but
// its compiler does produce the lowered traversal.  closest_hit is pinned against that: oracle/ref_interp.cpp
// executes the reference's own IR (reference parser, sema, planner, specialize_destructors, bit reader) on
// trees built by this repository and tests/test_ref_ir_golden.py requires this oracle (and the CUDA kernels)
// to reproduce its answers bit for bit for the 15 corpus layouts.  Also pinned: the reference's KATs
// (tests/test_oracle_kats.py) and the reference planner's slot tables (tests/golden/ref_plans.json).
// Still "parity unpinned": the arithmetic inside intrinsics (dot/cross/sum association, min/max on NaN),
// closest_point and collision_detection results (the reference's lowering of both is broken) — see DESIGN.md §4.
#include <omp.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "oracle_geometry.hpp"
#include "oracle_layouts.hpp"
#include "scion_b200.h"

using namespace oracle;

namespace {

constexpr int kStackDepth = 64;  // specialize.hpp:57

struct Best { float t; uint32_t prim; };
struct BestCp { float d2; V3 p; uint32_t prim; };

// logical-tree "layouts": buf[1] = scion_lnode[], buf[2] = dop_lo2, buf[3] = dop_hi2,
//                         buf[4] = scion_wnode[], buf[5] = scion_wleaf[]
constexpr int L_LOGICAL2 = 100, L_LOGICAL_DOP = 101, L_LOGICAL8 = 102;

inline Node2 decode_any2(const TreeBytes& T, int id, const Ref& ref) {
  if (id < 100) return decode2(T, (LayoutId)id, ref);
  const scion_lnode* nodes = (const scion_lnode*)T.buf[1];
  const scion_lnode& l = nodes[ref.r];
  Node2 n;
  n.box = {{l.lo[0], l.lo[1], l.lo[2]}, {l.hi[0], l.hi[1], l.hi[2]}};
  if (id == L_LOGICAL_DOP) {
    std::memcpy(&n.lo2, T.buf[2] + ref.r * 16, 16);
    std::memcpy(&n.hi2, T.buf[3] + ref.r * 16, 16);
  }
  if (l.left < 0) { n.leaf = true; n.nprims = l.nprims; n.prim_begin = l.first_prim; }
  else { n.left.r = (uint64_t)l.left; n.right.r = (uint64_t)l.right; }
  return n;
}
inline Node8 decode_any8(const TreeBytes& T, int id, uint64_t I) {
  if (id < 100) return decode8(T, (LayoutId)id, I);
  Node8 n;
  int32_t c = (int32_t)(uint32_t)I;
  const scion_wleaf* leaves = (const scion_wleaf*)T.buf[5];
  if (c < 0) {
    if (c == SCION_W_SENTINEL) { n.leaf = true; n.nprims = 0; return n; }
    n.leaf = true; n.prim_begin = leaves[~c].first_prim; n.nprims = leaves[~c].nprims;
    return n;
  }
  const scion_wnode& w = ((const scion_wnode*)T.buf[4])[c];
  for (int k = 0; k < 8; k++) {
    n.box[k] = {{w.lo[k][0], w.lo[k][1], w.lo[k][2]}, {w.hi[k][0], w.hi[k][1], w.hi[k][2]}};
    n.children[k] = (uint64_t)(uint32_t)w.child[k];
  }
  return n;
}

struct Query {
  const TreeBytes& T;
  int id;
  int family;
  scion_counters c{0, 0, 0, 0};
  uint32_t status = SCION_Q_OK;

  void note_stack(int occupancy) {
    if ((uint32_t)occupancy > c.max_stack) c.max_stack = (uint32_t)occupancy;
    if (occupancy > kStackDepth) status = SCION_Q_STACK_OVERFLOW;
  }
  void leaf_tris(const Ray& ray, uint64_t begin, uint32_t n, Best& best) {
    for (uint64_t i = begin; i < begin + n; i++) {
      TriHit h = ray_tri_mt(ray, load_tri(T, i));  // intersects(ray,t) && distmin(ray,t) < best[0]
      c.prim_tests++;
      if (h.some && h.t < best.t) best = {h.t, (uint32_t)i};
    }
  }
  // chrt.scion:2-17 / chrt_dop14.scion:3-18.  `pending` = explicit-stack entries below this call.
  void chrt2(const Ray& ray, const Ref& ref, Best& best, int pending) {
    if (status) return;
    Node2 n = decode_any2(T, id, ref);
    c.node_visits++;
    bool hit;
    float tn;
    if (family == SCION_FAMILY_DOP14) {
      if (ray_aabb(ray, n.box).some) c.cold_loads++;
      hit = intersects_dop(ray, n.box.lo, n.box.hi, n.lo2, n.hi2);
      tn = distmin_dop(ray, n.box.lo, n.box.hi, n.lo2, n.hi2);
    } else {
      hit = intersects(ray, n.box);
      tn = distmin(ray, n.box);
      if ((hit || n.bounds_cold) && n.segments_touched > 1) c.cold_loads++;
    }
    if (!n.leaf) {
      if (hit && tn < best.t) {
        note_stack(pending + 2);  // pop self, push right then left
        chrt2(ray, n.left, best, pending + 1);
        chrt2(ray, n.right, best, pending);
      }
    } else if (hit) {
      leaf_tris(ray, n.prim_begin, n.nprims, best);
    }
  }
  // chrt8.scion:3-21
  void chrt8(const Ray& ray, uint64_t I, Best& best, int pending) {
    if (status) return;
    Node8 n = decode_any8(T, id, I);
    if (n.leaf) { leaf_tris(ray, n.prim_begin, n.nprims, best); return; }
    c.node_visits++;
    // children that pass at entry: the deferred-cull stack form pushes exactly these
    uint32_t mask = 0;
    for (int k = 0; k < 8; k++)
      if (intersects(ray, n.box[k]) && distmin(ray, n.box[k]) < best.t) mask |= 1u << k;
    note_stack(pending + __builtin_popcount(mask));
    for (int k = 0; k < 8; k++) {
      if (intersects(ray, n.box[k]) && distmin(ray, n.box[k]) < best.t) {
        int later = __builtin_popcount(mask >> (k + 1));  // entries of this node still stacked while child k runs
        chrt8(ray, n.children[k], best, pending + later);
      }
    }
  }
  float node_distmin(V3 p, const Node2& n) const {
    return family == SCION_FAMILY_DOP14 ? distmin_dop_point(p, n.box.lo, n.box.hi, n.lo2, n.hi2) : sqdist_point_aabb(p, n.box);
  }
  // cpq.scion:3-33 / cpq_dop14.scion:2-31
  void cpq(V3 p, const Ref& ref, BestCp& best, int pending) {
    if (status) return;
    Node2 n = decode_any2(T, id, ref);
    c.node_visits++;
    if (n.segments_touched > 1) c.cold_loads++;
    if (!n.leaf) {
      if (node_distmin(p, n) < best.d2) {
        float ub = distmax_point_aabb(p, n.box);
        if (ub < best.d2) best.d2 = ub;  // best = (upper_bound, best[1])
        Node2 ln = decode_any2(T, id, n.left), rn = decode_any2(T, id, n.right);
        c.node_visits += 2;
        if (ln.segments_touched > 1) c.cold_loads += 2;
        float L = node_distmin(p, ln), R = node_distmin(p, rn);
        note_stack(pending + 2);
        if (L < R) { cpq(p, n.left, best, pending + 1); cpq(p, n.right, best, pending); }
        else { cpq(p, n.right, best, pending + 1); cpq(p, n.left, best, pending); }
      }
    } else if (node_distmin(p, n) < best.d2) {
      for (uint64_t i = n.prim_begin; i < n.prim_begin + n.nprims; i++) {
        ClosestPt ps = point_triangle(p, load_tri(T, i));
        V3 x = sub(p, ps.p);
        float d2 = dot(x, x);
        c.prim_tests++;
        if (d2 < best.d2) best = {d2, ps.p, (uint32_t)i};
      }
    }
  }
};

int resolve(const char* layout, int* id, int* family) {
  std::string n = layout;
  if (n == "@logical2") { *id = L_LOGICAL2; *family = SCION_FAMILY_BVH2; return 0; }
  if (n == "@logical-dop14") { *id = L_LOGICAL_DOP; *family = SCION_FAMILY_DOP14; return 0; }
  if (n == "@logical8") { *id = L_LOGICAL8; *family = SCION_FAMILY_BVH8; return 0; }
  const LayoutDesc* d = find_layout(layout);
  if (!d) return 1;
  *id = (int)d->id;
  *family = d->family;
  return 0;
}

}  // namespace

extern "C" {

int oracle_layout_count() { return (int)(sizeof(kLayouts) / sizeof(kLayouts[0])); }
const char* oracle_layout_name(int i) { return kLayouts[i].name; }
int oracle_layout_stride(const char* name) { const LayoutDesc* d = find_layout(name); return d ? (int)d->stride : -1; }
int oracle_layout_family(const char* name) { const LayoutDesc* d = find_layout(name); return d ? d->family : -1; }

// closest_hit over a PhysicalTree byte image or a LogicalTree ("@logical2", "@logical-dop14", "@logical8").
int oracle_closest_hit(const TreeBytes* T, const scion_ray* rays, uint64_t n, scion_hit* hits, uint32_t* status,
                       scion_counters* counters, int nthreads) {
  int id, family;
  if (resolve(T->layout, &id, &family)) return 1;
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads)
  for (int64_t q = 0; q < (int64_t)n; q++) {
    Query Q{*T, id, family};
    Ray ray{{rays[q].ox, rays[q].oy, rays[q].oz}, {rays[q].dx, rays[q].dy, rays[q].dz}, rays[q].tmax};
    Best best{INF, SCION_MISS_PRIM};
    if (family == SCION_FAMILY_BVH8) Q.chrt8(ray, id == L_LOGICAL8 ? (uint64_t)(uint32_t)(int32_t)T->root0 : T->root0, best, 0);
    else Q.chrt2(ray, id >= 100 ? Ref{T->root0} : root_ref(*T, (LayoutId)id), best, 0);
    hits[q] = {best.t, best.prim};
    if (status) status[q] = Q.status;
    if (counters) counters[q] = Q.c;
  }
  return 0;
}

int oracle_closest_point(const TreeBytes* T, const float* pts, uint64_t n, scion_cp* out, uint32_t* status,
                         scion_counters* counters, int nthreads) {
  int id, family;
  if (resolve(T->layout, &id, &family)) return 1;
  if (family == SCION_FAMILY_BVH8) return 2;  // corpus.cpp:83 "cpq requires a binary layout"
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads)
  for (int64_t q = 0; q < (int64_t)n; q++) {
    Query Q{*T, id, family};
    V3 p{pts[3 * q], pts[3 * q + 1], pts[3 * q + 2]};
    BestCp best{INF, {0, 0, 0}, SCION_MISS_PRIM};
    Q.cpq(p, id >= 100 ? Ref{T->root0} : root_ref(*T, (LayoutId)id), best, 0);
    out[q] = {best.d2, best.p.x, best.p.y, best.p.z, best.prim};
    if (status) status[q] = Q.status;
    if (counters) counters[q] = Q.c;
  }
  return 0;
}

// Brute force over the primitive array (ground truth for small scenes): first triangle in array
// order attaining the strict minimum — what the DFS order yields when no box test mis-prunes.
int oracle_brute_hit(const float* tris9, uint64_t ntris, const scion_ray* rays, uint64_t n, scion_hit* hits) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t q = 0; q < (int64_t)n; q++) {
    Ray ray{{rays[q].ox, rays[q].oy, rays[q].oz}, {rays[q].dx, rays[q].dy, rays[q].dz}, rays[q].tmax};
    Best best{INF, SCION_MISS_PRIM};
    for (uint64_t i = 0; i < ntris; i++) {
      Tri t;
      std::memcpy(&t, tris9 + 9 * i, 36);
      TriHit h = ray_tri_mt(ray, t);
      if (h.some && h.t < best.t) best = {h.t, (uint32_t)i};
    }
    hits[q] = {best.t, best.prim};
  }
  return 0;
}
int oracle_brute_point(const float* tris9, uint64_t ntris, const float* pts, uint64_t n, scion_cp* out) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t q = 0; q < (int64_t)n; q++) {
    V3 p{pts[3 * q], pts[3 * q + 1], pts[3 * q + 2]};
    BestCp best{INF, {0, 0, 0}, SCION_MISS_PRIM};
    for (uint64_t i = 0; i < ntris; i++) {
      Tri t;
      std::memcpy(&t, tris9 + 9 * i, 36);
      ClosestPt ps = point_triangle(p, t);
      V3 x = sub(p, ps.p);
      float d2 = dot(x, x);
      if (d2 < best.d2) best = {d2, ps.p, (uint32_t)i};
    }
    out[q] = {best.d2, best.p.x, best.p.y, best.p.z, best.prim};
  }
  return 0;
}

// ------------------------------------------------------------------ KAT entry points
int oracle_ray_aabb(const float o[3], const float d[3], float tmax, const float lo[3], const float hi[3], float out[2]) {
  Interval I = ray_aabb(Ray{{o[0], o[1], o[2]}, {d[0], d[1], d[2]}, tmax}, Box{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}});
  out[0] = I.low; out[1] = I.high;
  return I.some ? 1 : 0;
}
int oracle_ray_tri(const float o[3], const float d[3], float tmax, const float tri9[9], float out[4]) {
  Tri t;
  std::memcpy(&t, tri9, 36);
  TriHit h = ray_tri_mt(Ray{{o[0], o[1], o[2]}, {d[0], d[1], d[2]}, tmax}, t);
  out[0] = h.b0; out[1] = h.b1; out[2] = h.b2; out[3] = h.t;
  return h.some ? 1 : 0;
}
// batch form, method 0 = Moeller-Trumbore (geometry.scion:25-38), 1 = Pluecker (geometry.scion:40-55);
// rays are scion_ray records (8 floats), out = (b0, b1, b2, t, hit as 0/1 bits) per pair
void oracle_ray_tri_batch(const float* rays8, const float* tris9, uint64_t n, int method, float* out5) {
  for (uint64_t i = 0; i < n; i++) {
    const float* r = rays8 + 8 * i;
    Tri t;
    std::memcpy(&t, tris9 + 9 * i, 36);
    const Ray ray{{r[0], r[1], r[2]}, {r[4], r[5], r[6]}, r[3]};
    const TriHit h = method == 1 ? ray_tri_pc(ray, t) : ray_tri_mt(ray, t);
    float* o = out5 + 5 * i;
    o[0] = h.b0; o[1] = h.b1; o[2] = h.b2; o[3] = h.t;
    const uint32_t hit = h.some ? 1u : 0u;
    std::memcpy(o + 4, &hit, 4);
  }
}
void oracle_point_tri(const float p[3], const float tri9[9], float out_pt[3], float out_bary[3]) {
  Tri t;
  std::memcpy(&t, tri9, 36);
  ClosestPt c = point_triangle(V3{p[0], p[1], p[2]}, t);
  out_pt[0] = c.p.x; out_pt[1] = c.p.y; out_pt[2] = c.p.z;
  out_bary[0] = c.bary.x; out_bary[1] = c.bary.y; out_bary[2] = c.bary.z;
}
float oracle_sqdist_point_aabb(const float p[3], const float lo[3], const float hi[3]) {
  return sqdist_point_aabb(V3{p[0], p[1], p[2]}, Box{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}});
}
float oracle_distmax_point_aabb(const float p[3], const float lo[3], const float hi[3]) {
  return distmax_point_aabb(V3{p[0], p[1], p[2]}, Box{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}});
}
float oracle_fmul_rd(float a, float b) { return fmul_rd(a, b); }
float oracle_fadd_rd(float a, float b) { return fadd_rd(a, b); }
float oracle_fsub_rd(float a, float b) { return fsub_rd(a, b); }
float oracle_fsub_ru(float a, float b) { return fsub_ru(a, b); }
float oracle_fdiv_rd(float a, float b) { return fdiv_rd(a, b); }
float oracle_frcp_rd(float a) { return frcp_rd(a); }
uint64_t oracle_read_bits(const uint8_t* buf, uint64_t bit, uint32_t width) { return read_bits(buf, bit, width); }
uint64_t oracle_read_bits_naive(const uint8_t* buf, uint64_t bit, uint32_t width) { return read_bits_naive(buf, bit, width); }

// Quantise + dequantise one box with one scheme (restating the build-side helper funcs):
//   scheme 0: sg-eq   (sg_eq.scion:9-30: construct_bins_inverse/construct_bins/quantize_lo/quantize_hi + :5-8,:40-41)
//   scheme 1: q16     (pbrt_q16.scion:14-23,:49-52 quantize_bounds/vu_floor/vu_ceil + :6-13)
//   scheme 2: q8      (bvh8_q8.scion:23-24,:40-53 tfloor/tceil/quantize_bounds + :5-22), frame = the given world box
// out_codes: 6 integer codes (lo xyz, hi xyz); out_box: dequantised lo xyz, hi xyz.
void oracle_quantize_roundtrip(int scheme, const float wlo[3], const float whi[3], const float lo[3], const float hi[3],
                               uint32_t out_codes[6], float out_box[6]) {
  if (scheme == 0) {
    for (int a = 0; a < 3; a++) {
      float l1 = fsub_ru(whi[a], wlo[a]);
      float l2 = l1 > 0.0f ? l1 : 1.0f;
      float binv = fdiv_rd(1023.0f, l2), bins = frcp_rd(binv);
      uint32_t ql = (uint32_t)floorf(fmul_rd(fsub_rd(lo[a], wlo[a]), binv)) & 1023u;
      uint32_t qh = (uint32_t)floorf(fmul_rd(fsub_rd(whi[a], hi[a]), binv)) & 1023u;
      out_codes[a] = ql; out_codes[3 + a] = qh;
      out_box[a] = fadd_rd(wlo[a], fmul_rd((float)ql, bins));
      out_box[3 + a] = fsub_ru(whi[a], fmul_rd((float)qh, bins));
    }
  } else {
    const float top = scheme == 1 ? 65535.0f : 255.0f;
    const float step = scheme == 1 ? 1.0f / 65535.0f : 1 / 255.0f;
    for (int a = 0; a < 3; a++) {
      float mex = whi[a] - wlo[a];
      float rcp = (1.0f / mex) * top;
      float ql = fmaxf(0.0f, fminf(floorf((lo[a] - wlo[a]) * rcp), top));
      float qh = fmaxf(0.0f, fminf(ceilf((hi[a] - wlo[a]) * rcp), top));
      out_codes[a] = (uint32_t)ql; out_codes[3 + a] = (uint32_t)qh;
      out_box[a] = wlo[a] + ((float)out_codes[a] * step) * mex;
      out_box[3 + a] = wlo[a] + ((float)out_codes[3 + a] * step) * mex;
    }
  }
}

// ------------------------------------------------------------------ encoding check
// Walks the LogicalTree and the encoded tree in lockstep (decode o encode must be the identity on
// topology, leaf ranges and — for float32 layouts — bounds; quantised layouts must reproduce the
// oracle's own codes, i.e. the build blocks restated in oracle_quantize_roundtrip).
// Returns the number of mismatching nodes; writes a description of the first into msg.
uint64_t oracle_check_encoding(const TreeBytes* T, const scion_lnode* lnodes, uint64_t nnodes, const float* dop_lo2, const float* dop_hi2,
                               const scion_wnode* wnodes, const scion_wleaf* wleaves, int32_t wroot, char* msg, int msg_len, uint64_t* enclosure_violations) {
  const LayoutDesc* d = find_layout(T->layout);
  if (!d) return ~0ull;
  uint64_t bad = 0, loose = 0;
  // RNE dequantisation (q16 / q8 schemes) is not conservative to the last ulp (SURVEY App. A,
  // "L2 parity"): enclosure violations are COUNTED and reported, not treated as encoder faults.
  auto not_enclosed = [&]() { loose++; };
  auto fail = [&](const char* what, uint64_t node) {
    if (bad++ == 0 && msg) snprintf(msg, (size_t)msg_len, "%s: %s at logical node %llu", T->layout, what, (unsigned long long)node);
  };
  auto same3 = [](V3 a, const float* b) { return bits_of(a.x) == bits_of(b[0]) && bits_of(a.y) == bits_of(b[1]) && bits_of(a.z) == bits_of(b[2]); };
  if (d->family != SCION_FAMILY_BVH8) {
    const bool q16 = d->id == L_PBRT_Q16 || d->id == L_PBRT_Q16_SOAOS;
    const bool quant = q16 || d->id == L_SG_EQ || d->id == L_SG_EQ_ALIGN16;
    const float* wlo = lnodes[0].lo;
    const float* whi = lnodes[0].hi;
    struct Item { uint64_t l; Ref r; V3 elo, ehi; };
    std::vector<Item> st;
    V3 rl{wlo[0], wlo[1], wlo[2]}, rh{whi[0], whi[1], whi[2]};
    st.push_back({0, root_ref(*T, d->id), rl, rh});
    uint64_t visited = 0;
    while (!st.empty()) {
      Item it = st.back();
      st.pop_back();
      visited++;
      const scion_lnode& l = lnodes[it.l];
      Node2 n = decode2(*T, d->id, it.r);
      if (n.leaf != (l.left < 0)) { fail("variant", it.l); continue; }
      if (d->id == L_SHARED_SLAB) {
        // boxes are inherited: expected = accumulated (elo, ehi) (shared_slab.scion:24-33)
        float e[3] = {it.elo.x, it.elo.y, it.elo.z}, f[3] = {it.ehi.x, it.ehi.y, it.ehi.z};
        if (!same3(n.box.lo, e) || !same3(n.box.hi, f)) fail("inherited bounds", it.l);
      } else if (!quant) {
        if (!same3(n.box.lo, l.lo) || !same3(n.box.hi, l.hi)) fail("bounds", it.l);
      } else {
        uint32_t codes[6];
        float box[6];
        oracle_quantize_roundtrip(q16 ? 1 : 0, wlo, whi, l.lo, l.hi, codes, box);
        if (!same3(n.box.lo, box) || !same3(n.box.hi, box + 3)) fail("quantised bounds", it.l);
        // enclosure: decoded box must contain the original
        if (!(n.box.lo.x <= l.lo[0] && n.box.lo.y <= l.lo[1] && n.box.lo.z <= l.lo[2] && n.box.hi.x >= l.hi[0] && n.box.hi.y >= l.hi[1] && n.box.hi.z >= l.hi[2]))
          not_enclosed();
      }
      if (d->family == SCION_FAMILY_DOP14) {
        const float* a = dop_lo2 + it.l * 4;
        const float* b = dop_hi2 + it.l * 4;
        if (std::memcmp(&n.lo2, a, 16) || std::memcmp(&n.hi2, b, 16)) fail("diagonal slabs", it.l);
      }
      if (n.leaf) {
        if (n.nprims != l.nprims || n.prim_begin != l.first_prim) fail("leaf range", it.l);
      } else {
        Item L{(uint64_t)l.left, n.left, it.elo, it.ehi}, R{(uint64_t)l.right, n.right, it.elo, it.ehi};
        if (d->id == L_SHARED_SLAB) {
          float e[3] = {l.hi[0] - l.lo[0], l.hi[1] - l.lo[1], l.hi[2] - l.lo[2]};
          int ax = (e[0] >= e[1] && e[0] >= e[2]) ? 0 : (e[1] >= e[2] ? 1 : 2);  // longest_axis, shared_slab.scion:7-12
          V3 lo2v = it.elo, hi2v = it.ehi;
          (ax == 0 ? lo2v.x : ax == 1 ? lo2v.y : lo2v.z) = l.lo[ax];
          (ax == 0 ? hi2v.x : ax == 1 ? hi2v.y : hi2v.z) = l.hi[ax];
          L.elo = R.elo = lo2v;
          L.ehi = R.ehi = hi2v;
        }
        if (d->id == L_PBRT || d->id == L_PBRT_ALIGN16 || d->id == L_PBRT_SOA || d->id == L_PBRT_SOAOS || d->id == L_PBRT_SOAOS_ALIGN16 || q16 || d->id == L_SG_EQ ||
            d->id == L_SG_EQ_ALIGN16 || d->id == L_DOP14) {
          // index-referenced preorder builds: references ARE the preorder indices
          if (n.left.r != (uint64_t)l.left || n.right.r != (uint64_t)l.right) fail("child index", it.l);
        }
        st.push_back(R);
        st.push_back(L);
      }
    }
    if (visited != nnodes) fail("node count reached from the root", visited);
  } else {
    struct Item { int32_t c; uint64_t r; };
    std::vector<Item> st;
    st.push_back({wroot, T->root0});
    while (!st.empty()) {
      Item it = st.back();
      st.pop_back();
      Node8 n = decode8(*T, d->id, it.r);
      if (it.c < 0) {
        if (!n.leaf) { fail("variant", (uint64_t)(uint32_t)it.c); continue; }
        const scion_wleaf& l = wleaves[~it.c];
        if (n.nprims != l.nprims || n.prim_begin != l.first_prim) fail("leaf reference (App. C.2 encoding)", (uint64_t)(~it.c));
        continue;
      }
      if (n.leaf) { fail("variant", (uint64_t)it.c); continue; }
      const scion_wnode& w = wnodes[it.c];
      if (it.r != (((uint64_t)it.c << 2) | 1)) fail("interior reference", (uint64_t)it.c);
      // expected boxes
      float mlo[3], mhi[3];
      for (int a = 0; a < 3; a++) {
        mlo[a] = w.lo[7][a]; mhi[a] = w.hi[7][a];
        for (int k = 6; k >= 0; k--) { mlo[a] = fminf(w.lo[k][a], mlo[a]); mhi[a] = fmaxf(w.hi[k][a], mhi[a]); }
      }
      for (int k = 0; k < 8; k++) {
        if (d->id == L_BVH8 || d->id == L_BVH8_ALIGN16) {
          if (!same3(n.box[k].lo, w.lo[k]) || !same3(n.box[k].hi, w.hi[k])) fail("child bounds", (uint64_t)it.c);
        } else {
          uint32_t codes[6];
          float box[6];
          oracle_quantize_roundtrip((d->id == L_BVH8_Q8 || d->id == L_BVH8_Q8_CI || d->id == L_BVH8_Q8_ALIGN16 || d->id == L_BVH8_Q8_CI_ALIGN16) ? 2 : 1, mlo, mhi, w.lo[k], w.hi[k], codes, box);
          if (!same3(n.box[k].lo, box) || !same3(n.box[k].hi, box + 3)) fail("quantised child bounds", (uint64_t)it.c);
          if (w.child[k] != SCION_W_SENTINEL &&
              !(n.box[k].lo.x <= w.lo[k][0] && n.box[k].lo.y <= w.lo[k][1] && n.box[k].lo.z <= w.lo[k][2] && n.box[k].hi.x >= w.hi[k][0] && n.box[k].hi.y >= w.hi[k][1] && n.box[k].hi.z >= w.hi[k][2]))
            not_enclosed();
        }
        if (w.child[k] == SCION_W_SENTINEL) {
          if (n.children[k] != 0) fail("sentinel reference", (uint64_t)it.c);
        } else {
          st.push_back({w.child[k], n.children[k]});
        }
      }
    }
  }
  if (enclosure_violations) *enclosure_violations = loose;
  return bad;
}

}  // extern "C"

// ------------------------------------------------------------------ decode entry points (tests of the
// generated decoders): out_f = lo xyz, hi xyz, lo2 xyzw, hi2 xyzw, left.plo xyz, left.phi xyz (20 floats);
// out_u = leaf, left, right, prim_begin, nprims
extern "C" int oracle_decode2(const TreeBytes* T, uint64_t ref, const float* carried6, float* out_f, uint64_t* out_u) {
  const LayoutDesc* d = find_layout(T->layout);
  if (!d || d->family == SCION_FAMILY_BVH8) return 1;
  Ref r;
  r.r = ref;
  r.plo = {carried6[0], carried6[1], carried6[2]};
  r.phi = {carried6[3], carried6[4], carried6[5]};
  Node2 n = decode2(*T, d->id, r);
  const float f[20] = {n.box.lo.x, n.box.lo.y, n.box.lo.z, n.box.hi.x, n.box.hi.y, n.box.hi.z, n.lo2.x, n.lo2.y, n.lo2.z, n.lo2.w,
                       n.hi2.x, n.hi2.y, n.hi2.z, n.hi2.w, n.left.plo.x, n.left.plo.y, n.left.plo.z, n.left.phi.x, n.left.phi.y, n.left.phi.z};
  std::memcpy(out_f, f, sizeof(f));
  out_u[0] = n.leaf; out_u[1] = n.left.r; out_u[2] = n.right.r; out_u[3] = n.prim_begin; out_u[4] = n.nprims;
  return 0;
}
// out_f = 8 x (lo xyz, hi xyz); out_u = leaf, prim_begin, nprims, children[8]
extern "C" int oracle_decode8(const TreeBytes* T, uint64_t ref, float* out_f, uint64_t* out_u) {
  const LayoutDesc* d = find_layout(T->layout);
  if (!d || d->family != SCION_FAMILY_BVH8) return 1;
  Node8 n = decode8(*T, d->id, ref);
  out_u[0] = n.leaf; out_u[1] = n.prim_begin; out_u[2] = n.nprims;
  for (int k = 0; k < 8; k++) {
    out_u[3 + k] = n.leaf ? 0 : n.children[k];
    const float f[6] = {n.box[k].lo.x, n.box[k].lo.y, n.box[k].lo.z, n.box[k].hi.x, n.box[k].hi.y, n.box[k].hi.z};
    std::memcpy(out_f + 6 * k, f, sizeof(f));
  }
  return 0;
}


// ------------------------------------------------------------------ collision detection
// /root/reference/proj/corpus/alg/cd.scion:2-31 and cd_dop14.scion:2-31, kept recursive like the DSL
// ([recursive], depth guard 10^4 frames).  Result = set of (triangle index in tree 1,
// triangle index in tree 2); returned sorted so that set equality is a plain comparison.
namespace {
struct CdRun {
  const TreeBytes& A;
  const TreeBytes& B;
  int id, family;
  std::vector<uint64_t> pairs;
  uint64_t node_pairs = 0, tri_tests = 0;
  bool too_deep = false;
  void rec(const Ref& ra, const Ref& rb, int depth) {
    if (depth > 10000) { too_deep = true; return; }
    Node2 a = decode_any2(A, id, ra), b = decode_any2(B, id, rb);
    node_pairs++;
    const bool hit = family == SCION_FAMILY_DOP14 ? dop_overlap(a.box, a.lo2, a.hi2, b.box, b.lo2, b.hi2) : aabb_overlap(a.box, b.box);
    if (!hit) return;
    if (!a.leaf && !b.leaf) {
      rec(a.left, b.left, depth + 1); rec(a.left, b.right, depth + 1);
      rec(a.right, b.left, depth + 1); rec(a.right, b.right, depth + 1);
    } else if (!a.leaf) {
      rec(a.left, rb, depth + 1); rec(a.right, rb, depth + 1);
    } else if (!b.leaf) {
      rec(ra, b.left, depth + 1); rec(ra, b.right, depth + 1);
    } else {
      for (uint64_t i = a.prim_begin; i < a.prim_begin + a.nprims; i++)
        for (uint64_t j = b.prim_begin; j < b.prim_begin + b.nprims; j++) {
          tri_tests++;
          if (sat_triangles(load_tri(A, i), load_tri(B, j))) pairs.push_back((i << 32) | j);
        }
    }
  }
};
}  // namespace

extern "C" {
// returns the number of colliding pairs (written sorted, up to `capacity`), or -1 on error
int64_t oracle_collision_detection(const TreeBytes* A, const TreeBytes* B, uint64_t* out_pairs, uint64_t capacity, uint64_t* stats3) {
  int id, family, id2, family2;
  if (resolve(A->layout, &id, &family) || resolve(B->layout, &id2, &family2) || id != id2 || family == SCION_FAMILY_BVH8) return -1;
  CdRun run{*A, *B, id, family};
  run.rec(id >= 100 ? Ref{A->root0} : root_ref(*A, (LayoutId)id), id >= 100 ? Ref{B->root0} : root_ref(*B, (LayoutId)id), 0);
  if (run.too_deep) return -2;
  std::sort(run.pairs.begin(), run.pairs.end());
  for (size_t i = 0; i < run.pairs.size() && i < capacity; i++) out_pairs[i] = run.pairs[i];
  if (stats3) { stats3[0] = run.node_pairs; stats3[1] = run.tri_tests; stats3[2] = run.pairs.size(); }
  return (int64_t)run.pairs.size();
}
// O(n*m) SAT brute force
int64_t oracle_brute_collisions(const float* tris_a, uint64_t na, const float* tris_b, uint64_t nb, uint64_t* out_pairs, uint64_t capacity) {
  std::vector<std::vector<uint64_t>> per((size_t)omp_get_max_threads());
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < (int64_t)na; i++) {
    Tri a;
    std::memcpy(&a, tris_a + 9 * i, 36);
    auto& v = per[(size_t)omp_get_thread_num()];
    for (uint64_t j = 0; j < nb; j++) {
      Tri b;
      std::memcpy(&b, tris_b + 9 * j, 36);
      if (sat_triangles(a, b)) v.push_back(((uint64_t)i << 32) | j);
    }
  }
  std::vector<uint64_t> all;
  for (auto& v : per) all.insert(all.end(), v.begin(), v.end());
  std::sort(all.begin(), all.end());
  for (size_t i = 0; i < all.size() && i < capacity; i++) out_pairs[i] = all[i];
  return (int64_t)all.size();
}
int oracle_sat(const float* a9, const float* b9) {
  Tri a, b;
  std::memcpy(&a, a9, 36);
  std::memcpy(&b, b9, 36);
  return sat_triangles(a, b) ? 1 : 0;
}
}
