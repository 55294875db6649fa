// TEST-ONLY: compiles the GENERATED layout headers (csrc/gen/*.cuh) in the host mode of
// device/scion_rt.cuh so that emit_cuda's output can be checked against the oracle's independent
// decoders on a machine without a GPU.  Not part of the product library.
#include <cstring>
#include <string>

#include "device/geometry.cuh"
#include "gen/bvh8.cuh"
#include "gen/bvh8_align16.cuh"
#include "gen/bvh8_q16_align16.cuh"
#include "gen/bvh8_q16_ci_align16.cuh"
#include "gen/bvh8_q8_align16.cuh"
#include "gen/bvh8_q8_ci_align16.cuh"
#include "gen/bvh8_q16.cuh"
#include "gen/bvh8_q16_ci.cuh"
#include "gen/bvh8_q8.cuh"
#include "gen/bvh8_q8_ci.cuh"
#include "gen/dop14.cuh"
#include "gen/identity.cuh"
#include "gen/pbrt.cuh"
#include "gen/pbrt_align16.cuh"
#include "gen/pbrt_post.cuh"
#include "gen/pbrt_q16.cuh"
#include "gen/pbrt_q16_soaos.cuh"
#include "gen/pbrt_soa.cuh"
#include "gen/pbrt_soaos.cuh"
#include "gen/pbrt_soaos_align16.cuh"
#include "gen/ptr.cuh"
#include "gen/sg_eq.cuh"
#include "gen/sg_eq_align16.cuh"
#include "gen/shared_slab.cuh"

using scion::TreeView;
namespace g = scion_gen;

template <class R> R make_ref(uint64_t r, const float* c) {
  if constexpr (sizeof(R) <= 8) return (R)r;
  else { R x; x.P = r; x.plo = {c[0], c[1], c[2]}; x.phi = {c[3], c[4], c[5]}; return x; }
}
template <class R> uint64_t ref_id(const R& r) {
  if constexpr (sizeof(R) <= 8) return (uint64_t)r;
  else return r.P;
}
template <class L> int dec2(const TreeView* T, uint64_t ref, const float* carried, float* f, uint64_t* u) {
  typename L::Node n{};
  auto r = make_ref<typename L::Ref>(ref, carried);
  L::decode(*T, r, n);
  L::decode_cold(*T, r, n);
  if constexpr (L::kCanFetch) {  // split form: fetch() + decode_fetched() must be decode()
    typename L::Fetched w;
    typename L::Node m{};
    L::fetch(*T, r, w);
    L::decode_fetched(*T, r, w, m);
    if (m.variant != n.variant || std::memcmp(&m.low, &n.low, sizeof(n.low)) != 0 || std::memcmp(&m.high, &n.high, sizeof(n.high)) != 0) return 3;
    if (n.variant == L::kLeaf ? (m.data.begin != n.data.begin || m.data.end != n.data.end) : (ref_id(m.left) != ref_id(n.left) || ref_id(m.right) != ref_id(n.right))) return 3;
  }
  std::memset(f, 0, 20 * sizeof(float));
  if constexpr (L::kFamily == 1) {
    float v[14] = {n.lo1.x, n.lo1.y, n.lo1.z, n.hi1.x, n.hi1.y, n.hi1.z, n.lo2.x, n.lo2.y, n.lo2.z, n.lo2.w, n.hi2.x, n.hi2.y, n.hi2.z, n.hi2.w};
    std::memcpy(f, v, sizeof(v));
  } else {
    float v[6] = {n.low.x, n.low.y, n.low.z, n.high.x, n.high.y, n.high.z};
    std::memcpy(f, v, sizeof(v));
  }
  u[0] = n.variant == L::kLeaf;
  u[1] = u[2] = u[3] = u[4] = 0;
  if (n.variant == L::kLeaf) { u[3] = n.data.begin; u[4] = n.nprims; if (n.data.end - n.data.begin != n.nprims) return 2; }
  else {
    u[1] = ref_id(n.left); u[2] = ref_id(n.right);
    if constexpr (sizeof(typename L::Ref) > 8) { float v[6] = {n.left.plo.x, n.left.plo.y, n.left.plo.z, n.left.phi.x, n.left.phi.y, n.left.phi.z}; std::memcpy(f + 14, v, sizeof(v)); }
  }
  return 0;
}
template <class L> int dec8(const TreeView* T, uint64_t ref, float* f, uint64_t* u) {
  typename L::Node n{};
  L::decode(*T, (typename L::Ref)ref, n);
  std::memset(f, 0, 48 * sizeof(float));
  std::memset(u, 0, 11 * sizeof(uint64_t));
  u[0] = n.variant == L::kLeaf;
  if (n.variant == L::kLeaf) { u[1] = n.data.begin; u[2] = n.nprims; return 0; }
  for (int k = 0; k < 8; k++) {
    u[3 + k] = (uint64_t)n.children[k];
    float v[6] = {n.lo[k].x, n.lo[k].y, n.lo[k].z, n.hi[k].x, n.hi[k].y, n.hi[k].z};
    std::memcpy(f + 6 * k, v, sizeof(v));
  }
  return 0;
}

// the per-child record view of the lane-cooperative kernel (scion::LaneRecord): decode_slot<0>() over the view of slot k
// must give child k of decode(), for every k
template <class L> int dec8_lane(const TreeView* T, uint64_t ref, float* f, uint64_t* u) {
  std::memset(f, 0, 48 * sizeof(float));
  std::memset(u, 0, 11 * sizeof(uint64_t));
  const typename L::Ref r = (typename L::Ref)ref;
  u[0] = L::ref_variant(r) == L::kLeaf;
  if (u[0]) {
    typename L::Node n{};
    L::decode(*T, r, n);
    u[1] = n.data.begin; u[2] = n.nprims;
    return 0;
  }
  // a padded private copy: the host compiler may keep the (dead) reads of the other slots, which reach past the record
  unsigned char copy[3 * 256] = {0};
  static_assert(L::kSlotRecordBytes <= 256, "interior record");
  std::memcpy(copy, L::slot_record(*T, r), L::kSlotUsedBytes);
  for (uint32_t k = 0; k < 8; k++) {
    scion::f32x3 lo, hi;
    typename L::Ref ch;
    const scion::LaneRecord<L> rec{copy, k};
    L::template decode_slot<0>(*T, r, rec, lo, hi, ch);
    u[3 + k] = (uint64_t)ch;
    float v[6] = {lo.x, lo.y, lo.z, hi.x, hi.y, hi.z};
    std::memcpy(f + 6 * k, v, sizeof(v));
  }
  return 0;
}
extern "C" int host_decode8_lane(const char* layout, const TreeView* T, uint64_t ref, float* f, uint64_t* u) {
  std::string n = layout;
#define L8(NAME, T_) if (n == NAME) return dec8_lane<g::T_>(T, ref, f, u);
  L8("bvh8", L_bvh8) L8("bvh8-q8", L_bvh8_q8) L8("bvh8-q8-ci", L_bvh8_q8_ci) L8("bvh8-q16", L_bvh8_q16) L8("bvh8-q16-ci", L_bvh8_q16_ci)
  L8("bvh8-align16", L_bvh8_align16) L8("bvh8-q8-align16", L_bvh8_q8_align16) L8("bvh8-q8-ci-align16", L_bvh8_q8_ci_align16) L8("bvh8-q16-align16", L_bvh8_q16_align16)
  L8("bvh8-q16-ci-align16", L_bvh8_q16_ci_align16)
#undef L8
  return -1;
}

extern "C" int host_decode2(const char* layout, const TreeView* T, uint64_t ref, const float* carried, float* f, uint64_t* u) {
  std::string n = layout;
#define L2(NAME, T_) if (n == NAME) return dec2<g::T_>(T, ref, carried, f, u);
  L2("pbrt", L_pbrt) L2("pbrt-align16", L_pbrt_align16) L2("pbrt-soa", L_pbrt_soa) L2("pbrt-post", L_pbrt_post) L2("pbrt-q16", L_pbrt_q16)
  L2("sg-eq", L_sg_eq) L2("sg-eq-align16", L_sg_eq_align16) L2("ptr", L_ptr) L2("identity", L_identity) L2("shared-slab", L_shared_slab) L2("dop14", L_dop14)
  L2("pbrt-soaos", L_pbrt_soaos) L2("pbrt-soaos-align16", L_pbrt_soaos_align16) L2("pbrt-q16-soaos", L_pbrt_q16_soaos)
#undef L2
  return -1;
}
extern "C" int host_decode8(const char* layout, const TreeView* T, uint64_t ref, float* f, uint64_t* u) {
  std::string n = layout;
#define L8(NAME, T_) if (n == NAME) return dec8<g::T_>(T, ref, f, u);
  L8("bvh8", L_bvh8) L8("bvh8-q8", L_bvh8_q8) L8("bvh8-q8-ci", L_bvh8_q8_ci) L8("bvh8-q16", L_bvh8_q16) L8("bvh8-q16-ci", L_bvh8_q16_ci)
  L8("bvh8-align16", L_bvh8_align16) L8("bvh8-q8-align16", L_bvh8_q8_align16) L8("bvh8-q8-ci-align16", L_bvh8_q8_ci_align16) L8("bvh8-q16-align16", L_bvh8_q16_align16)
  L8("bvh8-q16-ci-align16", L_bvh8_q16_ci_align16)
#undef L8
  return -1;
}
// ---- emitted-code differential (SPEC acceptance 8): closest_hit on the HOST through the generated
// decoders and the product's geometry header — a plain recursive restatement of chrt.scion / chrt8.scion /
// chrt_dop14.scion, nothing shared with the kernels' state machines.  TEST-ONLY.
struct Hit { float t; uint32_t prim; };
template <class L> void leaf_tris(const TreeView& T, const scion::RayCtx& ray, uint64_t b, uint64_t e, Hit& best) {
  for (uint64_t i = b; i < e; i++) {
    float tri[9];
    std::memcpy(tri, T.buf[L::kBuf_primitives] + i * 36ull, 36);
    float t;
    if (scion::ray_tri_mt(ray, tri, t) && t < best.t) best = Hit{t, (uint32_t)i};
  }
}
template <class L> void visit2(const TreeView& T, const scion::RayCtx& ray, const typename L::Ref& ref, Hit& best) {
  typename L::Node n{};
  L::decode(T, ref, n);
  float tn, tf;
  bool hit;
  if constexpr (L::kFamily == 1) {
    bool some = scion::ray_aabb(ray, n.lo1, n.hi1, tn, tf);
    if (some) { L::decode_cold(T, ref, n); some = scion::dop_diagonals(ray, n.lo2, n.hi2, tn, tf); }
    hit = scion::interval_intersects(ray, some, tn, tf);
  } else {
    if constexpr (L::kBoundsCold) L::decode_cold(T, ref, n);  // part of the box lies behind `---`
    const bool some = scion::ray_aabb(ray, n.low, n.high, tn, tf);
    hit = scion::interval_intersects(ray, some, tn, tf);
    if (hit && !L::kBoundsCold) L::decode_cold(T, ref, n);
  }
  if (!hit) return;
  if (n.variant == L::kLeaf) { leaf_tris<L>(T, ray, n.data.begin, n.data.end, best); return; }
  if (!(tn < best.t)) return;
  visit2<L>(T, ray, n.left, best);
  visit2<L>(T, ray, n.right, best);
}
template <class L> void visit8(const TreeView& T, const scion::RayCtx& ray, const typename L::Ref& ref, Hit& best) {
  typename L::Node n{};
  L::decode(T, ref, n);
  if (n.variant == L::kLeaf) { leaf_tris<L>(T, ray, n.data.begin, n.data.end, best); return; }
  for (int k = 0; k < 8; k++) {
    float tn, tf;
    const bool some = scion::ray_aabb(ray, n.lo[k], n.hi[k], tn, tf);
    if (scion::interval_intersects(ray, some, tn, tf) && tn < best.t) visit8<L>(T, ray, n.children[k], best);
  }
}
template <class L, bool WIDE> int run_chrt(const TreeView* T, const float* rays8, uint64_t nrays, Hit* out) {
  for (uint64_t q = 0; q < nrays; q++) {
    const float* r = rays8 + 8 * q;
    const scion::RayCtx ray = scion::make_ray(r[0], r[1], r[2], r[3], r[4], r[5], r[6]);
    Hit best{scion::inf(), 0xFFFFFFFFu};
    if constexpr (WIDE) visit8<L>(*T, ray, L::root(*T), best);
    else visit2<L>(*T, ray, L::root(*T), best);
    out[q] = best;
  }
  return 0;
}
extern "C" int host_closest_hit(const char* layout, const TreeView* T, const float* rays8, uint64_t nrays, void* hits) {
  std::string n = layout;
  Hit* out = (Hit*)hits;
#define L2(NAME, T_) if (n == NAME) return run_chrt<g::T_, false>(T, rays8, nrays, out);
  L2("pbrt", L_pbrt) L2("pbrt-align16", L_pbrt_align16) L2("pbrt-soa", L_pbrt_soa) L2("pbrt-post", L_pbrt_post) L2("pbrt-q16", L_pbrt_q16)
  L2("sg-eq", L_sg_eq) L2("sg-eq-align16", L_sg_eq_align16) L2("ptr", L_ptr) L2("identity", L_identity) L2("shared-slab", L_shared_slab) L2("dop14", L_dop14)
  L2("pbrt-soaos", L_pbrt_soaos) L2("pbrt-soaos-align16", L_pbrt_soaos_align16) L2("pbrt-q16-soaos", L_pbrt_q16_soaos)
#undef L2
#define L8(NAME, T_) if (n == NAME) return run_chrt<g::T_, true>(T, rays8, nrays, out);
  L8("bvh8", L_bvh8) L8("bvh8-q8", L_bvh8_q8) L8("bvh8-q8-ci", L_bvh8_q8_ci) L8("bvh8-q16", L_bvh8_q16) L8("bvh8-q16-ci", L_bvh8_q16_ci)
  L8("bvh8-align16", L_bvh8_align16) L8("bvh8-q8-align16", L_bvh8_q8_align16) L8("bvh8-q8-ci-align16", L_bvh8_q8_ci_align16) L8("bvh8-q16-align16", L_bvh8_q16_align16)
  L8("bvh8-q16-ci-align16", L_bvh8_q16_ci_align16)
#undef L8
  return -1;
}
extern "C" unsigned host_treeview_size() { return (unsigned)sizeof(TreeView); }
