// Build context of the GENERATED constructors (gen/<layout>.cuh build_<Variant>(): the layout's `build` block compiled
// by emit_cuda — SPEC.md:276-284 specialize_constructors, :387-395 build_physical).
//
// The emitted code is a template over this class and uses exactly:
//   Node               the logical fields of one LogicalTree node, by the names the ADTs of the corpus use
//                      (low high | lo1 hi1 lo2 hi2 | lo hi children | left right | nprims data)
//   reserve(b, bytes)  this node's slot in buffer b: next element index (next arena byte offset for ptr-referenced groups)
//   commit(b, s, this, image, bytes)   the staged record image of segment s -> the buffer
//   append(data, n)    copy the leaf's primitives behind the cursor of the global primitive array, return the start
//   child<L>(c)        build the subtree c with L::build_node, return its reference (0 for an empty 8-wide slot)
//   is_root, set_global, glob<T>, set_root_component
// Buffers are sized by a count pass over the LogicalTree (variant_home of the plan: which buffer a variant
// materialises in) and allocated exactly once; a reserve / append beyond the counted size is a hard fault
// ("count pass disagreement ... indicates a compiler bug").
// Host only, sequential (recursive emit pass in the order of the build block); the hand-written per-family encoders of
// encode_node.hpp are the fast path (OpenMP / device) and are checked byte for byte against this one.
#pragma once
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../device/scion_rt.cuh"
#include "physical.hpp"

namespace scion {

struct BuildNode {
  int variant = 0;            // index in the ADT's variant list: 0 = Interior, 1 = Leaf for every ADT of the corpus
  int64_t id = 0;             // binary: node index; 8-wide: child code (>= 0 interior index, < 0 leaf id = ~code)
  f32x3 low{}, high{};        // BVH2: node box
  f32x3 lo1{}, hi1{};         // DOP-14: axis slabs (= the box)
  f32x4 lo2{}, hi2{};         // DOP-14: diagonal slabs
  vec<f32x3, 8> lo{}, hi{};   // 8-wide interior: child boxes (empty slots: inverted)
  int64_t left = -1, right = -1;
  int64_t children[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint32_t nprims = 0;
  uint64_t data = 0;          // first primitive of the leaf in the LogicalTree's tree-ordered array
};

struct BuildCtx {
  using Node = BuildNode;
  static constexpr int64_t kNoChild = INT64_MIN;

  const scion_ltree& lt;
  const lc::Plan& plan;
  scion_ptree& pt;
  bool wide;
  std::vector<uint64_t> cursor;   // per buffer: next free element (arena: byte)
  int prim_buffer = -1;
  int64_t root_id = 0;

  BuildCtx(const scion_ltree& t, const lc::Plan& p, scion_ptree& out) : lt(t), plan(p), pt(out), wide(p.family == lc::Family::Bvh8) {
    cursor.assign(plan.buffers.size(), 0);
    for (auto& b : plan.buffers)
      if (b.is_global_array) prim_buffer = b.id;
  }

  static void fault(const std::string& what) { throw std::runtime_error("build fault: " + what); }

  Node view(int64_t id) const {
    Node n;
    n.id = id;
    if (!wide) {
      const scion_lnode& s = lt.nodes[(size_t)id];
      n.variant = s.left < 0 ? 1 : 0;
      n.low = n.lo1 = f32x3{s.lo[0], s.lo[1], s.lo[2]};
      n.high = n.hi1 = f32x3{s.hi[0], s.hi[1], s.hi[2]};
      if (!lt.dop_lo2.empty()) {
        const float* a = &lt.dop_lo2[4 * (size_t)id];
        const float* b = &lt.dop_hi2[4 * (size_t)id];
        n.lo2 = f32x4{a[0], a[1], a[2], a[3]};
        n.hi2 = f32x4{b[0], b[1], b[2], b[3]};
      }
      n.left = s.left;
      n.right = s.right;
      n.nprims = s.nprims;
      n.data = s.first_prim;
    } else if (id >= 0) {
      const scion_wnode& s = lt.wnodes[(size_t)id];
      n.variant = 0;
      for (int k = 0; k < 8; k++) {
        n.lo[k] = f32x3{s.lo[k][0], s.lo[k][1], s.lo[k][2]};
        n.hi[k] = f32x3{s.hi[k][0], s.hi[k][1], s.hi[k][2]};
        n.children[k] = s.child[k] == SCION_W_SENTINEL ? kNoChild : (int64_t)s.child[k];
      }
    } else {
      const scion_wleaf& l = lt.wleaves[(size_t)(~id)];
      n.variant = 1;
      n.nprims = l.nprims;
      n.data = l.first_prim;
    }
    return n;
  }
  bool is_root(const Node& n) const { return n.id == root_id; }

  uint64_t reserve(int b, uint64_t bytes) {
    const lc::Buffer& B = plan.buffers[(size_t)b];
    const uint64_t at = cursor[(size_t)b];
    if (B.is_arena) {
      cursor[(size_t)b] += bytes;
      if (at + B.segments[0].stride_bytes > pt.sizes[(size_t)b]) fault("arena '" + B.name + "' overflows its counted size");
    } else {
      cursor[(size_t)b] += 1;
      if (at >= pt.counts[(size_t)b]) fault("buffer '" + B.name + "' overflows its counted size");
    }
    return at;
  }
  void commit(int b, int seg, uint64_t self, const uint32_t* image, uint64_t bytes) {
    const lc::Buffer& B = plan.buffers[(size_t)b];
    uint8_t* base = pt.buffers[(size_t)b].data();
    const uint64_t off = B.is_arena ? self : pt.seg_bases[(size_t)b][(size_t)seg] + self * B.segments[(size_t)seg].stride_bytes;
    if (off + bytes > pt.buffers[(size_t)b].size()) fault("record outside buffer '" + B.name + "'");
    std::memcpy(base + off, image, bytes);
  }
  uint64_t append(uint64_t first, uint64_t n) {
    if (prim_buffer < 0) fault("append without a global primitive array");
    const uint64_t at = cursor[(size_t)prim_buffer];
    if (at + n > pt.counts[(size_t)prim_buffer]) fault("primitive array overflows its counted size");
    std::memcpy(pt.buffers[(size_t)prim_buffer].data() + at * 36, lt.tris.data() + first * 9, n * 36);
    cursor[(size_t)prim_buffer] += n;
    return at;
  }
  template <class L>
  uint64_t child(int64_t c) {
    if (c == kNoChild) return 0;  // empty 8-wide slot: reference 0
    return L::build_node(*this, view(c));
  }

  template <class T>
  void set_global(int g, const T& v) {
    static_assert(sizeof(T) <= 16, "global cells are 16 bytes");
    pt.globals[(size_t)g].fill(0);
    std::memcpy(pt.globals[(size_t)g].data(), &v, sizeof(T));
  }
  template <class T>
  T glob(int g) const {
    T v;
    std::memcpy(&v, pt.globals[(size_t)g].data(), sizeof(T));
    return v;
  }
  void set_root_component(int r, const f32x3& v) {  // tree-carried components of the root reference, in declaration order
    int k = 0;
    for (int i = 1; i < r; i++) k += (int)(plan.type_bits(plan.ref[(size_t)i].type) / 32);
    if (k + 3 > 6) fault("more than 6 tree-carried floats in the root reference");
    pt.carried[k] = v.x; pt.carried[k + 1] = v.y; pt.carried[k + 2] = v.z;
  }
  void set_root_component(int r, float v) {
    int k = 0;
    for (int i = 1; i < r; i++) k += (int)(plan.type_bits(plan.ref[(size_t)i].type) / 32);
    if (k + 1 > 6) fault("more than 6 tree-carried floats in the root reference");
    pt.carried[k] = v;
  }
};

// one generated builder per layout compiled into the library (build/build_<layout>.cpp, stamped from
// host/build_inst.cpp.in and compiled by the HOST compiler with -frounding-math: the directed-rounding
// intrinsics of scion_rt.cuh are exact only in its plain-host mode)
typedef uint64_t (*build_root_fn)(BuildCtx&);
struct BuilderEntry {
  const char* layout;
  build_root_fn build_root;  // null: the layout file carries no build block
};
const BuilderEntry* find_builder(const char* layout);

// build_physical through the layout's own build block (count pass + generated emit pass); throws on build faults
void encode_tree_generated(const scion_ltree& t, const LayoutEntry& layout, scion_ptree& out);
// the same with an explicit constructor set (tests: constructors emitted from ANOTHER file of the same layout — the
// reference's own corpus file — run against this library's plan)
void encode_tree_with(const scion_ltree& t, const LayoutEntry& layout, build_root_fn build_root, scion_ptree& out);

}  // namespace scion
