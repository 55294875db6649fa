// Node encoding: LogicalTree -> PhysicalTree byte buffers (build_physical).
//
// The reference's constructor specialiser (src/specialize_build.cpp) and src/build_physical.cpp
// are missing/placeholder, so each encoder below restates the `build` block of the corresponding
// corpus layout (cited per function) by hand.  Field *placement* is never hard-coded: every write
// goes through the slot table produced by our planner from the .scion layout text, so the byte
// image is the planner's (and therefore the reference planner's) by construction.
// Bit packing is little-endian, LSB first: the inverse of read_bits_raw,
// /root/reference/proj/src/bits.cpp:7-19.
//
// Compiled with -ffp-contract=off -frounding-math (directed-rounding quantisers).
#include <cfenv>
#include <cmath>
#include <cstring>
#include <functional>
#include <limits>
#include <stdexcept>

#include "build_ctx.hpp"
#include "encode_node.hpp"
#include "physical.hpp"

namespace scion {

// embedded layout sources: generated at build time from paper_2511_15028_b200/layouts/*.scion
struct EmbeddedLayout {
  const char* name;
  const char* source;
};
extern const EmbeddedLayout kEmbeddedLayouts[];
extern const int kEmbeddedLayoutCount;

const std::vector<LayoutEntry>& layout_registry() {
  static const std::vector<LayoutEntry> reg = [] {
    std::vector<LayoutEntry> v;
    for (int i = 0; i < kEmbeddedLayoutCount; i++) {
      LayoutEntry e;
      e.name = kEmbeddedLayouts[i].name;
      e.source = kEmbeddedLayouts[i].source;
      e.program = std::make_unique<lc::Program>(lc::parse_program({e.source}));
      e.plan = std::make_unique<lc::Plan>(lc::plan_layout(*e.program, e.name));
      e.has_cpq = e.plan->family != lc::Family::Bvh8;  // corpus.cpp:83 "cpq requires a binary layout"
      v.push_back(std::move(e));
    }
    return v;
  }();
  return reg;
}
const LayoutEntry* dyn_find_layout(const std::string& name);  // host/plugin.cpp: layouts registered at run time
const LayoutEntry* find_layout(const std::string& name) {
  for (auto& e : layout_registry())
    if (e.name == name) return &e;
  return dyn_find_layout(name);
}
static bool is_builtin(const LayoutEntry& layout) {
  for (auto& e : layout_registry())
    if (&e == &layout) return true;
  return false;
}

namespace {

using enc::EncodeJob;
using enc::Field;

struct Writer {
  scion_ptree& pt;
  const lc::Plan& plan;
  bool shell;  // sizes, globals and root only: the buffers are filled elsewhere (device-side encode)
  Writer(scion_ptree& p, const lc::Plan& pl, bool sh) : pt(p), plan(pl), shell(sh) {}
  void alloc(const std::string& buffer, uint64_t count, uint64_t arena_bytes = 0) {
    const lc::Buffer* b = plan.buffer_named(buffer);
    if (!b) throw std::runtime_error("encode: no buffer '" + buffer + "' in layout " + plan.layout_name);
    std::vector<uint64_t> bases;
    uint64_t bytes = b->is_arena ? arena_bytes : b->bytes(count, &bases);
    if (b->is_arena) bases = {0};
    if (!shell) pt.buffers[(size_t)b->id].assign(bytes, 0);
    pt.sizes[(size_t)b->id] = bytes;
    pt.counts[(size_t)b->id] = count;
    pt.seg_bases[(size_t)b->id] = bases;
  }
  Field field(const std::string& name) const {
    const lc::Slot& s = plan.slot(name);
    const lc::Buffer& b = plan.buffers[(size_t)s.buffer];
    Field f;
    f.base = shell ? nullptr : pt.buffers[(size_t)s.buffer].data();
    f.buffer = s.buffer;
    f.arena = b.is_arena;
    f.off = s.offset;
    f.width = s.width;
    if (!b.is_arena) {
      f.seg_base_bits = pt.seg_bases[(size_t)s.buffer][(size_t)s.segment] * 8;
      f.stride_bits = b.segments[(size_t)s.segment].stride_bytes * 8;
    }
    return f;
  }
  int global_index(const std::string& name) const {
    for (size_t i = 0; i < plan.globals.size(); i++)
      if (plan.globals[i].name == name) return (int)i;
    throw std::runtime_error("encode: no global '" + name + "' in layout " + plan.layout_name);
  }
  void global_u(const std::string& name, uint64_t v) { std::memcpy(pt.globals[(size_t)global_index(name)].data(), &v, 8); }
  void global_f3(const std::string& name, const float* f) { std::memcpy(pt.globals[(size_t)global_index(name)].data(), f, 12); }
  void copy_primitives(const scion_ltree& t, const std::string& buffer, const std::string& count_global) {
    alloc(buffer, t.tris.size() / 9);
    if (!shell) std::memcpy(pt.buffers[(size_t)plan.buffer_named(buffer)->id].data(), t.tris.data(), t.tris.size() * 4);
    global_u(count_global, t.tris.size() / 9);
  }
};

void require(bool ok, const std::string& what) {
  if (!ok) throw std::runtime_error("build fault: " + what);
}
void check_leaf_capacity(const scion_ltree& t, const lc::Plan& plan) {
  for (auto& n : t.nodes)
    if (n.left < 0) require(n.nprims >= 1 && n.nprims <= plan.max_leaf, "leaf with " + std::to_string(n.nprims) + " primitives exceeds the nprims capacity of layout " + plan.layout_name);
}
void check_preorder(const scion_ltree& t) {
  for (size_t i = 0; i < t.nodes.size(); i++)
    if (t.nodes[i].left >= 0) require((uint64_t)t.nodes[i].left == i + 1, "preorder build must place the left child at this+1");
}

// arena (ptr-referenced) layouts: node address = byte offset inside the arena (plan.cpp:315-318),
// preorder allocation, each node rounded up to the group alignment
uint64_t arena_stride(const lc::Buffer& b) { return (b.segments[0].stride_bytes + b.align - 1) / b.align * b.align; }
uint64_t arena_bytes(const scion_ltree& t, const lc::Buffer& b) {
  const uint64_t n = t.nodes.size();
  return (n ? (n - 1) * arena_stride(b) + b.segments[0].stride_bytes : 0) + 8;  // put_bits/readers may touch one trailing word
}

// postorder numbering of the preorder array (pbrt-post)
std::vector<uint32_t> postorder(const scion_ltree& t) {
  const uint64_t N = t.nodes.size();
  std::vector<uint32_t> post(N);
  std::vector<std::pair<uint32_t, int>> st;
  st.push_back({0, 0});
  uint32_t next = 0;
  while (!st.empty()) {
    auto& [node, state] = st.back();
    const scion_lnode& n = t.nodes[node];
    if (n.left < 0 || state == 2) {
      post[node] = next++;
      st.pop_back();
    } else if (state == 0) {
      state = 1;
      st.push_back({(uint32_t)n.left, 0});
    } else {
      state = 2;
      st.push_back({(uint32_t)n.right, 0});
    }
  }
  return post;
}

// Everything of a build except the per-node loop: buffer sizes, globals (root blocks of the
// layouts: pbrt_q16.scion:49-56, sg_eq.scion:9-30, shared_slab.scion:40-46), root reference,
// capacity checks, and the slot table + constants of the per-node encoder (enc::EncodeJob).
void prepare(const scion_ltree& t, const std::string& name, Writer& w, EncodeJob& j, std::vector<uint32_t>& post) {
  const uint64_t N = t.nodes.size();
  j = EncodeJob();
  j.count = N;
  j.nodes = t.nodes.data();
  if (name == "pbrt" || name == "pbrt-align16" || name == "pbrt-soa" || name == "pbrt-soaos" || name == "pbrt-soaos-align16") {
    check_preorder(t);
    w.copy_primitives(t, "primitives", "P");
    w.alloc("nodes", N);
    w.global_u("N", N);
    j.kind = enc::kPbrt;
    j.f[0] = w.field("low"); j.f[1] = w.field("high"); j.f[2] = w.field("nprims"); j.f[3] = w.field("c_o"); j.f[4] = w.field("p_o");
    w.pt.root0 = 0;
  } else if (name == "pbrt-post") {
    w.copy_primitives(t, "primitives", "P");
    w.alloc("nodes", N);
    w.global_u("N", N);
    post = postorder(t);
    j.kind = enc::kPbrtPost;
    j.post = post.data();
    j.f[0] = w.field("low"); j.f[1] = w.field("high"); j.f[2] = w.field("nprims"); j.f[3] = w.field("c_l"); j.f[4] = w.field("c_r"); j.f[5] = w.field("p_o");
    w.pt.root0 = post[0];
  } else if (name == "pbrt-q16" || name == "pbrt-q16-soaos") {
    require(N < (1ull << 28), name + ": node count exceeds the u28 child offset");
    require(t.tris.size() / 9 < (1ull << 28), name + ": primitive count exceeds the u28 primitive offset");
    check_preorder(t);
    w.copy_primitives(t, "primitives", "primitive_count");
    w.alloc("nodes", N);
    w.global_u("node_count", N);
    float we[3];
    for (int a = 0; a < 3; a++) {  // root block: world_low = low, world_extent = high - low; rcp = (1.0 / mex) * 65535.0
      j.c0[a] = t.nodes[0].lo[a];
      we[a] = t.nodes[0].hi[a] - t.nodes[0].lo[a];
      j.c1[a] = (1.0f / we[a]) * 65535.0f;
    }
    w.global_f3("world_low", j.c0);
    w.global_f3("world_extent", we);
    j.kind = enc::kQ16;
    j.f[0] = w.field("bounds_q"); j.f[1] = w.field("nprims"); j.f[2] = w.field("c_offset"); j.f[3] = w.field("p_offset");
    w.pt.root0 = 0;
  } else if (name == "sg-eq" || name == "sg-eq-align16") {
    check_preorder(t);
    w.copy_primitives(t, "primitives", "primitive_count");
    w.alloc("nodes", N);
    w.global_u("node_count", N);
    float bins[3];
    for (int a = 0; a < 3; a++) {  // root block: bins_inv = fdiv_rd(1023, guarded fsub_ru(high, low)), bins = frcp_rd(bins_inv)
      j.c0[a] = t.nodes[0].lo[a];
      j.c1[a] = t.nodes[0].hi[a];
      float l1 = enc::fsub_ru(j.c1[a], j.c0[a]);
      float l2 = l1 > 0.0f ? l1 : 1.0f;
      j.c2[a] = enc::fdiv_rd(1023.0f, l2);
      bins[a] = enc::frcp_rd(j.c2[a]);
    }
    w.global_f3("wlow", j.c0);
    w.global_f3("whigh", j.c1);
    w.global_f3("bins", bins);
    w.global_f3("bins_inv", j.c2);
    j.kind = enc::kSgEq;
    j.f[0] = w.field("q_min"); j.f[1] = w.field("q_max"); j.f[2] = w.field("nprims"); j.f[3] = w.field("offset"); j.f[4] = w.field("poffset");
    w.pt.root0 = 0;
  } else if (name == "dop14") {
    require(N < (1ull << 31), "dop14: node count exceeds i32 references");
    require(t.tris.size() / 9 < (1ull << 27), "dop14: primitive count exceeds the 27-bit offset");
    w.copy_primitives(t, "primitives", "P");
    w.alloc("nodes", N);
    w.global_u("N", N);
    j.kind = enc::kDop14;
    j.dop_lo2 = t.dop_lo2.data();
    j.dop_hi2 = t.dop_hi2.data();
    j.f[0] = w.field("lo1"); j.f[1] = w.field("hi1"); j.f[2] = w.field("c0"); j.f[3] = w.field("c1"); j.f[4] = w.field("lo2"); j.f[5] = w.field("hi2");
    w.pt.root0 = 0;
  } else if (name == "ptr" || name == "identity" || name == "shared-slab") {
    const lc::Buffer& b = *w.plan.buffer_named("node");
    w.copy_primitives(t, "primitives", name == "shared-slab" ? "N" : "NP");
    w.alloc("node", N, arena_bytes(t, b));
    j.arena_stride = arena_stride(b);
    if (name == "ptr") {  // ptr.scion:17-31
      j.kind = enc::kPtr;
      j.f[0] = w.field("low"); j.f[1] = w.field("high"); j.f[2] = w.field("nprims"); j.f[3] = w.field("L"); j.f[4] = w.field("R"); j.f[5] = w.field("p_o");
    } else if (name == "identity") {  // identity.scion:19-33
      j.kind = enc::kIdentity;
      j.f[0] = w.field("low"); j.f[1] = w.field("high"); j.f[2] = w.field("tag"); j.f[3] = w.field("left"); j.f[4] = w.field("right"); j.f[5] = w.field("nprims"); j.f[6] = w.field("p_o");
    } else {  // shared_slab.scion:40-67 — root block: plo = low, phi = high (carried in the root reference)
      j.kind = enc::kSharedSlab;
      j.f[0] = w.field("L"); j.f[1] = w.field("R"); j.f[2] = w.field("slo"); j.f[3] = w.field("shi"); j.f[4] = w.field("o"); j.f[5] = w.field("axis"); j.f[6] = w.field("is_leaf"); j.f[7] = w.field("nprims");
      std::memcpy(w.pt.carried, t.nodes[0].lo, 12);
      std::memcpy(w.pt.carried + 3, t.nodes[0].hi, 12);
      std::memcpy(w.pt.globals[(size_t)w.global_index("__ref_plo")].data(), t.nodes[0].lo, 12);
      std::memcpy(w.pt.globals[(size_t)w.global_index("__ref_phi")].data(), t.nodes[0].hi, 12);
    }
    w.pt.root0 = 0;  // address of node 0
  } else if (name.rfind("bvh8", 0) == 0) {
    const int qbits = name.find("-q8") != std::string::npos ? 8 : (name.find("-q16") != std::string::npos ? 16 : 0);  // bvh8, bvh8-align16: f32 boxes
    const int ref_bits = name.find("-ci") != std::string::npos ? 32 : 64;  // bvh8-q8-ci, bvh8-q8-ci-align16, ...
    require(t.has_wide, "8-wide layouts need a collapsed tree (scion_ltree_collapse8)");
    const uint64_t NI = t.wnodes.size();
    const uint64_t P = t.tris.size() / 9;
    require(ref_bits == 64 || NI < (1ull << 30), "8-wide: interior count exceeds the 30-bit index");
    require(ref_bits == 64 || P < (1ull << 25), "8-wide: primitive count exceeds the 25-bit offset of compressed references");
    for (auto& l : t.wleaves) require(l.nprims >= 1 && l.nprims <= 32, "8-wide leaf capacity is 32 primitives");
    w.copy_primitives(t, "primitives", "primitive_count");
    w.alloc("Interiors", NI);
    w.global_u("interior_count", NI);
    j.kind = enc::kBvh8;
    j.count = NI;
    j.qbits = qbits;
    j.ref_bits = ref_bits;
    j.wnodes = t.wnodes.data();
    j.wleaves = t.wleaves.data();
    j.f[0] = w.field("children");
    if (qbits == 0) { j.f[1] = w.field("lo"); j.f[2] = w.field("hi"); }
    else { j.f[1] = w.field("mlo"); j.f[2] = w.field("mex"); j.f[3] = w.field("child_bounds"); }
    w.pt.root0 = enc::wide_ref(j, t.wroot);
  } else {
    throw std::runtime_error("no encoder registered for layout '" + name + "'");
  }
}

void init_ptree(const scion_ltree& t, const LayoutEntry& layout, scion_ptree& out) {
  const lc::Plan& plan = *layout.plan;
  out = scion_ptree();
  out.layout = layout.name;
  out.plan = &plan;
  out.buffers.resize(plan.buffers.size());
  out.sizes.assign(plan.buffers.size(), 0);
  out.counts.assign(plan.buffers.size(), 0);
  out.seg_bases.resize(plan.buffers.size());
  out.globals.resize(plan.globals.size());
  for (auto& g : out.globals) g.fill(0);
  out.nprims = t.tris.size() / 9;
  if (plan.family != lc::Family::Bvh8) check_leaf_capacity(t, plan);
}

}  // namespace

void encode_tree(const scion_ltree& t, const LayoutEntry& layout, scion_ptree& out) {
  if (!is_builtin(layout)) {  // a layout registered at run time: its own build block is its only encoder
    encode_tree_generated(t, layout, out);
    return;
  }
  init_ptree(t, layout, out);
  Writer w(out, *layout.plan, false);
  EncodeJob job;
  std::vector<uint32_t> post;
  prepare(t, layout.name, w, job, post);
  const int64_t n = (int64_t)job.count;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; i++) enc::encode_one(job, (uint64_t)i);
}

// build_physical through the layout's own `build` block, compiled by emit_cuda into gen/<layout>.cuh build_node()
// (SPEC.md:276-284, :387-395).  (a) count pass: every buffer is sized from the LogicalTree and the plan's variant_home
// (which buffer a variant materialises in) and allocated exactly once; (b) recursive emit pass in the order the build
// block prescribes; (c) count / emit agreement is checked — a mismatch is a hard fault.
void encode_tree_generated(const scion_ltree& t, const LayoutEntry& layout, scion_ptree& out) {
  const BuilderEntry* be = find_builder(layout.name.c_str());
  if (!be || !be->build_root) throw std::runtime_error("layout '" + layout.name + "' carries no build block");
  encode_tree_with(t, layout, be->build_root, out);
}
void encode_tree_with(const scion_ltree& t, const LayoutEntry& layout, build_root_fn build_root, scion_ptree& out) {
  const lc::Plan& plan = *layout.plan;
  init_ptree(t, layout, out);
  const bool wide = plan.family == lc::Family::Bvh8;
  if (wide) require(t.has_wide, "8-wide layouts need a collapsed tree (scion_ltree_collapse8)");
  // logical nodes per variant (variant 0 = Interior, 1 = Leaf in every ADT of the corpus)
  uint64_t per_variant[2] = {0, 0};
  if (wide) {
    per_variant[0] = t.wnodes.size();
    per_variant[1] = t.wleaves.size();
    for (auto& l : t.wleaves) require(l.nprims >= 1 && l.nprims <= plan.max_leaf, "8-wide leaf exceeds the nprims capacity of layout " + plan.layout_name);
  } else {
    for (auto& n : t.nodes) per_variant[n.left < 0 ? 1 : 0]++;
  }
  Writer w(out, plan, false);
  for (auto& b : plan.buffers) {
    uint64_t count = 0;
    if (b.is_global_array) {
      count = t.tris.size() / 9;
    } else {
      for (size_t v = 0; v < plan.adt->variants.size() && v < 2; v++) {
        auto it = plan.variant_home.find(plan.adt->variants[v].name);
        if (it != plan.variant_home.end() && it->second == b.id) count += per_variant[v];
      }
    }
    const uint64_t arena = b.is_arena ? (count ? (count - 1) * arena_stride(b) + b.segments[0].stride_bytes : 0) + 8 : 0;
    w.alloc(b.name, count, arena);
    for (size_t g = 0; g < plan.globals.size(); g++)
      if (plan.globals[g].name == b.count_name) w.global_u(b.count_name, count);
  }
  BuildCtx ctx(t, plan, out);
  ctx.root_id = wide ? (int64_t)t.wroot : 0;
  if (wide ? t.wroot == SCION_W_SENTINEL : t.nodes.empty()) throw std::runtime_error("build fault: empty tree");
  out.root0 = build_root(ctx);
  for (auto& b : plan.buffers) {
    const uint64_t used = ctx.cursor[(size_t)b.id];
    const uint64_t want = b.is_arena ? (out.counts[(size_t)b.id] ? out.counts[(size_t)b.id] * arena_stride(b) : 0) : out.counts[(size_t)b.id];
    require(used == want, "count pass and emit pass disagree on buffer '" + b.name + "' (" + std::to_string(used) + " vs " + std::to_string(want) + ")");
  }
}

void encode_shell(const scion_ltree& t, const LayoutEntry& layout, scion_ptree& out, enc::EncodeJob& job, std::vector<uint32_t>& post) {
  init_ptree(t, layout, out);
  Writer w(out, *layout.plan, true);
  prepare(t, layout.name, w, job, post);
}

}  // namespace scion
