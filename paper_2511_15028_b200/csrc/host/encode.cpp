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
const LayoutEntry* find_layout(const std::string& name) {
  for (auto& e : layout_registry())
    if (e.name == name) return &e;
  return nullptr;
}

namespace {

// ------------------------------------------------------------------ directed rounding (host)
// true directed rounding through the FP environment
struct RoundingScope {
  int old;
  explicit RoundingScope(int mode) : old(fegetround()) { fesetround(mode); }
  ~RoundingScope() { fesetround(old); }
};
float fmul_rd(float a, float b) { volatile float x = a, y = b; RoundingScope s(FE_DOWNWARD); volatile float r = x * y; return r; }
float fsub_rd(float a, float b) { volatile float x = a, y = b; RoundingScope s(FE_DOWNWARD); volatile float r = x - y; return r; }
float fsub_ru(float a, float b) { volatile float x = a, y = b; RoundingScope s(FE_UPWARD); volatile float r = x - y; return r; }
float fdiv_rd(float a, float b) { volatile float x = a, y = b; RoundingScope s(FE_DOWNWARD); volatile float r = x / y; return r; }
float frcp_rd(float a) { volatile float x = a; RoundingScope s(FE_DOWNWARD); volatile float r = 1.0f / x; return r; }

// ------------------------------------------------------------------ bit writer
inline void put_bits(uint8_t* buf, uint64_t bit, uint32_t width, uint64_t value) {
  uint64_t byte = bit >> 3;
  uint32_t sh = (uint32_t)(bit & 7);
  uint32_t left = width;
  if (width < 64) value &= (1ull << width) - 1ull;
  while (left > 0) {
    uint32_t take = std::min<uint32_t>(8 - sh, left);
    uint8_t m = (uint8_t)(((1u << take) - 1u) << sh);
    buf[byte] = (uint8_t)((buf[byte] & ~m) | (((uint8_t)(value & ((1u << take) - 1u))) << sh));
    value >>= take;
    left -= take;
    sh = 0;
    byte++;
  }
}

struct Field {  // resolved slot of one stored field
  uint8_t* base = nullptr;
  uint64_t seg_base_bits = 0, stride_bits = 0, off = 0;
  uint32_t width = 0;
  bool arena = false;
  uint64_t pos(uint64_t idx) const { return arena ? idx * 8 + off : seg_base_bits + idx * stride_bits + off; }
  void set(uint64_t idx, uint64_t v) const { put_bits(base, pos(idx), width, v); }
  void set_lane(uint64_t idx, uint32_t lane, uint32_t lane_bits, uint64_t v) const { put_bits(base, pos(idx) + (uint64_t)lane * lane_bits, lane_bits, v); }
  void set_f(uint64_t idx, uint32_t lane, float f) const {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    set_lane(idx, lane, 32, u);
  }
  void set_f3(uint64_t idx, const float* f) const { for (uint32_t a = 0; a < 3; a++) set_f(idx, a, f[a]); }
};

struct Writer {
  scion_ptree& pt;
  const lc::Plan& plan;
  Writer(scion_ptree& p, const lc::Plan& pl) : pt(p), plan(pl) {}
  void alloc(const std::string& buffer, uint64_t count, uint64_t arena_bytes = 0) {
    const lc::Buffer* b = plan.buffer_named(buffer);
    if (!b) throw std::runtime_error("encode: no buffer '" + buffer + "' in layout " + plan.layout_name);
    std::vector<uint64_t> bases;
    uint64_t bytes = b->is_arena ? arena_bytes : b->bytes(count, &bases);
    if (b->is_arena) bases = {0};
    pt.buffers[(size_t)b->id].assign(bytes, 0);
    pt.counts[(size_t)b->id] = count;
    pt.seg_bases[(size_t)b->id] = bases;
  }
  Field field(const std::string& name) const {
    const lc::Slot& s = plan.slot(name);
    const lc::Buffer& b = plan.buffers[(size_t)s.buffer];
    Field f;
    f.base = pt.buffers[(size_t)s.buffer].data();
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
    std::memcpy(pt.buffers[(size_t)plan.buffer_named(buffer)->id].data(), t.tris.data(), t.tris.size() * 4);
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

// ------------------------------------------------------------------ bvh2, preorder, index refs
// pbrt.scion:21-33 / pbrt_align16.scion (same build) / authored pbrt-soa: `build low; build high;
// build nprims [= 0]; c_o = R - this | p_o = append(data, nprims)`
void encode_pbrt(const scion_ltree& t, Writer& w) {
  const uint64_t N = t.nodes.size();
  w.copy_primitives(t, "primitives", "P");
  w.alloc("nodes", N);
  w.global_u("N", N);
  Field low = w.field("low"), high = w.field("high"), nprims = w.field("nprims"), c_o = w.field("c_o"), p_o = w.field("p_o");
  for (uint64_t i = 0; i < N; i++) {
    const scion_lnode& n = t.nodes[i];
    low.set_f3(i, n.lo);
    high.set_f3(i, n.hi);
    if (n.left >= 0) {
      require((uint64_t)n.left == i + 1, "preorder build must place the left child at this+1");
      nprims.set(i, 0);
      c_o.set(i, (uint64_t)n.right - i);
    } else {
      nprims.set(i, n.nprims);
      p_o.set(i, n.first_prim);
    }
  }
  w.pt.root0 = 0;
}

// pbrt_post.scion:21-35: order=post, `c_l = this - L; c_r = this - R`
void encode_pbrt_post(const scion_ltree& t, Writer& w) {
  const uint64_t N = t.nodes.size();
  w.copy_primitives(t, "primitives", "P");
  w.alloc("nodes", N);
  w.global_u("N", N);
  // postorder numbering of the preorder array
  std::vector<uint32_t> post(N);
  {
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
  }
  Field low = w.field("low"), high = w.field("high"), nprims = w.field("nprims"), c_l = w.field("c_l"), c_r = w.field("c_r"), p_o = w.field("p_o");
  for (uint64_t i = 0; i < N; i++) {
    const scion_lnode& n = t.nodes[i];
    uint64_t me = post[i];
    low.set_f3(me, n.lo);
    high.set_f3(me, n.hi);
    if (n.left >= 0) {
      nprims.set(me, 0);
      c_l.set(me, me - post[(size_t)n.left]);
      c_r.set(me, me - post[(size_t)n.right]);
    } else {
      nprims.set(me, n.nprims);
      p_o.set(me, n.first_prim);
    }
  }
  w.pt.root0 = post[0];
}

// pbrt_q16.scion:49-73 — root block: world_low = low, world_extent = high - low;
// quantize_bounds: rcp = (1.0 / mex) * 65535.0; vu_floor((low - mlo) * rcp), vu_ceil((high - mlo) * rcp)
inline float clamp_code(float f, float top) { return std::fmax(0.0f, std::fmin(f, top)); }
void encode_pbrt_q16(const scion_ltree& t, Writer& w) {
  const uint64_t N = t.nodes.size();
  require(N < (1ull << 28), "pbrt-q16: node count exceeds the u28 child offset");
  require(t.tris.size() / 9 < (1ull << 28), "pbrt-q16: primitive count exceeds the u28 primitive offset");
  w.copy_primitives(t, "primitives", "primitive_count");
  w.alloc("nodes", N);
  w.global_u("node_count", N);
  float wl[3], we[3], rcp[3];
  for (int a = 0; a < 3; a++) {
    wl[a] = t.nodes[0].lo[a];
    we[a] = t.nodes[0].hi[a] - t.nodes[0].lo[a];
    rcp[a] = (1.0f / we[a]) * 65535.0f;
  }
  w.global_f3("world_low", wl);
  w.global_f3("world_extent", we);
  Field bq = w.field("bounds_q"), nprims = w.field("nprims"), c_off = w.field("c_offset"), p_off = w.field("p_offset");
  for (uint64_t i = 0; i < N; i++) {
    const scion_lnode& n = t.nodes[i];
    for (uint32_t a = 0; a < 3; a++) {
      float lo = clamp_code(std::floor((n.lo[a] - wl[a]) * rcp[a]), 65535.0f);
      float hi = clamp_code(std::ceil((n.hi[a] - wl[a]) * rcp[a]), 65535.0f);
      bq.set_lane(i, a, 16, (uint64_t)(uint32_t)lo);      // q16x3.lo lanes
      bq.set_lane(i, 3 + a, 16, (uint64_t)(uint32_t)hi);  // q16x3.hi lanes
    }
    if (n.left >= 0) {
      require((uint64_t)n.left == i + 1, "preorder build must place the left child at this+1");
      nprims.set(i, 0);
      c_off.set(i, (uint64_t)n.right - i);
    } else {
      nprims.set(i, n.nprims);
      p_off.set(i, n.first_prim);
    }
  }
  w.pt.root0 = 0;
}

// sg_eq.scion:9-30, :53-76 — root block: wlow, whigh, bins_inv = fdiv_rd(1023, guarded
// fsub_ru(high, low)), bins = frcp_rd(bins_inv); quantize_lo/hi = floorf(fmul_rd(fsub_rd(..), bin_inv))
void encode_sg_eq(const scion_ltree& t, Writer& w) {
  const uint64_t N = t.nodes.size();
  w.copy_primitives(t, "primitives", "primitive_count");
  w.alloc("nodes", N);
  w.global_u("node_count", N);
  float wl[3], wh[3], bins_inv[3], bins[3];
  for (int a = 0; a < 3; a++) {
    wl[a] = t.nodes[0].lo[a];
    wh[a] = t.nodes[0].hi[a];
    float l1 = fsub_ru(wh[a], wl[a]);
    float l2 = l1 > 0.0f ? l1 : 1.0f;
    bins_inv[a] = fdiv_rd(1023.0f, l2);
    bins[a] = frcp_rd(bins_inv[a]);
  }
  w.global_f3("wlow", wl);
  w.global_f3("whigh", wh);
  w.global_f3("bins", bins);
  w.global_f3("bins_inv", bins_inv);
  Field qmin = w.field("q_min"), qmax = w.field("q_max"), nprims = w.field("nprims"), off = w.field("offset"), poff = w.field("poffset");
  for (uint64_t i = 0; i < N; i++) {
    const scion_lnode& n = t.nodes[i];
    uint32_t lo[3], hi[3];
    for (int a = 0; a < 3; a++) {
      lo[a] = (uint32_t)std::floor(fmul_rd(fsub_rd(n.lo[a], wl[a]), bins_inv[a]));
      hi[a] = (uint32_t)std::floor(fmul_rd(fsub_rd(wh[a], n.hi[a]), bins_inv[a]));
    }
    qmin.set(i, ((lo[0] & 1023u) << 20) | ((lo[1] & 1023u) << 10) | (lo[2] & 1023u));
    qmax.set(i, ((hi[0] & 1023u) << 20) | ((hi[1] & 1023u) << 10) | (hi[2] & 1023u));
    if (n.left >= 0) {
      require((uint64_t)n.left == i + 1, "preorder build must place the left child at this+1");
      nprims.set(i, 0);
      off.set(i, (uint64_t)n.right - i);
    } else {
      nprims.set(i, n.nprims);
      poff.set(i, n.first_prim);
    }
  }
  w.pt.root0 = 0;
}

// dop14.scion:24-40 — `c0 = L; c1 = R` | `c0 = 0; c1 = 0x80000000 | (off << 4) | nprims`
void encode_dop14(const scion_ltree& t, Writer& w) {
  const uint64_t N = t.nodes.size();
  require(N < (1ull << 31), "dop14: node count exceeds i32 references");
  require(t.tris.size() / 9 < (1ull << 27), "dop14: primitive count exceeds the 27-bit offset");
  w.copy_primitives(t, "primitives", "P");
  w.alloc("nodes", N);
  w.global_u("N", N);
  Field lo1 = w.field("lo1"), hi1 = w.field("hi1"), c0 = w.field("c0"), c1 = w.field("c1"), lo2 = w.field("lo2"), hi2 = w.field("hi2");
  for (uint64_t i = 0; i < N; i++) {
    const scion_lnode& n = t.nodes[i];
    lo1.set_f3(i, n.lo);
    hi1.set_f3(i, n.hi);
    for (uint32_t k = 0; k < 4; k++) {
      lo2.set_f(i, k, t.dop_lo2[i * 4 + k]);
      hi2.set_f(i, k, t.dop_hi2[i * 4 + k]);
    }
    if (n.left >= 0) {
      c0.set(i, (uint32_t)n.left);
      c1.set(i, (uint32_t)n.right);
    } else {
      c0.set(i, 0);
      c1.set(i, 0x80000000u | (n.first_prim << 4) | n.nprims);
    }
  }
  w.pt.root0 = 0;
}

// ------------------------------------------------------------------ arena (ptr-referenced) layouts
// node address = byte offset inside the arena (plan.cpp:315-318), preorder allocation,
// each node rounded up to the group alignment.
struct Arena {
  std::vector<uint64_t> addr;
  uint64_t bytes = 0;
};
Arena place_arena(const scion_ltree& t, const lc::Buffer& b) {
  Arena a;
  a.addr.resize(t.nodes.size());
  uint64_t stride = b.segments[0].stride_bytes, cur = 0;
  for (size_t i = 0; i < t.nodes.size(); i++) {
    cur = (cur + b.align - 1) / b.align * b.align;
    a.addr[i] = cur;
    cur += stride;
  }
  a.bytes = cur + 8;  // put_bits/readers may touch one trailing word
  return a;
}

// ptr.scion:17-31
void encode_ptr(const scion_ltree& t, Writer& w) {
  w.copy_primitives(t, "primitives", "NP");
  Arena a = place_arena(t, *w.plan.buffer_named("node"));
  w.alloc("node", t.nodes.size(), a.bytes);
  Field low = w.field("low"), high = w.field("high"), nprims = w.field("nprims"), L = w.field("L"), R = w.field("R"), p_o = w.field("p_o");
  for (size_t i = 0; i < t.nodes.size(); i++) {
    const scion_lnode& n = t.nodes[i];
    uint64_t me = a.addr[i];
    low.set_f3(me, n.lo);
    high.set_f3(me, n.hi);
    if (n.left >= 0) {
      nprims.set(me, 0);
      L.set(me, a.addr[(size_t)n.left]);
      R.set(me, a.addr[(size_t)n.right]);
    } else {
      nprims.set(me, n.nprims);
      p_o.set(me, n.first_prim);
    }
  }
  w.pt.root0 = a.addr[0];
}

// identity.scion:19-33
void encode_identity(const scion_ltree& t, Writer& w) {
  w.copy_primitives(t, "primitives", "NP");
  Arena a = place_arena(t, *w.plan.buffer_named("node"));
  w.alloc("node", t.nodes.size(), a.bytes);
  Field low = w.field("low"), high = w.field("high"), tag = w.field("tag"), left = w.field("left"), right = w.field("right"), nprims = w.field("nprims"), p_o = w.field("p_o");
  for (size_t i = 0; i < t.nodes.size(); i++) {
    const scion_lnode& n = t.nodes[i];
    uint64_t me = a.addr[i];
    low.set_f3(me, n.lo);
    high.set_f3(me, n.hi);
    if (n.left >= 0) {
      tag.set(me, 0);
      left.set(me, a.addr[(size_t)n.left]);
      right.set(me, a.addr[(size_t)n.right]);
    } else {
      tag.set(me, 1);
      nprims.set(me, n.nprims);
      p_o.set(me, n.first_prim);
    }
  }
  w.pt.root0 = a.addr[0];
}

// shared_slab.scion:40-67 — root block: plo = low, phi = high (carried in the root reference);
// Interior: axis = longest_axis(low, high), slo = low[axis], shi = high[axis]
void encode_shared_slab(const scion_ltree& t, Writer& w) {
  w.copy_primitives(t, "primitives", "N");
  Arena a = place_arena(t, *w.plan.buffer_named("node"));
  w.alloc("node", t.nodes.size(), a.bytes);
  Field L = w.field("L"), R = w.field("R"), slo = w.field("slo"), shi = w.field("shi"), o = w.field("o"), axis = w.field("axis"), is_leaf = w.field("is_leaf"), nprims = w.field("nprims");
  for (size_t i = 0; i < t.nodes.size(); i++) {
    const scion_lnode& n = t.nodes[i];
    uint64_t me = a.addr[i];
    if (n.left >= 0) {
      float e[3] = {n.hi[0] - n.lo[0], n.hi[1] - n.lo[1], n.hi[2] - n.lo[2]};
      uint32_t ax = (e[0] >= e[1] && e[0] >= e[2]) ? 0 : (e[1] >= e[2] ? 1 : 2);
      is_leaf.set(me, 0);
      nprims.set(me, 0);
      o.set(me, 0);
      axis.set(me, ax);
      slo.set_f(me, 0, n.lo[ax]);
      shi.set_f(me, 0, n.hi[ax]);
      L.set(me, a.addr[(size_t)n.left]);
      R.set(me, a.addr[(size_t)n.right]);
    } else {
      is_leaf.set(me, 1);
      axis.set(me, 0);
      slo.set_f(me, 0, 0.0f);
      shi.set_f(me, 0, 0.0f);
      L.set(me, 0);
      R.set(me, 0);
      nprims.set(me, n.nprims);
      o.set(me, n.first_prim);
    }
  }
  w.pt.root0 = a.addr[0];
  std::memcpy(w.pt.carried, t.nodes[0].lo, 12);
  std::memcpy(w.pt.carried + 3, t.nodes[0].hi, 12);
  std::memcpy(w.pt.globals[(size_t)w.global_index("__ref_plo")].data(), t.nodes[0].lo, 12);
  std::memcpy(w.pt.globals[(size_t)w.global_index("__ref_phi")].data(), t.nodes[0].hi, 12);
}

// ------------------------------------------------------------------ 8-wide family
// bvh8.scion:19-30, bvh8_q8.scion:40-77, bvh8_q8_ci.scion:42-79, bvh8_q16*.scion:
// Interior -> ((this << 2) | 1); Leaf -> ((poffset << 7) | ((nprims - 1) << 2) | 0).
// SENTINEL slots: inverted box, child reference 0.
void encode_bvh8(const scion_ltree& t, Writer& w, int qbits, int ref_bits) {
  require(t.has_wide, "8-wide layouts need a collapsed tree (scion_ltree_collapse8)");
  const uint64_t NI = t.wnodes.size();
  const uint64_t P = t.tris.size() / 9;
  require(ref_bits == 64 || NI < (1ull << 30), "8-wide: interior count exceeds the 30-bit index");
  require(ref_bits == 64 || P < (1ull << 25), "8-wide: primitive count exceeds the 25-bit offset of compressed references");
  w.copy_primitives(t, "primitives", "primitive_count");
  w.alloc("Interiors", NI);
  w.global_u("interior_count", NI);
  auto ref_of = [&](int32_t c) -> uint64_t {
    if (c == SCION_W_SENTINEL) return 0;
    if (c >= 0) return ((uint64_t)c << 2) | 1ull;
    const scion_wleaf& l = t.wleaves[(size_t)(~c)];
    require(l.nprims >= 1 && l.nprims <= 32, "8-wide leaf capacity is 32 primitives");
    return ((uint64_t)l.first_prim << 7) | ((uint64_t)(l.nprims - 1) << 2);
  };
  Field children = w.field("children");
  if (qbits == 0) {
    Field lo = w.field("lo"), hi = w.field("hi");
    for (uint64_t i = 0; i < NI; i++) {
      const scion_wnode& n = t.wnodes[i];
      for (uint32_t k = 0; k < 8; k++) {
        for (uint32_t a = 0; a < 3; a++) {
          lo.set_f(i, 3 * k + a, n.lo[k][a]);
          hi.set_f(i, 3 * k + a, n.hi[k][a]);
        }
        children.set_lane(i, k, (uint32_t)ref_bits, ref_of(n.child[k]));
      }
    }
  } else {
    const float top = qbits == 8 ? 255.0f : 65535.0f;
    Field mlo_f = w.field("mlo"), mex_f = w.field("mex"), cb = w.field("child_bounds");
    for (uint64_t i = 0; i < NI; i++) {
      const scion_wnode& n = t.wnodes[i];
      float mlo[3], mex[3], rcp[3];
      for (int a = 0; a < 3; a++) {
        float l = n.lo[7][a], h = n.hi[7][a];
        for (int k = 6; k >= 0; k--) {  // min(lo[0], min(lo[1], ... min(lo[6], lo[7])))
          l = std::fmin(n.lo[k][a], l);
          h = std::fmax(n.hi[k][a], h);
        }
        mlo[a] = l;
        mex[a] = h - l;
        rcp[a] = (1.0f / mex[a]) * top;
      }
      mlo_f.set_f3(i, mlo);
      mex_f.set_f3(i, mex);
      for (uint32_t k = 0; k < 8; k++) {
        for (uint32_t a = 0; a < 3; a++) {
          float ql = clamp_code(std::floor((n.lo[k][a] - mlo[a]) * rcp[a]), top);
          float qh = clamp_code(std::ceil((n.hi[k][a] - mlo[a]) * rcp[a]), top);
          cb.set_lane(i, k * 6 + a, (uint32_t)qbits, (uint64_t)(uint32_t)ql);      // qbox.lo lanes
          cb.set_lane(i, k * 6 + 3 + a, (uint32_t)qbits, (uint64_t)(uint32_t)qh);  // qbox.hi lanes
        }
        children.set_lane(i, k, (uint32_t)ref_bits, ref_of(n.child[k]));
      }
    }
  }
  w.pt.root0 = ref_of(t.wroot);
}

}  // namespace

void encode_tree(const scion_ltree& t, const LayoutEntry& layout, scion_ptree& out) {
  const lc::Plan& plan = *layout.plan;
  out = scion_ptree();
  out.layout = layout.name;
  out.plan = &plan;
  out.buffers.resize(plan.buffers.size());
  out.counts.assign(plan.buffers.size(), 0);
  out.seg_bases.resize(plan.buffers.size());
  out.globals.resize(plan.globals.size());
  for (auto& g : out.globals) g.fill(0);
  out.nprims = t.tris.size() / 9;
  if (plan.family != lc::Family::Bvh8) check_leaf_capacity(t, plan);
  Writer w(out, plan);
  const std::string& n = layout.name;
  if (n == "pbrt" || n == "pbrt-align16" || n == "pbrt-soa") encode_pbrt(t, w);
  else if (n == "pbrt-post") encode_pbrt_post(t, w);
  else if (n == "pbrt-q16") encode_pbrt_q16(t, w);
  else if (n == "sg-eq" || n == "sg-eq-align16") encode_sg_eq(t, w);
  else if (n == "dop14") encode_dop14(t, w);
  else if (n == "ptr") encode_ptr(t, w);
  else if (n == "identity") encode_identity(t, w);
  else if (n == "shared-slab") encode_shared_slab(t, w);
  else if (n == "bvh8") encode_bvh8(t, w, 0, 64);
  else if (n == "bvh8-q8") encode_bvh8(t, w, 8, 64);
  else if (n == "bvh8-q8-ci") encode_bvh8(t, w, 8, 32);
  else if (n == "bvh8-q16") encode_bvh8(t, w, 16, 64);
  else if (n == "bvh8-q16-ci") encode_bvh8(t, w, 16, 32);
  else throw std::runtime_error("no encoder registered for layout '" + n + "'");
}

}  // namespace scion
