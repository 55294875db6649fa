// C ABI of the backend (include/scion_b200.h): thin extern "C" layer over the host C++ (layout
// compiler, scene tools, encoders) and the CUDA kernels.  Nothing here falls back to a CPU
// traversal: without a CUDA device every query entry point fails with SCION_ERR_NO_DEVICE.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "device/geometry.cuh"
#include "device/launch.cuh"
#include "host/build_ctx.hpp"
#include "host/dtree.hpp"
#include "host/encode_node.hpp"
#include "host/physical.hpp"
#include "host/rng.hpp"
#include "host/scene.hpp"
#include "scion_b200.h"

namespace {

thread_local std::string g_error;
std::atomic<uint64_t> g_launches{0};

int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}
#define SCION_TRY(...)                                              \
  try {                                                             \
    __VA_ARGS__                                                     \
  } catch (const scion::lc::LayoutError& e) {                       \
    return fail(SCION_ERR_LAYOUT, e.what());                        \
  } catch (const std::bad_alloc&) {                                 \
    return fail(SCION_ERR_BUILD, "out of host memory");             \
  } catch (const std::exception& e) {                               \
    return fail(SCION_ERR_BUILD, e.what());                         \
  }
#define CUDA_OK(expr)                                                                                  \
  do {                                                                                                 \
    cudaError_t e__ = (expr);                                                                          \
    if (e__ != cudaSuccess) return fail(e__ == cudaErrorNoDevice || e__ == cudaErrorInsufficientDriver ? SCION_ERR_NO_DEVICE : SCION_ERR_CUDA, \
                                        std::string(#expr) + ": " + cudaGetErrorString(e__));          \
  } while (0)

char* dup_string(const std::string& s) {
  char* p = (char*)malloc(s.size() + 1);
  if (p) memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

}  // namespace

using scion::ImageHeader;
using scion::kHeaderBytes;
using scion::kImageMagic;
using scion::CounterPool;
using scion::fill_view;
using scion::finish_dtree;
int scion::abi_fail(int code, const std::string& msg) { return fail(code, msg); }

void scion::fill_view(scion_dtree& t) {
  const ImageHeader& h = t.header;
  memset(&t.view, 0, sizeof(t.view));
  for (int b = 0; b < h.nbuf; b++) {
    t.view.buf[b] = t.image + h.offset[b];
    t.view.count[b] = h.count[b];
    for (int s = 0; s < SCION_MAX_SEGMENTS; s++) t.view.seg_base[b][s] = h.seg_base[b][s];
  }
  memcpy(t.view.glob, h.glob, sizeof(h.glob));
  t.view.root0 = h.root0;
  memcpy(t.view.root_carried, h.carried, sizeof(h.carried));
}

namespace {
int header_from_ptree(const scion_ptree& p, ImageHeader& h) {
  memset(&h, 0, sizeof(h));
  h.magic = kImageMagic;
  if (p.buffers.size() > SCION_MAX_BUFFERS || p.globals.size() > SCION_MAX_GLOBALS) return fail(SCION_ERR_LAYOUT, "layout exceeds the device view limits");
  strncpy(h.layout, p.layout.c_str(), sizeof(h.layout) - 1);
  h.nbuf = (int32_t)p.buffers.size();
  h.nglob = (int32_t)p.globals.size();
  uint64_t off = kHeaderBytes;
  for (size_t b = 0; b < p.buffers.size(); b++) {
    if (p.seg_bases[b].size() > SCION_MAX_SEGMENTS) return fail(SCION_ERR_LAYOUT, "too many segments");
    const uint64_t sz = p.sizes.size() == p.buffers.size() ? p.sizes[b] : p.buffers[b].size();
    h.offset[b] = off;
    h.bytes[b] = sz;
    h.count[b] = p.counts[b];
    for (size_t s = 0; s < p.seg_bases[b].size(); s++) h.seg_base[b][s] = p.seg_bases[b][s];
    off += (sz + 32 + 255) / 256 * 256;  // >= 32 bytes of slack behind every buffer: covering vector loads (scion_rt.cuh load_record, geometry.cuh load_triangle36)
  }
  for (size_t g = 0; g < p.globals.size(); g++) memcpy(h.glob[g], p.globals[g].data(), 16);
  h.root0 = p.root0;
  memcpy(h.carried, p.carried, sizeof(h.carried));
  h.nprims = p.nprims;
  h.total_bytes = off;
  return SCION_OK;
}

}  // namespace

int scion::finish_dtree(scion_dtree* t) {
  t->kernels = scion::find_kernels(t->layout->name.c_str());
  if (!t->kernels) return fail(SCION_ERR_LAYOUT, "no kernels were compiled for layout '" + t->layout->name + "'");
  {
    std::lock_guard<std::mutex> lock(t->counters.mu);
    CUDA_OK(t->counters.grow());
  }
  fill_view(*t);
  // side treelet of the top levels for the layouts whose kernel can stage it (north_star: top levels in shared memory via
  // TMA bulk copies).  The image is complete on the device here (every caller has synchronised).
  if (t->kernels->build_treelet && t->header.nbuf > 1 && t->header.count[1] > 0 && t->header.count[1] < (1ull << 31)) {
    uint32_t slots = 0;
    CUDA_OK(cudaSetDevice(t->device));
    CUDA_OK(t->kernels->build_treelet(t->view, &t->treelet, &slots));
    t->view.treelet = t->treelet;
    t->view.treelet_slots = slots;
  }
  return SCION_OK;
}

namespace {
struct FileW {
  FILE* f;
  bool ok = true;
  void raw(const void* p, size_t n) { if (n && fwrite(p, 1, n, f) != n) ok = false; }
  template <class T> void val(T v) { raw(&v, sizeof(T)); }
  void str(const std::string& s) { val<uint32_t>((uint32_t)s.size()); raw(s.data(), s.size()); }
};
struct FileR {
  FILE* f;
  bool ok = true;
  void raw(void* p, size_t n) { if (n && fread(p, 1, n, f) != n) ok = false; }
  template <class T> T val() { T v{}; raw(&v, sizeof(T)); return v; }
  std::string str() { uint32_t n = val<uint32_t>(); if (!ok || n > 4096) { ok = false; return ""; } std::string s(n, 0); raw(s.data(), n); return s; }
};
}  // namespace

namespace scion {
__global__ void ray_triangle_kernel(const scion_ray* __restrict__ rays, const float* __restrict__ tris, uint64_t n, int method, scion_trihit* __restrict__ out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const scion_ray r = rays[i];
  const RayCtx ray = make_ray(r.ox, r.oy, r.oz, r.tmax, r.dx, r.dy, r.dz);
  float tri[9];
#pragma unroll
  for (int k = 0; k < 9; k++) tri[k] = tris[9 * i + k];
  scion_trihit h{0.0f, 0.0f, 0.0f, 0.0f, 0u};
  float b0, b1, b2, t;
  const bool hit = method == SCION_TRI_PLUECKER ? ray_tri_pc_full(ray, tri, b0, b1, b2, t) : ray_tri_mt_full(ray, tri, b0, b1, b2, t);
  if (hit) h = scion_trihit{b0, b1, b2, t, 1u};
  out[i] = h;
}
// device-side encode: one thread per node (host/encode_node.hpp)
__global__ void encode_nodes_kernel(const enc::EncodeJob job) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < job.count) enc::encode_one(job, i);
}
int device_sm_count() {
  static int sms[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (sms[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    sms[dev] = v;
  }
  return sms[dev];
}
}  // namespace scion

extern "C" {

const char* scion_last_error(void) { return g_error.c_str(); }
int scion_abi_version(void) { return SCION_ABI_VERSION; }
void scion_free(void* p) { free(p); }
uint64_t scion_kernel_launches(void) { return g_launches.load(); }

// ------------------------------------------------------------------ layout registry
static void info_of(const scion::LayoutEntry& e, scion_layout_info* out) {
  const scion::lc::Plan& p = *e.plan;
  out->name = e.name.c_str();
  out->family = (int)p.family;
  out->arity = p.family == scion::lc::Family::Bvh8 ? 8 : 2;
  const scion::lc::Buffer* nb = p.buffer_named(p.node_group);
  out->node_stride = nb ? (uint32_t)nb->node_stride() : 0;
  out->node_align = nb ? nb->align : 1;
  out->n_segments = nb ? (uint32_t)nb->segments.size() : 0;
  out->ref_bits = (uint32_t)p.type_bits(p.ref[0].type);
  out->max_leaf = p.max_leaf;
  out->has_cpq = e.has_cpq ? 1 : 0;
}
int scion_layout_count(void) {
  SCION_TRY(return (int)scion::layout_registry().size();)
}
int scion_layout_info_at(int index, scion_layout_info* out) {
  SCION_TRY(auto& r = scion::layout_registry(); if (index < 0 || index >= (int)r.size() || !out) return fail(SCION_ERR_ARG, "layout index out of range"); info_of(r[(size_t)index], out); return SCION_OK;)
}
int scion_layout_registered_count(void) { return scion::dyn_layout_count(); }
int scion_layout_registered_at(int index, scion_layout_info* out) {
  SCION_TRY(const scion::LayoutEntry* e = scion::dyn_layout_at(index); if (!e || !out) return fail(SCION_ERR_ARG, "layout index out of range"); info_of(*e, out); return SCION_OK;)
}
int scion_layout_find(const char* name, scion_layout_info* out) {
  SCION_TRY(const scion::LayoutEntry* e = name ? scion::find_layout(name) : nullptr; if (!e) return fail(SCION_ERR_ARG, std::string("unknown layout '") + (name ? name : "") + "'"); if (out) info_of(*e, out); return SCION_OK;)
}
int scion_layout_plan_json(const char* name, char** out_json) {
  SCION_TRY(const scion::LayoutEntry* e = name ? scion::find_layout(name) : nullptr; if (!e || !out_json) return fail(SCION_ERR_ARG, "unknown layout"); *out_json = dup_string(e->plan->to_json()); return SCION_OK;)
}
int scion_layout_emit_cuda(const char* name, char** out_text) {
  SCION_TRY(const scion::LayoutEntry* e = name ? scion::find_layout(name) : nullptr; if (!e || !out_text) return fail(SCION_ERR_ARG, "unknown layout"); *out_text = dup_string(scion::lc::emit_cuda(*e->plan)); return SCION_OK;)
}
int scion_layout_emit_c(const char* name, char** out_text) {
  SCION_TRY(const scion::LayoutEntry* e = name ? scion::find_layout(name) : nullptr; if (!e || !out_text) return fail(SCION_ERR_ARG, "unknown layout"); *out_text = dup_string(scion::lc::emit_c_records(*e->plan)); return SCION_OK;)
}
int scion_layout_stats_json(const char* name, char** out_json) {
  SCION_TRY(const scion::LayoutEntry* e = name ? scion::find_layout(name) : nullptr; if (!e || !out_json) return fail(SCION_ERR_ARG, "unknown layout"); *out_json = dup_string(scion::lc::decode_stats_json(*e->plan)); return SCION_OK;)
}
int scion_compile_layout_text(const char* src, char** out_plan_json, char** out_cuda) {
  if (!src) return fail(SCION_ERR_ARG, "null source");
  SCION_TRY(scion::lc::Program prog = scion::lc::parse_program({std::string(src)}); scion::lc::Plan plan = scion::lc::plan_layout(prog, "user-layout");
            if (out_plan_json) *out_plan_json = dup_string(plan.to_json()); if (out_cuda) *out_cuda = dup_string(scion::lc::emit_cuda(plan)); return SCION_OK;)
}

int scion_layout_register(const char* name, const char* src, const char* work_dir, char** out_log) {
  if (!name || !src) return fail(SCION_ERR_ARG, "null argument");
  std::string log;
  int rc = SCION_OK;
  try {
    scion::register_layout_plugin(name, src, work_dir ? work_dir : "", log);
  } catch (const scion::lc::LayoutError& e) {
    rc = fail(SCION_ERR_LAYOUT, e.what());
  } catch (const std::exception& e) {
    rc = fail(SCION_ERR_BUILD, e.what());
  }
  if (out_log) *out_log = dup_string(log);
  return rc;
}

// ------------------------------------------------------------------ scene tools
int scion_scene_terrain(uint32_t grid, uint64_t seed, scion_scene** out) {
  if (!out) return fail(SCION_ERR_ARG, "null out");
  SCION_TRY(auto* s = new scion_scene(); scion::make_terrain(grid, seed, *s); *out = s; return SCION_OK;)
}
int scion_scene_sphere(uint32_t grid, uint64_t seed, scion_scene** out) {
  if (!out) return fail(SCION_ERR_ARG, "null out");
  SCION_TRY(auto* s = new scion_scene(); scion::make_sphere(grid, seed, *s); *out = s; return SCION_OK;)
}
int scion_scene_cloud(uint64_t npoints, uint64_t seed, scion_scene** out) {
  if (!out) return fail(SCION_ERR_ARG, "null out");
  SCION_TRY(auto* s = new scion_scene(); scion::make_cloud(npoints, seed, *s); *out = s; return SCION_OK;)
}
int scion_scene_from_triangles(const float* xyz9, uint64_t ntris, scion_scene** out) {
  if (!out || (!xyz9 && ntris)) return fail(SCION_ERR_ARG, "null argument");
  SCION_TRY(auto* s = new scion_scene(); s->name = "user"; s->tris.assign(xyz9, xyz9 + ntris * 9); *out = s; return SCION_OK;)
}
uint64_t scion_scene_ntris(const scion_scene* s) { return s ? s->ntris() : 0; }
const float* scion_scene_triangles(const scion_scene* s) { return s ? s->tris.data() : nullptr; }
void scion_scene_bounds(const scion_scene* s, float lo[3], float hi[3]) { if (s) scion::scene_bounds(*s, lo, hi); }
void scion_scene_free(scion_scene* s) { delete s; }

int scion_build_sah(const scion_scene* s, uint32_t bins, uint32_t max_leaf, uint32_t max_depth, scion_ltree** out) {
  if (!s || !out) return fail(SCION_ERR_ARG, "null argument");
  SCION_TRY(auto* t = new scion_ltree(); try { scion::build_binary(*s, scion::Builder::SAH, bins, max_leaf, max_depth, *t); } catch (...) { delete t; throw; } *out = t; return SCION_OK;)
}
int scion_build_median(const scion_scene* s, uint32_t max_leaf, scion_ltree** out) {
  if (!s || !out) return fail(SCION_ERR_ARG, "null argument");
  SCION_TRY(auto* t = new scion_ltree(); try { scion::build_binary(*s, scion::Builder::Median, 2, max_leaf, 0, *t); } catch (...) { delete t; throw; } *out = t; return SCION_OK;)
}
int scion_ltree_from_arrays(const scion_lnode* nodes, uint64_t nnodes, const float* tris9, uint64_t ntris, scion_ltree** out) {
  if (!out) return fail(SCION_ERR_ARG, "null out");
  SCION_TRY(auto* t = new scion_ltree(); try { scion::import_binary(nodes, nnodes, tris9, ntris, *t); } catch (...) { delete t; throw; } *out = t; return SCION_OK;)
}
int scion_ltree_collapse8(scion_ltree* t) {
  if (!t) return fail(SCION_ERR_ARG, "null tree");
  SCION_TRY(scion::collapse8(*t); return SCION_OK;)
}
uint64_t scion_ltree_nnodes(const scion_ltree* t) { return t->nodes.size(); }
const scion_lnode* scion_ltree_nodes(const scion_ltree* t) { return t->nodes.data(); }
uint64_t scion_ltree_nprims(const scion_ltree* t) { return t->tris.size() / 9; }
const float* scion_ltree_triangles(const scion_ltree* t) { return t->tris.data(); }
const uint32_t* scion_ltree_prim_ids(const scion_ltree* t) { return t->prim_ids.data(); }
const float* scion_ltree_dop_lo2(const scion_ltree* t) { return t->dop_lo2.data(); }
const float* scion_ltree_dop_hi2(const scion_ltree* t) { return t->dop_hi2.data(); }
uint32_t scion_ltree_depth(const scion_ltree* t) { return t->depth; }
uint64_t scion_ltree_nwnodes(const scion_ltree* t) { return t->wnodes.size(); }
const scion_wnode* scion_ltree_wnodes(const scion_ltree* t) { return t->wnodes.data(); }
uint64_t scion_ltree_nwleaves(const scion_ltree* t) { return t->wleaves.size(); }
const scion_wleaf* scion_ltree_wleaves(const scion_ltree* t) { return t->wleaves.data(); }
int32_t scion_ltree_wroot(const scion_ltree* t) { return t->wroot; }
void scion_ltree_free(scion_ltree* t) { delete t; }

// ------------------------------------------------------------------ build_physical
int scion_encode(const scion_ltree* t, const char* layout, scion_ptree** out) {
  if (!t || !layout || !out) return fail(SCION_ERR_ARG, "null argument");
  SCION_TRY(const scion::LayoutEntry* e = scion::find_layout(layout); if (!e) return fail(SCION_ERR_ARG, std::string("unknown layout '") + layout + "'");
            if (e->plan->family == scion::lc::Family::Bvh8 && !t->has_wide) return fail(SCION_ERR_BUILD, "8-wide layouts need scion_ltree_collapse8 first");
            auto* p = new scion_ptree(); try { scion::encode_tree(*t, *e, *p); } catch (...) { delete p; throw; } *out = p; return SCION_OK;)
}
int scion_encode_generated(const scion_ltree* t, const char* layout, scion_ptree** out) {
  if (!t || !layout || !out) return fail(SCION_ERR_ARG, "null argument");
  SCION_TRY(const scion::LayoutEntry* e = scion::find_layout(layout); if (!e) return fail(SCION_ERR_ARG, std::string("unknown layout '") + layout + "'");
            if (e->plan->family == scion::lc::Family::Bvh8 && !t->has_wide) return fail(SCION_ERR_BUILD, "8-wide layouts need scion_ltree_collapse8 first");
            auto* p = new scion_ptree(); try { scion::encode_tree_generated(*t, *e, *p); } catch (...) { delete p; throw; } *out = p; return SCION_OK;)
}
int scion_layout_has_build(const char* layout) {
  const scion::BuilderEntry* b = layout ? scion::find_builder(layout) : nullptr;
  return b && b->build_root ? 1 : 0;
}
const char* scion_ptree_layout(const scion_ptree* p) { return p->layout.c_str(); }
int scion_ptree_nbuffers(const scion_ptree* p) { return (int)p->buffers.size(); }
int scion_ptree_buffer(const scion_ptree* p, int i, const char** name, const uint8_t** data, uint64_t* bytes, uint64_t* count) {
  if (!p || i < 0 || i >= (int)p->buffers.size()) return fail(SCION_ERR_ARG, "buffer index out of range");
  if (name) *name = p->plan->buffers[(size_t)i].name.c_str();
  if (data) *data = p->buffers[(size_t)i].data();
  if (bytes) *bytes = p->buffers[(size_t)i].size();
  if (count) *count = p->counts[(size_t)i];
  return SCION_OK;
}
int scion_ptree_segment_bases(const scion_ptree* p, int i, uint64_t* bases, int max) {
  if (!p || i < 0 || i >= (int)p->buffers.size()) return 0;
  int n = (int)p->seg_bases[(size_t)i].size();
  for (int s = 0; s < n && s < max; s++) bases[s] = p->seg_bases[(size_t)i][(size_t)s];
  return n;
}
int scion_ptree_nglobals(const scion_ptree* p) { return (int)p->globals.size(); }
int scion_ptree_global(const scion_ptree* p, int i, const char** name, uint8_t raw[16], uint32_t* nbytes) {
  if (!p || i < 0 || i >= (int)p->globals.size()) return fail(SCION_ERR_ARG, "global index out of range");
  if (name) *name = p->plan->globals[(size_t)i].name.c_str();
  if (raw) memcpy(raw, p->globals[(size_t)i].data(), 16);
  if (nbytes) *nbytes = (uint32_t)((p->plan->type_bits(p->plan->globals[(size_t)i].type) + 7) / 8);
  return SCION_OK;
}
int scion_ptree_root(const scion_ptree* p, uint64_t* ref0, float* carried6) {
  if (!p) return fail(SCION_ERR_ARG, "null tree");
  if (ref0) *ref0 = p->root0;
  if (carried6) memcpy(carried6, p->carried, sizeof(p->carried));
  return SCION_OK;
}
uint64_t scion_ptree_total_bytes(const scion_ptree* p) {
  uint64_t s = 0;
  for (auto& b : p->buffers) s += b.size();
  return s;
}
uint64_t scion_ptree_node_bytes(const scion_ptree* p) {
  uint64_t s = 0;
  for (size_t b = 0; b < p->buffers.size(); b++)
    if (!p->plan->buffers[b].is_global_array) s += p->buffers[b].size();
  return s;
}
// ---- validation shared by every way a PhysicalTree built elsewhere enters the library (container file,
// in-memory import): sizes must be the planner's footprint() for the stated counts (plan.cpp:333-347), segment
// bases the planner's, the primitive range and the root reference inside their buffers — a tree that passes
// cannot make a kernel read outside the device image through its ROOT; child links inside node records are the
// producer's contract ("buffers sized exactly footprint()").
static int validate_ptree(scion_ptree& p, std::string& why) {
  const scion::lc::Plan& plan = *p.plan;
  const size_t nb = plan.buffers.size();
  if (p.buffers.size() != nb || p.counts.size() != nb || p.seg_bases.size() != nb) { why = "buffer table does not match the layout's plan"; return 1; }
  if (p.globals.size() != plan.globals.size()) { why = "global slot table does not match the layout's plan"; return 1; }
  if (nb > SCION_MAX_BUFFERS || plan.globals.size() > SCION_MAX_GLOBALS) { why = "layout exceeds the device view limits"; return 1; }
  p.sizes.resize(nb);
  for (size_t b = 0; b < nb; b++) {
    const scion::lc::Buffer& pb = plan.buffers[b];
    const uint64_t have = p.buffers[b].size();
    p.sizes[b] = have;
    if (pb.is_arena) {
      if (p.seg_bases[b].empty()) p.seg_bases[b] = {0};
      if (p.seg_bases[b].size() != 1 || p.seg_bases[b][0] != 0) { why = "arena buffer '" + pb.name + "' must have the single segment base 0"; return 1; }
      continue;
    }
    if (pb.segments.size() > SCION_MAX_SEGMENTS) { why = "too many segments"; return 1; }
    std::vector<uint64_t> bases;
    const uint64_t stride = pb.node_stride();
    if (stride && p.counts[b] > (~0ull >> 8) / stride) { why = "element count of buffer '" + pb.name + "' is absurd"; return 1; }
    const uint64_t want = pb.bytes(p.counts[b], &bases);
    if (have != want) { why = "buffer '" + pb.name + "': " + std::to_string(have) + " bytes, footprint() says " + std::to_string(want) + " for " + std::to_string(p.counts[b]) + " elements"; return 1; }
    if (p.seg_bases[b].empty()) p.seg_bases[b] = bases;
    if (p.seg_bases[b] != bases) { why = "segment bases of buffer '" + pb.name + "' disagree with the plan (plan.cpp:333-347)"; return 1; }
  }
  const scion::lc::Buffer* prim = plan.buffer_named("primitives");
  if (!prim) { why = "layout has no primitives array"; return 1; }
  if (p.nprims == 0) p.nprims = p.counts[(size_t)prim->id];
  if (p.nprims != p.counts[(size_t)prim->id]) { why = "nprims disagrees with the primitives buffer"; return 1; }
  const scion::lc::Buffer* nodes = plan.buffer_named(plan.node_group);
  if (!nodes) { why = "layout has no node group"; return 1; }
  const uint64_t ncount = p.counts[(size_t)nodes->id], nbytes = p.buffers[(size_t)nodes->id].size();
  if (plan.family == scion::lc::Family::Bvh8) {  // tagged reference: bit 0 = Interior, else Leaf(O, nprims) (bvh8*.scion)
    const bool ci = plan.type_bits(plan.ref[0].type) <= 32;
    const uint64_t r = p.root0;
    if (r & 1ull) {
      const uint64_t key = ci ? ((r & 0xffffffffull) >> 2) : (r >> 2);
      if (key >= ncount) { why = "root reference names interior " + std::to_string(key) + " of " + std::to_string(ncount); return 1; }
    } else {
      const uint64_t o = ci ? ((r & 0xffffffffull) >> 7) : (r >> 7), n = ((r >> 2) & 31ull) + 1ull;
      if (p.nprims && o + n > p.nprims) { why = "root leaf reference exceeds the primitives array"; return 1; }
    }
  } else if (nodes->is_arena) {
    if (ncount && p.root0 + nodes->segments[0].stride_bytes > nbytes) { why = "root reference lies outside the node arena"; return 1; }
  } else {
    if (ncount == 0 || p.root0 >= ncount) { why = "root reference " + std::to_string(p.root0) + " is not a node index (node count " + std::to_string(ncount) + ")"; return 1; }
  }
  return 0;
}

// In-memory import of a PhysicalTree produced by someone else's build_physical (buffer id ->
// byte array; global slot -> scalar; root reference): one descriptor per BufferDesc / GlobalDesc of the plan
// (/root/reference/proj/include/layoutc/plan.hpp:31-48), matched by NAME, any order.  The library copies.
int scion_ptree_from_buffers(const scion_tree_desc* d, scion_ptree** out) {
  if (!d || !out || !d->layout || (!d->buffers && d->nbuffers) || (!d->globals && d->nglobals)) return fail(SCION_ERR_ARG, "null argument");
  SCION_TRY(
    const scion::LayoutEntry* e = scion::find_layout(d->layout);
    if (!e) return fail(SCION_ERR_ARG, std::string("unknown layout '") + d->layout + "'");
    const scion::lc::Plan& plan = *e->plan;
    auto p = std::make_unique<scion_ptree>();
    p->layout = e->name;
    p->plan = &plan;
    const size_t nb = plan.buffers.size();
    p->buffers.resize(nb); p->counts.assign(nb, 0); p->seg_bases.resize(nb);
    p->globals.resize(plan.globals.size());
    for (auto& g : p->globals) g.fill(0);
    std::vector<char> seen_b(nb, 0), seen_g(plan.globals.size(), 0);
    for (uint32_t i = 0; i < d->nbuffers; i++) {
      const scion_buffer_desc& bd = d->buffers[i];
      if (!bd.name) return fail(SCION_ERR_ARG, "buffer descriptor without a name");
      const scion::lc::Buffer* pb = plan.buffer_named(bd.name);
      if (!pb) return fail(SCION_ERR_ARG, std::string("layout '") + e->name + "' has no buffer '" + bd.name + "'");
      if (seen_b[(size_t)pb->id]) return fail(SCION_ERR_ARG, std::string("buffer '") + bd.name + "' given twice");
      if (!bd.data && bd.bytes) return fail(SCION_ERR_ARG, std::string("buffer '") + bd.name + "' has bytes but no data");
      seen_b[(size_t)pb->id] = 1;
      p->buffers[(size_t)pb->id].assign((const uint8_t*)bd.data, (const uint8_t*)bd.data + bd.bytes);
      p->counts[(size_t)pb->id] = bd.count;
      if (bd.seg_bases) p->seg_bases[(size_t)pb->id].assign(bd.seg_bases, bd.seg_bases + bd.n_seg_bases);
    }
    for (size_t b = 0; b < nb; b++)
      if (!seen_b[b] && plan.buffers[b].node_stride() != 0) return fail(SCION_ERR_ARG, "missing buffer '" + plan.buffers[b].name + "'");
    for (uint32_t i = 0; i < d->nglobals; i++) {
      const scion_global_desc& gd = d->globals[i];
      if (!gd.name) return fail(SCION_ERR_ARG, "global descriptor without a name");
      size_t g = 0;
      while (g < plan.globals.size() && plan.globals[g].name != gd.name) g++;
      if (g == plan.globals.size()) return fail(SCION_ERR_ARG, std::string("layout '") + e->name + "' has no global slot '" + gd.name + "'");
      if (seen_g[g]) return fail(SCION_ERR_ARG, std::string("global '") + gd.name + "' given twice");
      seen_g[g] = 1;
      memcpy(p->globals[g].data(), gd.raw, 16);
    }
    for (size_t g = 0; g < plan.globals.size(); g++)
      if (!seen_g[g]) return fail(SCION_ERR_ARG, "missing global slot '" + plan.globals[g].name + "'");
    p->root0 = d->root_ref;
    memcpy(p->carried, d->carried, sizeof(p->carried));
    p->nprims = d->nprims;
    std::string why;
    if (validate_ptree(*p, why)) return fail(SCION_ERR_ARG, "scion_ptree_from_buffers: " + why);
    *out = p.release();
    return SCION_OK;
  )
}
// the survey's one-call form: import + upload; the host descriptor stays the caller's
int scion_tree_upload(const scion_tree_desc* host, int device, scion_dtree** out) {
  scion_ptree* p = nullptr;
  int rc = scion_ptree_from_buffers(host, &p);
  if (rc) return rc;
  rc = scion_dtree_upload(p, device, out);
  scion_ptree_free(p);
  return rc;
}

// ---- container file: "SCIONPT1" | u32 version | u32 name_len | name | u64 nprims | u64 root0 | 6 x f32 carried |
//      u32 nglob | nglob x { u32 len, name, 16 raw bytes } | u32 nbuf | nbuf x { u32 len, name, u64 count, u64 bytes,
//      u32 nseg, nseg x u64 base } | raw buffers, each padded to 16 bytes.  Little-endian throughout.
int scion_ptree_save(const scion_ptree* p, const char* path) {
  if (!p || !path) return fail(SCION_ERR_ARG, "null argument");
  FILE* f = fopen(path, "wb");
  if (!f) return fail(SCION_ERR_ARG, std::string("cannot open ") + path);
  FileW w{f};
  w.raw("SCIONPT1", 8);
  w.val<uint32_t>(1);
  w.str(p->layout);
  w.val<uint64_t>(p->nprims);
  w.val<uint64_t>(p->root0);
  w.raw(p->carried, sizeof(p->carried));
  w.val<uint32_t>((uint32_t)p->globals.size());
  for (size_t g = 0; g < p->globals.size(); g++) { w.str(p->plan->globals[g].name); w.raw(p->globals[g].data(), 16); }
  w.val<uint32_t>((uint32_t)p->buffers.size());
  for (size_t b = 0; b < p->buffers.size(); b++) {
    w.str(p->plan->buffers[b].name);
    w.val<uint64_t>(p->counts[b]);
    w.val<uint64_t>(p->buffers[b].size());
    w.val<uint32_t>((uint32_t)p->seg_bases[b].size());
    for (uint64_t x : p->seg_bases[b]) w.val<uint64_t>(x);
  }
  static const char zeros[16] = {0};
  for (auto& b : p->buffers) { w.raw(b.data(), b.size()); w.raw(zeros, (16 - b.size() % 16) % 16); }
  bool ok = w.ok;
  if (fclose(f) != 0) ok = false;
  return ok ? SCION_OK : fail(SCION_ERR_ARG, std::string("write failed: ") + path);
}
int scion_ptree_load(const char* path, scion_ptree** out) {
  if (!path || !out) return fail(SCION_ERR_ARG, "null argument");
  struct Closer { void operator()(FILE* f) const { if (f) fclose(f); } };
  std::unique_ptr<FILE, Closer> file(fopen(path, "rb"));  // closed on every path, exceptions included
  if (!file) return fail(SCION_ERR_ARG, std::string("cannot open ") + path);
  FileR r{file.get()};
  auto bail = [&](const std::string& why) { return fail(SCION_ERR_ARG, std::string(path) + ": " + why); };
  uint64_t file_bytes = 0;
  if (fseek(file.get(), 0, SEEK_END) == 0) { long e = ftell(file.get()); if (e > 0) file_bytes = (uint64_t)e; }
  if (fseek(file.get(), 0, SEEK_SET) != 0) return bail("cannot seek");
  char magic[8];
  r.raw(magic, 8);
  if (!r.ok || memcmp(magic, "SCIONPT1", 8) != 0) return bail("not a scion PhysicalTree container");
  if (r.val<uint32_t>() != 1) return bail("unsupported container version");
  std::string layout = r.str();
  SCION_TRY(
    const scion::LayoutEntry* e = scion::find_layout(layout);
    if (!e) return bail("container names unknown layout '" + layout + "'");
    auto p = std::make_unique<scion_ptree>();
    p->layout = layout;
    p->plan = e->plan.get();
    p->nprims = r.val<uint64_t>();
    p->root0 = r.val<uint64_t>();
    r.raw(p->carried, sizeof(p->carried));
    uint32_t ng = r.val<uint32_t>();
    if (!r.ok || ng != p->plan->globals.size()) return bail("global slot table does not match the layout's plan");
    p->globals.resize(ng);
    for (uint32_t g = 0; g < ng; g++) { if (r.str() != p->plan->globals[g].name) return bail("global slot name mismatch"); r.raw(p->globals[g].data(), 16); }
    uint32_t nb = r.val<uint32_t>();
    if (!r.ok || nb != p->plan->buffers.size()) return bail("buffer table does not match the layout's plan");
    p->buffers.resize(nb); p->counts.resize(nb); p->seg_bases.resize(nb);
    std::vector<uint64_t> sizes(nb);
    uint64_t payload = 0;
    for (uint32_t b = 0; b < nb; b++) {
      if (r.str() != p->plan->buffers[b].name) return bail("buffer name mismatch");
      p->counts[b] = r.val<uint64_t>();
      sizes[b] = r.val<uint64_t>();
      uint32_t ns = r.val<uint32_t>();
      const scion::lc::Buffer& pb = p->plan->buffers[b];
      if (!r.ok || ns != (pb.is_arena ? 1u : (uint32_t)pb.segments.size())) return bail("segment table does not match the layout's plan");
      for (uint32_t s = 0; s < ns; s++) p->seg_bases[b].push_back(r.val<uint64_t>());
      if (!r.ok || sizes[b] > file_bytes || payload + sizes[b] > file_bytes) return bail("buffer sizes exceed the file");  // before any allocation
      payload += sizes[b];
    }
    for (uint32_t b = 0; b < nb; b++) {
      p->buffers[b].resize(sizes[b]);
      r.raw(p->buffers[b].data(), sizes[b]);
      char pad[16];
      r.raw(pad, (16 - sizes[b] % 16) % 16);
    }
    if (!r.ok) return bail("truncated container");
    std::string why;
    if (validate_ptree(*p, why)) return bail(why);
    *out = p.release();
    return SCION_OK;
  )
}
int scion_ptree_corrupt(scion_ptree* p, int buffer, uint64_t byte_offset, uint8_t xor_mask) {
  if (!p || buffer < 0 || buffer >= (int)p->buffers.size() || byte_offset >= p->buffers[(size_t)buffer].size()) return fail(SCION_ERR_ARG, "corrupt: out of range");
  p->buffers[(size_t)buffer][byte_offset] ^= xor_mask;
  return SCION_OK;
}
void scion_ptree_free(scion_ptree* p) { delete p; }

// ------------------------------------------------------------------ device residency
int scion_device_count(int* out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) { if (out) *out = 0; return fail(SCION_ERR_NO_DEVICE, cudaGetErrorString(e)); }
  if (out) *out = n;
  return SCION_OK;
}

static int dtree_create(const scion_ptree* p, int device, bool copy, scion_dtree** out, void* into = nullptr, uint64_t into_bytes = 0) {
  if (!p || !out) return fail(SCION_ERR_ARG, "null argument");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(SCION_ERR_NO_DEVICE, "no CUDA device: the B200 backend has no CPU fallback");
  if (device < 0 || device >= ndev) return fail(SCION_ERR_ARG, "device index out of range");
  const scion::LayoutEntry* e = scion::find_layout(p->layout);
  if (!e) return fail(SCION_ERR_ARG, "unknown layout");
  auto* t = new scion_dtree();
  t->layout = e;
  t->device = device;
  int rc = header_from_ptree(*p, t->header);
  if (rc) { delete t; return rc; }
  // every failure below releases what was acquired so far (scion_dtree_free respects owns_image)
#define CREATE_OK(expr) do { cudaError_t ce__ = (expr); if (ce__ != cudaSuccess) { scion_dtree_free(t); \
    return fail(ce__ == cudaErrorNoDevice || ce__ == cudaErrorInsufficientDriver ? SCION_ERR_NO_DEVICE : SCION_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(ce__)); } } while (0)
  CREATE_OK(cudaSetDevice(device));
  if (into) {
    if (into_bytes < t->header.total_bytes || ((uintptr_t)into & 255u)) { delete t; return fail(SCION_ERR_ARG, "upload_into: buffer too small or not 256-byte aligned"); }
    t->image = (uint8_t*)into;
    t->owns_image = false;
  } else {
    CREATE_OK(cudaMalloc(&t->image, t->header.total_bytes));
  }
  CREATE_OK(cudaMemset(t->image, 0, t->header.total_bytes));
  CREATE_OK(cudaMemcpy(t->image, &t->header, sizeof(ImageHeader), cudaMemcpyHostToDevice));
  if (copy)
    for (size_t b = 0; b < p->buffers.size(); b++)
      if (!p->buffers[b].empty()) CREATE_OK(cudaMemcpy(t->image + t->header.offset[b], p->buffers[b].data(), p->buffers[b].size(), cudaMemcpyHostToDevice));
#undef CREATE_OK
  rc = finish_dtree(t);
  if (rc) { scion_dtree_free(t); return rc; }
  *out = t;
  return SCION_OK;
}
int scion_dtree_upload(const scion_ptree* p, int device, scion_dtree** out) { return dtree_create(p, device, true, out); }
int scion_dtree_upload_into(const scion_ptree* p, int device, void* d_image, uint64_t bytes, scion_dtree** out) {
  if (!d_image) return fail(SCION_ERR_ARG, "null image buffer");
  return dtree_create(p, device, true, out, d_image, bytes);
}
uint64_t scion_ptree_image_bytes(const scion_ptree* p) {
  ImageHeader h;
  if (!p || header_from_ptree(*p, h)) return 0;
  return h.total_bytes;
}
int scion_dtree_alloc_like(const scion_ptree* p, int device, scion_dtree** out) { return dtree_create(p, device, false, out); }

// Device-side encode: the per-node encoders of host/encode_node.hpp run as one
// CUDA thread per node on the uploaded LogicalTree arrays and write the records straight into the
// device image; sizes, globals and the root reference come from the same prepare() as the host path,
// so the image is byte-identical to scion_encode + scion_dtree_upload (tests/test_device_encode.py).
int scion_encode_device(const scion_ltree* t, const char* layout, int device, scion_dtree** out) {
  if (!t || !layout || !out) return fail(SCION_ERR_ARG, "null argument");
  const scion::LayoutEntry* e = nullptr;
  scion_ptree shell;
  scion::enc::EncodeJob job;
  std::vector<uint32_t> post;
  SCION_TRY(e = scion::find_layout(layout); if (!e) return fail(SCION_ERR_ARG, std::string("unknown layout '") + layout + "'");
            if (e->plan->family == scion::lc::Family::Bvh8 && !t->has_wide) return fail(SCION_ERR_BUILD, "8-wide layouts need scion_ltree_collapse8 first");
            scion::encode_shell(*t, *e, shell, job, post);)
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) { cudaGetLastError(); return fail(SCION_ERR_NO_DEVICE, "no CUDA device: this backend has no CPU fallback"); }
  if (device < 0 || device >= ndev) return fail(SCION_ERR_ARG, "device index out of range");
  CUDA_OK(cudaSetDevice(device));
  auto* d = new scion_dtree();
  d->device = device;
  d->layout = e;
  int rc = header_from_ptree(shell, d->header);
  if (rc) { delete d; return rc; }
  std::vector<void*> temps;
  auto bail = [&](int code) { for (void* p : temps) cudaFree(p); scion_dtree_free(d); return code; };
  auto up = [&](const void* src, size_t bytes, const void** dst) -> cudaError_t {
    void* p = nullptr;
    cudaError_t ce = cudaMalloc(&p, bytes ? bytes : 16);
    if (ce != cudaSuccess) return ce;
    temps.push_back(p);
    *dst = p;
    return bytes ? cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice) : cudaSuccess;
  };
#define ENC_OK(x) do { cudaError_t ce__ = (x); if (ce__ != cudaSuccess) return bail(fail(SCION_ERR_CUDA, cudaGetErrorString(ce__))); } while (0)
  ENC_OK(cudaMalloc(&d->image, d->header.total_bytes));
  ENC_OK(cudaMemset(d->image, 0, d->header.total_bytes));
  ENC_OK(cudaMemcpy(d->image, &d->header, sizeof(ImageHeader), cudaMemcpyHostToDevice));
  const scion::lc::Buffer* prim = e->plan->buffer_named("primitives");
  if (!prim) return bail(fail(SCION_ERR_LAYOUT, "layout has no primitives array"));
  if (!t->tris.empty()) ENC_OK(cudaMemcpy(d->image + d->header.offset[prim->id], t->tris.data(), t->tris.size() * 4, cudaMemcpyHostToDevice));
  const void* p = nullptr;
  if (job.kind == scion::enc::kBvh8) {
    ENC_OK(up(t->wnodes.data(), t->wnodes.size() * sizeof(scion_wnode), &p)); job.wnodes = (const scion_wnode*)p;
    ENC_OK(up(t->wleaves.data(), t->wleaves.size() * sizeof(scion_wleaf), &p)); job.wleaves = (const scion_wleaf*)p;
    job.nodes = nullptr;
  } else {
    ENC_OK(up(t->nodes.data(), t->nodes.size() * sizeof(scion_lnode), &p)); job.nodes = (const scion_lnode*)p;
    if (job.kind == scion::enc::kDop14) {
      ENC_OK(up(t->dop_lo2.data(), t->dop_lo2.size() * 4, &p)); job.dop_lo2 = (const float*)p;
      ENC_OK(up(t->dop_hi2.data(), t->dop_hi2.size() * 4, &p)); job.dop_hi2 = (const float*)p;
    }
    if (job.kind == scion::enc::kPbrtPost) { ENC_OK(up(post.data(), post.size() * 4, &p)); job.post = (const uint32_t*)p; }
  }
  for (auto& f : job.f)
    if (f.buffer >= 0) f.base = d->image + d->header.offset[f.buffer];
  if (job.count) {
    scion::encode_nodes_kernel<<<(unsigned)((job.count + 127) / 128), 128>>>(job);
    ENC_OK(cudaGetLastError());
    g_launches.fetch_add(1);
  }
  ENC_OK(cudaDeviceSynchronize());
#undef ENC_OK
  for (void* q : temps) cudaFree(q);
  temps.clear();
  rc = finish_dtree(d);
  if (rc) { scion_dtree_free(d); return rc; }
  *out = d;
  return SCION_OK;
}
int scion_dtree_download_image(const scion_dtree* t, void* h_dst, uint64_t bytes) {
  if (!t || !h_dst) return fail(SCION_ERR_ARG, "null argument");
  if (bytes < t->header.total_bytes) return fail(SCION_ERR_ARG, "destination smaller than the image");
  CUDA_OK(cudaSetDevice(t->device));
  CUDA_OK(cudaMemcpy(h_dst, t->image, t->header.total_bytes, cudaMemcpyDeviceToHost));
  return SCION_OK;
}

int scion_dtree_image(const scion_dtree* t, void** d_ptr, uint64_t* bytes) {
  if (!t) return fail(SCION_ERR_ARG, "null tree");
  if (d_ptr) *d_ptr = t->image;
  if (bytes) *bytes = t->header.total_bytes;
  return SCION_OK;
}
int scion_dtree_from_image(const char* layout, void* d_image, uint64_t bytes, int device, int adopt, scion_dtree** out) {
  if (!d_image || !out || bytes < sizeof(ImageHeader)) return fail(SCION_ERR_ARG, "bad image");
  CUDA_OK(cudaSetDevice(device));
  auto* t = new scion_dtree();
  t->device = device;
  t->image = (uint8_t*)d_image;
  t->owns_image = adopt != 0;
  cudaError_t ce = cudaMemcpy(&t->header, d_image, sizeof(ImageHeader), cudaMemcpyDeviceToHost);
  if (ce != cudaSuccess) { t->owns_image = false; delete t; return fail(SCION_ERR_CUDA, cudaGetErrorString(ce)); }
  if (t->header.magic != kImageMagic || t->header.total_bytes > bytes) { t->owns_image = false; delete t; return fail(SCION_ERR_ARG, "not a scion device image"); }
  {  // the header came from device memory someone else filled: range-check it before fill_view indexes fixed-size arrays
    const ImageHeader& h = t->header;
    bool ok = ((uintptr_t)d_image & 255u) == 0 && h.nbuf >= 1 && h.nbuf <= SCION_MAX_BUFFERS && h.nglob >= 0 && h.nglob <= SCION_MAX_GLOBALS && h.total_bytes >= kHeaderBytes;
    for (int b = 0; ok && b < h.nbuf; b++)
      ok = h.offset[b] >= kHeaderBytes && (h.offset[b] & 255u) == 0 && h.bytes[b] <= h.total_bytes && h.offset[b] <= h.total_bytes - h.bytes[b];
    if (!ok) { t->owns_image = false; delete t; return fail(SCION_ERR_ARG, "corrupt device image header (buffer table out of range, or image not 256-byte aligned)"); }
  }
  t->header.layout[sizeof(t->header.layout) - 1] = 0;
  if (layout && strcmp(layout, t->header.layout) != 0) { t->owns_image = false; delete t; return fail(SCION_ERR_ARG, "image holds a different layout"); }
  t->layout = scion::find_layout(t->header.layout);
  if (!t->layout) { t->owns_image = false; delete t; return fail(SCION_ERR_ARG, "image names an unknown layout"); }
  int rc = finish_dtree(t);
  if (rc) { t->owns_image = false; scion_dtree_free(t); return rc; }  // adoption takes effect on success only
  *out = t;
  return SCION_OK;
}
void scion_dtree_free(scion_dtree* t) {
  if (!t) return;
  cudaSetDevice(t->device);
  for (int i = 0; i < scion_dtree::kSlots; i++) {
    if (t->streams[i]) { cudaStreamSynchronize(t->streams[i]); cudaStreamDestroy(t->streams[i]); }
    if (t->ev_in[i]) cudaEventDestroy(t->ev_in[i]);
    if (t->ev_run[i]) cudaEventDestroy(t->ev_run[i]);
    if (t->ev_out[i]) cudaEventDestroy(t->ev_out[i]);
    if (t->h2d[i]) cudaFree(t->h2d[i]);
    if (t->d2h[i]) cudaFree(t->d2h[i]);
    if (t->pk[i]) cudaFree(t->pk[i]);
    if (t->d_status[i]) cudaFree(t->d_status[i]);
  }
  t->counters.destroy();
  if (t->cd_scratch.ptr) cudaFree(t->cd_scratch.ptr);
  if (t->treelet) cudaFree(t->treelet);
  if (t->image && t->owns_image) cudaFree(t->image);
  delete t;
}

// ------------------------------------------------------------------ queries
static int run_query(const scion_dtree* t, bool hit, const void* in, uint64_t n, void* out, uint32_t* status, scion_counters* counters, int variant, void* stream) {
  if (!t || (!in && n) || (!out && n)) return fail(SCION_ERR_ARG, "null argument");
  if (n == 0) return SCION_OK;
  scion::launch_fn fn = hit ? t->kernels->closest_hit : t->kernels->closest_point;
  if (!fn) return fail(SCION_ERR_ARG, "closest_point requires a binary layout (8-wide layouts have no CPQ, corpus.cpp:83)");
  CUDA_OK(cudaSetDevice(t->device));
  scion::LaunchArgs a;
  a.view = t->view;
  a.in = in;
  a.n = n;
  a.out = out;
  a.status = status;
  a.counters = counters;
  CounterPool& pool = const_cast<scion_dtree*>(t)->counters;
  size_t slot = 0;
  CUDA_OK(pool.take(&slot, &a.next));
  a.stream = (cudaStream_t)stream;
  a.variant = variant;
  a.grid = 0;
  {
    cudaError_t e0 = cudaMemsetAsync(a.next, 0, sizeof(unsigned long long), a.stream);
    if (e0 != cudaSuccess) { pool.release(slot, a.stream, false); CUDA_OK(e0); }
  }
  // Experiment (SCION_L2_PERSIST=1): pin the node buffer in the persisting L2 carve-out.
  static const bool l2_persist = [] { const char* e = getenv("SCION_L2_PERSIST"); return e && e[0] == '1'; }();
  if (l2_persist && t->header.nbuf > 1) {
    static bool limit_set = false;
    if (!limit_set) {
      cudaDeviceProp prop;
      cudaGetDeviceProperties(&prop, t->device);
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prop.persistingL2CacheMaxSize);
      limit_set = true;
    }
    cudaStreamAttrValue attr;
    memset(&attr, 0, sizeof(attr));
    attr.accessPolicyWindow.base_ptr = (void*)t->view.buf[1];
    size_t bytes = t->header.bytes[1];
    int maxw = 0;
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, t->device);
    if (maxw > 0 && bytes > (size_t)maxw) bytes = (size_t)maxw;
    attr.accessPolicyWindow.num_bytes = bytes;
    // hitRatio: the fraction of the window's lines that may persist; window > carve-out with ratio 1 thrashes the carve-out
    static const float ratio = [] { const char* e = getenv("SCION_L2_PERSIST_RATIO"); float r = e ? (float)atof(e) : 1.0f; return r > 0.0f && r <= 1.0f ? r : 1.0f; }();
    attr.accessPolicyWindow.hitRatio = ratio;
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    const cudaError_t pe = cudaStreamSetAttribute(a.stream, cudaStreamAttributeAccessPolicyWindow, &attr);
    static bool told = false;
    if (!told && getenv("SCION_DEBUG")) {
      told = true;
      cudaDeviceProp prop;
      cudaGetDeviceProperties(&prop, t->device);
      fprintf(stderr, "[scion] L2 persistence: window %zu B of %zu B, ratio %.2f, carve-out max %d B, max window %d B, rc %d\n", bytes, (size_t)t->header.bytes[1], ratio,
              prop.persistingL2CacheMaxSize, maxw, (int)pe);
    }
  }
  {
    const cudaError_t e1 = fn(a);
    // the guard event goes behind the memset even if the launch itself failed
    const cudaError_t e2 = pool.release(slot, a.stream, true);
    CUDA_OK(e1);
    CUDA_OK(e2);
  }
  g_launches.fetch_add(1);
  return SCION_OK;
}
int scion_closest_hit(const scion_dtree* t, const scion_ray* d_rays, uint64_t n, scion_hit* d_hits, uint32_t* d_status, scion_counters* d_counters, int variant, void* stream) {
  return run_query(t, true, d_rays, n, d_hits, d_status, d_counters, variant, stream);
}
int scion_closest_point(const scion_dtree* t, const float* d_points, uint64_t n, scion_cp* d_out, uint32_t* d_status, scion_counters* d_counters, int variant, void* stream) {
  return run_query(t, false, d_points, n, d_out, d_status, d_counters, variant, stream);
}

int scion_ray_triangle(const scion_ray* d_rays, const float* d_tris9, uint64_t n, int method, scion_trihit* d_out, void* stream) {
  if ((!d_rays || !d_tris9 || !d_out) && n) return fail(SCION_ERR_ARG, "null argument");
  if (method != SCION_TRI_MT && method != SCION_TRI_PLUECKER) return fail(SCION_ERR_ARG, "unknown triangle test");
  if (n == 0) return SCION_OK;
  scion::ray_triangle_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(d_rays, d_tris9, n, method, d_out);
  CUDA_OK(cudaGetLastError());
  g_launches.fetch_add(1);
  return SCION_OK;
}

int scion_collision_detection(const scion_dtree* a, const scion_dtree* b, scion_pair* d_out, uint64_t capacity, uint64_t* out_count,
                              scion_cd_stats* stats, uint64_t frontier_capacity, void* stream) {
  if (!a || !b || (!d_out && capacity) || !out_count) return fail(SCION_ERR_ARG, "null argument");
  if (a->layout != b->layout) return fail(SCION_ERR_ARG, "collision_detection needs two trees of the same layout");
  if (a->device != b->device) return fail(SCION_ERR_ARG, "collision_detection needs both trees on the same device");
  if (!a->kernels->collide) return fail(SCION_ERR_ARG, "cd requires a binary layout (corpus.cpp:86)");
  CUDA_OK(cudaSetDevice(a->device));
  scion_dtree* owner = const_cast<scion_dtree*>(a);
  std::lock_guard<std::mutex> lock(owner->host_mutex);
  scion::CdArgs args{a->view, b->view, d_out, capacity, frontier_capacity, out_count, stats, (cudaStream_t)stream, &owner->cd_scratch};
  int overflow = 0;
  CUDA_OK(a->kernels->collide(args, &overflow));
  g_launches.fetch_add(1);
  if (overflow) return fail(SCION_ERR_QUERY, "collision_detection: node-pair frontier exceeded its capacity (pass a larger frontier_capacity)");
  return SCION_OK;
}
int scion_collision_detection_host(const scion_dtree* a, const scion_dtree* b, scion_pair* h_out, uint64_t capacity, uint64_t* out_count,
                                   scion_cd_stats* stats) {
  if (!a || (!h_out && capacity) || !out_count) return fail(SCION_ERR_ARG, "null argument");
  CUDA_OK(cudaSetDevice(a->device));
  scion_pair* d = nullptr;
  CUDA_OK(cudaMalloc(&d, (capacity ? capacity : 1) * sizeof(scion_pair)));
  int rc = scion_collision_detection(a, b, d, capacity, out_count, stats, 0, nullptr);
  if (rc == SCION_OK) {
    uint64_t m = *out_count < capacity ? *out_count : capacity;
    cudaError_t e = m ? cudaMemcpy(h_out, d, m * sizeof(scion_pair), cudaMemcpyDeviceToHost) : cudaSuccess;
    if (e != cudaSuccess) rc = fail(SCION_ERR_CUDA, cudaGetErrorString(e));
  }
  cudaFree(d);
  return rc;
}

// Host entry points.  The query array is cut into chunks that flow through three dedicated
// streams — uploads, kernels, downloads — tied together by events, over kSlots staging slots:
//   upload(c)   waits for kernel(c - kSlots)   (its input slot is free again)
//   kernel(c)   waits for upload(c) and download(c - kSlots)   (its output slot is drained)
//   download(c) waits for kernel(c)
// so the H2D copy engine never idles behind a kernel or a D2H copy of its own slot: the call runs at
// the speed of the slowest of the three (on a PCIe Gen5 x16 B200 the 32-byte rays: ~55 GB/s).
}  // extern "C"
namespace scion {
// the reference's packed Ray record (corpus/lib/geometry.scion:4: origin, direction, tmax — 7 x f32, 28 bytes) -> scion_ray
// FLOATS = 7: origin, direction, tmax;  FLOATS = 6: origin, direction with the DSL's default tmax = inf (geometry.scion:4 `tmax = inf`)
template <int FLOATS>
__global__ void unpack_rays_kernel(const float* __restrict__ packed, uint64_t n, scion_ray* __restrict__ rays) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* p = packed + FLOATS * i;
  const float ox = __ldcs(p), oy = __ldcs(p + 1), oz = __ldcs(p + 2), dx = __ldcs(p + 3), dy = __ldcs(p + 4), dz = __ldcs(p + 5);
  const float tmax = FLOATS == 7 ? __ldcs(p + 6) : __uint_as_float(0x7f800000u);
  float4* o = reinterpret_cast<float4*>(rays + i);
  o[0] = make_float4(ox, oy, oz, tmax);
  o[1] = make_float4(dx, dy, dz, 0.0f);
}
}  // namespace scion
extern "C" {
static int run_query_host(const scion_dtree* ct, bool hit, const void* h_in, uint64_t n, void* h_out, uint32_t* h_status, int packed_floats = 0) {
  const bool packed_rays = packed_floats != 0;
  if (!ct || (!h_in && n) || (!h_out && n)) return fail(SCION_ERR_ARG, "null argument");
  scion_dtree* t = const_cast<scion_dtree*>(ct);
  std::lock_guard<std::mutex> lock(t->host_mutex);
  CUDA_OK(cudaSetDevice(t->device));
  const uint64_t in_sz = hit ? (packed_rays ? 4u * (uint64_t)packed_floats : sizeof(scion_ray)) : 12, out_sz = hit ? sizeof(scion_hit) : sizeof(scion_cp);
  // chunk size: an eighth of the call, between 2^17 and 2^23 queries (every chunk kernel pays ~0.5 ms of
  // ramp-up and ragged tail, so small chunks are kernel-bound: 2^28 rays run in 225 / 224 / 185 / 183 ms
  // with 2^20 / 2^21 / 2^22 / 2^23-query chunks; a small call wants its copies overlapped all the same: 2^20 rays of C1
  // run in 0.84 / 0.72 / 0.69 / 0.87 ms with 2^19 / 2^18 / 2^17 / 2^16-query chunks); SCION_HOST_CHUNK_LOG2 overrides
  static const int forced_log2 = [] { const char* e = getenv("SCION_HOST_CHUNK_LOG2"); int l = e ? atoi(e) : 0; return l ? (l < 10 ? 10 : (l > 26 ? 26 : l)) : 0; }();
  uint64_t kChunk = 1ull << 17;
  if (forced_log2) kChunk = 1ull << forced_log2;
  else while (kChunk < (1ull << 23) && kChunk * 8 < n) kChunk <<= 1;
  constexpr int S = scion_dtree::kSlots;
  if (t->chunk < kChunk) {
    t->chunk = 0;  // a failure below must not leave a stale size next to freed / null staging slots
    for (int i = 0; i < S; i++) {
      if (!t->streams[i]) {
        CUDA_OK(cudaStreamCreateWithFlags(&t->streams[i], cudaStreamNonBlocking));
        CUDA_OK(cudaEventCreateWithFlags(&t->ev_in[i], cudaEventDisableTiming));
        CUDA_OK(cudaEventCreateWithFlags(&t->ev_run[i], cudaEventDisableTiming));
        CUDA_OK(cudaEventCreateWithFlags(&t->ev_out[i], cudaEventDisableTiming));
      }
      if (t->h2d[i]) { cudaFree(t->h2d[i]); t->h2d[i] = nullptr; }
      if (t->d2h[i]) { cudaFree(t->d2h[i]); t->d2h[i] = nullptr; }
      if (t->d_status[i]) { cudaFree(t->d_status[i]); t->d_status[i] = nullptr; }
      CUDA_OK(cudaMalloc(&t->h2d[i], kChunk * sizeof(scion_ray)));
      CUDA_OK(cudaMalloc(&t->d2h[i], kChunk * sizeof(scion_cp)));
      CUDA_OK(cudaMalloc(&t->d_status[i], kChunk * sizeof(uint32_t)));
    }
    t->chunk = kChunk;
  }
  if (packed_rays && t->pk_chunk < t->chunk) {  // 28-byte staging of the packed entry point, first use only
    t->pk_chunk = 0;
    for (int i = 0; i < S; i++) {
      if (t->pk[i]) { cudaFree(t->pk[i]); t->pk[i] = nullptr; }
      CUDA_OK(cudaMalloc(&t->pk[i], t->chunk * 28));
    }
    t->pk_chunk = t->chunk;
  }
  // kernels alternate between two streams: the ragged tail of chunk c (a persistent grid drains at the
  // pace of its longest queries) overlaps the head of chunk c + 1
  cudaStream_t s_in = t->streams[0], s_out = t->streams[3];
  // on any failure the four streams are drained before returning: async D2H copies into the caller's
  // h_out / h_status may still be in flight
  auto pipeline = [&]() -> int {
    uint64_t c = 0;
    for (uint64_t off = 0; off < n; off += kChunk, c++) {
      const int k = (int)(c % S);
      cudaStream_t s_run = t->streams[1 + (c & 1)];
      const uint64_t m = std::min(kChunk, n - off);
      if (c >= (uint64_t)S) CUDA_OK(cudaStreamWaitEvent(s_in, t->ev_run[k], 0));
      CUDA_OK(cudaMemcpyAsync(packed_rays ? t->pk[k] : t->h2d[k], (const uint8_t*)h_in + off * in_sz, m * in_sz, cudaMemcpyHostToDevice, s_in));
      CUDA_OK(cudaEventRecord(t->ev_in[k], s_in));
      CUDA_OK(cudaStreamWaitEvent(s_run, t->ev_in[k], 0));
      if (c >= (uint64_t)S) CUDA_OK(cudaStreamWaitEvent(s_run, t->ev_out[k], 0));
      if (packed_rays) {  // 28 -> 32 bytes on the device: ~0.1 ms per 2^23-ray chunk, behind the upload of the next chunk
        if (packed_floats == 7) scion::unpack_rays_kernel<7><<<(unsigned)((m + 255) / 256), 256, 0, s_run>>>((const float*)t->pk[k], m, (scion_ray*)t->h2d[k]);
        else scion::unpack_rays_kernel<6><<<(unsigned)((m + 255) / 256), 256, 0, s_run>>>((const float*)t->pk[k], m, (scion_ray*)t->h2d[k]);
        CUDA_OK(cudaGetLastError());
        g_launches.fetch_add(1);
      }
      int rc = run_query(t, hit, t->h2d[k], m, t->d2h[k], h_status ? t->d_status[k] : nullptr, nullptr, 0, s_run);
      if (rc) return rc;
      CUDA_OK(cudaEventRecord(t->ev_run[k], s_run));
      CUDA_OK(cudaStreamWaitEvent(s_out, t->ev_run[k], 0));
      CUDA_OK(cudaMemcpyAsync((uint8_t*)h_out + off * out_sz, t->d2h[k], m * out_sz, cudaMemcpyDeviceToHost, s_out));
      if (h_status) CUDA_OK(cudaMemcpyAsync(h_status + off, t->d_status[k], m * sizeof(uint32_t), cudaMemcpyDeviceToHost, s_out));
      CUDA_OK(cudaEventRecord(t->ev_out[k], s_out));
    }
    return SCION_OK;
  };
  const int rc = pipeline();
  const std::string why = rc ? g_error : std::string();
  cudaError_t se = cudaSuccess;
  for (int i = 0; i < S; i++) {
    const cudaError_t e = cudaStreamSynchronize(t->streams[i]);
    if (e != cudaSuccess && se == cudaSuccess) se = e;
  }
  if (rc) return fail(rc, why);
  CUDA_OK(se);
  return SCION_OK;
}
int scion_closest_hit_host(const scion_dtree* t, const scion_ray* h_rays, uint64_t n, scion_hit* h_hits, uint32_t* h_status) {
  return run_query_host(t, true, h_rays, n, h_hits, h_status);
}
int scion_closest_hit_host_packed(const scion_dtree* t, const float* h_rays7, uint64_t n, scion_hit* h_hits, uint32_t* h_status) {
  return run_query_host(t, true, h_rays7, n, h_hits, h_status, 7);
}
int scion_closest_hit_host_od(const scion_dtree* t, const float* h_rays6, uint64_t n, scion_hit* h_hits, uint32_t* h_status) {
  return run_query_host(t, true, h_rays6, n, h_hits, h_status, 6);
}
int scion_rays_unpack(const float* d_rays7, uint64_t n, scion_ray* d_rays, void* stream) {
  if ((!d_rays7 || !d_rays) && n) return fail(SCION_ERR_ARG, "null argument");
  if (n == 0) return SCION_OK;
  scion::unpack_rays_kernel<7><<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(d_rays7, n, d_rays);
  CUDA_OK(cudaGetLastError());
  g_launches.fetch_add(1);
  return SCION_OK;
}
int scion_closest_point_host(const scion_dtree* t, const float* h_points, uint64_t n, scion_cp* h_out, uint32_t* h_status) {
  return run_query_host(t, false, h_points, n, h_out, h_status);
}

// ------------------------------------------------------------------ generators
static scion::CameraBasis basis_of(const scion_camera& c) {
  scion::CameraBasis b;
  double f[3], r[3], u[3], up[3] = {c.up[0], c.up[1], c.up[2]};
  for (int a = 0; a < 3; a++) f[a] = (double)c.target[a] - c.eye[a];
  double fl = std::sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
  for (int a = 0; a < 3; a++) f[a] /= fl;
  r[0] = f[1] * up[2] - f[2] * up[1]; r[1] = f[2] * up[0] - f[0] * up[2]; r[2] = f[0] * up[1] - f[1] * up[0];
  double rl = std::sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  for (int a = 0; a < 3; a++) r[a] /= rl;
  u[0] = r[1] * f[2] - r[2] * f[1]; u[1] = r[2] * f[0] - r[0] * f[2]; u[2] = r[0] * f[1] - r[1] * f[0];
  for (int a = 0; a < 3; a++) { b.eye[a] = c.eye[a]; b.fwd[a] = (float)f[a]; b.right[a] = (float)r[a]; b.up[a] = (float)u[a]; }
  double th = std::tan(0.5 * c.fov_y_deg * 3.14159265358979323846 / 180.0);
  b.tan_half_y = (float)th;
  b.tan_half_x = (float)(th * (double)c.width / (double)c.height);
  b.width = c.width;
  b.height = c.height;
  return b;
}
void scion_camera_default(const float lo[3], const float hi[3], int look_down_y, uint32_t w, uint32_t h, scion_camera* out) {
  float c[3], e[3];
  for (int a = 0; a < 3; a++) { c[a] = 0.5f * (lo[a] + hi[a]); e[a] = hi[a] - lo[a]; }
  float diag = std::sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
  for (int a = 0; a < 3; a++) { out->target[a] = c[a]; out->eye[a] = c[a]; }
  if (look_down_y) {  // terrains: above the +y face, looking down at a slant
    out->eye[1] = hi[1] + 0.9f * diag;
    out->eye[2] = hi[2] + 0.35f * diag;
    out->up[0] = 0; out->up[1] = 1; out->up[2] = 0;
  } else {  // outside the +z face
    out->eye[2] = hi[2] + 0.55f * diag;
    out->eye[0] = c[0] + 0.07f * diag;
    out->eye[1] = c[1] + 0.05f * diag;
    out->up[0] = 0; out->up[1] = 1; out->up[2] = 0;
  }
  out->fov_y_deg = 42.0f;
  out->width = w;
  out->height = h;
}

}  // extern "C"

namespace scion {
__global__ void gen_primary_kernel(CameraBasis cam, uint64_t first, uint64_t n, scion_ray* rays) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rays[i] = primary_ray(cam, first + i);
}
__global__ void gen_secondary_kernel(const float* tris, uint64_t ntris, uint64_t seed, uint64_t first, uint64_t n, scion_ray* rays) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rays[i] = secondary_ray(tris, ntris, seed, first + i);
}
__global__ void gen_points_kernel(float3 lo, float3 hi, uint64_t seed, uint64_t first, uint64_t n, float* pts) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    float l[3] = {lo.x, lo.y, lo.z}, h[3] = {hi.x, hi.y, hi.z}, o[3];
    query_point(l, h, seed, first + i, o);
    pts[3 * i] = o[0]; pts[3 * i + 1] = o[1]; pts[3 * i + 2] = o[2];
  }
}
}  // namespace scion

extern "C" {

int scion_gen_primary(const scion_camera* cam, uint64_t first, uint64_t n, scion_ray* d_rays, void* stream) {
  if (!cam || (!d_rays && n)) return fail(SCION_ERR_ARG, "null argument");
  if (n == 0) return SCION_OK;
  scion::gen_primary_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(basis_of(*cam), first, n, d_rays);
  CUDA_OK(cudaGetLastError());
  g_launches.fetch_add(1);
  return SCION_OK;
}
int scion_gen_secondary(const scion_dtree* t, uint64_t seed, uint64_t first, uint64_t n, scion_ray* d_rays, void* stream) {
  if (!t || (!d_rays && n)) return fail(SCION_ERR_ARG, "null argument");
  if (n == 0) return SCION_OK;
  CUDA_OK(cudaSetDevice(t->device));
  // buffer 0 is the primitives array in every layout of the registry (Triangle stride 36, 4-byte aligned)
  scion::gen_secondary_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>((const float*)t->view.buf[0], t->header.nprims, seed, first, n, d_rays);
  CUDA_OK(cudaGetLastError());
  g_launches.fetch_add(1);
  return SCION_OK;
}
int scion_gen_points(const float lo[3], const float hi[3], uint64_t seed, uint64_t first, uint64_t n, float* d_points, void* stream) {
  if (!lo || !hi || (!d_points && n)) return fail(SCION_ERR_ARG, "null argument");
  if (n == 0) return SCION_OK;
  scion::gen_points_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(make_float3(lo[0], lo[1], lo[2]), make_float3(hi[0], hi[1], hi[2]), seed, first, n, d_points);
  CUDA_OK(cudaGetLastError());
  g_launches.fetch_add(1);
  return SCION_OK;
}
int scion_gen_primary_host(const scion_camera* cam, uint64_t first, uint64_t n, scion_ray* h_rays) {
  if (!cam || (!h_rays && n)) return fail(SCION_ERR_ARG, "null argument");
  scion::CameraBasis b = basis_of(*cam);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; i++) h_rays[i] = scion::primary_ray(b, first + (uint64_t)i);
  return SCION_OK;
}
int scion_gen_secondary_host(const float* tris9, uint64_t ntris, uint64_t seed, uint64_t first, uint64_t n, scion_ray* h_rays) {
  if (!tris9 || !ntris || (!h_rays && n)) return fail(SCION_ERR_ARG, "null argument");
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; i++) h_rays[i] = scion::secondary_ray(tris9, ntris, seed, first + (uint64_t)i);
  return SCION_OK;
}
int scion_gen_points_host(const float lo[3], const float hi[3], uint64_t seed, uint64_t first, uint64_t n, float* h_points) {
  if (!lo || !hi || (!h_points && n)) return fail(SCION_ERR_ARG, "null argument");
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; i++) scion::query_point(lo, hi, seed, first + (uint64_t)i, h_points + 3 * i);
  return SCION_OK;
}

void scion_partition(uint64_t n, int rank, int nranks, uint64_t* first, uint64_t* count) {
  if (nranks < 1) nranks = 1;
  uint64_t a = n * (uint64_t)rank / (uint64_t)nranks, b = n * (uint64_t)(rank + 1) / (uint64_t)nranks;
  if (first) *first = a;
  if (count) *count = b - a;
}

}  // extern "C"
