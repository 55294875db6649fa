/*
 * scion_b200.h — C ABI of the B200-native traversal backend for Scion BVH layouts.
 *
 * This is the drop-in boundary for ONE path of the reference (arxiv 2511.15028,
 * `layoutc`): executing closest-hit ray/triangle and closest-point queries over
 * a PhysicalTree whose node layout was chosen by a Scion layout specification.
 *
 * The reference ships no header for its exec layer (include/layoutc/ has no
 * interp/harness/scene/emit header; src/interp.cpp, src/emit_c.cpp,
 * src/build_physical.cpp, src/scene.cpp, src/logical.cpp, src/rng.cpp and
 * src/harness.cpp are placeholders).  Every entry point below therefore cites the
 * SPEC.md contract (and, where one exists, the reference header) it stands in for.
 *
 * Conventions
 *   - every function returns int: 0 = SCION_OK, otherwise a scion_status code;
 *     nothing throws across the boundary; scion_last_error() gives the message
 *     of the calling thread's last failure.
 *   - plain pointers and sizes only; no torch / STL types.
 *   - "d_" pointers are device pointers on the tree's device, "h_" pointers are
 *     host pointers.  Device launches are asynchronous on the given stream
 *     (cudaStream_t passed as void*; NULL = the legacy default stream).
 *   - a scion_dtree is immutable after creation: concurrent launches on
 *     different streams are legal.
 */
#ifndef SCION_B200_H
#define SCION_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCION_ABI_VERSION 1

typedef enum scion_status {
  SCION_OK = 0,
  SCION_ERR_ARG = 1,       /* bad argument / unknown name (CLI exit code 2 class)  */
  SCION_ERR_LAYOUT = 2,    /* layout spec rejected (PlanError class, plan.hpp:89)              */
  SCION_ERR_BUILD = 3,     /* builder hard fault: count/emit disagreement, capacity */
  SCION_ERR_CUDA = 4,      /* CUDA runtime failure                                              */
  SCION_ERR_NO_DEVICE = 5, /* no CUDA device: the product path has NO CPU fallback              */
  SCION_ERR_QUERY = 6      /* at least one query reported an error status        */
} scion_status;

/* per-query status word (overflow / OOB are query errors, never silent) */
#define SCION_Q_OK 0u
#define SCION_Q_STACK_OVERFLOW 1u

/* layout families — /root/reference/proj/include/layoutc/corpus.hpp:11 (enum Family) */
#define SCION_FAMILY_BVH2 0
#define SCION_FAMILY_DOP14 1
#define SCION_FAMILY_BVH8 2

#define SCION_MISS_PRIM 0xFFFFFFFFu
#define SCION_STACK_DEPTH 64 /* specialize.hpp:57 CompileOptions::stack_depth */

/* ------------------------------------------------------------------------- */
/* Query / result records                                                     */
/* ------------------------------------------------------------------------- */

/* Ray(origin, direction, tmax = inf) — corpus/lib/geometry.scion:4, padded to 32 B
 * so that one ray is two 16-byte vector loads. */
typedef struct scion_ray {
  float ox, oy, oz, tmax;
  float dx, dy, dz, pad;
} scion_ray;

/* closest_hit's `best: mut (f32, Triangle)` (corpus/alg/chrt.scion:2): the triangle
 * is reported as its index in the tree-ordered primitives array.  Miss:
 * t = +inf, prim = SCION_MISS_PRIM. */
typedef struct scion_hit {
  float t;
  uint32_t prim;
} scion_hit;

/* closest_point's `best: mut (f32, Point)` (corpus/alg/cpq.scion:3) plus the chosen
 * primitive (harness contract "identical chosen primitive").
 * prim = SCION_MISS_PRIM when d2 was only ever tightened by the farthest-corner
 * bound and no primitive improved it. */
typedef struct scion_cp {
  float d2;
  float x, y, z;
  uint32_t prim;
} scion_cp;

typedef struct scion_counters { /* interpreter cost counters */
  uint32_t node_visits; /* node decodes (CPQ: incl. the two child peeks per interior; 8-wide: interiors only) */
  uint32_t prim_tests;  /* triangle tests */
  uint32_t cold_loads;  /* reads of segments behind `---` (dop14 diagonals, pbrt-soa topology) */
  uint32_t max_stack;   /* peak occupancy of the 64-entry explicit stack */
} scion_counters;

/* ------------------------------------------------------------------------- */
/* Logical tree interchange (what oracle and GPU both consume)                */
/* ------------------------------------------------------------------------- */

/* Binary LogicalTree node, nodes stored in preorder. */
typedef struct scion_lnode {
  float lo[3], hi[3];
  int32_t left, right;  /* node indices, or -1/-1 for a Leaf */
  uint32_t first_prim;  /* Leaf: first triangle in the tree-ordered array */
  uint32_t nprims;      /* Leaf: count (>0); Interior: 0 */
} scion_lnode;

/* 8-wide LogicalTree interior (collapse_to_wide). Children are
 * left-packed; unused slots are SENTINELs with an inverted box (lo=+inf, hi=-inf). */
#define SCION_W_SENTINEL INT32_MIN
typedef struct scion_wnode {
  float lo[8][3], hi[8][3];
  int32_t child[8]; /* >=0: interior index; <0 (and != SENTINEL): leaf id = ~child */
} scion_wnode;

typedef struct scion_wleaf {
  uint32_t first_prim, nprims;
} scion_wleaf;

typedef struct scion_scene scion_scene; /* triangle soup                          */
typedef struct scion_ltree scion_ltree; /* LogicalTree (binary, optional 8-wide)  */
typedef struct scion_ptree scion_ptree; /* PhysicalTree on the host */
typedef struct scion_dtree scion_dtree; /* PhysicalTree resident on one device    */

const char* scion_last_error(void);
int scion_abi_version(void);

/* ------------------------------------------------------------------------- */
/* Layout registry — replaces corpus_layouts()/find_corpus_layout(),          */
/* /root/reference/proj/src/corpus.cpp:9-34, and plan_layout()/footprint(),   */
/* /root/reference/proj/include/layoutc/plan.hpp:94, :110                     */
/* ------------------------------------------------------------------------- */
typedef struct scion_layout_info {
  const char* name;        /* CLI-facing name, same strings as corpus.cpp:11-25 */
  int family;              /* SCION_FAMILY_*                                    */
  int arity;               /* 2 or 8                                            */
  uint32_t node_stride;    /* node bytes = sum of segment strides (plan.cpp:327) */
  uint32_t node_align;
  uint32_t n_segments;
  uint32_t ref_bits;       /* width of the primary reference component          */
  uint32_t max_leaf;       /* capacity of the nprims field                      */
  int has_cpq;             /* closest_point available (binary families only, corpus.cpp:83) */
} scion_layout_info;

int scion_layout_count(void);
int scion_layout_info_at(int index, scion_layout_info* out);
int scion_layout_find(const char* name, scion_layout_info* out);
/* JSON dump of the MemoryPlan (buffers, segments, slots @bit offset:width), the
 * counterpart of the `footprint` report. Caller frees with scion_free. */
int scion_layout_plan_json(const char* name, char** out_json);
/* emit_cuda: the CUDA sibling of emit_c — deterministic text. */
int scion_layout_emit_cuda(const char* name, char** out_text);
/* emit_c, record half ("packed record declarations matching MemoryPlan strides bit-for-bit ... a
 * static assertion on node size"): a C11 header with the typed packed node records, their assertions and the slot table. */
int scion_layout_emit_c(const char* name, char** out_text);
/* op-count report of the layout's decode, per variant (the CLI's --dump-stats): JSON. */
int scion_layout_stats_json(const char* name, char** out_json);
/* Compile a layout spec from source text (layout-language subset of the
 * reference grammar, src/parser.cpp:790-955) and return plan JSON / CUDA text. */
int scion_compile_layout_text(const char* scion_source, char** out_plan_json, char** out_cuda);
/* Open-world layouts (constructor + destructor specialisation at run time): compile a layout the
 * library was not built with and register it under `name`.  The text goes through the front end (SCION_ERR_LAYOUT with
 * the reference's diagnostic classes when it is ill-formed), emit_cuda produces its header (decode, typed records, the
 * constructors of its build block), nvcc instantiates every traversal kernel for it with the library's own flags, and
 * the plugin is loaded into the process.  Afterwards scion_encode (through the layout's build block), scion_dtree_upload,
 * scion_ptree_from_buffers, scion_closest_hit / _point, scion_collision_detection accept the name like a built-in's.
 * Needs nvcc (SCION_NVCC, default /usr/local/cuda/bin/nvcc) and the library's device sources (SCION_B200_SRC, default
 * csrc/ next to the library) at run time; 10-25 s.  work_dir: where the sources and the plugin are kept (null: a fresh
 * directory under $TMPDIR); a plugin found there that was compiled from the same text with the same compiler, flags and
 * library is reused without compiling.  *out_log (nullable, scion_free) receives the build log. */
int scion_layout_register(const char* name, const char* scion_text, const char* work_dir, char** out_log);
/* layouts registered at run time, in registration order (scion_layout_count / _info_at enumerate the built-in registry,
 * i.e. the corpus of corpus_layouts(); scion_layout_find resolves both) */
int scion_layout_registered_count(void);
int scion_layout_registered_at(int index, scion_layout_info* out);
void scion_free(void* p);

/* ------------------------------------------------------------------------- */
/* Scene tools — stand in for src/scene.cpp, src/logical.cpp */
/* ------------------------------------------------------------------------- */
int scion_scene_terrain(uint32_t grid, uint64_t seed, scion_scene** out);  /* 2*grid^2 triangles */
int scion_scene_sphere(uint32_t grid, uint64_t seed, scion_scene** out);   /* 2*grid^2 triangles */
int scion_scene_cloud(uint64_t npoints, uint64_t seed, scion_scene** out); /* degenerate triangles p0=p1=p2 */
int scion_scene_from_triangles(const float* xyz9, uint64_t ntris, scion_scene** out);
uint64_t scion_scene_ntris(const scion_scene* s);
const float* scion_scene_triangles(const scion_scene* s); /* 9 floats per triangle */
void scion_scene_bounds(const scion_scene* s, float lo[3], float hi[3]);
void scion_scene_free(scion_scene* s);

/* build_sah: binned SAH, `bins` bins, C_trav = C_isect = 1, ties ->
 * lowest axis then lowest bin, coincident centroids -> index halves. Depth is capped at
 * max_depth (<= 64) by switching to median splits.  build_median: SPEC.md:556-561. */
int scion_build_sah(const scion_scene* s, uint32_t bins, uint32_t max_leaf, uint32_t max_depth,
                    scion_ltree** out);
int scion_build_median(const scion_scene* s, uint32_t max_leaf, scion_ltree** out);
/* Import an externally built binary LogicalTree (the reference's `build-tree` artefact):
 * any node order, root = node 0, leaves reference ranges of tris9.  The tree is re-flattened to
 * preorder with primitives in left-first leaf order; bounds are taken as given.  No depth cap:
 * trees deeper than the 64-entry stack make queries report SCION_Q_STACK_OVERFLOW. */
int scion_ltree_from_arrays(const scion_lnode* nodes, uint64_t nnodes, const float* tris9, uint64_t ntris, scion_ltree** out);
/* collapse_to_wide; idempotent, result cached inside the ltree. */
int scion_ltree_collapse8(scion_ltree* t);

uint64_t scion_ltree_nnodes(const scion_ltree* t);
const scion_lnode* scion_ltree_nodes(const scion_ltree* t);
uint64_t scion_ltree_nprims(const scion_ltree* t);
const float* scion_ltree_triangles(const scion_ltree* t);     /* tree order, 9 floats each */
const uint32_t* scion_ltree_prim_ids(const scion_ltree* t);   /* tree order -> scene index */
const float* scion_ltree_dop_lo2(const scion_ltree* t);       /* 4 floats per node (DOP-14 diagonals) */
const float* scion_ltree_dop_hi2(const scion_ltree* t);
uint32_t scion_ltree_depth(const scion_ltree* t);
uint64_t scion_ltree_nwnodes(const scion_ltree* t);
const scion_wnode* scion_ltree_wnodes(const scion_ltree* t);
uint64_t scion_ltree_nwleaves(const scion_ltree* t);
const scion_wleaf* scion_ltree_wleaves(const scion_ltree* t);
int32_t scion_ltree_wroot(const scion_ltree* t); /* child-style code of the 8-wide root */
void scion_ltree_free(scion_ltree* t);

/* ------------------------------------------------------------------------- */
/* build_physical: LogicalTree -> byte buffers + globals + root ref */
/* ------------------------------------------------------------------------- */
int scion_encode(const scion_ltree* t, const char* layout, scion_ptree** out);
/* The same through the layout's own `build` block (constructor specialisation):
 * the layout compiler turns the block into per-variant constructors (gen/<layout>.cuh build_<Variant>()) that run a
 * count pass + a recursive emit pass on the host.  scion_encode is the fast path (hand-restated per family, OpenMP or
 * device-side); the two must produce byte-identical trees (tests/test_generated_build.py).  SCION_ERR_BUILD when the
 * layout file carries no build block (scion_layout_has_build) or on a build fault (count / emit disagreement). */
int scion_encode_generated(const scion_ltree* t, const char* layout, scion_ptree** out);
int scion_layout_has_build(const char* layout);
const char* scion_ptree_layout(const scion_ptree* p);
int scion_ptree_nbuffers(const scion_ptree* p);
int scion_ptree_buffer(const scion_ptree* p, int i, const char** name, const uint8_t** data,
                       uint64_t* bytes, uint64_t* count);
/* segment base byte offsets of buffer i (plan.cpp:333-347); returns the count written */
int scion_ptree_segment_bases(const scion_ptree* p, int i, uint64_t* bases, int max);
int scion_ptree_nglobals(const scion_ptree* p);
/* global slot: name + raw little-endian bits (up to 16 bytes: f32x3 / f32x4 / u64) */
int scion_ptree_global(const scion_ptree* p, int i, const char** name, uint8_t raw[16], uint32_t* nbytes);
/* root reference: component 0 as u64, tree-carried components as raw floats */
int scion_ptree_root(const scion_ptree* p, uint64_t* ref0, float* carried6);
uint64_t scion_ptree_total_bytes(const scion_ptree* p); /* footprint().total_bytes */
uint64_t scion_ptree_node_bytes(const scion_ptree* p);  /* all buffers except primitives */
/* PhysicalTree container file ("versioned container file = header (magic, version, layout
 * name, global slots) + raw little-endian buffers"; read by the `run` subcommand) */
int scion_ptree_save(const scion_ptree* p, const char* path);
int scion_ptree_load(const char* path, scion_ptree** out);
/* In-memory import of a PhysicalTree produced by another build_physical (one descriptor per
 * BufferDesc / GlobalDesc of the MemoryPlan, /root/reference/proj/include/layoutc/plan.hpp:31-48).  Descriptors
 * are matched by name, in any order; the library copies, the caller keeps ownership.  Sizes are validated against
 * the plan (buffer bytes == footprint() for the stated count, /root/reference/proj/src/plan.cpp:333-347; segment
 * bases; root reference inside the node group); anything else is SCION_ERR_ARG, never a silent upload. */
typedef struct scion_buffer_desc {
  const char* name;          /* plan buffer name: "primitives", "nodes", "Interiors", "node" (arena) ... */
  const void* data;
  uint64_t bytes;
  uint64_t count;            /* elements (arena: nodes allocated in it; not checked against the bytes) */
  const uint64_t* seg_bases; /* nullable: byte offset of every segment; must equal the plan's if given */
  uint32_t n_seg_bases;
} scion_buffer_desc;
typedef struct scion_global_desc {
  const char* name;          /* plan global slot name: "world_low", "N", "__ref_plo" ... */
  uint8_t raw[16];           /* little-endian bits, zero padded */
} scion_global_desc;
typedef struct scion_tree_desc {
  const char* layout;
  const scion_buffer_desc* buffers;
  uint32_t nbuffers;
  const scion_global_desc* globals;
  uint32_t nglobals;
  uint64_t root_ref;         /* primary component of the root reference */
  float carried[6];          /* tree-carried components (shared-slab: plo, phi), else zeros */
  uint64_t nprims;           /* 0 = take the primitives buffer's count */
} scion_tree_desc;
int scion_ptree_from_buffers(const scion_tree_desc* desc, scion_ptree** out);
/* import + upload in one call (the host descriptor stays the caller's) */
int scion_tree_upload(const scion_tree_desc* host, int device, scion_dtree** out);
/* fault injection for verify tests: xor one byte of a buffer */
int scion_ptree_corrupt(scion_ptree* p, int buffer, uint64_t byte_offset, uint8_t xor_mask);
void scion_ptree_free(scion_ptree* p);

/* ------------------------------------------------------------------------- */
/* Device residency                                                           */
/* ------------------------------------------------------------------------- */
int scion_device_count(int* out);
/* host -> device copy of every buffer (the library owns the device memory) */
int scion_dtree_upload(const scion_ptree* p, int device, scion_dtree** out);
/* allocate an empty device tree with p's shapes (for receiving a broadcast) */
int scion_dtree_alloc_like(const scion_ptree* p, int device, scion_dtree** out);
/* bytes of the packed device image of p (header + 256-byte aligned buffers + slack) */
uint64_t scion_ptree_image_bytes(const scion_ptree* p);
/* upload INTO caller-owned device memory (>= scion_ptree_image_bytes, 256-byte aligned), e.g. a
 * torch tensor that is then replicated with ncclBroadcast; the caller keeps ownership */
int scion_dtree_upload_into(const scion_ptree* p, int device, void* d_image, uint64_t bytes, scion_dtree** out);
/* Packed wire image used for replication: [header | globals | buffers...] in ONE
 * contiguous device allocation so that a single ncclBroadcast replicates the tree. */
int scion_dtree_image(const scion_dtree* t, void** d_ptr, uint64_t* bytes);
/* Copy the whole device image (header + buffers, scion_dtree_image bytes) to host memory. */
int scion_dtree_download_image(const scion_dtree* t, void* h_dst, uint64_t bytes);
/* Device-side build_physical (SPEC.md:276-284 constructor specialisation): the
 * LogicalTree arrays are uploaded once and every node record is encoded by one CUDA thread; the
 * resulting image is byte-identical to scion_encode + scion_dtree_upload.  Same builder faults
 * (SCION_ERR_BUILD) as scion_encode; SCION_ERR_NO_DEVICE without a GPU. */
int scion_encode_device(const scion_ltree* t, const char* layout, int device, scion_dtree** out);
/* rebuild a device tree around a received image (no copy; image owned by caller unless adopt=1; on failure the
 * image always stays the caller's).  The image must be 256-byte aligned. */
int scion_dtree_from_image(const char* layout, void* d_image, uint64_t bytes, int device, int adopt,
                           scion_dtree** out);
void scion_dtree_free(scion_dtree* t);

/* ------------------------------------------------------------------------- */
/* Queries — stand in for interpret(program, tree, "closest_hit"|"closest_point", args)
 * specialised per layout at build time by emit_cuda.        */
/* ------------------------------------------------------------------------- */
/* variant: 0 = default (tuned) kernel; other values select documented experimental
 * kernel variants that must produce identical results. */
int scion_closest_hit(const scion_dtree* t, const scion_ray* d_rays, uint64_t n, scion_hit* d_hits,
                      uint32_t* d_status /* nullable */, scion_counters* d_counters /* nullable */,
                      int variant, void* stream);
int scion_closest_point(const scion_dtree* t, const float* d_points_xyz, uint64_t n, scion_cp* d_out,
                        uint32_t* d_status, scion_counters* d_counters, int variant, void* stream);
/* collision_detection(bvh1, bvh2, r: mut set[(Triangle, Triangle)]) — corpus/alg/cd.scion:2-31,
 * cd_dop14.scion (binary layouts only, corpus.cpp:86).  Both trees must use the same layout and live on the
 * same device (the same tree twice = self-collision).  The result is a SET: up to `capacity` pairs
 * (primitive index in tree a, primitive index in tree b) are written to d_out in unspecified order and
 * *out_count receives the true set size (> capacity means the caller must retry with a larger buffer).
 * Synchronous (level-synchronous frontier expansion).  Frontier exhaustion is an error, never silent. */
typedef struct scion_pair {
  uint32_t a, b;
} scion_pair;
typedef struct scion_cd_stats {
  uint64_t node_pairs; /* node pairs tested (= recursive calls of the DSL) */
  uint64_t tri_tests;  /* SAT tests */
  uint64_t levels;
  uint64_t max_frontier;
} scion_cd_stats;
int scion_collision_detection(const scion_dtree* a, const scion_dtree* b, scion_pair* d_out, uint64_t capacity, uint64_t* out_count,
                              scion_cd_stats* stats /* nullable */, uint64_t frontier_capacity /* 0 = default 2^24 */, void* stream);
/* host-buffer form: pairs copied back (D2H) */
int scion_collision_detection_host(const scion_dtree* a, const scion_dtree* b, scion_pair* h_out, uint64_t capacity, uint64_t* out_count,
                                   scion_cd_stats* stats);
/* Batch ray/triangle primitive test: pair i = (d_rays[i], d_tris9[9*i .. 9*i+8]).  method 0 = Moeller-Trumbore
 * (geometry.scion:25-38, the test every traversal uses), 1 = Pluecker coordinates (geometry.scion:40-55; never
 * selected by the corpus dispatcher :57-59 — exposed for the Appendix F fidelity check, SPEC acceptance 9). */
typedef struct scion_trihit {
  float b0, b1, b2, t; /* TriangleIntersection (geometry.scion:9); zeros on a miss */
  uint32_t hit;
} scion_trihit;
#define SCION_TRI_MT 0
#define SCION_TRI_PLUECKER 1
int scion_ray_triangle(const scion_ray* d_rays, const float* d_tris9, uint64_t n, int method, scion_trihit* d_out, void* stream);
/* Host-buffer entry points (the reference-facing call: host in, host out). H2D copy,
 * kernel, D2H copy, stream sync; chunked + double-buffered over two streams. */
int scion_closest_hit_host(const scion_dtree* t, const scion_ray* h_rays, uint64_t n, scion_hit* h_hits,
                           uint32_t* h_status /* nullable */);
int scion_closest_point_host(const scion_dtree* t, const float* h_points_xyz, uint64_t n, scion_cp* h_out,
                             uint32_t* h_status);
/* The same call for rays in the reference's own packed record — Ray(origin, direction, tmax), 7 x f32 = 224 bits
 * (corpus/lib/geometry.scion:4, packed sum of members: src/sema.cpp:47-87) — i.e. exactly what an array of the DSL's
 * Ray values is on the host.  28 instead of 32 bytes cross the PCIe link per ray (the call is H2D-bound); the rays are
 * widened to scion_ray on the device (scion_rays_unpack, also usable on its own for device-resident packed rays). */
int scion_closest_hit_host_packed(const scion_dtree* t, const float* h_rays7, uint64_t n, scion_hit* h_hits,
                                  uint32_t* h_status /* nullable */);
int scion_rays_unpack(const float* d_rays7, uint64_t n, scion_ray* d_rays, void* stream);
/* ... and for rays that carry the DSL's default tmax (`Ray(origin, direction)`: tmax = inf, geometry.scion:4): origin and
 * direction only, 6 x f32 = 24 bytes per ray — with this form the call is no longer bound by the PCIe link on C5 */
int scion_closest_hit_host_od(const scion_dtree* t, const float* h_rays6, uint64_t n, scion_hit* h_hits,
                              uint32_t* h_status /* nullable */);

/* ------------------------------------------------------------------------- */
/* Query generators (src/rng.cpp placeholder): every query is
 * a pure function of (seed, global index) so any rank count sees identical inputs. */
/* ------------------------------------------------------------------------- */
typedef struct scion_camera {
  float eye[3];
  float target[3];
  float up[3];
  float fov_y_deg;
  uint32_t width, height;
} scion_camera;
/* default pinhole camera looking at the bounds (outside the +z face; +y for terrains) */
void scion_camera_default(const float lo[3], const float hi[3], int look_down_y, uint32_t w, uint32_t h,
                          scion_camera* out);
int scion_gen_primary(const scion_camera* cam, uint64_t first, uint64_t n, scion_ray* d_rays, void* stream);
/* secondary: origin = uniform point on a hash-chosen triangle + eps*normal, direction =
 * uniform hemisphere about the geometric normal */
int scion_gen_secondary(const scion_dtree* t, uint64_t seed, uint64_t first, uint64_t n, scion_ray* d_rays,
                        void* stream);
int scion_gen_points(const float lo[3], const float hi[3], uint64_t seed, uint64_t first, uint64_t n,
                     float* d_points_xyz, void* stream);
/* host twins of the generators (bit-identical results), used by CPU callers and tests */
int scion_gen_primary_host(const scion_camera* cam, uint64_t first, uint64_t n, scion_ray* h_rays);
int scion_gen_secondary_host(const float* tris9, uint64_t ntris, uint64_t seed, uint64_t first, uint64_t n,
                             scion_ray* h_rays);
int scion_gen_points_host(const float lo[3], const float hi[3], uint64_t seed, uint64_t first, uint64_t n,
                          float* h_points_xyz);

/* contiguous query partition for rank r of nranks: [first, first+count) */
void scion_partition(uint64_t n, int rank, int nranks, uint64_t* first, uint64_t* count);

/* ------------------------------------------------------------------------- */
/* Multi-GPU (SPEC.md:416 concurrent queries on a shared immutable tree; :645 "the query loop may fan out across
 * workers ... reports are merged deterministically by query index").  The tree is replicated with ONE
 * ncclBroadcast of its packed image, queries are partitioned contiguously (scion_partition), results are gathered
 * by query index; no collective runs inside a traversal launch.  NCCL is bound at run time (libnccl.so.2 of the
 * process): without it these calls return SCION_ERR_ARG and everything else keeps working. */
/* ------------------------------------------------------------------------- */
#define SCION_NCCL_UNIQUE_ID_BYTES 128
typedef struct scion_comm scion_comm; /* one NCCL communicator bound to one device */
int scion_nccl_version(int* out);
/* one process per GPU: rank 0 creates the id, ships it to the others out of band, every rank calls init_rank */
int scion_comm_unique_id(uint8_t id[SCION_NCCL_UNIQUE_ID_BYTES]);
int scion_comm_init_rank(const uint8_t id[SCION_NCCL_UNIQUE_ID_BYTES], int nranks, int rank, int device, scion_comm** out);
/* one process, ndev GPUs (ncclCommInitAll): fills out[0..ndev); devices NULL = 0..ndev-1 */
int scion_comm_init_all(int ndev, const int* devices, scion_comm** out);
/* wrap a communicator the caller created (an ncclComm_t of the same libnccl instance); never destroyed by us */
int scion_comm_adopt(void* nccl_comm, scion_comm** out);
int scion_comm_rank(const scion_comm* c);
int scion_comm_size(const scion_comm* c);
int scion_comm_device(const scion_comm* c);
void scion_comm_free(scion_comm* c);
/* Replicate a resident tree.  Exactly the root rank passes its tree (others NULL); every rank returns with a tree on
 * its communicator's device (*out == root_tree on the root).  Collective: all ranks must call. */
int scion_dtree_broadcast(scion_dtree* root_tree, int root, scion_comm* comm, void* stream, scion_dtree** out);
/* single-process form over the array of scion_comm_init_all: out[root] = root_tree, the others are created */
int scion_dtree_broadcast_all(scion_dtree* root_tree, int root, scion_comm* const* comms, int n, void* const* streams, scion_dtree** out);
/* Gather result records by query index: this rank's d_part holds the records of scion_partition(n_total, rank,
 * nranks); d_full (n_total records, may contain d_part at its own offset) receives all of them on every rank. */
int scion_gather_results(scion_comm* comm, const void* d_part, uint64_t n_total, uint32_t record_bytes, void* d_full, void* stream);
int scion_gather_results_all(scion_comm* const* comms, int n, const void* const* d_parts, uint64_t n_total, uint32_t record_bytes,
                             void* const* d_fulls, void* const* streams);

/* number of product kernels launched by this process so far (bench `gpu_launches`) */
uint64_t scion_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* SCION_B200_H */
