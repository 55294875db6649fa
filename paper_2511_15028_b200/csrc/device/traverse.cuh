// Traversal kernels, one query per thread, templated over the emitted layout struct
// (gen/<layout>.cuh).  They restate, in explicit-stack form (LIFO, children
// pushed in reverse visit order, overflow = query error):
//   closest_hit, binary   /root/reference/proj/corpus/alg/chrt.scion:2-17
//   closest_hit, DOP-14   /root/reference/proj/corpus/alg/chrt_dop14.scion:3-18
//   closest_hit, 8-wide   /root/reference/proj/corpus/alg/chrt8.scion:3-21
//   closest_point         /root/reference/proj/corpus/alg/cpq.scion:3-33, cpq_dop14.scion:2-31
// The visit ORDER is the reference's (left first, slot order, near child first with ties to the
// right child), because hit ids are only bit-exact when pruning sees the same `best` at the same
// moment.
//
// Execution model (justified by profiles/r1_ncu_v1_c5_q16.txt: the first, one-warp-32-rays kernel
// ran at 6.2 of 32 active threads per instruction, its triangle loop at 1 of 32; evolution v1..v9 in
// DESIGN.md §5):
//   * persistent warps; every LANE is refilled with a new query once enough lanes have retired
//     (ballot + prefix popcount over a warp-private chunk of the global work counter);
//   * per-lane state machine — FETCH, NODE, PRIM — so that lanes in the same state execute the same
//     instructions: a NODE step decodes and tests one node and pushes / pops on one predicated
//     straight-line path; leaf ranges are parked and resolved by all 32 lanes together once enough
//     lanes wait (cooperative PRIM phase), which batches the rare Moeller-Trumbore evaluations;
//   * state that only the PRIM / retire paths need (ray direction, query index, leaf range) lives in
//     shared memory, so the NODE step runs in 56 registers (9 CTAs/SM).
// Stack: LaneStack below — first entries in shared memory laid out [entry][word][thread] (lane l
// always hits bank l, so any mix of per-lane depths is conflict free) and addressed by one register,
// deeper entries in local memory.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>

#include "geometry.cuh"
#include "scion_b200.h"

namespace scion {

#ifndef SCION_MINB2
#define SCION_MINB2 9   /* 56 registers, 36 warps/SM: +7 % over the compiler's own 61-63 (8 blocks); 10 blocks (48 regs) spills and halves throughput */
#endif
#ifndef SCION_CHUNK
#define SCION_CHUNK 128
#endif
#ifndef SCION_STACK_SMEM
// Shared memory and L1 share 256 KB per SM: at 9 CTAs/SM a 16 KB window leaves ~60 KB of L1, 12 KB
// ~92 KB, 8 KB ~124 KB.  Measured (C5 probe, pbrt-q16, kernel v7): 20 KB 1265, 16 KB 2106, 12 KB
// 2178, 10 KB 2183, 8 KB 2176, 6 KB 1979, 4 KB 1747 Mrays/s (small windows send pushes to local memory).
#define SCION_STACK_SMEM (12 * 1024)
#endif
#ifndef SCION_BLOCK_THREADS
#define SCION_BLOCK_THREADS 128
#endif
constexpr int kBlockThreads = SCION_BLOCK_THREADS;
constexpr unsigned kFullMask = 0xffffffffu;
constexpr int kChunk = SCION_CHUNK;     // queries a warp takes from the global counter at a time
#ifndef SCION_STREAM_HITS
#define SCION_STREAM_HITS 1
#endif
#ifndef SCION_GUIDED_CHUNKS
#define SCION_GUIDED_CHUNKS 1
#endif
#ifndef SCION_GUIDED_NUM  /* switch to 32-query chunks when fewer than NUM/DEN full chunks per warp remain */
#define SCION_GUIDED_NUM 2ull
#define SCION_GUIDED_DEN 1ull
#endif
#ifndef SCION_REFILL_MIN
#define SCION_REFILL_MIN 4
#endif
#ifndef SCION_PRIM_MIN
#define SCION_PRIM_MIN 6
#endif
constexpr int kRefillMin = SCION_REFILL_MIN;   // refill when at least this many lanes are idle (or all of them)
constexpr int kPrimMin = SCION_PRIM_MIN;       // run the PRIM phase when at least this many lanes wait in it

constexpr int kStackSmemBytesPerBlock = SCION_STACK_SMEM;  // shared-memory share of the per-lane stacks of one CTA (LaneStack below)

template <bool COUNT>
struct Tally {
  uint32_t node_visits = 0, prim_tests = 0, cold_loads = 0, max_stack = 0;
  SCION_DEV void reset() { node_visits = prim_tests = cold_loads = max_stack = 0; }
  SCION_DEV void visit() { if (COUNT) node_visits++; }
  SCION_DEV void prim() { if (COUNT) prim_tests++; }
  SCION_DEV void cold(uint32_t k = 1) { if (COUNT) cold_loads += k; }
  SCION_DEV void stack(uint32_t occ) { if (COUNT) max_stack = occ > max_stack ? occ : max_stack; }
  SCION_DEV void store(scion_counters* out, uint64_t q) const {
    if (COUNT && out) out[q] = scion_counters{node_visits, prim_tests, cold_loads, max_stack};
  }
};

// Warp-private window on the global work counter.  All 32 lanes call refill(); lanes that pass
// want=true and for which work is left get a query index.  All members are warp-uniform.
template <bool GUIDED>
struct WorkFetcherT {
  unsigned long long chunk_base = 0;
  unsigned chunk_left = 0;
  bool exhausted = false;
  SCION_DEV bool refill(bool want, unsigned long long* next, uint64_t n, uint64_t& q) {
    const unsigned lane = threadIdx.x & 31u;
    const unsigned lt = (1u << lane) - 1u;
    bool got = false;
    unsigned idle = __ballot_sync(kFullMask, want);
    while (idle) {
      if (chunk_left == 0) {
        if (exhausted) break;
        // guided chunk size: full chunks while plenty of work is left, 32-query chunks once fewer than two full
        // chunks per warp of the grid remain — small launches (2^16 rays: 212 -> ~60 us) and the ragged tail of
        // big ones no longer leave three quarters of the warps without work
        unsigned long long base = 0;
        unsigned take = (unsigned)kChunk;
        if (lane == 0) {
#if SCION_GUIDED_CHUNKS
          if (GUIDED) {
#if SCION_GUIDED_CHUNKS == 2
          const unsigned long long seen = *reinterpret_cast<volatile unsigned long long*>(next);
#else
          const unsigned long long seen = chunk_base;  // end of this warp's previous chunk: a lower bound of the global progress, no extra load
#endif
          const unsigned long long rem = seen < n ? n - seen : 0ull;
          if (rem * SCION_GUIDED_DEN < (unsigned long long)gridDim.x * (blockDim.x >> 5) * SCION_GUIDED_NUM * (unsigned long long)kChunk) take = 32u;
          }
#endif
          base = atomicAdd(next, (unsigned long long)take);
        }
        base = __shfl_sync(kFullMask, base, 0);
        take = __shfl_sync(kFullMask, take, 0);
        if (base >= n) { exhausted = true; break; }
        chunk_base = base;
        chunk_left = (unsigned)(n - base < (uint64_t)take ? n - base : (uint64_t)take);
      }
      const unsigned rank = __popc(idle & lt);
      if (want && !got && rank < chunk_left) { q = chunk_base + rank; got = true; }
      const unsigned cnt = __popc(idle);
      const unsigned taken = cnt < chunk_left ? cnt : chunk_left;
      chunk_base += taken;
      chunk_left -= taken;
      idle = __ballot_sync(kFullMask, want && !got);
    }
    return got;
  }
};
using WorkFetcher = WorkFetcherT<true>;        // closest_hit kernels
// closest_point keeps fixed 128-query chunks: with the guided rule C4 drops from 1246 to 1134 Mq/s (measured twice,
// with and without the extra counter load; the cause is in the generated code, not in the policy)
using WorkFetcherFixed = WorkFetcherT<false>;

// results are written once and never read by the kernel: streaming store (evict-first), so that 2 GB of hit
// records do not displace node records in L2
SCION_DEV void store_hit(scion_hit* dst, float t, uint32_t prim) {
#if SCION_STREAM_HITS
  __stcs(reinterpret_cast<float2*>(dst), make_float2(t, __uint_as_float(prim)));
#else
  *dst = scion_hit{t, prim};
#endif
}
SCION_DEV RayCtx load_ray(const scion_ray* rays, uint64_t q) {
  const float4* p = reinterpret_cast<const float4*>(rays + q);
  const float4 a = __ldcs(p), b = __ldcs(p + 1);  // streaming: read once
  return make_ray(a.x, a.y, a.z, a.w, b.x, b.y, b.z);
}

// bounds test of one binary / DOP node against the ray.  Loads the cold segment only when the
// reference semantics would evaluate it (dop.scion:20-21 `if I {...}`).
template <class L, class TallyT>
SCION_DEV bool node_test(const TreeView& T, const RayCtx& ray, const typename L::Ref& ref, typename L::Node& n, float& t_near, TallyT& tally) {
  float t_far;
  // kBoundsCold: the box itself lies (partly) behind `---` (pbrt-soaos-align16), so the cold segment is part of every visit
  constexpr bool kEager = L::kHasCold && L::kBoundsCold;
  if constexpr (kEager) L::decode_cold(T, ref, n);
  if constexpr (L::kFamily == SCION_FAMILY_DOP14) {
    bool some = ray_aabb(ray, n.lo1, n.hi1, t_near, t_far);
    if (some) {
      if constexpr (!kEager) L::decode_cold(T, ref, n);
      tally.cold();
      some = dop_diagonals(ray, n.lo2, n.hi2, t_near, t_far);
    }
    return interval_intersects(ray, some, t_near, t_far);
  } else {
    const bool some = ray_aabb(ray, n.low, n.high, t_near, t_far);
    const bool hit = interval_intersects(ray, some, t_near, t_far);
    if constexpr (L::kHasCold) {
      if (hit || L::kBoundsCold) {
        if constexpr (!kEager) L::decode_cold(T, ref, n);
        tally.cold();
      }
    }
    return hit;
  }
}

enum : int { kFetch = 0, kNode = 1, kPrim = 2 };  // lane modes (3 = kPop of the closest-point kernel)
#ifndef SCION_PREFETCH
#define SCION_PREFETCH 1
#endif
#ifndef SCION_CPQ_GUIDED  /* 1: closest_point uses the guided (128 -> 32 query) work-fetch chunks of the closest-hit kernels */
#define SCION_CPQ_GUIDED 0
#endif
#ifndef SCION_INNER
#define SCION_INNER 4
#endif
#ifndef SCION_DUMMY_LD
#define SCION_DUMMY_LD 0
#endif
#ifndef SCION_PF_TRI
#define SCION_PF_TRI 0
#endif
#ifndef SCION_PF8
#define SCION_PF8 0
#endif
#ifndef SCION_CPQ_BOTH
#define SCION_CPQ_BOTH -1  // -1: per layout (records fetched by ONE vector load), 0: never, 1: always
#endif
constexpr bool kPrefetch = SCION_PREFETCH != 0;  // L2-prefetch a node record when its reference is pushed (+3-4 % on C5, binary)
constexpr int kInner = SCION_INNER;  // node steps between two looks at the warp (idle lanes to refill, lanes waiting with a leaf)

// L2 prefetch of a parked leaf's triangles (SCION_PF_TRI: 1 = the line of the first triangle, 2 = first and last
// line): the cooperative leaf phase runs a few steps after the lane parks, the prefetch covers that gap.
template <class L>
SCION_DEV void prefetch_triangles(const TreeView& T, uint32_t begin, uint32_t end) {
#if SCION_PF_TRI > 0
  const uint8_t* p = T.buf[L::kBuf_primitives] + (uint64_t)begin * 36ull;
  prefetch_to<2>(p);
#if SCION_PF_TRI > 1
  prefetch_to<2>(p + (uint64_t)(end - begin) * 36ull - 1ull);
#endif
#else
  (void)T; (void)begin; (void)end;
#endif
}

// keeps the result-store address arithmetic inside the (rare) retire branch instead of letting the
// compiler hoist it into every loop iteration (9 SASS instructions per iteration in v3)
SCION_DEV uint64_t opaque(uint64_t q) {
  asm volatile("" : "+l"(q));
  return q;
}

// ------------------------------------------------------------------------------------------
// Lane-private LIFO addressed by ONE register (kernel v6).  `top` is the shared-space byte address
// of the slot the next push writes: window + 4*tid + depth*kSlot; word w of an entry lives at
// +w*4*kBlockThreads, so every 32-bit access of a warp hits 32 different banks whatever the mix of
// depths.  Depth tests compare (top - window) with constants (4*tid < kSlot), so neither the depth
// nor the thread's base address occupies a register.  Entries beyond the shared-memory share go
// to a local array (rare: the window holds the first 32 references of a 4-byte-reference layout).
// ------------------------------------------------------------------------------------------
template <class Entry, int kWindowBytes = kStackSmemBytesPerBlock, int BT = kBlockThreads>
struct LaneStack {
  static_assert(sizeof(Entry) % 4 == 0, "stack entries are stored as 32-bit words");
  static constexpr int kWords = (int)sizeof(Entry) / 4;
  static constexpr uint32_t kSlot = (uint32_t)BT * 4u * (uint32_t)kWords;
  static constexpr int kFit = (int)((uint32_t)kWindowBytes / kSlot);
  static constexpr int kSmem = kFit < SCION_STACK_DEPTH ? kFit : SCION_STACK_DEPTH;
  static_assert(kSmem >= 1, "the shared-memory window must hold at least one entry per thread");
  static constexpr int kDeep = SCION_STACK_DEPTH - kSmem > 0 ? SCION_STACK_DEPTH - kSmem : 1;
  static constexpr uint32_t kSmemBytes = (uint32_t)kSmem * kSlot;

  SCION_DEV static void store(uint32_t a, const Entry& e) {
    uint32_t w[kWords];
    memcpy(w, &e, sizeof(Entry));
#pragma unroll
    for (int i = 0; i < kWords; i++) asm volatile("st.shared.b32 [%0], %1;" ::"r"(a + (uint32_t)(i * 4 * BT)), "r"(w[i]));
  }
  SCION_DEV static void load(uint32_t a, Entry& e) {
    uint32_t w[kWords];
#pragma unroll
    for (int i = 0; i < kWords; i++) asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w[i]) : "r"(a + (uint32_t)(i * 4 * BT)));
    memcpy(&e, w, sizeof(Entry));
  }
};

// Warp-cooperative leaf phase, v6.  Same contract as coop_triangles (owners fold the results of
// their own range in ascending primitive order with the strict `t < best` rule = the sequential
// foreach of chrt.scion:10-15), cheaper bookkeeping: an owner publishes only the FIRST slot of its
// run (one byte store) and the OR of the start bits (one REDUX); a worker finds its run with one
// FLO over the start mask.  The owner's direction comes from the per-thread stash in shared
// memory (it is not needed by the node phase, so it does not occupy registers there).
struct CoopScratch2 {
  float t[32];
  uint8_t owner[32];
};
struct alignas(16) RayStash {
  float dx, dy, dz;
  uint32_t pad;
};
template <class L>
SCION_DEV uint32_t coop_triangles2(const TreeView& T, bool own, float ox, float oy, float oz, float tmax, const RayStash* __restrict__ warp_stash,
                                   uint32_t& prim_i, uint32_t prim_end, float& best_t, uint32_t& best_prim, CoopScratch2& sc) {
  static_assert(L::kStride_primitives == 36, "Triangle stride");
  const unsigned lane = threadIdx.x & 31u;
  uint32_t tested = 0;
  for (;;) {
    const uint32_t remaining = own ? prim_end - prim_i : 0u;
    if (__ballot_sync(kFullMask, remaining != 0u) == 0u) break;
    const uint32_t c = remaining < 32u ? remaining : 32u;
    uint32_t incl = c;  // inclusive prefix sum over lanes
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_up_sync(kFullMask, incl, d);
      if (lane >= (unsigned)d) incl += v;
    }
    const uint32_t excl = incl - c;
    const bool starts_run = c != 0u && excl < 32u;
    const uint32_t take = starts_run ? (c < 32u - excl ? c : 32u - excl) : 0u;
    if (starts_run) sc.owner[excl] = (uint8_t)lane;
    const unsigned starts = __reduce_or_sync(kFullMask, starts_run ? (1u << excl) : 0u);
    const uint32_t total = __shfl_sync(kFullMask, incl, 31);
    __syncwarp();
    const bool work = lane < total;  // total may exceed 32; lanes are 0..31
    // the run that covers slot `lane` starts at the highest start bit at or below it
    const unsigned below = starts & (0xffffffffu >> (31u - lane));
    const unsigned first = 31u - (unsigned)__clz((int)(below | 1u));
    const unsigned o = sc.owner[first];
    const uint32_t kk = lane - first;
    RayCtx r;
    r.ox = __shfl_sync(kFullMask, ox, o);
    r.oy = __shfl_sync(kFullMask, oy, o);
    r.oz = __shfl_sync(kFullMask, oz, o);
    r.tmax = __shfl_sync(kFullMask, tmax, o);
    const uint32_t pi = __shfl_sync(kFullMask, prim_i, o) + kk;
    float t = scion::inf();
    if (work) {
      const RayStash d = warp_stash[o];
      r.dx = d.dx; r.dy = d.dy; r.dz = d.dz;
      float tri[9];
      load_triangle36(T.buf[L::kBuf_primitives], pi, tri);
      float th;
      if (ray_tri_mt(r, tri, th)) t = th;
    }
    sc.t[lane] = t;
    __syncwarp();
    for (uint32_t k = 0; k < take; k++) {
      const float th = sc.t[excl + k];
      if (th < best_t) {  // a miss is +inf and never passes
        best_t = th;
        best_prim = prim_i + k;
      }
    }
    prim_i += take;
    tested += take;
    __syncwarp();
  }
  return tested;
}

// SCION_LEAF_NOINLINE (experiment): the cooperative leaf phase as an out-of-line function with by-value arguments and
// results, so that its ~35 live registers (triangle, Moeller-Trumbore temporaries) no longer count towards the register
// allocation of the node step: the step's state is saved around the CALL only, and the kernel can be bounded to fewer
// registers / more CTAs per SM (SCION_MINB2) without spilling inside the step.
#ifndef SCION_LEAF_NOINLINE
#define SCION_LEAF_NOINLINE 0
#endif
struct LeafOut {
  float best_t;
  uint32_t best_prim, tested;
};
template <class L>
__device__ __noinline__ LeafOut coop_triangles2_call(const uint8_t* prims, bool own, float ox, float oy, float oz, float tmax, const RayStash* warp_stash, uint32_t prim_i,
                                                     uint32_t prim_end, float best_t, uint32_t best_prim, CoopScratch2* sc) {
  TreeView T;
  T.buf[L::kBuf_primitives] = prims;
  const uint32_t tested = coop_triangles2<L>(T, own, ox, oy, oz, tmax, warp_stash, prim_i, prim_end, best_t, best_prim, *sc);
  return LeafOut{best_t, best_prim, tested};
}

// ------------------------------------------------------------------------------------------
// closest_hit, binary + DOP-14 families (kernel v6)
//
// Per-lane state machine.  A *step* (lanes in kNode) is: decode one node -> bounds test ->
// interior hit: push right, continue with left | leaf hit: park the primitive range (kPrim) |
// otherwise pop the next pending reference.  Push and pop are predicated STS / LDS on ONE
// straight-line path; in v5 they were two divergent branches that each ran at ~12/32 lanes
// (profiles/r1_ncu_v5_c5_q16.txt).  Retiring a query, entries beyond the shared-memory window
// and overflow share one rarely taken branch.
// kInner steps run back to back; only then does the warp look for idle lanes (refill) and for
// lanes waiting with a leaf (cooperative PRIM phase).
//
// TL > 0 (kernel variant 2, north_star "stage the BVH's top levels into shared memory with TMA bulk copies"): the top TL
// levels of the tree — a side treelet in heap order built once per tree by build_treelet_kernel (treelet.cuh): slot s
// holds the record of one node and its index in the main array, its children sit in slots 2s+1 / 2s+2 — are copied
// into shared memory with ONE cp.async.bulk per CTA (mbarrier completion; SASS UBLKCP) and visits of those nodes are
// served by LDS instead of a global load.  A reference with bit 31 set designates a treelet slot; the children of a
// slot in the last staged level are ordinary main-array references (the "escape").  The visit order, every decode
// and every test are unchanged (the records are byte copies), so results and counters are identical.
// The treelet is a cache, not part of the layout: it is not counted in bytes/prim.
// BT / WIN / MINB: CTA size, shared-memory stack window and CTAs per SM — a treelet is staged once per CTA, so the
// staged variant runs larger CTAs than the default 128 threads (see launch_hit_t).
// ------------------------------------------------------------------------------------------
template <class L>
inline constexpr bool kTreeletOk = L::kCanFetch && !L::kHasCold && L::kFamily == SCION_FAMILY_BVH2 && std::is_same<typename L::Ref, uint32_t>::value;
template <class L>
constexpr bool treelet_ok() {
  return kTreeletOk<L>;
}
constexpr uint32_t kTreeletBit = 0x80000000u;
template <class L, bool COUNT, int TL = 0, int BT = kBlockThreads, int WIN = kStackSmemBytesPerBlock, int MINB = SCION_MINB2>
__global__ void __launch_bounds__(BT, MINB) chrt2_kernel(const TreeView T, const scion_ray* __restrict__ rays, uint64_t n,
                                                              scion_hit* __restrict__ hits, uint32_t* __restrict__ status,
                                                              scion_counters* __restrict__ counters, unsigned long long* __restrict__ next, const int tune) {
  using Ref = typename L::Ref;
  using LS = LaneStack<Ref, WIN, BT>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr uint32_t kTlSlots = TL > 0 ? (1u << TL) - 1u : 0u;
  uint32_t tl_rec = 0, tl_orig = 0;  // shared-space addresses of the staged records / main-array indices
  bool tl_on = false;
  if constexpr (TL > 0) {
    static_assert(kTreeletOk<L>, "the treelet needs single-vector-load records and 32-bit index references");
    __shared__ __align__(8) unsigned long long mbar;
    constexpr uint32_t kRecBytes = kTlSlots * L::kStageStride;
    constexpr uint32_t kBytes = (kRecBytes + kTlSlots * 4u + 15u) & ~15u;
    tl_rec = (uint32_t)__cvta_generic_to_shared(smem_raw + WIN);
    tl_on = T.treelet != nullptr && T.treelet_slots == kTlSlots;
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (tl_on) {
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(kBytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(tl_rec), "l"(T.treelet), "r"(kBytes), "r"(mb)
                     : "memory");
      }
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(mb), "r"(0u) : "memory");
    }
  }
  __shared__ CoopScratch2 coop[BT / 32];
  __shared__ RayStash stash[BT];          // ray direction: only the leaf phase needs it
  __shared__ unsigned long long stash_q[BT];  // query index: only the retire path needs it
  __shared__ uint2 stash_leaf[BT];        // parked primitive range [begin, end)
  Ref deep[LS::kDeep];
  uint32_t window = (uint32_t)__cvta_generic_to_shared(smem_raw);
  asm volatile("" : "+r"(window));  // opaque: kept in a register instead of being re-derived (S2R CgaCtaId + 3) at every push and pop
  uint32_t top = window + threadIdx.x * 4u;
  if constexpr (TL > 0) {  // addresses of the staged treelet as constant offsets from the register that holds `window`
    tl_rec = window + (uint32_t)WIN;
    tl_orig = tl_rec + kTlSlots * (uint32_t)L::kStageStride;
  }
  uint32_t my_leaf = (uint32_t)__cvta_generic_to_shared(&stash_leaf[threadIdx.x]);
  asm volatile("" : "+r"(my_leaf));  // one register; re-deriving the address costs 7 instructions in a divergent branch
  WorkFetcher work;
  (void)tune;
  Tally<COUNT> tally;
  int mode = kFetch;
  RayCtx ray = make_ray(0, 0, 0, 0, 1, 1, 1);
  float best_t = 0;
  uint32_t best_prim = 0;
  Ref cur = L::root(T);

  auto retire = [&](uint32_t st) {
    const uint64_t qq = opaque(stash_q[threadIdx.x]);
    store_hit(hits + qq, best_t, best_prim);
    if (status) status[qq] = st;
    tally.store(counters, qq);
    mode = kFetch;
  };

  // next pending reference, or retire the query when the stack is empty (used after a leaf phase
  // and on the rare paths of step())
  auto pop_or_retire = [&]() {
    const uint32_t rel = top - window;  // depth * kSlot + 4 * tid, 4 * tid < kSlot
    if (rel - LS::kSlot < LS::kSmemBytes) {  // 1 <= depth <= kSmem: the entry is in shared memory
      top -= LS::kSlot;
      LS::load(top, cur);
      mode = kNode;
    } else if (rel < LS::kSlot) {  // empty: the query is done
      retire(SCION_Q_OK);
    } else {
      top -= LS::kSlot;
      cur = deep[rel / LS::kSlot - 1u - (uint32_t)LS::kSmem];
      mode = kNode;
    }
  };

  const Ref root = [&]() -> Ref {
    if constexpr (TL > 0) return tl_on ? (Ref)kTreeletBit : L::root(T);  // slot 0 of the treelet is the root
    else return L::root(T);
  }();
  auto step = [&]() {
    typename L::Node node;
    if constexpr (TL > 0) {
      typename L::Fetched w;
      const bool in_t = ((uint32_t)cur & kTreeletBit) != 0u;
      const uint32_t slot = (uint32_t)cur & ~kTreeletBit;
      Ref idx = cur;
      if (in_t) {
        constexpr int NW = (int)(sizeof(typename L::Fetched) / 4);
        const uint32_t a = tl_rec + slot * (uint32_t)L::kStageStride;  // tl_rec = window + WIN: one IMAD off the register that holds `window`
#pragma unroll
        for (int i = 0; i < NW; i += 4)
          asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(w.w[i]), "=r"(w.w[i + 1]), "=r"(w.w[i + 2]), "=r"(w.w[i + 3]) : "r"(a + 4u * (uint32_t)i));
        uint32_t o;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(o) : "r"(tl_orig + slot * 4u));
        idx = (Ref)o;
      } else {
        L::fetch(T, idx, w);
      }
      L::decode_fetched(T, idx, w, node);
      const uint32_t c = 2u * slot + 1u;
      if (in_t && c + 1u < kTlSlots) {  // both children are staged too (an interior node always has both)
        node.left = (Ref)(kTreeletBit | c);
        node.right = (Ref)(kTreeletBit | (c + 1u));
      }
    } else {
      L::decode(T, cur, node);
    }
#if SCION_DUMMY_LD  // diagnostic: N extra loads of the record's own first word (an L1 hit on the sector just requested, nobody waits for them)
    if constexpr (L::kCanStage && std::is_integral<Ref>::value) {
      const uint8_t* a__ = T.buf[L::kStageBuffer] + (uint64_t)cur * L::kStageStride;
#pragma unroll
      for (int i__ = 0; i__ < SCION_DUMMY_LD; i__++) {
        uint32_t d__;
        asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(d__) : "l"(a__ + 4 * i__));
      }
    }
#endif
    tally.visit();
    float t_near;
    const bool hit = node_test<L>(T, ray, cur, node, t_near, tally);
    const bool leaf = node.variant == L::kLeaf;
    const bool p_prim = hit && leaf && (uint32_t)node.data.begin < (uint32_t)node.data.end;
    const bool p_push = hit && !leaf && t_near < best_t;
    const uint32_t rel = top - window;
    // the common push (depth < kSmem) and pop (1 <= depth <= kSmem) are straight-line predicated
    // code; everything else (empty stack = retire, entries beyond the shared-memory window,
    // overflow) is one rarely taken branch
    const bool fast = p_push ? rel < LS::kSmemBytes : rel - LS::kSlot < LS::kSmemBytes;
    if (COUNT && p_push) tally.stack(rel / LS::kSlot + 2u);  // reference discipline: pop self, push right, push left
    if (!(fast || p_prim)) {
      if (p_push) {
        const uint32_t depth = rel / LS::kSlot;
        if (depth + 2u > (uint32_t)SCION_STACK_DEPTH) {
          retire(SCION_Q_STACK_OVERFLOW);
        } else {
          deep[depth - (uint32_t)LS::kSmem] = node.right;
          top += LS::kSlot;
          cur = node.left;
        }
      } else {
        pop_or_retire();
      }
      return;
    }
    if (p_prim) {  // park the primitive range (shared memory: the leaf phase reads it, the step keeps no register for it)
      asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(my_leaf), "r"((uint32_t)node.data.begin), "r"((uint32_t)node.data.end));
      prefetch_triangles<L>(T, (uint32_t)node.data.begin, (uint32_t)node.data.end);
      mode = kPrim;
    } else if (p_push) {
      LS::store(top, node.right);
      if constexpr (kPrefetch) {
        // L2-prefetch the pushed child (+4 %; gating it by distance loses 3-7 %: even a sibling four records away profits)
        if constexpr (TL > 0) {
          if (((uint32_t)node.right & kTreeletBit) == 0u) L::prefetch(T, node.right);  // staged children need no prefetch
        } else {
          L::prefetch(T, node.right);
        }
      }
      top += LS::kSlot;
      cur = node.left;
    } else {
      top -= LS::kSlot;
      LS::load(top, cur);
    }
  };

  for (;;) {
    // ---- NODE: kInner steps per lane without looking at the rest of the warp
#pragma unroll 1
    for (int k = 0; k < kInner; k++) {
      if (mode == kNode) step();
    }
    // ---- FETCH: refill idle lanes
    const unsigned idle = __ballot_sync(kFullMask, mode == kFetch);
    if (idle && (__popc(idle) >= kRefillMin || work.exhausted)) {
      uint64_t nq;
      if (!work.exhausted && work.refill(mode == kFetch, next, n, nq)) {
        ray = load_ray(rays, nq);
        stash[threadIdx.x] = RayStash{ray.dx, ray.dy, ray.dz, 0u};
        stash_q[threadIdx.x] = nq;
        best_t = scion::inf();
        best_prim = SCION_MISS_PRIM;
        tally.reset();
        top = window + threadIdx.x * 4u;
        cur = root;
        mode = kNode;
      }
      if (work.exhausted && __ballot_sync(kFullMask, mode != kFetch) == 0u) break;
    }
    // ---- PRIM: all 32 lanes test the parked (owner, triangle) pairs
    const unsigned pmask = __ballot_sync(kFullMask, mode == kPrim);
    if (pmask && (__popc(pmask) >= kPrimMin || __ballot_sync(kFullMask, mode == kNode) == 0u)) {
      const bool own = mode == kPrim;
      uint2 range = make_uint2(0u, 0u);
      if (own) asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(range.x), "=r"(range.y) : "r"(my_leaf));
      uint32_t prim_i = range.x;
#if SCION_LEAF_NOINLINE
      const LeafOut lo_ = coop_triangles2_call<L>(T.buf[L::kBuf_primitives], own, ray.ox, ray.oy, ray.oz, ray.tmax, stash + (threadIdx.x & ~31u), prim_i, range.y, best_t,
                                                  best_prim, &coop[threadIdx.x >> 5]);
      best_t = lo_.best_t;
      best_prim = lo_.best_prim;
      const uint32_t done = lo_.tested;
#else
      const uint32_t done = coop_triangles2<L>(T, own, ray.ox, ray.oy, ray.oz, ray.tmax, stash + (threadIdx.x & ~31u), prim_i, range.y, best_t,
                                               best_prim, coop[threadIdx.x >> 5]);
#endif
      if (COUNT) tally.prim_tests += done;
      if (own) pop_or_retire();
    }
  }
}


// ------------------------------------------------------------------------------------------
// closest_hit, 8-wide family.  Stack entries are (child reference, t_near); the cull
// `t_near < best` is re-applied at pop time, which is result-equivalent to the reference's
// in-loop test because t_near is a pure function of (ray, box).
// ------------------------------------------------------------------------------------------
template <class Ref>
struct WideEntry {
  Ref ref;
  float t_near;
};

#ifndef SCION_MINB8
#define SCION_MINB8 4
#endif
#ifndef SCION_STACK_SMEM8
// 4 CTAs/SM (124 registers) leave shared memory to spare, and the entries are 8 bytes (16 with 64-bit
// references).  C5 probe, bvh8 / bvh8-q16 (64-bit references): 12 KB 1433 / 1391, 16 KB 1494 / 1451,
// 24 KB 1531 / 1493, 32 KB 1529 / 1491 Mrays/s; the -ci layouts (32-bit references) do not care.
#define SCION_STACK_SMEM8 (24 * 1024)
#endif
constexpr int kStackSmemBytesPerBlock8 = SCION_STACK_SMEM8;
#ifndef SCION_INNER8
#define SCION_INNER8 1
#endif
#ifndef SCION_PRIM_MIN8
#define SCION_PRIM_MIN8 6
#endif
#ifndef SCION_REFILL_MIN8
#define SCION_REFILL_MIN8 4
#endif
// 8-wide kernel v7.  Same lane state machine as chrt2_kernel with three differences that follow from
// the shape of an 8-wide visit (one ~500-instruction interior step instead of ~100):
//   * a step only ever decodes INTERIOR records: where the variant is encoded in the reference
//     (every 8-wide layout of the corpus, L::kVariantInRef) a leaf reference is recognised when it is
//     popped and the lane parks its primitive range at once, instead of spending a whole step slot on it;
//   * the first passing child is continued with directly (registers); only the other passing children
//     are stored, at their final positions, so that they pop in slot order (chrt8.scion:7);
//   * the warp looks for idle / parked lanes after every step (SCION_INNER8 = 1): a waiting lane costs
//     1/32 of a 500-instruction step.
template <class L, bool COUNT>
__global__ void __launch_bounds__(kBlockThreads, SCION_MINB8) chrt8_kernel(const TreeView T, const scion_ray* __restrict__ rays, uint64_t n,
                                                              scion_hit* __restrict__ hits, uint32_t* __restrict__ status,
                                                              scion_counters* __restrict__ counters, unsigned long long* __restrict__ next, const int tune) {
  using Ref = typename L::Ref;
  using Entry = WideEntry<Ref>;
  using LS = LaneStack<Entry, kStackSmemBytesPerBlock8>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ CoopScratch2 coop[kBlockThreads / 32];
  __shared__ RayStash stash[kBlockThreads];
  __shared__ unsigned long long stash_q[kBlockThreads];
  Entry deep[LS::kDeep];
  uint32_t window = (uint32_t)__cvta_generic_to_shared(smem_raw);
  asm volatile("" : "+r"(window));
  uint32_t top = window + threadIdx.x * 4u;
  WorkFetcher work;
  (void)tune;
  Tally<COUNT> tally;
  int mode = kFetch;
  RayCtx ray = make_ray(0, 0, 0, 0, 1, 1, 1);
  float best_t = 0;
  uint32_t best_prim = 0, prim_i = 0, prim_end = 0;
  Ref cur = L::root(T);

  auto retire = [&](uint32_t st) {
    const uint64_t qq = opaque(stash_q[threadIdx.x]);
    store_hit(hits + qq, best_t, best_prim);
    if (status) status[qq] = st;
    tally.store(counters, qq);
    mode = kFetch;
  };
  // `cur` was just chosen: park it if the reference itself says it is a leaf
  auto enter = [&]() {
    mode = kNode;
    if constexpr (L::kVariantInRef) {
      if (L::ref_variant(cur) == L::kLeaf) {
        typename L::Node leaf;
        L::decode(T, cur, leaf);  // reference-only arm: no memory access
        prim_i = (uint32_t)leaf.data.begin;
        prim_end = (uint32_t)leaf.data.end;
        if (prim_i < prim_end) {
          mode = kPrim;
          prefetch_triangles<L>(T, prim_i, prim_end);
        } else {
          mode = -1;  // empty leaf: nothing to do, take the next entry
        }
      }
    }
  };
  // next pending entry whose deferred cull `t_near < best` still passes, or retire
  auto pop_next = [&]() {
    for (;;) {
      const uint32_t rel = top - window;
      Entry e;
      if (rel - LS::kSlot < LS::kSmemBytes) {
        top -= LS::kSlot;
        LS::load(top, e);
      } else if (rel < LS::kSlot) {
        retire(SCION_Q_OK);
        return;
      } else {
        top -= LS::kSlot;
        e = deep[rel / LS::kSlot - 1u - (uint32_t)LS::kSmem];
      }
      if (e.t_near < best_t) {
        cur = e.ref;
        enter();
        if (mode >= 0) return;
      }
    }
  };

  auto step = [&]() {
    typename L::Node node;
    L::decode(T, cur, node);
    if constexpr (!L::kVariantInRef) {
      if (node.variant == L::kLeaf) {
        prim_i = (uint32_t)node.data.begin;
        prim_end = (uint32_t)node.data.end;
        if (prim_i < prim_end) mode = kPrim;
        else pop_next();
        return;
      }
    }
    tally.visit();
    uint32_t mask = 0;
    float tn[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      float t_far;
      const bool some = ray_aabb(ray, node.lo[k], node.hi[k], tn[k], t_far);
      if (interval_intersects(ray, some, tn[k], t_far) && tn[k] < best_t) mask |= 1u << k;
    }
    if (mask == 0u) {
      pop_next();
      return;
    }
    const uint32_t m = (uint32_t)__popc(mask);
    const uint32_t rel = top - window;
    const uint32_t depth = rel / LS::kSlot;
    if (COUNT) tally.stack(depth + m);
    if (depth + m > (uint32_t)SCION_STACK_DEPTH) {  // the reference would hold all m passing children at once
      retire(SCION_Q_STACK_OVERFLOW);
      return;
    }
    // slot k1 = lowest passing slot is visited next; the others are stored so that they pop in slot
    // order: slot k lands above every passing slot with a larger index
    const uint32_t rest = mask & (mask - 1u);
    if (rel + (m - 1u) * LS::kSlot <= LS::kSmemBytes) {  // all stores land in the shared-memory window
#pragma unroll
      for (int k = 1; k < 8; k++) {
        if ((rest >> k) & 1u) LS::store(top + (uint32_t)__popc(mask >> (k + 1)) * LS::kSlot, Entry{node.children[k], tn[k]});
      }
    } else {
#pragma unroll
      for (int k = 1; k < 8; k++) {
        if ((rest >> k) & 1u) {
          const uint32_t pos = depth + (uint32_t)__popc(mask >> (k + 1));
          if (pos < (uint32_t)LS::kSmem) LS::store(window + threadIdx.x * 4u + pos * LS::kSlot, Entry{node.children[k], tn[k]});
          else deep[pos - (uint32_t)LS::kSmem] = Entry{node.children[k], tn[k]};
        }
      }
    }
#if SCION_PF8 == 1  // L2-prefetch the record of the entry that pops first (the second passing slot)
    if (rest) {
      Ref second = node.children[1];
#pragma unroll
      for (int k = 7; k >= 1; k--)
        if ((rest >> k) & 1u) second = node.children[k];
      L::prefetch(T, second);
    }
#elif SCION_PF8 == 2  // ... of every pushed entry
#pragma unroll
    for (int k = 1; k < 8; k++)
      if ((rest >> k) & 1u) L::prefetch(T, node.children[k]);
#endif
    top += (m - 1u) * LS::kSlot;
    Ref first = node.children[0];
#pragma unroll
    for (int k = 7; k >= 0; k--)
      if ((mask >> k) & 1u) first = node.children[k];
    cur = first;
    enter();
    if (mode < 0) pop_next();
  };

  for (;;) {
#pragma unroll 1
    for (int k = 0; k < SCION_INNER8; k++) {
      if (mode == kNode) step();
    }
    const unsigned idle = __ballot_sync(kFullMask, mode == kFetch);
    if (idle && (__popc(idle) >= SCION_REFILL_MIN8 || work.exhausted)) {
      uint64_t nq;
      if (!work.exhausted && work.refill(mode == kFetch, next, n, nq)) {
        ray = load_ray(rays, nq);
        stash[threadIdx.x] = RayStash{ray.dx, ray.dy, ray.dz, 0u};
        stash_q[threadIdx.x] = nq;
        best_t = scion::inf();
        best_prim = SCION_MISS_PRIM;
        tally.reset();
        top = window + threadIdx.x * 4u;
        cur = L::root(T);
        enter();
        if (mode < 0) retire(SCION_Q_OK);  // the root is an empty leaf
      }
      if (work.exhausted && __ballot_sync(kFullMask, mode != kFetch) == 0u) break;
    }
    const unsigned pmask = __ballot_sync(kFullMask, mode == kPrim);
    if (pmask && (__popc(pmask) >= SCION_PRIM_MIN8 || __ballot_sync(kFullMask, mode == kNode) == 0u)) {
      const bool own = mode == kPrim;
      const uint32_t done = coop_triangles2<L>(T, own, ray.ox, ray.oy, ray.oz, ray.tmax, stash + (threadIdx.x & ~31u), prim_i, prim_end, best_t,
                                               best_prim, coop[threadIdx.x >> 5]);
      if (COUNT) tally.prim_tests += done;
      if (own) pop_next();
    }
  }
}

// ------------------------------------------------------------------------------------------
// closest_hit, 8-wide family, STAGED RECORD (kernel v16) — for layouts whose interior record starts on a 16-byte
// boundary (L::kCanSlot: the paper's `-align16` files and the 256-byte f32 record).
//
// chrt8_kernel decodes a whole 104-256-byte record into registers: 124-128 registers, 4 CTAs/SM, 16 warps/SM, issue
// slots 55 % busy with nothing else saturated (profiles/r1_ncu_v11_c5_q8ci.txt: `wait` + `long_scoreboard` stalls of a
// kernel that has 4 warps per scheduler to hide them).  Here a lane copies its record into shared memory with 16-byte
// asynchronous copies (cp.async = SASS LDGSTS: global -> shared without passing through registers; chunk c of the 32
// lanes of a warp is contiguous, so reading a chunk back is a conflict-free LDS.128) and then decodes ONE child slot at a
// time from there with the emitted decode_slot<K>() (same expressions as decode(), dead slots removed by the compiler).
// Slots are visited 7 -> 0 and a passing child is pushed at once, so the entries pop in slot order (chrt8.scion:7) and no
// per-slot arrays stay live; the lowest passing slot is continued with in registers.  Same visit order, same deferred
// `t_near < best` cull at pop, same counters and overflow rule as chrt8_kernel (tests compare the two bit for bit).
// ------------------------------------------------------------------------------------------
#ifndef SCION_MINB8S
#define SCION_MINB8S 6
#endif
#ifndef SCION_STACK_SMEM8S
#define SCION_STACK_SMEM8S (16 * 1024)
#endif
#ifndef SCION_CPASYNC_CG  /* 1: cp.async.cg (L2 only) instead of .ca (allocate in L1) */
#define SCION_CPASYNC_CG 0
#endif
constexpr int kStackSmemBytesPerBlock8S = SCION_STACK_SMEM8S;
template <class L>
constexpr size_t staged_record_bytes() {  // shared memory of one CTA for the lanes' record copies
  if constexpr (L::kCanSlot) return (size_t)((L::kSlotUsedBytes + 15u) / 16u) * 16u * (size_t)kBlockThreads;
  else return 0;
}
template <class L, bool COUNT>
__global__ void __launch_bounds__(kBlockThreads, SCION_MINB8S) chrt8s_kernel(const TreeView T, const scion_ray* __restrict__ rays, uint64_t n,
                                                                scion_hit* __restrict__ hits, uint32_t* __restrict__ status,
                                                                scion_counters* __restrict__ counters, unsigned long long* __restrict__ next, const int tune) {
  static_assert(L::kCanSlot && L::kVariantInRef, "staged-record kernel: 16-byte aligned interior records, leaf variant in the reference");
  using Ref = typename L::Ref;
  using Entry = WideEntry<Ref>;
  using LS = LaneStack<Entry, kStackSmemBytesPerBlock8S>;
  constexpr int kChunks = (int)((L::kSlotUsedBytes + 15u) / 16u);
  constexpr int kPitch = 16 * kBlockThreads;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ CoopScratch2 coop[kBlockThreads / 32];
  __shared__ RayStash stash[kBlockThreads];
  __shared__ unsigned long long stash_q[kBlockThreads];
  Entry deep[LS::kDeep];
  uint32_t window = (uint32_t)__cvta_generic_to_shared(smem_raw);
  asm volatile("" : "+r"(window));
  uint32_t top = window + threadIdx.x * 4u;
  uint32_t rec_addr = (uint32_t)__cvta_generic_to_shared(smem_raw + kStackSmemBytesPerBlock8S + threadIdx.x * 16u);  // this lane's chunk 0
  WorkFetcher work;
  (void)tune;
  Tally<COUNT> tally;
  int mode = kFetch;
  RayCtx ray = make_ray(0, 0, 0, 0, 1, 1, 1);
  float best_t = 0;
  uint32_t best_prim = 0, prim_i = 0, prim_end = 0;
  Ref cur = L::root(T);

  auto retire = [&](uint32_t st) {
    const uint64_t qq = opaque(stash_q[threadIdx.x]);
    store_hit(hits + qq, best_t, best_prim);
    if (status) status[qq] = st;
    tally.store(counters, qq);
    mode = kFetch;
  };
  auto enter = [&]() {  // `cur` was just chosen: park it if the reference itself says it is a leaf
    mode = kNode;
    if (L::ref_variant(cur) == L::kLeaf) {
      typename L::Node leaf;
      L::decode(T, cur, leaf);  // reference-only arm: no memory access
      prim_i = (uint32_t)leaf.data.begin;
      prim_end = (uint32_t)leaf.data.end;
      mode = prim_i < prim_end ? kPrim : -1;  // -1: empty leaf, take the next entry
    }
  };
  auto pop_next = [&]() {  // next pending entry whose deferred cull `t_near < best` still passes, or retire
    for (;;) {
      const uint32_t rel = top - window;
      Entry e;
      if (rel - LS::kSlot < LS::kSmemBytes) {
        top -= LS::kSlot;
        LS::load(top, e);
      } else if (rel < LS::kSlot) {
        retire(SCION_Q_OK);
        return;
      } else {
        top -= LS::kSlot;
        e = deep[rel / LS::kSlot - 1u - (uint32_t)LS::kSmem];
      }
      if (e.t_near < best_t) {
        cur = e.ref;
        enter();
        if (mode >= 0) return;
      }
    }
  };
  auto step = [&]() {
    {  // stage the record: kChunks 16-byte asynchronous copies, global -> shared
      const uint8_t* p = L::slot_record(T, cur);
#pragma unroll
      for (int c = 0; c < kChunks; c++) {
#if SCION_CPASYNC_CG
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(rec_addr + (uint32_t)(c * kPitch)), "l"(p + 16 * c) : "memory");
#else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(rec_addr + (uint32_t)(c * kPitch)), "l"(p + 16 * c) : "memory");
#endif
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      asm volatile("" : "+r"(rec_addr)::"memory");  // the record loads below depend on THIS value of the address: they cannot move above the wait
    }
    const StagedRecord<kChunks * 4, kPitch> rec{rec_addr};
    tally.visit();
    const uint32_t rel0 = top - window;
    uint32_t m = 0;
    Ref pend = cur;
    float pend_t = 0.0f;
    // FAST: all (at most 7) pushes of this step land in the shared-memory window: predicated stores, no branch
    auto run_slots = [&](auto FAST) {
      constexpr bool kFast = decltype(FAST)::value;
      auto slot = [&](auto KC) {
        constexpr int K = decltype(KC)::value;
        f32x3 lo, hi;
        Ref ch;
        L::template decode_slot<K>(T, cur, rec, lo, hi, ch);
        float tn, t_far;
        const bool some = ray_aabb(ray, lo, hi, tn, t_far);
        if (interval_intersects(ray, some, tn, t_far) && tn < best_t) {
          if (m) {  // a slot with a larger index passed before: it pops after this one
            if constexpr (kFast) {
              LS::store(top, Entry{pend, pend_t});
            } else {  // entries beyond the reference capacity are dropped: the query retires with an overflow status below
              const uint32_t rel = top - window;
              if (rel < LS::kSmemBytes) {
                LS::store(top, Entry{pend, pend_t});
              } else {
                const uint32_t pos = rel / LS::kSlot - (uint32_t)LS::kSmem;
                if (pos < (uint32_t)LS::kDeep) deep[pos] = Entry{pend, pend_t};
              }
            }
            top += LS::kSlot;
          }
          pend = ch;
          pend_t = tn;
          m++;
        }
      };
      slot(std::integral_constant<int, 7>{});
      slot(std::integral_constant<int, 6>{});
      slot(std::integral_constant<int, 5>{});
      slot(std::integral_constant<int, 4>{});
      slot(std::integral_constant<int, 3>{});
      slot(std::integral_constant<int, 2>{});
      slot(std::integral_constant<int, 1>{});
      slot(std::integral_constant<int, 0>{});
    };
    if (rel0 + 7u * LS::kSlot <= LS::kSmemBytes) run_slots(std::true_type{});
    else run_slots(std::false_type{});
    if (m == 0u) {
      pop_next();
      return;
    }
    const uint32_t depth0 = rel0 / LS::kSlot;
    if (COUNT) tally.stack(depth0 + m);
    if (depth0 + m > (uint32_t)SCION_STACK_DEPTH) {  // the reference would hold all m passing children at once
      retire(SCION_Q_STACK_OVERFLOW);
      return;
    }
    cur = pend;  // the lowest passing slot is visited next
    enter();
    if (mode < 0) pop_next();
  };

  for (;;) {
#pragma unroll 1
    for (int k = 0; k < SCION_INNER8; k++) {
      if (mode == kNode) step();
    }
    const unsigned idle = __ballot_sync(kFullMask, mode == kFetch);
    if (idle && (__popc(idle) >= SCION_REFILL_MIN8 || work.exhausted)) {
      uint64_t nq;
      if (!work.exhausted && work.refill(mode == kFetch, next, n, nq)) {
        ray = load_ray(rays, nq);
        stash[threadIdx.x] = RayStash{ray.dx, ray.dy, ray.dz, 0u};
        stash_q[threadIdx.x] = nq;
        best_t = scion::inf();
        best_prim = SCION_MISS_PRIM;
        tally.reset();
        top = window + threadIdx.x * 4u;
        cur = L::root(T);
        enter();
        if (mode < 0) retire(SCION_Q_OK);  // the root is an empty leaf
      }
      if (work.exhausted && __ballot_sync(kFullMask, mode != kFetch) == 0u) break;
    }
    const unsigned pmask = __ballot_sync(kFullMask, mode == kPrim);
    if (pmask && (__popc(pmask) >= SCION_PRIM_MIN8 || __ballot_sync(kFullMask, mode == kNode) == 0u)) {
      const bool own = mode == kPrim;
      const uint32_t done = coop_triangles2<L>(T, own, ray.ox, ray.oy, ray.oz, ray.tmax, stash + (threadIdx.x & ~31u), prim_i, prim_end, best_t,
                                               best_prim, coop[threadIdx.x >> 5]);
      if (COUNT) tally.prim_tests += done;
      if (own) pop_next();
    }
  }
}

// ------------------------------------------------------------------------------------------
// closest_point, binary + DOP-14 families
// ------------------------------------------------------------------------------------------
template <class L, class TallyT>
SCION_DEV float cpq_node_distmin(const TreeView& T, const f32x3& p, const typename L::Ref& ref, typename L::Node& n, TallyT& tally) {
  L::decode(T, ref, n);
  tally.visit();
  if constexpr (L::kHasCold) {
    L::decode_cold(T, ref, n);
    tally.cold();
  }
  if constexpr (L::kFamily == SCION_FAMILY_DOP14) return distmin_dop_point(p, n.lo1, n.hi1, n.lo2, n.hi2);
  else return sqdist_point_aabb(p, n.low, n.high);
}

// Cooperative leaf phase of closest_point (cpq.scion:25-31), v7: same run bookkeeping as
// coop_triangles2; the worker returns (d2, closest point); owners fold with the strict
// `d2 < best[0]` rule in ascending primitive order.  The owner's best point lives in shared memory
// (`best_pt`, one float4 per thread: x, y, z, primitive index) — only the fold and the retire path
// touch it.
struct CoopScratchCp2 {
  float d2[32];
  float c[32][3];
  uint8_t owner[32];
};
template <class L>
SCION_DEV uint32_t coop_points2(const TreeView& T, bool own, const f32x3& p, uint32_t& prim_i, uint32_t prim_end, float& best_d, float4* __restrict__ best_pt,
                                CoopScratchCp2& sc) {
  static_assert(L::kStride_primitives == 36, "Triangle stride");
  const unsigned lane = threadIdx.x & 31u;
  uint32_t tested = 0;
  for (;;) {
    const uint32_t remaining = own ? prim_end - prim_i : 0u;
    if (__ballot_sync(kFullMask, remaining != 0u) == 0u) break;
    const uint32_t c = remaining < 32u ? remaining : 32u;
    uint32_t incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_up_sync(kFullMask, incl, d);
      if (lane >= (unsigned)d) incl += v;
    }
    const uint32_t excl = incl - c;
    const bool starts_run = c != 0u && excl < 32u;
    const uint32_t take = starts_run ? (c < 32u - excl ? c : 32u - excl) : 0u;
    if (starts_run) sc.owner[excl] = (uint8_t)lane;
    const unsigned starts = __reduce_or_sync(kFullMask, starts_run ? (1u << excl) : 0u);
    const uint32_t total = __shfl_sync(kFullMask, incl, 31);
    __syncwarp();
    const bool work = lane < total;
    const unsigned below = starts & (0xffffffffu >> (31u - lane));
    const unsigned first = 31u - (unsigned)__clz((int)(below | 1u));
    const unsigned o = sc.owner[first];
    const uint32_t kk = lane - first;
    const f32x3 q{__shfl_sync(kFullMask, p.x, o), __shfl_sync(kFullMask, p.y, o), __shfl_sync(kFullMask, p.z, o)};
    const uint32_t pi = __shfl_sync(kFullMask, prim_i, o) + kk;
    if (work) {
      float tri[9];
      load_triangle36(T.buf[L::kBuf_primitives], pi, tri);
      const f32x3 cp = closest_point_triangle(q, tri);
      const f32x3 x = q - cp;
      sc.d2[lane] = dot(x, x);
      sc.c[lane][0] = cp.x; sc.c[lane][1] = cp.y; sc.c[lane][2] = cp.z;
    }
    __syncwarp();
    int won = -1;
    for (uint32_t k = 0; k < take; k++) {
      const float d2 = sc.d2[excl + k];
      if (d2 < best_d) {
        best_d = d2;
        won = (int)k;
      }
    }
    if (won >= 0) *best_pt = make_float4(sc.c[excl + won][0], sc.c[excl + won][1], sc.c[excl + won][2], __uint_as_float(prim_i + (uint32_t)won));
    prim_i += take;
    tested += take;
    __syncwarp();
  }
  return tested;
}

#ifndef SCION_MINBC
#define SCION_MINBC 6
#endif
#ifndef SCION_STACK_SMEM_C  /* shared-memory stack window of one closest-point CTA */
#define SCION_STACK_SMEM_C SCION_STACK_SMEM
#endif
constexpr int kStackSmemBytesPerBlockC = SCION_STACK_SMEM_C;
#ifndef SCION_PRIM_MINC
#define SCION_PRIM_MINC 6
#endif
#ifndef SCION_INNERC
#define SCION_INNERC 8  // 4 -> 8 after v13: +1 % (pbrt-q16 1388 -> 1401, pbrt 1424 -> 1439), >= 0 on every other binary layout
#endif
// closest_point kernel v7.  The reference decodes a node three times on the way down: as the
// child peek of its parent (cpq.scion:9-16), again when it is visited, and its own two children.
// The value of every decode and of square_distance(p, box) is a pure function, and `best` does not
// change between the peek of the NEAR child and its visit, so the kernel carries the near child's
// decoded record and distance into the next step instead of fetching it again.  A step therefore
// has two decode slots: X = left child (descending lane) or the popped node (popping lane), and
// Y = right child (descending lanes only).  The instrumented build still counts every decode the
// reference performs (identical counters), it just does not repeat the work.
// Rejected: ONE decode per step (modes pop / peek-left / peek-right, every decode at ~25/32 lanes instead
// of the Y slot at ~12/32): 886 instead of 1247 Mq/s — the two child loads of a step overlap in the
// memory system, and the kernel is bound by that latency, not by issue slots.
template <class L, bool COUNT>
__global__ void __launch_bounds__(kBlockThreads, SCION_MINBC) cpq2_kernel(const TreeView T, const float* __restrict__ points, uint64_t n,
                                                             scion_cp* __restrict__ out, uint32_t* __restrict__ status,
                                                             scion_counters* __restrict__ counters, unsigned long long* __restrict__ next, const int tune) {
  using Ref = typename L::Ref;
  using Node = typename L::Node;
  using Entry = Ref;
  using LS = LaneStack<Entry, kStackSmemBytesPerBlockC>;
  enum : int { kPop = 3 };  // stepping lanes: kNode (record + distance of `node` are valid) or kPop (take the next pending reference first)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ CoopScratchCp2 coop[kBlockThreads / 32];
  __shared__ float4 best_pt[kBlockThreads];
  __shared__ unsigned long long stash_q[kBlockThreads];
  Entry deep[LS::kDeep];
  auto make_entry = [](const Ref& r, float) -> Entry { return r; };
  uint32_t window = (uint32_t)__cvta_generic_to_shared(smem_raw);
  asm volatile("" : "+r"(window));
  uint32_t top = window + threadIdx.x * 4u;
#if SCION_CPQ_GUIDED
  WorkFetcher work;
#else
  WorkFetcherFixed work;
#endif
  (void)tune;
  Tally<COUNT> tally;
  int mode = kFetch;
  f32x3 p{0.0f, 0.0f, 0.0f};
  float best_d = 0, d = 0;
  uint32_t prim_i = 0, prim_end = 0;
  bool carried = false;  // (instrumented build) `node` came from its parent's peek: its visit is a decode the reference repeats
  Node node;
  Ref root = L::root(T);
  Ref cur = root;  // reference of `node` (decode_cold of tree-carried layouts needs it)

  auto retire = [&](uint32_t st) {
    const uint64_t qq = opaque(stash_q[threadIdx.x]);
    const float4 b = best_pt[threadIdx.x];
    out[qq] = scion_cp{best_d, b.x, b.y, b.z, __float_as_uint(b.w)};
    if (status) status[qq] = st;
    tally.store(counters, qq);
    mode = kFetch;
  };

  auto step = [&]() {
    bool go = false;  // interior: decode both children
    Ref rx = cur, ry = cur;
    if (mode == kNode) {
      if (COUNT && carried) {
        tally.visit();
        if (L::kHasCold) tally.cold();
      }
      mode = kPop;
      if (d < best_d) {
        if (node.variant == L::kLeaf) {
          prim_i = (uint32_t)node.data.begin;
          prim_end = (uint32_t)node.data.end;
          if (prim_i < prim_end) {
            mode = kPrim;
            return;
          }
        } else {
          float ub;
          if constexpr (L::kFamily == SCION_FAMILY_DOP14) ub = distmax_point_aabb(p, node.lo1, node.hi1);
          else ub = distmax_point_aabb(p, node.low, node.high);
          if (ub < best_d) best_d = ub;  // best = (upper_bound, best[1])
          go = true;
          rx = node.left;
          ry = node.right;
        }
      }
    }
    const uint32_t rel = top - window;
    if (!go) {  // pop the next pending reference, or retire
      if (rel - LS::kSlot < LS::kSmemBytes) {
        top -= LS::kSlot;
        LS::load(top, rx);
      } else if (rel < LS::kSlot) {
        retire(SCION_Q_OK);
        return;
      } else {
        top -= LS::kSlot;
        rx = deep[rel / LS::kSlot - 1u - (uint32_t)LS::kSmem];
      }
    } else {
      const uint32_t depth = rel / LS::kSlot;
      if (COUNT) tally.stack(depth + 2u);  // reference discipline: pop self, push far, push near
      if (depth + 2u > (uint32_t)SCION_STACK_DEPTH) {
        retire(SCION_Q_STACK_OVERFLOW);
        return;
      }
    }
    // Both decode slots unconditional where the record is ONE vector load (pbrt, pbrt-align16, pbrt-q16, sg-eq-align16):
    // a popping lane decodes its X record twice (same address, no extra sector).  The Y instructions are issued for the
    // warp anyway as soon as one lane descends, and without the `go` branch around them the Y load is in flight together
    // with the X load instead of behind X's decode (r1_ncu_v11_c4_q16.txt: 24 % of the stall samples sat on that second,
    // serialised load): C4 pbrt-q16 1305 -> 1389, pbrt 1253 -> 1427 Mq/s.  Multi-load records lose (pbrt-soa -14 %,
    // pbrt-post -16 %, ptr -6 %, identity -11 %, dop14 -11 %, sg-eq -3 %): they keep the branch.
    constexpr bool kBoth = SCION_CPQ_BOTH < 0 ? (L::kCanStage && !L::kHasCold) : (SCION_CPQ_BOTH != 0);
    auto descend = [&](const Node& nx, float dx, const Node& ny, float dy) {
      const bool left_first = dx < dy;  // ties: the right child is visited first (cpq.scion:17 `L < R`)
      const Entry far = make_entry(left_first ? ry : rx, left_first ? dy : dx);
      if (rel < LS::kSmemBytes) LS::store(top, far);
      else deep[rel / LS::kSlot - (uint32_t)LS::kSmem] = far;
      top += LS::kSlot;
      if (left_first) { node = nx; d = dx; cur = rx; }
      else { node = ny; d = dy; cur = ry; }
      carried = true;
    };
    auto stay = [&](const Node& nx, float dx) {
      node = nx;
      d = dx;
      cur = rx;
      carried = false;
    };
    Node nx;
    if constexpr (kBoth) {
      Node ny;
      Tally<false> quiet;
      const float dx = cpq_node_distmin<L>(T, p, rx, nx, quiet);
      const float dy = cpq_node_distmin<L>(T, p, go ? ry : rx, ny, quiet);
      if (COUNT) {
        const uint32_t k = go ? 2u : 1u;
        tally.node_visits += k;
        if (L::kHasCold) tally.cold_loads += k;
      }
      if (go) descend(nx, dx, ny, dy);
      else stay(nx, dx);
    } else {
      const float dx = cpq_node_distmin<L>(T, p, rx, nx, tally);
      if (go) {
        Node ny;
        const float dy = cpq_node_distmin<L>(T, p, ry, ny, tally);
        descend(nx, dx, ny, dy);
      } else {
        stay(nx, dx);
      }
    }
    mode = kNode;
  };

  for (;;) {
#pragma unroll 1
    for (int k = 0; k < SCION_INNERC; k++) {
      if (mode == kNode || mode == kPop) step();
    }
    const unsigned idle = __ballot_sync(kFullMask, mode == kFetch);
    if (idle && (__popc(idle) >= kRefillMin || work.exhausted)) {
      uint64_t nq;
      if (!work.exhausted && work.refill(mode == kFetch, next, n, nq)) {
        p = f32x3{__ldcs(points + 3 * nq), __ldcs(points + 3 * nq + 1), __ldcs(points + 3 * nq + 2)};
        stash_q[threadIdx.x] = nq;
        best_pt[threadIdx.x] = make_float4(0.0f, 0.0f, 0.0f, __uint_as_float(SCION_MISS_PRIM));
        best_d = scion::inf();
        tally.reset();
        top = window + threadIdx.x * 4u;
        LS::store(top, make_entry(root, 0.0f));  // the root is "popped" by the first step (0 < inf: never culled there)
        top += LS::kSlot;
        mode = kPop;
      }
      if (work.exhausted && __ballot_sync(kFullMask, mode != kFetch) == 0u) break;
    }
    const unsigned pmask = __ballot_sync(kFullMask, mode == kPrim);
    if (pmask && (__popc(pmask) >= SCION_PRIM_MINC || __ballot_sync(kFullMask, mode == kNode || mode == kPop) == 0u)) {
      const bool own = mode == kPrim;
      const uint32_t done = coop_points2<L>(T, own, p, prim_i, prim_end, best_d, &best_pt[threadIdx.x], coop[threadIdx.x >> 5]);
      if (COUNT) tally.prim_tests += done;
      if (own) mode = kPop;
    }
  }
}

}  // namespace scion

#include "traverse_experiments.cuh"
#include "traverse_coop8.cuh"
