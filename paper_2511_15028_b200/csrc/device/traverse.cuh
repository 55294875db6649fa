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
// Stack: the traversal stack lives in shared memory, laid out [entry][thread] so that any mix
// of per-lane depths is bank-conflict free (lane l always hits bank l); the top of the tree walk
// never touches it for the left child (implicit next node).  See DESIGN.md for the measured
// comparison against a local-memory stack.
#pragma once
#include <cuda_runtime.h>

#include "geometry.cuh"
#include "scion_b200.h"

namespace scion {

constexpr int kBlockThreads = 128;

// ------------------------------------------------------------------------------------------
// work distribution: persistent CTAs; each warp grabs 32 queries at a time with one atomic
// issued by an elected lane and broadcast by shuffle (warp-aggregated dynamic fetch).
// ------------------------------------------------------------------------------------------
struct WorkQueue {
  unsigned long long* counter;  // device global, zeroed before launch
};

// Hybrid traversal stack: the first kSmem entries live in shared memory, laid out
// [entry][thread] (lane l always hits bank l => conflict-free for any mix of per-lane depths);
// deeper entries spill to a per-thread local-memory array that is only touched by the rare deep
// paths.  kSmem is sized so that one CTA uses 16 KB of shared memory whatever the entry size.
constexpr int kStackSmemBytesPerBlock = 16 * 1024;
template <class Entry>
struct HybridStack {
  static constexpr int kSmem = (kStackSmemBytesPerBlock / kBlockThreads / (int)sizeof(Entry)) < SCION_STACK_DEPTH
                                   ? (kStackSmemBytesPerBlock / kBlockThreads / (int)sizeof(Entry))
                                   : SCION_STACK_DEPTH;
  static constexpr int kDeep = SCION_STACK_DEPTH - kSmem > 0 ? SCION_STACK_DEPTH - kSmem : 1;
  Entry* base;  // &smem[threadIdx.x]; entry e lives at base[e * kBlockThreads]
  Entry deep[kDeep];
  int sp = 0;
  SCION_DEV void push(const Entry& r) {
    if (sp < kSmem) base[sp * kBlockThreads] = r;
    else deep[sp - kSmem] = r;
    sp++;
  }
  SCION_DEV Entry pop() {
    sp--;
    return sp < kSmem ? base[sp * kBlockThreads] : deep[sp - kSmem];
  }
};

template <bool COUNT>
struct Tally {
  uint32_t node_visits = 0, prim_tests = 0, cold_loads = 0, max_stack = 0;
  SCION_DEV void visit() { if (COUNT) node_visits++; }
  SCION_DEV void visits(uint32_t k) { if (COUNT) node_visits += k; }
  SCION_DEV void prim() { if (COUNT) prim_tests++; }
  SCION_DEV void cold(uint32_t k = 1) { if (COUNT) cold_loads += k; }
  SCION_DEV void stack(uint32_t occ) { if (COUNT) max_stack = occ > max_stack ? occ : max_stack; }
  SCION_DEV void store(scion_counters* out, uint64_t q) const {
    if (COUNT && out) out[q] = scion_counters{node_visits, prim_tests, cold_loads, max_stack};
  }
};

SCION_DEV RayCtx load_ray(const scion_ray* rays, uint64_t q) {
  const float4* p = reinterpret_cast<const float4*>(rays + q);
  const float4 a = __ldcs(p), b = __ldcs(p + 1);  // streaming: read once
  return make_ray(a.x, a.y, a.z, a.w, b.x, b.y, b.z);
}

template <class L, class TallyT>
SCION_DEV void leaf_triangles(const TreeView& T, const RayCtx& ray, const Slice& data, float& best_t, uint32_t& best_prim, TallyT& tally) {
  static_assert(L::kStride_primitives == 36, "Triangle stride");
  for (uint64_t i = data.begin; i < data.end; i++) {
    float tri[9];
    load_triangle36(T.buf[L::kBuf_primitives], i, tri);
    float t;
    tally.prim();
    // `intersects(ray, t) && distmin(ray, t) < best[0]` then `best = (distmin(ray, t), t)`
    if (ray_tri_mt(ray, tri, t) && t < best_t) {
      best_t = t;
      best_prim = (uint32_t)i;
    }
  }
}

// bounds test of one binary / DOP node against the ray.  Loads the cold segment only when the
// reference semantics would evaluate it (dop.scion:20-21 `if I {...}`).
template <class L, class TallyT>
SCION_DEV bool node_test(const TreeView& T, const RayCtx& ray, const typename L::Ref& ref, typename L::Node& n, float& t_near, TallyT& tally) {
  float t_far;
  if constexpr (L::kFamily == SCION_FAMILY_DOP14) {
    bool some = ray_aabb(ray, n.lo1, n.hi1, t_near, t_far);
    if (some) {
      L::decode_cold(T, ref, n);
      tally.cold();
      some = dop_diagonals(ray, n.lo2, n.hi2, t_near, t_far);
    }
    return interval_intersects(ray, some, t_near, t_far);
  } else {
    const bool some = ray_aabb(ray, n.low, n.high, t_near, t_far);
    const bool hit = interval_intersects(ray, some, t_near, t_far);
    if constexpr (L::kHasCold) {
      if (hit) {
        L::decode_cold(T, ref, n);
        tally.cold();
      }
    }
    return hit;
  }
}

// ------------------------------------------------------------------------------------------
// closest_hit, binary + DOP-14 families
// ------------------------------------------------------------------------------------------
template <class L, bool COUNT>
__global__ void __launch_bounds__(kBlockThreads) chrt2_kernel(const TreeView T, const scion_ray* __restrict__ rays, uint64_t n,
                                                              scion_hit* __restrict__ hits, uint32_t* __restrict__ status,
                                                              scion_counters* __restrict__ counters, unsigned long long* __restrict__ next) {
  using Ref = typename L::Ref;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  HybridStack<Ref> stack;
  stack.base = reinterpret_cast<Ref*>(smem_raw) + threadIdx.x;
  const unsigned lane = threadIdx.x & 31u;
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(next, 32ull);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= n) break;
    const uint64_t q = base + lane;
    if (q < n) {
      const RayCtx ray = load_ray(rays, q);
      float best_t = scion::inf();
      uint32_t best_prim = SCION_MISS_PRIM;
      uint32_t st = SCION_Q_OK;
      Tally<COUNT> tally;
      stack.sp = 0;
      Ref cur = L::root(T);
      for (;;) {
        typename L::Node node;
        L::decode(T, cur, node);
        tally.visit();
        float t_near;
        const bool hit = node_test<L>(T, ray, cur, node, t_near, tally);
        bool descend = false;
        if (hit) {
          if (node.variant == L::kLeaf) {
            leaf_triangles<L>(T, ray, node.data, best_t, best_prim, tally);
          } else if (t_near < best_t) {
            // reference discipline: pop self, push right, push left => occupancy sp + 2
            tally.stack((uint32_t)stack.sp + 2u);
            if (stack.sp + 2 > SCION_STACK_DEPTH) { st = SCION_Q_STACK_OVERFLOW; break; }
            stack.push(node.right);
            cur = node.left;
            descend = true;
          }
        }
        if (!descend) {
          if (stack.sp == 0) break;
          cur = stack.pop();
        }
      }
      hits[q] = scion_hit{best_t, best_prim};
      if (status) status[q] = st;
      tally.store(counters, q);
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

template <class L, bool COUNT>
__global__ void __launch_bounds__(kBlockThreads) chrt8_kernel(const TreeView T, const scion_ray* __restrict__ rays, uint64_t n,
                                                              scion_hit* __restrict__ hits, uint32_t* __restrict__ status,
                                                              scion_counters* __restrict__ counters, unsigned long long* __restrict__ next) {
  using Ref = typename L::Ref;
  using Entry = WideEntry<Ref>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  HybridStack<Entry> stack;
  stack.base = reinterpret_cast<Entry*>(smem_raw) + threadIdx.x;
  const unsigned lane = threadIdx.x & 31u;
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(next, 32ull);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= n) break;
    const uint64_t q = base + lane;
    if (q < n) {
      const RayCtx ray = load_ray(rays, q);
      float best_t = scion::inf();
      uint32_t best_prim = SCION_MISS_PRIM;
      uint32_t st = SCION_Q_OK;
      Tally<COUNT> tally;
      stack.sp = 0;
      Ref cur = L::root(T);
      for (;;) {
        typename L::Node node;
        L::decode(T, cur, node);
        if (node.variant == L::kLeaf) {
          leaf_triangles<L>(T, ray, node.data, best_t, best_prim, tally);
        } else {
          tally.visit();
          // test all eight child boxes; push the passing ones in reverse slot order
          uint32_t mask = 0;
          float tn[8];
#pragma unroll
          for (int k = 0; k < 8; k++) {
            float t_far;
            const bool some = ray_aabb(ray, node.lo[k], node.hi[k], tn[k], t_far);
            if (interval_intersects(ray, some, tn[k], t_far) && tn[k] < best_t) mask |= 1u << k;
          }
          const int m = __popc(mask);
          tally.stack((uint32_t)(stack.sp + m));
          if (stack.sp + m > SCION_STACK_DEPTH) { st = SCION_Q_STACK_OVERFLOW; break; }
#pragma unroll
          for (int k = 7; k >= 0; k--)
            if (mask & (1u << k)) stack.push(Entry{node.children[k], tn[k]});
        }
        bool found = false;
        while (stack.sp > 0) {
          const Entry e = stack.pop();
          if (e.t_near < best_t) { cur = e.ref; found = true; break; }
        }
        if (!found) break;
      }
      hits[q] = scion_hit{best_t, best_prim};
      if (status) status[q] = st;
      tally.store(counters, q);
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

template <class L, bool COUNT>
__global__ void __launch_bounds__(kBlockThreads) cpq2_kernel(const TreeView T, const float* __restrict__ points, uint64_t n,
                                                             scion_cp* __restrict__ out, uint32_t* __restrict__ status,
                                                             scion_counters* __restrict__ counters, unsigned long long* __restrict__ next) {
  using Ref = typename L::Ref;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  HybridStack<Ref> stack;
  stack.base = reinterpret_cast<Ref*>(smem_raw) + threadIdx.x;
  const unsigned lane = threadIdx.x & 31u;
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(next, 32ull);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= n) break;
    const uint64_t q = base + lane;
    if (q < n) {
      const f32x3 p{__ldcs(points + 3 * q), __ldcs(points + 3 * q + 1), __ldcs(points + 3 * q + 2)};
      float best_d = scion::inf();
      f32x3 best_p{0.0f, 0.0f, 0.0f};
      uint32_t best_prim = SCION_MISS_PRIM;
      uint32_t st = SCION_Q_OK;
      Tally<COUNT> tally;
      stack.sp = 0;
      Ref cur = L::root(T);
      for (;;) {
        typename L::Node node;
        const float d = cpq_node_distmin<L>(T, p, cur, node, tally);
        bool descend = false;
        if (d < best_d) {
          if (node.variant == L::kLeaf) {
            for (uint64_t i = node.data.begin; i < node.data.end; i++) {
              float tri[9];
              load_triangle36(T.buf[L::kBuf_primitives], i, tri);
              const f32x3 c = closest_point_triangle(p, tri);
              const f32x3 x = p - c;
              const float d2 = dot(x, x);
              tally.prim();
              if (d2 < best_d) { best_d = d2; best_p = c; best_prim = (uint32_t)i; }
            }
          } else {
            float ub;
            if constexpr (L::kFamily == SCION_FAMILY_DOP14) ub = distmax_point_aabb(p, node.lo1, node.hi1);
            else ub = distmax_point_aabb(p, node.low, node.high);
            if (ub < best_d) best_d = ub;  // best = (upper_bound, best[1])
            typename L::Node ln, rn;
            const Ref left = node.left, right = node.right;
            const float dl = cpq_node_distmin<L>(T, p, left, ln, tally);
            const float dr = cpq_node_distmin<L>(T, p, right, rn, tally);
            tally.stack((uint32_t)stack.sp + 2u);
            if (stack.sp + 2 > SCION_STACK_DEPTH) { st = SCION_Q_STACK_OVERFLOW; break; }
            if (dl < dr) { stack.push(right); cur = left; }
            else { stack.push(left); cur = right; }
            descend = true;
          }
        }
        if (!descend) {
          if (stack.sp == 0) break;
          cur = stack.pop();
        }
      }
      out[q] = scion_cp{best_d, best_p.x, best_p.y, best_p.z, best_prim};
      if (status) status[q] = st;
      tally.store(counters, q);
    }
  }
}

}  // namespace scion
