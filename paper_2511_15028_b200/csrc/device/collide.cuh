// Collision detection (dual-tree traversal) — the third algorithm of the reference
// (/root/reference/proj/corpus/alg/cd.scion:2-31, cd_dop14.scion:2-31; SAT triangle/triangle test
// /root/reference/proj/corpus/lib/geometry.scion:112-157; AABB/AABB :158-160; DOP/DOP dop.scion:81-90).
//
// The DSL is a recursion over node PAIRS whose result is a SET of triangle pairs, so there is no
// visit-order contract: the GPU form is a level-synchronous frontier expansion.  One thread per
// node pair decodes both nodes with the emitted decoders, tests the bounds and appends the 4 / 2 / 2
// child pairs to the next frontier (warp-aggregated atomics); leaf/leaf pairs go to a primitive-pair
// work list that a second kernel resolves with one SAT test per thread.  Every test is the pure
// function the DSL states, so the resulting set equals the recursion's.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "geometry.cuh"
#include "scion_b200.h"

namespace scion {

// project6, geometry.scion:112-118
SCION_DEV int project6(const f32x3& ax, const f32x3& p1, const f32x3& p2, const f32x3& p3, const f32x3& q1, const f32x3& q2, const f32x3& q3) {
  const float P1 = dot(ax, p1), P2 = dot(ax, p2), P3 = dot(ax, p3);
  const float Q1 = dot(ax, q1), Q2 = dot(ax, q2), Q3 = dot(ax, q3);
  const float mn1 = fminf(fminf(P1, P2), P3), mx2 = fmaxf(fmaxf(Q1, Q2), Q3);
  if (mn1 > mx2) return 0;
  const float mx1 = fmaxf(fmaxf(P1, P2), P3), mn2 = fminf(fminf(Q1, Q2), Q3);
  if (mn2 > mx1) return 0;
  return 1;
}
// SAT_triangle_intersection, geometry.scion:120-154
SCION_DEV bool sat_triangles(const float* A, const float* B) {
  const f32x3 P1{A[0], A[1], A[2]}, P2{A[3], A[4], A[5]}, P3{A[6], A[7], A[8]};
  const f32x3 Q1{B[0], B[1], B[2]}, Q2{B[3], B[4], B[5]}, Q3{B[6], B[7], B[8]};
  const f32x3 p1{0.0f, 0.0f, 0.0f}, p2 = P2 - P1, p3 = P3 - P1;
  const f32x3 q1 = Q1 - P1, q2 = Q2 - P1, q3 = Q3 - P1;
  const f32x3 e1 = p2 - p1, e2 = p3 - p2, n1 = cross(e1, e2);
  if (project6(n1, p1, p2, p3, q1, q2, q3) == 0) return false;
  const f32x3 f1 = q2 - q1, f2 = q3 - q2, m1 = cross(f1, f2);
  if (project6(m1, p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(e1, f1), p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(e1, f2), p1, p2, p3, q1, q2, q3) == 0) return false;
  const f32x3 f3 = q1 - q3;
  if (project6(cross(e1, f3), p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(e2, f1), p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(e2, f2), p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(e2, f3), p1, p2, p3, q1, q2, q3) == 0) return false;
  const f32x3 e3 = p1 - p3;
  if (project6(cross(e3, f1), p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(e3, f2), p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(e3, f3), p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(e1, n1), p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(e2, n1), p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(e3, n1), p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(f1, m1), p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(f2, m1), p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(f3, m1), p1, p2, p3, q1, q2, q3) == 0) return false;
  return true;
}
// intersects(AABB, AABB), geometry.scion:158-160
SCION_DEV bool aabb_overlap(const f32x3& alo, const f32x3& ahi, const f32x3& blo, const f32x3& bhi) {
  const f32x3 low = scion::max(alo, blo), high = scion::min(ahi, bhi);
  return low.x <= high.x && low.y <= high.y && low.z <= high.z;
}

template <class Ref>
struct NodePair {
  Ref a, b;
};
struct LeafPair {
  uint32_t a_begin, a_count, b_begin, b_count;
};

// append `k` items with one atomic per warp; returns this lane's first slot
SCION_DEV unsigned long long warp_append(unsigned long long* counter, unsigned k) {
  const unsigned lane = threadIdx.x & 31u;
  const unsigned active = __activemask();
  unsigned incl = k;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned v = __shfl_up_sync(active, incl, d);
    if (lane >= (unsigned)d && (active >> (lane - d)) & 1u) incl += v;
  }
  // the scan above assumes a contiguous active mask; fall back to per-lane atomics otherwise
  if (active != 0xffffffffu) return k ? atomicAdd(counter, (unsigned long long)k) : 0ull;
  const unsigned total = __shfl_sync(active, incl, 31);
  unsigned long long base = 0;
  if (lane == 31 && total) base = atomicAdd(counter, (unsigned long long)total);
  base = __shfl_sync(active, base, 31);
  return base + (incl - k);
}

// ------------------------------------------------------------------------------------------
// One cooperative launch runs the whole dual-tree traversal: a persistent grid walks the node-pair
// frontier level by level (grid-wide barrier between levels, three rotating counters so that one
// barrier per level suffices: level l reads n[l % 3], appends to n[(l + 1) % 3] and clears
// n[(l + 2) % 3]), leaf/leaf pairs are collected on the way and resolved by the same grid after the
// last level.  The first version launched one kernel and synchronised with the host once per level:
// 18-21 levels of ~5 us work cost 3-5 ms; this one needs no host round trip.
// ------------------------------------------------------------------------------------------
struct CdState {  // device-side queue heads + diagnostics
  unsigned long long n[3];           // rotating frontier counters
  unsigned long long leaf_pairs;     // leaf/leaf pairs appended
  unsigned long long out_pairs;      // colliding triangle pairs appended
  unsigned long long node_pairs_tested;
  unsigned long long tri_tests;
  unsigned long long max_frontier;
  unsigned int levels;
  unsigned int overflow;             // bit 0 frontier, bit 1 leaf list, bit 2 output
};

// queue contents and counters are written by other SMs in the previous level: read them from L2
template <class T>
SCION_DEV T load_cg(const T* p) {
  static_assert(sizeof(T) % 4 == 0, "word-sized records");
  T v;
  uint32_t w[sizeof(T) / 4];
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 4); i++) w[i] = __ldcg(reinterpret_cast<const unsigned int*>(p) + i);
  memcpy(&v, w, sizeof(T));
  return v;
}

template <class L>
__global__ void __launch_bounds__(128) cd_kernel(const TreeView TA, const TreeView TB, NodePair<typename L::Ref>* __restrict__ front0,
                                                 NodePair<typename L::Ref>* __restrict__ front1, uint64_t front_capacity, LeafPair* __restrict__ leaves,
                                                 uint64_t leaf_capacity, scion_pair* __restrict__ out, uint64_t capacity, CdState* __restrict__ st) {
  using Ref = typename L::Ref;
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  if (tid == 0) {
    front0[0] = NodePair<Ref>{L::root(TA), L::root(TB)};
    st->n[0] = 1;
  }
  grid.sync();
  NodePair<Ref>* cur = front0;
  NodePair<Ref>* nxt = front1;
  for (unsigned level = 0;; level++) {
    const uint64_t n = load_cg(&st->n[level % 3]);
    if (n == 0 || (load_cg(&st->overflow) & 3u)) break;  // uniform over the grid: written before the last barrier
    if (tid == 0) {
      st->n[(level + 2) % 3] = 0;
      st->node_pairs_tested += n;
      st->levels = level + 1;
      if (n > st->max_frontier) st->max_frontier = n;
    }
    unsigned long long* next_n = &st->n[(level + 1) % 3];
    for (uint64_t base = tid - (tid & 31u); base < n; base += nthreads) {  // warp-uniform trip count
      const uint64_t i = base + (tid & 31u);
      const bool live = i < n;
      unsigned emit = 0, emit_leaf = 0;
      typename L::Node na, nb;
      NodePair<Ref> p{};
      if (live) {
        p = load_cg(cur + i);
        L::decode(TA, p.a, na);
        L::decode_cold(TA, p.a, na);
        L::decode(TB, p.b, nb);
        L::decode_cold(TB, p.b, nb);
        bool hit;
        if constexpr (L::kFamily == SCION_FAMILY_DOP14) {
          // intersects_dop_dop, dop.scion:81-90
          hit = aabb_overlap(na.lo1, na.hi1, nb.lo1, nb.hi1) && !(na.lo2.x > nb.hi2.x || nb.lo2.x > na.hi2.x) && !(na.lo2.y > nb.hi2.y || nb.lo2.y > na.hi2.y) &&
                !(na.lo2.z > nb.hi2.z || nb.lo2.z > na.hi2.z) && !(na.lo2.w > nb.hi2.w || nb.lo2.w > na.hi2.w);
        } else {
          hit = aabb_overlap(na.low, na.high, nb.low, nb.high);
        }
        if (hit) {
          const bool la = na.variant == L::kLeaf, lb = nb.variant == L::kLeaf;
          if (la && lb) emit_leaf = 1;
          else emit = (!la && !lb) ? 4u : 2u;
        }
      }
      const unsigned long long slot = warp_append(next_n, emit);
      const unsigned long long lslot = warp_append(&st->leaf_pairs, emit_leaf);
      if (emit) {
        if (slot + emit > front_capacity) {
          atomicOr(&st->overflow, 1u);
        } else {
          const bool la = na.variant == L::kLeaf, lb = nb.variant == L::kLeaf;
          if (!la && !lb) {
            nxt[slot + 0] = NodePair<Ref>{na.left, nb.left};
            nxt[slot + 1] = NodePair<Ref>{na.left, nb.right};
            nxt[slot + 2] = NodePair<Ref>{na.right, nb.left};
            nxt[slot + 3] = NodePair<Ref>{na.right, nb.right};
          } else if (!la) {
            nxt[slot + 0] = NodePair<Ref>{na.left, p.b};
            nxt[slot + 1] = NodePair<Ref>{na.right, p.b};
          } else {
            nxt[slot + 0] = NodePair<Ref>{p.a, nb.left};
            nxt[slot + 1] = NodePair<Ref>{p.a, nb.right};
          }
        }
      }
      if (emit_leaf) {
        if (lslot + 1 > leaf_capacity) atomicOr(&st->overflow, 2u);
        else leaves[lslot] = LeafPair{(uint32_t)na.data.begin, (uint32_t)(na.data.end - na.data.begin), (uint32_t)nb.data.begin, (uint32_t)(nb.data.end - nb.data.begin)};
      }
    }
    grid.sync();
    NodePair<Ref>* t = cur; cur = nxt; nxt = t;
  }
  // foreach t1 in data1 { foreach t2 in data2 { if intersects(t1, t2) insert } } — one thread per leaf pair
  static_assert(L::kStride_primitives == 36, "Triangle stride");
  if (load_cg(&st->overflow) & 3u) return;
  const uint64_t nl = load_cg(&st->leaf_pairs);
  unsigned long long tests = 0;
  for (uint64_t i = tid; i < nl; i += nthreads) {
    const LeafPair lp = load_cg(leaves + i);
    for (uint32_t a = 0; a < lp.a_count; a++) {
      float ta[9];
      load_triangle36(TA.buf[L::kBuf_primitives], lp.a_begin + a, ta);
      for (uint32_t b = 0; b < lp.b_count; b++) {
        float tb[9];
        load_triangle36(TB.buf[L::kBuf_primitives], lp.b_begin + b, tb);
        tests++;
        if (sat_triangles(ta, tb)) {
          const unsigned long long slot = atomicAdd(&st->out_pairs, 1ull);
          if (slot < capacity) out[slot] = scion_pair{lp.a_begin + a, lp.b_begin + b};
          else atomicOr(&st->overflow, 4u);
        }
      }
    }
  }
  if (tests) atomicAdd(&st->tri_tests, tests);
}

}  // namespace scion
