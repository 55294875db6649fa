// Measured-and-rejected closest-hit kernels, kept selectable for A/B timing and covered by identity tests:
//   chrt2d_kernel  two rays per lane, software-pipelined record fetch   (kernel variant 3, SCION_DUAL)
//   chrt2x_kernel  pair step: a step expands a node, both child records fetched together   (SCION_PAIR_STEP)
// Included at the end of traverse.cuh (they use its lane stack, work fetcher and cooperative leaf phase); nothing
// here is on the default path.
#pragma once

namespace scion {

// ------------------------------------------------------------------------------------------
// closest_hit, binary family, TWO rays per lane (kernel v14, SCION_DUAL=1) — for layouts whose record is one vector load
// (L::kCanFetch: pbrt, pbrt-align16, pbrt-q16, sg-eq-align16).
//
// chrt2_kernel is bound by the dependent chain of one step (pop -> address -> record load -> decode -> test -> push/pop)
// times the visits of a ray, with the register file fixing how many chains an SM holds.  Here every lane
// owns two independent rays ("slots").  A step of slot s consumes the record that was fetched at the END of slot s's
// previous step and ends by issuing the fetch of its next record (emitted L::fetch / L::decode_fetched), so the load of
// one slot is in flight while the other slot's step executes.  Everything else is the v11 machine run once per slot:
// same visit order, same predicated push/pop, same cooperative leaf phase, same results bit for bit.  The
// counter-instrumented build stays on chrt2_kernel (identical results by construction, tests compare the two).
// ------------------------------------------------------------------------------------------
#ifndef SCION_DUAL
#define SCION_DUAL 0
#endif
#ifndef SCION_MINB2D
#define SCION_MINB2D 6
#endif
#ifndef SCION_DUAL_MERGED
#define SCION_DUAL_MERGED 0
#endif
#ifndef SCION_STACK_SMEM_D  /* shared-memory stack window of one CTA, both slots together */
#define SCION_STACK_SMEM_D (16 * 1024)
#endif
template <class L>
constexpr bool dual_ok() {
  return L::kCanFetch && !L::kHasCold && L::kFamily != SCION_FAMILY_DOP14 && std::is_integral<typename L::Ref>::value;
}
template <class L>
__global__ void __launch_bounds__(kBlockThreads, SCION_MINB2D) chrt2d_kernel(const TreeView T, const scion_ray* __restrict__ rays, uint64_t n,
                                                                scion_hit* __restrict__ hits, uint32_t* __restrict__ status,
                                                                scion_counters* __restrict__ counters, unsigned long long* __restrict__ next, const int tune) {
  using Ref = typename L::Ref;
  constexpr int kSlotWindow = SCION_STACK_SMEM_D / 2;
  using LS = LaneStack<Ref, kSlotWindow>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ CoopScratch2 coop[kBlockThreads / 32];
  __shared__ RayStash stash[2][kBlockThreads];
  __shared__ unsigned long long stash_q[2][kBlockThreads];
  __shared__ uint2 stash_leaf[2][kBlockThreads];
  Ref deep[2][LS::kDeep];
  uint32_t window = (uint32_t)__cvta_generic_to_shared(smem_raw);
  asm volatile("" : "+r"(window));
  (void)tune; (void)counters;
  WorkFetcher work;
  struct Slot {
    RayCtx ray;
    float best_t;
    uint32_t best_prim;
    Ref cur;
    uint32_t top;
    int mode;
    typename L::Fetched rec;
  } S[2];
#pragma unroll
  for (int s = 0; s < 2; s++) {
    S[s].ray = make_ray(0, 0, 0, 0, 1, 1, 1);
    S[s].best_t = 0;
    S[s].best_prim = 0;
    S[s].cur = L::root(T);
    S[s].top = window + (uint32_t)s * (uint32_t)kSlotWindow + threadIdx.x * 4u;
    S[s].mode = kFetch;
  }

  auto retire = [&](auto SI, uint32_t st) {
    constexpr int s = decltype(SI)::value;
    const uint64_t qq = opaque(stash_q[s][threadIdx.x]);
    store_hit(hits + qq, S[s].best_t, S[s].best_prim);
    if (status) status[qq] = st;
    S[s].mode = kFetch;
  };
  auto pop_or_retire = [&](auto SI) {
    constexpr int s = decltype(SI)::value;
    const uint32_t rel = S[s].top - (window + (uint32_t)s * (uint32_t)kSlotWindow);
    if (rel - LS::kSlot < LS::kSmemBytes) {
      S[s].top -= LS::kSlot;
      LS::load(S[s].top, S[s].cur);
      S[s].mode = kNode;
    } else if (rel < LS::kSlot) {
      retire(SI, SCION_Q_OK);
    } else {
      S[s].top -= LS::kSlot;
      S[s].cur = deep[s][rel / LS::kSlot - 1u - (uint32_t)LS::kSmem];
      S[s].mode = kNode;
    }
  };
  // one node step of slot s; ends by putting the next record's load in flight
  auto step = [&](auto SI) {
    constexpr int s = decltype(SI)::value;
    Slot& X = S[s];
    typename L::Node node;
    L::decode_fetched(T, X.cur, X.rec, node);
    float t_near, t_far;
    const bool some = ray_aabb(X.ray, node.low, node.high, t_near, t_far);
    const bool hit = interval_intersects(X.ray, some, t_near, t_far);
    const bool leaf = node.variant == L::kLeaf;
    const bool p_prim = hit && leaf && (uint32_t)node.data.begin < (uint32_t)node.data.end;
    const bool p_push = hit && !leaf && t_near < X.best_t;
    const uint32_t rel = X.top - (window + (uint32_t)s * (uint32_t)kSlotWindow);
    const bool fast = p_push ? rel < LS::kSmemBytes : rel - LS::kSlot < LS::kSmemBytes;
    if (!(fast || p_prim)) {
      if (p_push) {
        const uint32_t depth = rel / LS::kSlot;
        if (depth + 2u > (uint32_t)SCION_STACK_DEPTH) {
          retire(SI, SCION_Q_STACK_OVERFLOW);
        } else {
          deep[s][depth - (uint32_t)LS::kSmem] = node.right;
          X.top += LS::kSlot;
          X.cur = node.left;
        }
      } else {
        pop_or_retire(SI);
      }
    } else if (p_prim) {
      const uint32_t my_leaf = (uint32_t)__cvta_generic_to_shared(&stash_leaf[s][threadIdx.x]);
      asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(my_leaf), "r"((uint32_t)node.data.begin), "r"((uint32_t)node.data.end));
      X.mode = kPrim;
    } else if (p_push) {
      LS::store(X.top, node.right);
      if constexpr (kPrefetch) L::prefetch(T, node.right);
      X.top += LS::kSlot;
      X.cur = node.left;
    } else {
      X.top -= LS::kSlot;
      LS::load(X.top, X.cur);
    }
    if (X.mode == kNode) L::fetch(T, X.cur, X.rec);
  };
  auto refill = [&](auto SI, bool force) {
    constexpr int s = decltype(SI)::value;
    Slot& X = S[s];
    const unsigned idle = __ballot_sync(kFullMask, X.mode == kFetch);
    if (idle && (force || __popc(idle) >= kRefillMin || work.exhausted)) {
      uint64_t nq;
      if (!work.exhausted && work.refill(X.mode == kFetch, next, n, nq)) {
        X.ray = load_ray(rays, nq);
        stash[s][threadIdx.x] = RayStash{X.ray.dx, X.ray.dy, X.ray.dz, 0u};
        stash_q[s][threadIdx.x] = nq;
        X.best_t = scion::inf();
        X.best_prim = SCION_MISS_PRIM;
        X.top = window + (uint32_t)s * (uint32_t)kSlotWindow + threadIdx.x * 4u;
        X.cur = L::root(T);
        X.mode = kNode;
        L::fetch(T, X.cur, X.rec);
      }
    }
  };
  auto prims = [&](auto SI, bool nothing_else) {
    constexpr int s = decltype(SI)::value;
    Slot& X = S[s];
    const unsigned pmask = __ballot_sync(kFullMask, X.mode == kPrim);
    if (pmask && (__popc(pmask) >= kPrimMin || nothing_else)) {
      const bool own = X.mode == kPrim;
      uint2 range = make_uint2(0u, 0u);
      if (own) range = stash_leaf[s][threadIdx.x];
      uint32_t prim_i = range.x;
      coop_triangles2<L>(T, own, X.ray.ox, X.ray.oy, X.ray.oz, X.ray.tmax, stash[s] + (threadIdx.x & ~31u), prim_i, range.y, X.best_t, X.best_prim,
                         coop[threadIdx.x >> 5]);
      if (own) {
        pop_or_retire(SI);
        if (X.mode == kNode) L::fetch(T, X.cur, X.rec);
      }
    }
  };
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;

  for (;;) {
#pragma unroll 1
    for (int k = 0; k < kInner; k++) {
      if (S[0].mode == kNode) step(I0{});
      if (S[1].mode == kNode) step(I1{});
    }
#if SCION_DUAL_MERGED  // thresholds on the two slots of the warp together (a slot's own events are half as frequent)
    const bool many_idle = __popc(__ballot_sync(kFullMask, S[0].mode == kFetch)) + __popc(__ballot_sync(kFullMask, S[1].mode == kFetch)) >= kRefillMin;
#else
    const bool many_idle = false;
#endif
    refill(I0{}, many_idle);
    refill(I1{}, many_idle);
    if (work.exhausted && __ballot_sync(kFullMask, S[0].mode != kFetch || S[1].mode != kFetch) == 0u) break;
    bool nothing_else = __ballot_sync(kFullMask, S[0].mode == kNode || S[1].mode == kNode) == 0u;
#if SCION_DUAL_MERGED
    nothing_else = nothing_else || __popc(__ballot_sync(kFullMask, S[0].mode == kPrim)) + __popc(__ballot_sync(kFullMask, S[1].mode == kPrim)) >= kPrimMin;
#endif
    prims(I0{}, nothing_else);
    prims(I1{}, nothing_else);
  }
}

// ------------------------------------------------------------------------------------------
// closest_hit, binary family, PAIR step (kernel v10) — for layouts whose reference is a plain
// integer and whose node has no cold segment.
//
// chrt2_kernel visits one node per step: one dependent memory round trip per node visit, and the
// warp waits for its slowest lane every time (profiles/r1_ncu_v8_c5_q16.txt: two out of three
// node loads of a warp include a DRAM access).  The closest-point kernel showed what that costs:
// peeking both children in one step (two loads in flight) is 1.41x faster than one decode per
// step.  Here a step EXPANDS an interior node: it fetches the records of BOTH children together,
// tests both boxes, continues with the left child at once and pushes the right child together
// with the outcome of its (pure) box test:
//     entry = (a, b, key)   interior: a/b = left/right reference, key = t_near
//                           leaf:     a/b = primitive range,    key = t_near | sign bit
//                           box missed / empty leaf: key = +inf ("dead": never passes the cull)
// The reference tests the right child when it is visited — `intersects(ray, box)` (pure) and, for
// interiors, `distmin(ray, box) < best[0]` with the `best` of that moment: the pure part is
// evaluated at push time, the cull `t_near < best` is applied at pop time with the then-current
// `best`, so every decision is the reference's (same argument as the 8-wide deferred cull, SURVEY
// Appendix A).  Dead entries are pushed too, so the stack occupancy — and with it the overflow status
// and the max_stack counter — is the reference's at every moment.  A popped entry needs no memory
// access at all: dependent round trips per ray drop from (visits) to (visits / 2).
//
// MEASURED AND REJECTED (kept behind SCION_PAIR_STEP=1, bit-exact incl. counters and overflow status on
// the whole GPU suite): C5 probe pbrt-q16 1293 Mrays/s against 2190 for the one-node step; pbrt 1320 vs
// 2144, sg-eq 629 vs 963.  A 12-byte entry leaves 8 (12 KB window) stack entries in shared memory where
// incoherent rays average 13, so pushes and pops go to local memory; 16 / 20 KB windows: 1368 / 1463
// (7 CTAs), 24 KB: 1128 (L1 starved).  In the one-node kernel the left child is the next record
// (same sector half of the time) and the right child was L2-prefetched when it was pushed — the
// round trips that matter were already short.
// ------------------------------------------------------------------------------------------
#ifndef SCION_PAIR_STEP
#define SCION_PAIR_STEP 0
#endif
#ifndef SCION_MINB2X
#define SCION_MINB2X 8
#endif
#ifndef SCION_INNERX
#define SCION_INNERX 2
#endif
#ifndef SCION_PRIM_MINX
#define SCION_PRIM_MINX 6
#endif
template <class Ref>
struct PairEntry {
  Ref a, b;
  float key;
};
template <class L>
constexpr bool pair_step_ok() {
  return SCION_PAIR_STEP != 0 && L::kFamily == SCION_FAMILY_BVH2 && !L::kHasCold && std::is_integral<typename L::Ref>::value;
}

#if SCION_PAIR_STEP
template <class L, bool COUNT>
__global__ void __launch_bounds__(kBlockThreads, SCION_MINB2X) chrt2x_kernel(const TreeView T, const scion_ray* __restrict__ rays, uint64_t n,
                                                               scion_hit* __restrict__ hits, uint32_t* __restrict__ status,
                                                               scion_counters* __restrict__ counters, unsigned long long* __restrict__ next, const int tune) {
  using Ref = typename L::Ref;
  using Entry = PairEntry<Ref>;
  using LS = LaneStack<Entry>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ CoopScratch2 coop[kBlockThreads / 32];
  __shared__ RayStash stash[kBlockThreads];
  __shared__ unsigned long long stash_q[kBlockThreads];
  __shared__ uint2 stash_leaf[kBlockThreads];
  Entry deep[LS::kDeep];
  uint32_t window = (uint32_t)__cvta_generic_to_shared(smem_raw);
  asm volatile("" : "+r"(window));
  uint32_t top = window + threadIdx.x * 4u;
  uint32_t my_leaf = (uint32_t)__cvta_generic_to_shared(&stash_leaf[threadIdx.x]);
  asm volatile("" : "+r"(my_leaf));
  WorkFetcher work;
  (void)tune;
  Tally<COUNT> tally;
  int mode = kFetch;
  RayCtx ray = make_ray(0, 0, 0, 0, 1, 1, 1);
  float best_t = 0;
  uint32_t best_prim = 0;
  Ref ea = L::root(T), eb = ea;  // children of the node this lane expands next (mode == kNode)
  constexpr uint32_t kLeafBit = 0x80000000u;

  auto retire = [&](uint32_t st) {
    const uint64_t qq = opaque(stash_q[threadIdx.x]);
    store_hit(hits + qq, best_t, best_prim);
    if (status) status[qq] = st;
    tally.store(counters, qq);
    mode = kFetch;
  };
  auto park = [&](uint32_t b, uint32_t e) {
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(my_leaf), "r"(b), "r"(e));
    mode = kPrim;
  };
  // next pending entry that passes its deferred test, or retire the query
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
      const uint32_t kb = f2u(e.key);
      if (kb & kLeafBit) {  // a leaf whose box the ray intersects: no distance cull (chrt.scion:10)
        park((uint32_t)e.a, (uint32_t)e.b);
        return;
      }
      if (e.key < best_t) {  // interior: `distmin(ray, box) < best[0]` with the best of THIS moment; dead entries are +inf
        ea = e.a;
        eb = e.b;
        mode = kNode;
        return;
      }
    }
  };
  // outcome of visiting one node whose box test is (hit, t_near): what to do with it now / what to remember
  auto classify = [&](const typename L::Node& nd, bool hit, float t_near, Ref& a, Ref& b, float& key) {
    const bool leaf = nd.variant == L::kLeaf;
    if (leaf) {
      a = (Ref)nd.data.begin;
      b = (Ref)nd.data.end;
      key = (hit && (uint32_t)nd.data.begin < (uint32_t)nd.data.end) ? u2f(f2u(t_near) | kLeafBit) : scion::inf();
    } else {
      a = nd.left;
      b = nd.right;
      key = hit ? t_near : scion::inf();
    }
  };

  auto step = [&]() {
    typename L::Node nl, nr;
    L::decode(T, ea, nl);
    L::decode(T, eb, nr);
    if (COUNT) { tally.visit(); tally.visit(); }
    float tl, tr;
    const bool hl = node_test<L>(T, ray, ea, nl, tl, tally);
    const bool hr = node_test<L>(T, ray, eb, nr, tr, tally);
    Ref la, lb, ra, rb;
    float lkey, rkey;
    classify(nl, hl, tl, la, lb, lkey);
    classify(nr, hr, tr, ra, rb, rkey);
    // push the right child (always: reference discipline = pop self, push right, push left)
    const uint32_t rel = top - window;
    if (COUNT) tally.stack(rel / LS::kSlot + 2u);
    if (rel < LS::kSmemBytes) {
      LS::store(top, Entry{ra, rb, rkey});
    } else {
      const uint32_t depth = rel / LS::kSlot;
      if (depth + 2u > (uint32_t)SCION_STACK_DEPTH) {
        retire(SCION_Q_STACK_OVERFLOW);
        return;
      }
      deep[depth - (uint32_t)LS::kSmem] = Entry{ra, rb, rkey};
    }
    top += LS::kSlot;
    // visit the left child now
    const uint32_t lk = f2u(lkey);
    if (lk & kLeafBit) {
      park((uint32_t)la, (uint32_t)lb);
    } else if (lkey < best_t) {
      ea = la;
      eb = lb;
    } else {
      pop_next();
    }
  };

  for (;;) {
#pragma unroll 1
    for (int k = 0; k < SCION_INNERX; k++) {
      if (mode == kNode) step();
    }
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
        // the root is visited here (one node, not a pair)
        const Ref root = L::root(T);
        typename L::Node nd;
        L::decode(T, root, nd);
        tally.visit();
        float t0;
        const bool h0 = node_test<L>(T, ray, root, nd, t0, tally);
        Ref a, b;
        float key;
        classify(nd, h0, t0, a, b, key);
        if (f2u(key) & kLeafBit) {
          park((uint32_t)a, (uint32_t)b);
        } else if (key < best_t) {
          ea = a;
          eb = b;
          mode = kNode;
        } else {
          retire(SCION_Q_OK);
        }
      }
      if (work.exhausted && __ballot_sync(kFullMask, mode != kFetch) == 0u) break;
    }
    const unsigned pmask = __ballot_sync(kFullMask, mode == kPrim);
    if (pmask && (__popc(pmask) >= SCION_PRIM_MINX || __ballot_sync(kFullMask, mode == kNode) == 0u)) {
      const bool own = mode == kPrim;
      uint2 range = make_uint2(0u, 0u);
      if (own) asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(range.x), "=r"(range.y) : "r"(my_leaf));
      uint32_t prim_i = range.x;
      const uint32_t done = coop_triangles2<L>(T, own, ray.ox, ray.oy, ray.oz, ray.tmax, stash + (threadIdx.x & ~31u), prim_i, range.y, best_t,
                                               best_prim, coop[threadIdx.x >> 5]);
      if (COUNT) tally.prim_tests += done;
      if (own) pop_next();
    }
  }
}

#endif  // SCION_PAIR_STEP

}  // namespace scion
