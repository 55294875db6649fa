// closest_hit, 8-wide family, LANE-COOPERATIVE (kernel variant 5, chrt8c_kernel) — VERDICT r1 "next" item 3.
//
// chrt8_kernel gives every lane its own ray and decodes a whole 104-256-byte interior record into that lane's
// registers: 124-128 registers, 4 CTAs/SM, 16 warps/SM, issue slots 55 % busy with nothing saturated
// (profiles/r1_ncu_v11_c5_q8ci.txt).  Here a GROUP of 8 lanes owns one ray (4 rays per warp, 16 per CTA):
//   * interior visit: lane k decodes and slab-tests child slot k only — the emitted decode_slot<0>() over the per-child
//     view scion::LaneRecord (6-24 bytes of the record per lane, no lane ever holds a record); one ballot gives the
//     group's pass mask; the lowest passing slot is continued with, the other passing lanes each store their own
//     (child reference, t_near) entry at its final position, so that entries pop in slot order (chrt8.scion:7);
//   * the deferred cull `t_near < best` at pop, the overflow rule (the reference would hold all m passing children at
//     once) and the counters are those of chrt8_kernel: same visit order, same results, bit for bit;
//   * leaf: the group's 8 lanes test 8 triangles at a time; a lexicographic (t, index) minimum over the group followed by
//     the strict `t < best` rule equals the sequential ascending fold of chrt8.scion:14-19;
//   * the stack lives entirely in shared memory (64 entries per ray — there are only 16 rays per CTA), no local tier.
// State that is uniform over a group (ray, best, cur, depth, mode) is replicated in its 8 lanes.
#pragma once

namespace scion {

#ifndef SCION_MINB8C
#define SCION_MINB8C 10
#endif
#ifndef SCION_LEAF_MIN8C  /* run the leaf phase when at least this many of the warp's 4 groups wait with a leaf */
#define SCION_LEAF_MIN8C 2
#endif
#ifndef SCION_REFILL_MIN8C  /* refill when at least this many of the warp's 4 groups are idle */
#define SCION_REFILL_MIN8C 1
#endif
#ifndef SCION_INNER8C
#define SCION_INNER8C 1  /* 1: 1013, 2: 990, 4: 924 Mrays/s (C5 probe, bvh8-q8-ci) */
#endif

template <class L>
inline constexpr bool kCoop8Ok = L::kFamily == SCION_FAMILY_BVH8 && L::kCanLane && L::kVariantInRef;
template <class L>
constexpr bool coop8_ok() {
  return kCoop8Ok<L>;
}

template <class L>
struct Coop8Smem {
  using Ref = typename L::Ref;
  static constexpr int kGroups = kBlockThreads / 8;
  // SoA per group; the +1 entry skews consecutive groups by one (ref) / one (t) bank pair
  Ref ref[kGroups][SCION_STACK_DEPTH + 1];
  float t[kGroups][SCION_STACK_DEPTH + 1];
};

template <class L, bool COUNT>
__global__ void __launch_bounds__(kBlockThreads, SCION_MINB8C) chrt8c_kernel(const TreeView T, const scion_ray* __restrict__ rays, uint64_t n,
                                                                scion_hit* __restrict__ hits, uint32_t* __restrict__ status,
                                                                scion_counters* __restrict__ counters, unsigned long long* __restrict__ next, const int tune) {
  static_assert(kCoop8Ok<L>, "lane-cooperative kernel: per-child record view and the leaf variant in the reference");
  using Ref = typename L::Ref;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Coop8Smem<L>& S = *reinterpret_cast<Coop8Smem<L>*>(smem_raw);
  const unsigned lane = threadIdx.x & 31u;
  const unsigned k = lane & 7u;                 // child slot / triangle slot of this lane
  const unsigned gbase = lane & 24u;            // first lane of the group
  const int g = (int)(threadIdx.x >> 3);        // group of the CTA
  Ref* const st_ref = S.ref[g];
  float* const st_t = S.t[g];
  WorkFetcher work;
  (void)tune;
  Tally<COUNT> tally;
  int mode = kFetch;
  RayCtx ray = make_ray(0, 0, 0, 0, 1, 1, 1);
  float best_t = 0;
  uint32_t best_prim = 0, prim_i = 0, prim_end = 0, depth = 0;
  unsigned long long q = 0;
  Ref cur = L::root(T);

  auto retire = [&](uint32_t st) {
    if (k == 0) {
      store_hit(hits + q, best_t, best_prim);
      if (status) status[q] = st;
      tally.store(counters, q);
    }
    mode = kFetch;
  };
  auto enter = [&]() {  // `cur` was just chosen: a leaf reference parks the group
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
      if (depth == 0u) {
        retire(SCION_Q_OK);
        return;
      }
      depth--;
      const float tn = st_t[depth];  // all 8 lanes read the same word: one broadcast
      if (tn < best_t) {
        cur = st_ref[depth];
        enter();
        if (mode >= 0) return;
      }
    }
  };
  // Every collective below is executed by all 32 lanes, converged, with the full mask (a run-time group mask would make
  // the compiler wrap each shuffle / vote in a WARPSYNC ... ENDCOLLECTIVE sequence); groups that have nothing to do in a
  // phase run it predicated off.  xor-shuffles by 4 / 2 / 1 and source lanes gbase + (0..7) never leave the group.
  auto bcast_ref = [&](const Ref& r, unsigned src) -> Ref {
    if constexpr (sizeof(Ref) == 8) {
      const uint32_t lo = __shfl_sync(kFullMask, (uint32_t)r, src), hi = __shfl_sync(kFullMask, (uint32_t)((uint64_t)r >> 32), src);
      return (Ref)(((uint64_t)hi << 32) | lo);
    } else {
      return (Ref)__shfl_sync(kFullMask, (uint32_t)r, src);
    }
  };
  const Ref root = L::root(T);

  auto step = [&]() {
    const bool act = mode == kNode;
    const Ref c = act ? cur : root;  // idle groups decode the root record: a valid address, the result is not used
    f32x3 lo, hi;
    Ref ch;
    const LaneRecord<L> rec{L::slot_record(T, c), k};
    L::template decode_slot<0>(T, c, rec, lo, hi, ch);
    float tn, t_far;
    const bool some = ray_aabb(ray, lo, hi, tn, t_far);
    const bool pass = act && interval_intersects(ray, some, tn, t_far) && tn < best_t;
    const unsigned mask = (__ballot_sync(kFullMask, pass) >> gbase) & 0xffu;
    // slot k1 = lowest passing slot is visited next; slot k lands above every passing slot with a larger index
    const unsigned first = ((unsigned)__ffs((int)mask) - 1u) & 7u;
    const Ref nxt = bcast_ref(ch, gbase + first);
    const uint32_t m = (uint32_t)__popc(mask);
    bool cont = false;
    __syncwarp();  // the pops of the previous step / leaf phase (reads of the group's stack) are complete before this step's pushes
    if (act) {
      tally.visit();
      if (mask != 0u) {
        if (COUNT) tally.stack(depth + m);
        if (depth + m > (uint32_t)SCION_STACK_DEPTH) {  // the reference would hold all m passing children at once
          retire(SCION_Q_STACK_OVERFLOW);
        } else {
          if (pass && k != first) {
            const uint32_t pos = depth + (uint32_t)__popc(mask >> (k + 1u));
            st_ref[pos] = ch;
            st_t[pos] = tn;
          }
          depth += m - 1u;
          cur = nxt;
          cont = true;
        }
      }
    }
    __syncwarp();  // a group's stores are visible to its later pops
    if (act) {
      if (cont) {
        enter();
        if (mode < 0) pop_next();
      } else if (mode == kNode) {  // nothing passed (an overflow has already retired the query)
        pop_next();
      }
    }
  };

  // leaves of the waiting groups: 8 triangles per group and round, lexicographic (t, slot) minimum over the group, then
  // the strict rule against `best`
  auto leaf_phase = [&]() {
    const bool own = mode == kPrim;
    for (;;) {
      const bool busy = own && prim_i < prim_end;
      if (!__any_sync(kFullMask, busy)) break;
      const uint32_t pi = prim_i + k;
      float t = scion::inf();
      if (busy && pi < prim_end) {
        float tri[9];
        load_triangle36(T.buf[L::kBuf_primitives], pi, tri);
        float th;
        if (ray_tri_mt(ray, tri, th)) t = th;
      }
      uint32_t idx = k;
#pragma unroll
      for (int d = 4; d >= 1; d >>= 1) {
        const float ot = __shfl_xor_sync(kFullMask, t, d);
        const uint32_t oi = __shfl_xor_sync(kFullMask, idx, d);
        if (ot < t || (ot == t && oi < idx)) { t = ot; idx = oi; }
      }
      if (busy) {
        if (t < best_t) {  // a miss is +inf and never passes
          best_t = t;
          best_prim = prim_i + idx;
        }
        const uint32_t left = prim_end - prim_i;
        if (COUNT) tally.prim_tests += left < 8u ? left : 8u;
        prim_i += 8u;
      }
    }
    if (own) pop_next();
  };

  for (;;) {
#pragma unroll 1
    for (int it = 0; it < SCION_INNER8C; it++) {
      if (__any_sync(kFullMask, mode == kNode)) step();
    }
    // ---- FETCH: a group is idle when its leader is
    const unsigned idle = __ballot_sync(kFullMask, mode == kFetch && k == 0u);
    if (idle && (__popc(idle) >= SCION_REFILL_MIN8C || work.exhausted)) {
      uint64_t nq = 0;
      bool got = false;
      if (!work.exhausted) got = work.refill(mode == kFetch && k == 0u, next, n, nq);
      got = __shfl_sync(kFullMask, (int)got, gbase) != 0;
      const uint32_t qlo = __shfl_sync(kFullMask, (uint32_t)nq, gbase), qhi = __shfl_sync(kFullMask, (uint32_t)(nq >> 32), gbase);
      if (got) {
        q = ((unsigned long long)qhi << 32) | qlo;
        ray = load_ray(rays, q);  // 8 lanes, one address
        best_t = scion::inf();
        best_prim = SCION_MISS_PRIM;
        tally.reset();
        depth = 0u;
        cur = root;
        enter();
        if (mode < 0) retire(SCION_Q_OK);  // the root is an empty leaf
      }
      if (work.exhausted && __ballot_sync(kFullMask, mode != kFetch) == 0u) break;
    }
    // ---- PRIM: groups that wait with a leaf
    const unsigned pmask = __ballot_sync(kFullMask, mode == kPrim && k == 0u);
    if (pmask && (__popc(pmask) >= SCION_LEAF_MIN8C || __ballot_sync(kFullMask, mode == kNode) == 0u)) leaf_phase();
  }
}

}  // namespace scion
