// Side treelet of the TOP LEVELS of a binary tree (north_star: "stage the BVH's top levels into shared memory with
// TMA bulk copies").  The node array of every index-referenced binary layout is in preorder (left child
// at this+1), so a prefix of the array is the left spine, not the top of the tree; the top K levels are therefore
// gathered ONCE per tree into a small side buffer in heap order:
//     slot s            record of the node (byte copy of its main-array record, L::kStageStride bytes)
//     slot 2s+1, 2s+2   its left / right child, if the node is an interior
//   [ records: (2^K - 1) x stride ][ main-array index of every slot: (2^K - 1) x u32 ]   (0xffffffff = empty slot)
// chrt2_kernel<L, ..., TL = K> copies the buffer into shared memory with one cp.async.bulk per CTA and serves visits of
// those nodes from there.  The treelet is a cache: it is not counted in bytes/prim.
#pragma once
#include "scion_rt.cuh"

namespace scion {

constexpr uint32_t kTreeletEmpty = 0xffffffffu;

template <class L>
constexpr size_t treelet_bytes(int levels) {
  const size_t slots = ((size_t)1 << levels) - 1;
  return (slots * L::kStageStride + slots * 4 + 15) & ~(size_t)15;
}

// one CTA, level-synchronous: the slots of level l only read slots of level l-1
template <class L>
__global__ void build_treelet_kernel(const TreeView T, int levels, uint8_t* __restrict__ out) {
  constexpr int NW = (int)(sizeof(typename L::Fetched) / 4);
  const uint32_t slots = (1u << levels) - 1u;
  uint32_t* rec = reinterpret_cast<uint32_t*>(out);
  uint32_t* orig = reinterpret_cast<uint32_t*>(out + (size_t)slots * L::kStageStride);
  for (int l = 0; l < levels; l++) {
    const uint32_t first = (1u << l) - 1u, count = 1u << l;
    for (uint32_t k = threadIdx.x; k < count; k += blockDim.x) {
      const uint32_t s = first + k;
      uint32_t idx = kTreeletEmpty;
      if (s == 0u) {
        idx = (uint32_t)L::root(T);
      } else {
        const uint32_t pidx = orig[(s - 1u) >> 1];
        if (pidx != kTreeletEmpty) {
          typename L::Node pn;
          L::decode(T, (typename L::Ref)pidx, pn);
          if (pn.variant != L::kLeaf) idx = (uint32_t)((s & 1u) ? pn.left : pn.right);
        }
      }
      orig[s] = idx;
      typename L::Fetched w;
#pragma unroll
      for (int i = 0; i < NW; i++) w.w[i] = 0u;
      if (idx != kTreeletEmpty) L::fetch(T, (typename L::Ref)idx, w);
#pragma unroll
      for (int i = 0; i < NW; i++) rec[(size_t)s * NW + i] = w.w[i];
    }
    __syncthreads();
  }
}

}  // namespace scion
