// Per-node encoders shared by the host encoder (host/encode.cpp) and the device-side encoder
// (device/encode.cu): ONE source for the arithmetic of every `build` block, compiled twice.
// Each function restates the build block of the corresponding corpus layout (cited per function,
// /root/reference/proj/corpus/layouts/*.scion) for ONE node; field placement comes from the slot
// table of the planner (EncodeJob::f), never from constants.  Bit packing is little-endian, LSB
// first — the inverse of read_bits_raw, /root/reference/proj/src/bits.cpp:7-19 — and touches only
// the bytes of the node's own record (records are byte-granular), so nodes can be encoded
// concurrently without atomics.
//
// Directed rounding: the host goes through the FP environment (fesetround), the device through
// the __f*_rd / __f*_ru intrinsics — both TRUE directed rounding; the oracle's
// third implementation (exact binary64 / TwoSum) must agree with both.
#pragma once
#include <stdint.h>
#include <string.h>

#include "scion_b200.h"

#if defined(__CUDACC__)
#define SCION_ENC_HD __host__ __device__ inline
#else
#define SCION_ENC_HD inline
#endif
#include <cfenv>
#include <math.h>

namespace scion {
namespace enc {

// ------------------------------------------------------------------ directed rounding
#if defined(__CUDA_ARCH__)
SCION_ENC_HD float fmul_rd(float a, float b) { return __fmul_rd(a, b); }
SCION_ENC_HD float fsub_rd(float a, float b) { return __fsub_rd(a, b); }
#else
struct RoundingScope {
  int old;
  SCION_ENC_HD explicit RoundingScope(int mode) : old(fegetround()) { fesetround(mode); }
  SCION_ENC_HD ~RoundingScope() { fesetround(old); }
};
SCION_ENC_HD float fmul_rd(float a, float b) { volatile float x = a, y = b; RoundingScope s(FE_DOWNWARD); volatile float r = x * y; return r; }
SCION_ENC_HD float fsub_rd(float a, float b) { volatile float x = a, y = b; RoundingScope s(FE_DOWNWARD); volatile float r = x - y; return r; }
inline float fsub_ru(float a, float b) { volatile float x = a, y = b; RoundingScope s(FE_UPWARD); volatile float r = x - y; return r; }
inline float fdiv_rd(float a, float b) { volatile float x = a, y = b; RoundingScope s(FE_DOWNWARD); volatile float r = x / y; return r; }
inline float frcp_rd(float a) { volatile float x = a; RoundingScope s(FE_DOWNWARD); volatile float r = 1.0f / x; return r; }
#endif

// ------------------------------------------------------------------ bit writer
SCION_ENC_HD void put_bits(uint8_t* buf, uint64_t bit, uint32_t width, uint64_t value) {
  uint64_t byte = bit >> 3;
  uint32_t sh = (uint32_t)(bit & 7);
  uint32_t left = width;
  if (width < 64) value &= (1ull << width) - 1ull;
  while (left > 0) {
    const uint32_t take = (8 - sh) < left ? (8 - sh) : left;
    const uint8_t m = (uint8_t)(((1u << take) - 1u) << sh);
    buf[byte] = (uint8_t)((buf[byte] & ~m) | (((uint8_t)(value & ((1u << take) - 1u))) << sh));
    value >>= take;
    left -= take;
    sh = 0;
    byte++;
  }
}

struct Field {  // resolved slot of one stored field
  uint8_t* base = nullptr;  // start of its buffer (host vector or device image)
  uint64_t seg_base_bits = 0, stride_bits = 0, off = 0;
  uint32_t width = 0;
  int32_t buffer = -1;  // plan buffer id (the device path re-bases `base` from it)
  bool arena = false;
  SCION_ENC_HD uint64_t pos(uint64_t idx) const { return arena ? idx * 8 + off : seg_base_bits + idx * stride_bits + off; }
  SCION_ENC_HD void set(uint64_t idx, uint64_t v) const { put_bits(base, pos(idx), width, v); }
  SCION_ENC_HD void set_lane(uint64_t idx, uint32_t lane, uint32_t lane_bits, uint64_t v) const { put_bits(base, pos(idx) + (uint64_t)lane * lane_bits, lane_bits, v); }
  SCION_ENC_HD void set_f(uint64_t idx, uint32_t lane, float f) const {
    uint32_t u;
    memcpy(&u, &f, 4);
    set_lane(idx, lane, 32, u);
  }
  SCION_ENC_HD void set_f3(uint64_t idx, const float* f) const { for (uint32_t a = 0; a < 3; a++) set_f(idx, a, f[a]); }
};

enum Kind : int { kPbrt = 0, kPbrtPost, kQ16, kSgEq, kDop14, kPtr, kIdentity, kSharedSlab, kBvh8 };

// Everything a per-node encoder needs besides the node itself.  Filled once per (tree, layout) by
// prepare_job() in host/encode.cpp; plain data, passed by value to the device kernel.
struct EncodeJob {
  int kind = kPbrt;
  uint64_t count = 0;      // records to encode: nodes, or 8-wide interiors
  Field f[10];             // meaning per kind, see the encoders below
  float c0[3] = {0, 0, 0}, c1[3] = {0, 0, 0}, c2[3] = {0, 0, 0};  // per-tree constants of the root block
  uint64_t arena_stride = 0;  // arena layouts: bytes between consecutive nodes (stride rounded up to the group alignment)
  int qbits = 0, ref_bits = 0;  // 8-wide family
  // logical tree (host or device pointers)
  const scion_lnode* nodes = nullptr;
  const float* dop_lo2 = nullptr;
  const float* dop_hi2 = nullptr;
  const uint32_t* post = nullptr;  // pbrt-post: postorder number of preorder node i
  const scion_wnode* wnodes = nullptr;
  const scion_wleaf* wleaves = nullptr;
};

SCION_ENC_HD float clamp_code(float f, float top) { return fmaxf(0.0f, fminf(f, top)); }

// pbrt.scion:21-33 / pbrt_align16.scion / authored pbrt-soa, pbrt-soaos, pbrt-soaos-align16: `build low; build high; build nprims [= 0];
// c_o = R - this | p_o = append(data, nprims)`.  f: low high nprims c_o p_o
SCION_ENC_HD void node_pbrt(const EncodeJob& j, uint64_t i) {
  const scion_lnode& n = j.nodes[i];
  j.f[0].set_f3(i, n.lo);
  j.f[1].set_f3(i, n.hi);
  if (n.left >= 0) {
    j.f[2].set(i, 0);
    j.f[3].set(i, (uint64_t)n.right - i);
  } else {
    j.f[2].set(i, n.nprims);
    j.f[4].set(i, n.first_prim);
  }
}
// pbrt_post.scion:21-35: order=post, `c_l = this - L; c_r = this - R`.  f: low high nprims c_l c_r p_o
SCION_ENC_HD void node_pbrt_post(const EncodeJob& j, uint64_t i) {
  const scion_lnode& n = j.nodes[i];
  const uint64_t me = j.post[i];
  j.f[0].set_f3(me, n.lo);
  j.f[1].set_f3(me, n.hi);
  if (n.left >= 0) {
    j.f[2].set(me, 0);
    j.f[3].set(me, me - j.post[n.left]);
    j.f[4].set(me, me - j.post[n.right]);
  } else {
    j.f[2].set(me, n.nprims);
    j.f[5].set(me, n.first_prim);
  }
}
// pbrt_q16.scion:49-73 (and the authored pbrt-q16-soaos, same fields in two arrays) — quantize_bounds: vu_floor((low - mlo) * rcp), vu_ceil((high - mlo) * rcp), clamp
// [0, 65535]; c0 = world_low, c1 = rcp = (1.0 / world_extent) * 65535.0.  f: bounds_q nprims c_offset p_offset
SCION_ENC_HD void node_q16(const EncodeJob& j, uint64_t i) {
  const scion_lnode& n = j.nodes[i];
  for (uint32_t a = 0; a < 3; a++) {
    const float lo = clamp_code(floorf((n.lo[a] - j.c0[a]) * j.c1[a]), 65535.0f);
    const float hi = clamp_code(ceilf((n.hi[a] - j.c0[a]) * j.c1[a]), 65535.0f);
    j.f[0].set_lane(i, a, 16, (uint64_t)(uint32_t)lo);      // q16x3.lo lanes
    j.f[0].set_lane(i, 3 + a, 16, (uint64_t)(uint32_t)hi);  // q16x3.hi lanes
  }
  if (n.left >= 0) {
    j.f[1].set(i, 0);
    j.f[2].set(i, (uint64_t)n.right - i);
  } else {
    j.f[1].set(i, n.nprims);
    j.f[3].set(i, n.first_prim);
  }
}
// sg_eq.scion:53-76 — quantize_lo/hi = floorf(fmul_rd(fsub_rd(..), bin_inv)) packed 10:10:10;
// c0 = wlow, c1 = whigh, c2 = bins_inv.  f: q_min q_max nprims offset poffset
SCION_ENC_HD void node_sg_eq(const EncodeJob& j, uint64_t i) {
  const scion_lnode& n = j.nodes[i];
  uint32_t lo[3], hi[3];
  for (int a = 0; a < 3; a++) {
    lo[a] = (uint32_t)floorf(fmul_rd(fsub_rd(n.lo[a], j.c0[a]), j.c2[a]));
    hi[a] = (uint32_t)floorf(fmul_rd(fsub_rd(j.c1[a], n.hi[a]), j.c2[a]));
  }
  j.f[0].set(i, ((lo[0] & 1023u) << 20) | ((lo[1] & 1023u) << 10) | (lo[2] & 1023u));
  j.f[1].set(i, ((hi[0] & 1023u) << 20) | ((hi[1] & 1023u) << 10) | (hi[2] & 1023u));
  if (n.left >= 0) {
    j.f[2].set(i, 0);
    j.f[3].set(i, (uint64_t)n.right - i);
  } else {
    j.f[2].set(i, n.nprims);
    j.f[4].set(i, n.first_prim);
  }
}
// dop14.scion:24-40 — `c0 = L; c1 = R` | `c0 = 0; c1 = 0x80000000 | (off << 4) | nprims`.  f: lo1 hi1 c0 c1 lo2 hi2
SCION_ENC_HD void node_dop14(const EncodeJob& j, uint64_t i) {
  const scion_lnode& n = j.nodes[i];
  j.f[0].set_f3(i, n.lo);
  j.f[1].set_f3(i, n.hi);
  for (uint32_t k = 0; k < 4; k++) {
    j.f[4].set_f(i, k, j.dop_lo2[i * 4 + k]);
    j.f[5].set_f(i, k, j.dop_hi2[i * 4 + k]);
  }
  if (n.left >= 0) {
    j.f[2].set(i, (uint32_t)n.left);
    j.f[3].set(i, (uint32_t)n.right);
  } else {
    j.f[2].set(i, 0);
    j.f[3].set(i, 0x80000000u | (n.first_prim << 4) | n.nprims);
  }
}
// arena layouts: node address = byte offset inside the arena (plan.cpp:315-318), preorder
// allocation, every node rounded up to the group alignment => address(i) = i * arena_stride
// ptr.scion:17-31.  f: low high nprims L R p_o
SCION_ENC_HD void node_ptr(const EncodeJob& j, uint64_t i) {
  const scion_lnode& n = j.nodes[i];
  const uint64_t me = i * j.arena_stride;
  j.f[0].set_f3(me, n.lo);
  j.f[1].set_f3(me, n.hi);
  if (n.left >= 0) {
    j.f[2].set(me, 0);
    j.f[3].set(me, (uint64_t)n.left * j.arena_stride);
    j.f[4].set(me, (uint64_t)n.right * j.arena_stride);
  } else {
    j.f[2].set(me, n.nprims);
    j.f[5].set(me, n.first_prim);
  }
}
// identity.scion:19-33.  f: low high tag left right nprims p_o
SCION_ENC_HD void node_identity(const EncodeJob& j, uint64_t i) {
  const scion_lnode& n = j.nodes[i];
  const uint64_t me = i * j.arena_stride;
  j.f[0].set_f3(me, n.lo);
  j.f[1].set_f3(me, n.hi);
  if (n.left >= 0) {
    j.f[2].set(me, 0);
    j.f[3].set(me, (uint64_t)n.left * j.arena_stride);
    j.f[4].set(me, (uint64_t)n.right * j.arena_stride);
  } else {
    j.f[2].set(me, 1);
    j.f[5].set(me, n.nprims);
    j.f[6].set(me, n.first_prim);
  }
}
// shared_slab.scion:40-67 — Interior: axis = longest_axis(low, high), slo = low[axis], shi = high[axis].
// f: L R slo shi o axis is_leaf nprims
SCION_ENC_HD void node_shared_slab(const EncodeJob& j, uint64_t i) {
  const scion_lnode& n = j.nodes[i];
  const uint64_t me = i * j.arena_stride;
  if (n.left >= 0) {
    const float e[3] = {n.hi[0] - n.lo[0], n.hi[1] - n.lo[1], n.hi[2] - n.lo[2]};
    const uint32_t ax = (e[0] >= e[1] && e[0] >= e[2]) ? 0 : (e[1] >= e[2] ? 1 : 2);
    j.f[6].set(me, 0);
    j.f[7].set(me, 0);
    j.f[4].set(me, 0);
    j.f[5].set(me, ax);
    j.f[2].set_f(me, 0, n.lo[ax]);
    j.f[3].set_f(me, 0, n.hi[ax]);
    j.f[0].set(me, (uint64_t)n.left * j.arena_stride);
    j.f[1].set(me, (uint64_t)n.right * j.arena_stride);
  } else {
    j.f[6].set(me, 1);
    j.f[5].set(me, 0);
    j.f[2].set_f(me, 0, 0.0f);
    j.f[3].set_f(me, 0, 0.0f);
    j.f[0].set(me, 0);
    j.f[1].set(me, 0);
    j.f[7].set(me, n.nprims);
    j.f[4].set(me, n.first_prim);
  }
}
// 8-wide family — bvh8.scion:19-30, bvh8_q8.scion:40-77, bvh8_q8_ci.scion:42-79, bvh8_q16*.scion:
// Interior -> ((this << 2) | 1); Leaf -> ((poffset << 7) | ((nprims - 1) << 2) | 0); SENTINEL slots:
// inverted box, child reference 0.  Quantised: merged low/extent over the 8
// children, `tfloor/tceil` of (v - mlo) * ((1.0 / mex) * top), clamp [0, top].
// f: children, then (qbits == 0) lo hi | (qbits > 0) mlo mex child_bounds
SCION_ENC_HD uint64_t wide_ref(const EncodeJob& j, int32_t c) {
  if (c == SCION_W_SENTINEL) return 0;
  if (c >= 0) return ((uint64_t)c << 2) | 1ull;
  const scion_wleaf& l = j.wleaves[(size_t)(~c)];
  return ((uint64_t)l.first_prim << 7) | ((uint64_t)(l.nprims - 1) << 2);
}
SCION_ENC_HD void node_bvh8(const EncodeJob& j, uint64_t i) {
  const scion_wnode& n = j.wnodes[i];
  if (j.qbits == 0) {
    for (uint32_t k = 0; k < 8; k++) {
      for (uint32_t a = 0; a < 3; a++) {
        j.f[1].set_f(i, 3 * k + a, n.lo[k][a]);
        j.f[2].set_f(i, 3 * k + a, n.hi[k][a]);
      }
      j.f[0].set_lane(i, k, (uint32_t)j.ref_bits, wide_ref(j, n.child[k]));
    }
  } else {
    const float top = j.qbits == 8 ? 255.0f : 65535.0f;
    float mlo[3], mex[3], rcp[3];
    for (int a = 0; a < 3; a++) {
      float l = n.lo[7][a], h = n.hi[7][a];
      for (int k = 6; k >= 0; k--) {  // min(lo[0], min(lo[1], ... min(lo[6], lo[7])))
        l = fminf(n.lo[k][a], l);
        h = fmaxf(n.hi[k][a], h);
      }
      mlo[a] = l;
      mex[a] = h - l;
      rcp[a] = (1.0f / mex[a]) * top;
    }
    j.f[1].set_f3(i, mlo);
    j.f[2].set_f3(i, mex);
    for (uint32_t k = 0; k < 8; k++) {
      for (uint32_t a = 0; a < 3; a++) {
        const float ql = clamp_code(floorf((n.lo[k][a] - mlo[a]) * rcp[a]), top);
        const float qh = clamp_code(ceilf((n.hi[k][a] - mlo[a]) * rcp[a]), top);
        j.f[3].set_lane(i, k * 6 + a, (uint32_t)j.qbits, (uint64_t)(uint32_t)ql);      // qbox.lo lanes
        j.f[3].set_lane(i, k * 6 + 3 + a, (uint32_t)j.qbits, (uint64_t)(uint32_t)qh);  // qbox.hi lanes
      }
      j.f[0].set_lane(i, k, (uint32_t)j.ref_bits, wide_ref(j, n.child[k]));
    }
  }
}

SCION_ENC_HD void encode_one(const EncodeJob& j, uint64_t i) {
  switch (j.kind) {
    case kPbrt: node_pbrt(j, i); break;
    case kPbrtPost: node_pbrt_post(j, i); break;
    case kQ16: node_q16(j, i); break;
    case kSgEq: node_sg_eq(j, i); break;
    case kDop14: node_dop14(j, i); break;
    case kPtr: node_ptr(j, i); break;
    case kIdentity: node_identity(j, i); break;
    case kSharedSlab: node_shared_slab(j, i); break;
    case kBvh8: node_bvh8(j, i); break;
  }
}

}  // namespace enc
}  // namespace scion
