// scion_rt.cuh — the runtime the emitted layout headers (gen/*.cuh) are written against.
//
// It provides the DSL's value types (f32x3, u16x3, records are emitted), the intrinsic table
// of the reference (/root/reference/proj/include/layoutc/sema.hpp:16-34: dot cross select min
// max floorf ceilf abs sum all fmul_rd fadd_rd fsub_rd fsub_ru fdiv_rd frcp_rd), `as` / `to`
// casts (src/sema.cpp:753-786), bit ranges x[a:b], and the record loaders that turn a planned
// element (stride, alignment) into the widest legal read-only vector loads.
//
// Dual mode: under nvcc everything is __device__ code for sm_100a (the product path).  Under a
// plain host compiler the same text compiles with host twins of the intrinsics so that the
// *generated decoders* can be unit-tested on a machine without a GPU (tests only; nothing in the
// product calls the host mode).
#pragma once
#include <stddef.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define SCION_DEV __device__ __forceinline__
#define SCION_HOSTDEV __host__ __device__ __forceinline__
#else
#include <cfenv>
#include <cmath>
#define SCION_DEV inline
#define SCION_HOSTDEV inline
#endif

#ifndef SCION_LDG256
#define SCION_LDG256 1
#endif
#ifndef SCION_CACHE_HINTS
// 0: plain read-only loads.  4 (default): primitive loads bypass L1 allocation and carry an L2 evict_first
// policy — 360 MB of randomly accessed triangles otherwise push the 93 MB node array out of L2 (C5 probe:
// pbrt-q16 +2.0 %, sg-eq +1.1 %, bvh8-q8-ci +0.8 %, closest point +4 %, pbrt -1.5 %, dop14 -0.5 %).
// 1: node records L2 evict_last (±0);  2: 1 + primitives evict_first (+1.7 %);  3: 2 + L1::no_allocate (-3 %).
#define SCION_CACHE_HINTS 4
#endif
#ifndef SCION_LDG_COVER
// byte-granular strides (identity 41 B, pbrt-post 34 B, shared-slab 29 B): 1 = the covering 16-byte quads (3-4 LDG.128 per
// record), 2 = the covering 32-byte sectors (2-3 LDG.256: one L1 wavefront per lane each; identity is L1-tag-bound, l1tex
// 99 % in profiles/r2_ncu_c5_identity.txt).  C5 probe: identity 1225 -> 1273 (+3.9 %), pbrt-post 1436 -> 1448 (+0.8 %);
// bit-exact (profiles/r2_ldg256_probe.txt).
#define SCION_LDG_COVER 2
#endif
#ifndef SCION_I2F_MAGIC
#define SCION_I2F_MAGIC 0
#endif
#ifndef SCION_LDG_PARITY
#define SCION_LDG_PARITY 1
#endif

namespace scion {

// --------------------------------------------------------------------------- device tree view
// Generic, layout-agnostic view of a PhysicalTree resident on the device: buffer base pointers
// in plan order, segment base offsets (plan.cpp:333-347), element counts, and the global slots
// as raw 16-byte cells.  Passed by value as a kernel parameter (constant bank).
#define SCION_MAX_BUFFERS 6
#define SCION_MAX_SEGMENTS 4
#define SCION_MAX_GLOBALS 12
struct TreeView {
  const uint8_t* buf[SCION_MAX_BUFFERS];
  uint64_t seg_base[SCION_MAX_BUFFERS][SCION_MAX_SEGMENTS];
  uint64_t count[SCION_MAX_BUFFERS];
  uint32_t glob[SCION_MAX_GLOBALS][4];
  uint64_t root0;      // root reference, primary component
  float root_carried[6];  // tree-carried components of the root reference (shared-slab)
  // side treelet of the top levels (device/treelet.cuh; a cache, not part of the layout): `treelet_slots` records in
  // heap order followed by their main-array indices, or null
  const uint8_t* treelet;
  uint32_t treelet_slots;
};

// --------------------------------------------------------------------------- vectors
template <class T, int N>
struct vec {
  T v[N];
  SCION_HOSTDEV T& operator[](int i) { return v[i]; }
  SCION_HOSTDEV const T& operator[](int i) const { return v[i]; }
};
template <class T>
struct vec<T, 2> {
  T x, y;
  SCION_HOSTDEV T& operator[](int i) { return i == 0 ? x : y; }
  SCION_HOSTDEV const T& operator[](int i) const { return i == 0 ? x : y; }
};
template <class T>
struct vec<T, 3> {
  T x, y, z;
  SCION_HOSTDEV T& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
  SCION_HOSTDEV const T& operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};
template <class T>
struct vec<T, 4> {
  T x, y, z, w;
  SCION_HOSTDEV T& operator[](int i) { return i == 0 ? x : (i == 1 ? y : (i == 2 ? z : w)); }
  SCION_HOSTDEV const T& operator[](int i) const { return i == 0 ? x : (i == 1 ? y : (i == 2 ? z : w)); }
};
using f32x3 = vec<float, 3>;
using f32x4 = vec<float, 4>;

template <class T> struct is_vec { static constexpr bool value = false; };
template <class T, int N> struct is_vec<vec<T, N>> { static constexpr bool value = true; };

#define SCION_VEC_BINOP(OP)                                                                                  \
  template <class T, int N> SCION_HOSTDEV vec<T, N> operator OP(const vec<T, N>& a, const vec<T, N>& b) {     \
    vec<T, N> r;                                                                                             \
    _Pragma("unroll") for (int i = 0; i < N; i++) r[i] = a[i] OP b[i];                                        \
    return r;                                                                                                \
  }                                                                                                          \
  template <class T, int N, class S> SCION_HOSTDEV vec<T, N> operator OP(const vec<T, N>& a, S b) {           \
    vec<T, N> r;                                                                                             \
    _Pragma("unroll") for (int i = 0; i < N; i++) r[i] = a[i] OP (T)b;                                        \
    return r;                                                                                                \
  }                                                                                                          \
  template <class T, int N, class S> SCION_HOSTDEV vec<T, N> operator OP(S a, const vec<T, N>& b) {           \
    vec<T, N> r;                                                                                             \
    _Pragma("unroll") for (int i = 0; i < N; i++) r[i] = (T)a OP b[i];                                        \
    return r;                                                                                                \
  }
SCION_VEC_BINOP(+)
SCION_VEC_BINOP(-)
SCION_VEC_BINOP(*)
SCION_VEC_BINOP(/)
SCION_VEC_BINOP(&)
SCION_VEC_BINOP(|)
SCION_VEC_BINOP(^)
#undef SCION_VEC_BINOP

struct Slice {  // T[a : b] over a global array: element indices [begin, end)
  uint64_t begin, end;
};
SCION_HOSTDEV Slice make_slice(uint64_t a, uint64_t b) { return Slice{a, b}; }

// --------------------------------------------------------------------------- scalar intrinsics
SCION_HOSTDEV uint32_t f2u(float f) {
#if defined(__CUDA_ARCH__)
  return __float_as_uint(f);
#else
  uint32_t u; memcpy(&u, &f, 4); return u;
#endif
}
SCION_HOSTDEV float u2f(uint32_t u) {
#if defined(__CUDA_ARCH__)
  return __uint_as_float(u);
#else
  float f; memcpy(&f, &u, 4); return f;
#endif
}
SCION_HOSTDEV float inf() { return u2f(0x7f800000u); }

// min/max: IEEE minNum/maxNum == C fminf/fmaxf == CUDA fminf/fmaxf
SCION_HOSTDEV float min(float a, float b) { return fminf(a, b); }
SCION_HOSTDEV float max(float a, float b) { return fmaxf(a, b); }
SCION_HOSTDEV uint32_t min(uint32_t a, uint32_t b) { return a < b ? a : b; }
SCION_HOSTDEV uint32_t max(uint32_t a, uint32_t b) { return a > b ? a : b; }
SCION_HOSTDEV float floorf_(float a) { return ::floorf(a); }
SCION_HOSTDEV float ceilf_(float a) { return ::ceilf(a); }
SCION_HOSTDEV float abs(float a) { return u2f(f2u(a) & 0x7fffffffu); }
template <class T> SCION_HOSTDEV T select(bool m, T a, T b) { return m ? a : b; }

#define SCION_VEC_FN2(NAME)                                                                          \
  template <class T, int N> SCION_HOSTDEV vec<T, N> NAME(const vec<T, N>& a, const vec<T, N>& b) {    \
    vec<T, N> r;                                                                                     \
    _Pragma("unroll") for (int i = 0; i < N; i++) r[i] = NAME(a[i], b[i]);                            \
    return r;                                                                                        \
  }                                                                                                  \
  template <class T, int N> SCION_HOSTDEV vec<T, N> NAME(const vec<T, N>& a, T b) {                   \
    vec<T, N> r;                                                                                     \
    _Pragma("unroll") for (int i = 0; i < N; i++) r[i] = NAME(a[i], b);                               \
    return r;                                                                                        \
  }                                                                                                  \
  template <class T, int N> SCION_HOSTDEV vec<T, N> NAME(T a, const vec<T, N>& b) {                   \
    vec<T, N> r;                                                                                     \
    _Pragma("unroll") for (int i = 0; i < N; i++) r[i] = NAME(a, b[i]);                               \
    return r;                                                                                        \
  }
SCION_VEC_FN2(min)
SCION_VEC_FN2(max)
#undef SCION_VEC_FN2
template <int N> SCION_HOSTDEV vec<float, N> floorf_(const vec<float, N>& a) {
  vec<float, N> r;
#pragma unroll
  for (int i = 0; i < N; i++) r[i] = floorf_(a[i]);
  return r;
}
template <int N> SCION_HOSTDEV vec<float, N> ceilf_(const vec<float, N>& a) {
  vec<float, N> r;
#pragma unroll
  for (int i = 0; i < N; i++) r[i] = ceilf_(a[i]);
  return r;
}
SCION_HOSTDEV float dot(const f32x3& a, const f32x3& b) { return ((a.x * b.x) + (a.y * b.y)) + (a.z * b.z); }
SCION_HOSTDEV f32x3 cross(const f32x3& a, const f32x3& b) {
  return f32x3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
SCION_HOSTDEV float sum(const f32x3& a) { return (a.x + a.y) + a.z; }

// directed rounding (geometry-runtime): TRUE directed rounding, not the
// binary64 shortcut.
#if defined(__CUDA_ARCH__)
SCION_DEV float fmul_rd(float a, float b) { return __fmul_rd(a, b); }
SCION_DEV float fadd_rd(float a, float b) { return __fadd_rd(a, b); }
SCION_DEV float fsub_rd(float a, float b) { return __fsub_rd(a, b); }
SCION_DEV float fsub_ru(float a, float b) { return __fsub_ru(a, b); }
SCION_DEV float fdiv_rd(float a, float b) { return __fdiv_rd(a, b); }
SCION_DEV float frcp_rd(float a) { return __frcp_rd(a); }
#elif !defined(__CUDACC__)
namespace host_rounding {
template <class F> inline float with_mode(int mode, F f) {
  int old = fegetround();
  fesetround(mode);
  volatile float r = f();
  fesetround(old);
  return r;
}
}  // namespace host_rounding
inline float fmul_rd(float a, float b) { volatile float x = a, y = b; return host_rounding::with_mode(FE_DOWNWARD, [&] { return x * y; }); }
inline float fadd_rd(float a, float b) { volatile float x = a, y = b; return host_rounding::with_mode(FE_DOWNWARD, [&] { return x + y; }); }
inline float fsub_rd(float a, float b) { volatile float x = a, y = b; return host_rounding::with_mode(FE_DOWNWARD, [&] { return x - y; }); }
inline float fsub_ru(float a, float b) { volatile float x = a, y = b; return host_rounding::with_mode(FE_UPWARD, [&] { return x - y; }); }
inline float fdiv_rd(float a, float b) { volatile float x = a, y = b; return host_rounding::with_mode(FE_DOWNWARD, [&] { return x / y; }); }
inline float frcp_rd(float a) { volatile float x = a; return host_rounding::with_mode(FE_DOWNWARD, [&] { return 1.0f / x; }); }
#else
// host pass of nvcc over device-only code: never called
__host__ __device__ inline float fmul_rd(float a, float b) { return a * b; }
__host__ __device__ inline float fadd_rd(float a, float b) { return a + b; }
__host__ __device__ inline float fsub_rd(float a, float b) { return a - b; }
__host__ __device__ inline float fsub_ru(float a, float b) { return a - b; }
__host__ __device__ inline float fdiv_rd(float a, float b) { return a / b; }
__host__ __device__ inline float frcp_rd(float a) { return 1.0f / a; }
#endif
#define SCION_VEC_RD2(NAME)                                                                      \
  template <int N> SCION_HOSTDEV vec<float, N> NAME(const vec<float, N>& a, const vec<float, N>& b) { \
    vec<float, N> r;                                                                             \
    _Pragma("unroll") for (int i = 0; i < N; i++) r[i] = NAME(a[i], b[i]);                        \
    return r;                                                                                    \
  }
SCION_VEC_RD2(fmul_rd)
SCION_VEC_RD2(fadd_rd)
SCION_VEC_RD2(fsub_rd)
SCION_VEC_RD2(fsub_ru)
SCION_VEC_RD2(fdiv_rd)
#undef SCION_VEC_RD2

// --------------------------------------------------------------------------- casts
// `e as T` value cast (sema.cpp:753-770); `e to T` equal-width bit cast (:771-786)
template <class To> struct as_impl;
template <> struct as_impl<float> {
  // SCION_I2F_MAGIC: integers below 2^23 convert exactly as bits(0x4B000000 | x) - 2^23 — one logic op and one FADD on
  // the full-rate pipes instead of one I2F on the quarter-rate conversion unit; the range test folds away when the
  // compiler knows the operand is a narrow bit field (every quantised layout), the value is identical.
  SCION_HOSTDEV static float go(uint32_t x) {
#if defined(__CUDA_ARCH__) && SCION_I2F_MAGIC
    if (x < 0x800000u) return __uint_as_float(0x4B000000u | x) - 8388608.0f;
#endif
    return (float)x;
  }
  SCION_HOSTDEV static float go(int32_t x) { return (float)x; }
  SCION_HOSTDEV static float go(uint64_t x) { return (float)x; }
  SCION_HOSTDEV static float go(float x) { return x; }
};
template <int N> struct as_impl<vec<float, N>> {
  template <class S> SCION_HOSTDEV static vec<float, N> go(const vec<S, N>& x) {
    vec<float, N> r;
#pragma unroll
    for (int i = 0; i < N; i++) r[i] = as_impl<float>::go(x[i]);
    return r;
  }
};
template <class To, class From> SCION_HOSTDEV To as_(const From& x) { return as_impl<To>::go(x); }

SCION_HOSTDEV uint64_t mask64(int w) { return w >= 64 ? ~0ull : ((1ull << w) - 1ull); }
// unsigned integer target of width W (float source truncates toward zero; inputs are
// pre-floored and clamped by the DSL code)
template <int W> SCION_HOSTDEV uint32_t as_uint(float x) { return (uint32_t)x & (uint32_t)mask64(W); }
template <int W> SCION_HOSTDEV uint32_t as_uint(uint32_t x) { return x & (uint32_t)mask64(W); }
template <int W> SCION_HOSTDEV uint32_t as_uint(int32_t x) { return (uint32_t)x & (uint32_t)mask64(W); }
template <int W> SCION_HOSTDEV uint32_t as_uint(uint64_t x) { return (uint32_t)(x & mask64(W)); }
template <int W> SCION_HOSTDEV uint64_t as_uint64(uint64_t x) { return x & mask64(W); }
template <int W> SCION_HOSTDEV uint64_t as_uint64(uint32_t x) { return (uint64_t)x & mask64(W); }
template <int W, class S, int N> SCION_HOSTDEV vec<uint32_t, N> as_uint(const vec<S, N>& x) {
  vec<uint32_t, N> r;
#pragma unroll
  for (int i = 0; i < N; i++) r[i] = as_uint<W>(x[i]);
  return r;
}
template <int W> SCION_HOSTDEV int32_t as_sint(uint32_t x) {
  return W >= 32 ? (int32_t)x : (int32_t)(x << (32 - W)) >> (32 - W);
}
template <int W> SCION_HOSTDEV int32_t as_sint(int32_t x) { return as_sint<W>((uint32_t)x); }

SCION_HOSTDEV float bit_to_f32(uint32_t x) { return u2f(x); }
SCION_HOSTDEV uint32_t bit_to_u32(float x) { return f2u(x); }
SCION_HOSTDEV uint32_t bit_to_u32(int32_t x) { return (uint32_t)x; }
SCION_HOSTDEV uint32_t bit_to_u32(uint32_t x) { return x; }
SCION_HOSTDEV int32_t bit_to_i32(uint32_t x) { return (int32_t)x; }
SCION_HOSTDEV int32_t bit_to_i32(int32_t x) { return x; }

// x[a:b] — inclusive bit range (bvh8_q8_ci.scion: I[2:31], I[7:31], I[2:6])
template <int LO, int HI> SCION_HOSTDEV uint32_t bits(uint32_t x) { return (x >> LO) & (uint32_t)mask64(HI - LO + 1); }
template <int LO, int HI> SCION_HOSTDEV uint32_t bits(int32_t x) { return bits<LO, HI>((uint32_t)x); }
template <int LO, int HI> SCION_HOSTDEV uint64_t bits(uint64_t x) { return (x >> LO) & mask64(HI - LO + 1); }

// dynamic lane update: `t[axis] = S` (shared_slab.scion upd)
template <class T, int N, class I> SCION_HOSTDEV void set_lane(vec<T, N>& v, I lane, T s) {
#pragma unroll
  for (int i = 0; i < N; i++)
    if ((int)lane == i) v[i] = s;
}
template <class T, int N, class I> SCION_HOSTDEV T get_lane(const vec<T, N>& v, I lane) {
  T r = v[0];
#pragma unroll
  for (int i = 1; i < N; i++)
    if ((int)lane == i) r = v[i];
  return r;
}

// --------------------------------------------------------------------------- record loads
template <int NW>
struct Words {
  uint32_t w[NW];
  static constexpr int kWords = NW;
  template <int I>
  SCION_HOSTDEV uint32_t word() const { return w[I]; }
};
SCION_HOSTDEV uint32_t ld32(const uint8_t* p) {
#if defined(__CUDA_ARCH__)
  return __ldg(reinterpret_cast<const uint32_t*>(p));
#else
  uint32_t v; memcpy(&v, p, 4); return v;
#endif
}
SCION_HOSTDEV void ld64(const uint8_t* p, uint32_t* o) {
#if defined(__CUDA_ARCH__)
  uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
  o[0] = v.x; o[1] = v.y;
#else
  memcpy(o, p, 8);
#endif
}
#if defined(__CUDA_ARCH__)
// L2 eviction policies (experiment SCION_CACHE_HINTS): node records evict_last, primitives evict_first
__device__ __forceinline__ uint64_t l2_policy_keep() { uint64_t p; asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t l2_policy_stream() { uint64_t p; asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
#endif
// SCION_L2_PROMO (0 | 64 | 128 | 256): L2 sector promotion of node-record loads — a miss fetches the whole 64 / 128 /
// 256-byte block into L2, so a left descent through a cold stretch of the preorder array pays one DRAM access per block
// instead of one per 32-byte sector.
#ifndef SCION_L2_PROMO
#define SCION_L2_PROMO 0
#endif
#define SCION_STR2(x) #x
#define SCION_STR(x) SCION_STR2(x)
#if SCION_L2_PROMO > 0
#define SCION_PROMO_Q ".L2::" SCION_STR(SCION_L2_PROMO) "B"
#else
#define SCION_PROMO_Q ""
#endif
SCION_HOSTDEV void ld128(const uint8_t* p, uint32_t* o) {
#if defined(__CUDA_ARCH__) && SCION_L2_PROMO > 0
  asm volatile("ld.global.nc" SCION_PROMO_Q ".v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]) : "l"(p));
#elif defined(__CUDA_ARCH__) && (SCION_CACHE_HINTS == 1 || SCION_CACHE_HINTS == 2 || SCION_CACHE_HINTS == 3)
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]) : "l"(p), "l"(l2_policy_keep()));
#elif defined(__CUDA_ARCH__)
  uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
#else
  memcpy(o, p, 16);
#endif
}
// 256-bit read-only load (sm_100: LDG.E.256): one L1 wavefront per lane where two LDG.128 take two —
// the f32 layouts are L1-tag-bound (profiles/r1_ncu_v8_c5_pbrt.txt: l1tex throughput 98 %)
SCION_HOSTDEV void ld256(const uint8_t* p, uint32_t* o) {
#if defined(__CUDA_ARCH__)
  asm volatile("ld.global.nc" SCION_PROMO_Q ".v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]), "=r"(o[4]), "=r"(o[5]), "=r"(o[6]), "=r"(o[7])
               : "l"(p));
#else
  memcpy(o, p, 32);
#endif
}
SCION_HOSTDEV uint32_t funnel_r(uint32_t lo, uint32_t hi, uint32_t shift_bits) {
#if defined(__CUDA_ARCH__)
  return __funnelshift_r(lo, hi, shift_bits);
#else
  return shift_bits == 0 ? lo : (lo >> shift_bits) | (hi << (32 - shift_bits));
#endif
}

template <int LEVEL>
SCION_HOSTDEV void prefetch_to(const void* p) {
#if defined(__CUDA_ARCH__)
  if constexpr (LEVEL == 1) asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
  else asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
#else
  (void)p;
#endif
}

// Load one planned element of BYTES bytes whose address is known to be ALIGN-aligned
// (ALIGN = gcd of the buffer base alignment, the segment base and the stride, computed by
// emit_cuda).  16-byte read-only vector loads whenever the plan allows them; 8- and 4-byte
// loads otherwise; byte-granular strides (pbrt-post 34 B, identity 41 B, shared-slab 29 B) read
// the covering aligned 16-byte quads, re-align words and funnel-shift.  Every device buffer is over-allocated by
// 32 bytes so the covering reads stay inside the allocation.
// load_record for the records of the *cold* part of a tree (experiment SCION_HOT_L1, traverse.cuh): same bytes, but the
// line is not allocated in L1, so that the few thousand records of the top levels stay there.  Only for records that
// are one 16- or 32-byte vector load.
// A record staged in shared memory by 16-byte async copies (traverse.cuh chrt8s_kernel): 16-byte chunk c of this lane's
// record lives at base + c * kChunkPitch (the 32 lanes' copies of one chunk are contiguous, so a warp's LDS.128 of one
// chunk is conflict free).  Same word<I>() interface as Words: the extraction templates below serve both.
template <int NW, int PITCH>
struct StagedRecord {
#if defined(__CUDA_ARCH__)
  // shared-space byte address of this lane's chunk 0.  The loads are NON-volatile asm: a pure function of the address for
  // the compiler, so repeated extractions of one chunk are merged and dead ones removed.  What orders them behind the
  // asynchronous copies is a data dependence: the kernel passes `addr` through an opaque asm after cp.async.wait_all.
  uint32_t addr;
  template <int I>
  SCION_HOSTDEV uint32_t word() const {
    uint32_t x, y, z, w;
    asm("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(addr + (uint32_t)((I / 4) * PITCH)));
    return I % 4 == 0 ? x : (I % 4 == 1 ? y : (I % 4 == 2 ? z : w));
  }
#else
  const uint8_t* base;
  template <int I>
  SCION_HOSTDEV uint32_t word() const {
    uint32_t v;
    memcpy(&v, base + (I / 4) * PITCH + (I % 4) * 4, 4);
    return v;
  }
#endif
  static constexpr int kWords = NW;
};
template <int BYTES, int ALIGN>
SCION_HOSTDEV void load_record_na(const uint8_t* p, Words<(BYTES + 3) / 4>& r) {
  static_assert((BYTES == 16 && ALIGN % 16 == 0) || (BYTES == 32 && ALIGN % 32 == 0), "single vector load records only");
#if defined(__CUDA_ARCH__)
  if constexpr (BYTES == 16) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]) : "l"(p));
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]), "=r"(r.w[7])
                 : "l"(p));
  }
#else
  memcpy(r.w, p, BYTES);
#endif
}
template <int BYTES, int ALIGN>
SCION_HOSTDEV void load_record(const uint8_t* p, Words<(BYTES + 3) / 4>& r) {
  constexpr int NW = (BYTES + 3) / 4;
  if constexpr (SCION_LDG256 && ALIGN % 32 == 0 && BYTES % 32 == 0) {
#pragma unroll
    for (int i = 0; i < NW; i += 8) ld256(p + 4 * i, r.w + i);
  } else if constexpr (ALIGN % 16 == 0 && BYTES % 16 == 0) {
#pragma unroll
    for (int i = 0; i < NW; i += 4) ld128(p + 4 * i, r.w + i);
  } else if constexpr (SCION_LDG_PARITY && ALIGN % 8 == 0 && BYTES % 8 == 0 && BYTES >= 24) {
    // 8-byte-aligned record (bvh8-q8-ci 104 B = 13 x 8): 16-byte loads from whichever 16-byte phase the
    // record starts at — 7 loads per lane instead of 13 (half the L1 wavefronts); the two phases diverge
    if ((reinterpret_cast<uintptr_t>(p) & 8u) == 0u) {
      constexpr int kQuads = NW / 4;
#pragma unroll
      for (int i = 0; i < kQuads; i++) ld128(p + 16 * i, r.w + 4 * i);
      if constexpr (NW % 4 == 2) ld64(p + 16 * kQuads, r.w + 4 * kQuads);
    } else {
      constexpr int kQuads = (NW - 2) / 4;
      ld64(p, r.w);
#pragma unroll
      for (int i = 0; i < kQuads; i++) ld128(p + 8 + 16 * i, r.w + 2 + 4 * i);
      if constexpr ((NW - 2) % 4 == 2) ld64(p + 8 + 16 * kQuads, r.w + 2 + 4 * kQuads);
    }
  } else if constexpr (ALIGN % 8 == 0 && BYTES % 8 == 0) {
#pragma unroll
    for (int i = 0; i < NW; i += 2) ld64(p + 4 * i, r.w + i);
  } else if constexpr (ALIGN % 4 == 0 && BYTES % 4 == 0) {
#pragma unroll
    for (int i = 0; i < NW; i++) r.w[i] = ld32(p + 4 * i);
  } else if constexpr (SCION_LDG_COVER == 2 && BYTES > 16 && BYTES <= 64) {
    // byte-granular stride, 256-bit variant: the 32-byte aligned sectors that cover the record (2, sometimes 3, loads of
    // one L1 wavefront per lane each, where the 16-byte quads below take 3-4), word re-alignment by a three-level select,
    // byte re-alignment by funnel shifts.  The last sector is only read when the record's bytes reach into it, so the read
    // never goes more than 31 bytes past the record (buffers carry 32 bytes of slack).
    const uint64_t a = (uint64_t)p;
    const uint8_t* q = (const uint8_t*)(a & ~31ull);
    const uint32_t wsh = (uint32_t)(a >> 2) & 7u;
    const uint32_t bsh = (uint32_t)(a & 3ull) * 8u;
    constexpr int NR = NW + 1;           // words needed before the funnel shift
    constexpr int K = (NR + 7 + 7) / 8;  // sectors covering words [wsh, wsh + NR)
    uint32_t w[8 * K + 8];
#pragma unroll
    for (int k = 0; k < K - 1; k++) ld256(q + 32 * k, w + 8 * k);
#pragma unroll
    for (int i = 8 * (K - 1); i < 8 * K + 8; i++) w[i] = 0u;
    // the last sector is only read when the record's bytes (not the extra funnel word) reach into it
    if ((uint32_t)(a & 31ull) + (uint32_t)BYTES > 32u * (uint32_t)(K - 1)) ld256(q + 32 * (K - 1), w + 8 * (K - 1));
    const bool s1 = (wsh & 1u) != 0u, s2 = (wsh & 2u) != 0u, s4 = (wsh & 4u) != 0u;
    uint32_t x[NR + 3];
#pragma unroll
    for (int i = 0; i < NR + 3; i++) x[i] = s4 ? w[i + 4] : w[i];
    uint32_t raw[NR];
#pragma unroll
    for (int i = 0; i < NR; i++) {
      const uint32_t lo = s1 ? x[i + 1] : x[i];
      const uint32_t hi = s1 ? x[i + 3] : x[i + 2];
      raw[i] = s2 ? hi : lo;
    }
#pragma unroll
    for (int i = 0; i < NW; i++) r.w[i] = funnel_r(raw[i], raw[i + 1], bsh);
  } else if constexpr (SCION_LDG_COVER && BYTES > 16) {
    // byte-granular stride (identity 41 B, pbrt-post 34 B, shared-slab 29 B): the 16-byte-aligned quads that
    // cover the record (4 instead of 12 loads for identity), word re-alignment by a two-level select, byte
    // re-alignment by funnel shifts.  The last quad is only read when the record reaches into it, so the read
    // never goes more than 31 bytes past the record (buffers carry 32 bytes of slack).
    const uint64_t a = (uint64_t)p;
    const uint8_t* q = (const uint8_t*)(a & ~15ull);
    const uint32_t wsh = (uint32_t)(a >> 2) & 3u;
    const uint32_t bsh = (uint32_t)(a & 3ull) * 8u;
    constexpr int NR = NW + 1;           // words needed before the funnel shift
    constexpr int K = (NR + 3 + 3) / 4;  // quads covering words [wsh, wsh + NR)
    uint32_t w[4 * K + 3];
#pragma unroll
    for (int k = 0; k < K - 1; k++) ld128(q + 16 * k, w + 4 * k);
    w[4 * (K - 1)] = w[4 * (K - 1) + 1] = w[4 * (K - 1) + 2] = w[4 * (K - 1) + 3] = 0u;
    if (wsh + (uint32_t)NR > 4u * (uint32_t)(K - 1)) ld128(q + 16 * (K - 1), w + 4 * (K - 1));
    w[4 * K] = w[4 * K + 1] = w[4 * K + 2] = 0u;
    const bool s1 = (wsh & 1u) != 0u, s2 = (wsh & 2u) != 0u;
    uint32_t raw[NR];
#pragma unroll
    for (int i = 0; i < NR; i++) {
      const uint32_t lo = s1 ? w[i + 1] : w[i];
      const uint32_t hi = s1 ? w[i + 3] : w[i + 2];
      raw[i] = s2 ? hi : lo;
    }
#pragma unroll
    for (int i = 0; i < NW; i++) r.w[i] = funnel_r(raw[i], raw[i + 1], bsh);
  } else {
    const uint64_t a = (uint64_t)p;
    const uint8_t* q = (const uint8_t*)(a & ~3ull);
    const uint32_t sh = (uint32_t)(a & 3ull) * 8u;
    uint32_t raw[NW + 1];
#pragma unroll
    for (int i = 0; i <= NW; i++) raw[i] = ld32(q + 4 * i);
#pragma unroll
    for (int i = 0; i < NW; i++) r.w[i] = funnel_r(raw[i], raw[i + 1], sh);
  }
}

// Staged prefix of a node array (see traverse.cuh): records [0, count) live at `base` (shared memory,
// generic address).  load_record_generic uses plain generic loads so that one instruction serves
// both the shared and the global window.
struct Stage {
  const uint8_t* base = nullptr;
  uint32_t count = 0;
};
template <int BYTES, int ALIGN>
SCION_HOSTDEV void load_record_generic(const uint8_t* p, Words<(BYTES + 3) / 4>& r) {
  constexpr int NW = (BYTES + 3) / 4;
  static_assert(ALIGN % 16 == 0 && BYTES % 16 == 0, "staging needs 16-byte records");
#pragma unroll
  for (int i = 0; i < NW; i += 4) {
#if defined(__CUDA_ARCH__)
    const uint4 v = *reinterpret_cast<const uint4*>(p + 4 * i);
    r.w[i] = v.x; r.w[i + 1] = v.y; r.w[i + 2] = v.z; r.w[i + 3] = v.w;
#else
    memcpy(r.w + i, p + 4 * i, 16);
#endif
  }
}

// Per-child view of an 8-wide interior record, for lane-cooperative traversal (traverse_coop8.cuh: lane k of a group of 8
// lanes decodes and tests child slot k only).  The view presents the record AS IF child slot `k` were slot 0: a bit range
// that lies in a field shared by all children (kLaneFieldElem == 0: mlo, mex) is read where it is, a bit range of an
// 8-element per-child field (child_bounds, children, lo, hi) is read k elements further on.  The emitted
// decode_slot<0>() evaluated over this view therefore yields the bounds and the reference of child k — the emitted
// expressions are the same for every slot (tests/test_generated_decoders.py checks all 8 slots of every 8-wide layout
// against decode()).  Loads go straight to global memory through the read-only path with the width of the field
// (LDG.U8 / .U16 / .32; shared fields by 8-byte pairs): the 8 lanes of a group touch one record, i.e. 1-3 lines per
// request instead of the 32 lines of a one-ray-per-lane gather.  The asm is not volatile: a pure function of the
// address for the compiler, so repeated reads are merged and the reads of the 7 other slots are removed as dead code.
template <class L>
struct LaneRecord {
  const uint8_t* p;  // address of the record
  uint32_t k;        // child slot this lane looks at
  static constexpr bool kDynamic = true;
  static constexpr int kWords = (int)((L::kSlotUsedBytes + 3u) / 4u);
  SCION_HOSTDEV static constexpr int field_of(uint32_t off) {
    for (int f = 0; f < L::kLaneFields; f++)
      if (off >= L::kLaneFieldOff[f] && off < L::kLaneFieldEnd[f]) return f;
    return -1;
  }
  template <int BYTES>
  SCION_HOSTDEV static uint32_t ld(const uint8_t* a) {  // BYTES in {1, 2, 4}, a is BYTES-aligned
#if defined(__CUDA_ARCH__)
    uint32_t v;
    if constexpr (BYTES == 1) asm("ld.global.nc.u8 %0, [%1];" : "=r"(v) : "l"(a));
    else if constexpr (BYTES == 2) asm("ld.global.nc.u16 %0, [%1];" : "=r"(v) : "l"(a));
    else asm("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(a));
    return v;
#else
    uint32_t v = 0;
    memcpy(&v, a, BYTES);
    return v;
#endif
  }
  SCION_HOSTDEV static uint32_t ld_pair(const uint8_t* a, int half) {  // one 32-bit half of an 8-byte aligned pair
#if defined(__CUDA_ARCH__)
    uint32_t x, y;
    asm("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "l"(a));
    return half ? y : x;
#else
    uint32_t v;
    memcpy(&v, a + 4 * half, 4);
    return v;
#endif
  }
  // bits [OFF, OFF + W) of the view
  template <int OFF, int W>
  SCION_HOSTDEV uint32_t field() const {
    constexpr int f = field_of((uint32_t)OFF);
    static_assert(f >= 0, "bit range outside the stored fields");
    constexpr uint32_t E = L::kLaneFieldElem[f];
    constexpr uint32_t mask = (uint32_t)((1ull << W) - 1ull);
    if constexpr (E == 0) {  // shared by all children: static address
      if constexpr (OFF % 32 == 0 && W == 32) {
        if constexpr (L::kLaneAlign % 8 == 0) return ld_pair(p + (OFF / 64) * 8, (OFF / 32) % 2);
        else return ld<4>(p + OFF / 8);
      } else {
        static_assert(OFF % 8 == 0 && (W == 8 || W == 16) && (OFF / 8) % (W / 8) == 0, "shared field: unsupported bit range");
        return ld<W / 8>(p + OFF / 8);
      }
    } else {
      static_assert(E % 8 == 0 && OFF % 8 == 0, "per-child elements are whole bytes");
      const uint8_t* a = p + OFF / 8 + k * (E / 8);
      if constexpr (W == 32 && (OFF / 8) % 4 == 0 && (E / 8) % 4 == 0) return ld<4>(a);
      else if constexpr (W == 16 && (OFF / 8) % 2 == 0 && (E / 8) % 2 == 0) return ld<2>(a);
      else if constexpr (W == 8) return ld<1>(a);
      else {  // any other byte-aligned range: assembled from bytes
        uint32_t v = 0;
#pragma unroll
        for (int i = 0; i < (W + 7) / 8; i++) v |= ld<1>(a + i) << (8 * i);
        return v & mask;
      }
    }
  }
};
template <class S, class = void> struct is_dynamic_src { static constexpr bool value = false; };
template <class S> struct is_dynamic_src<S, decltype((void)S::kDynamic)> { static constexpr bool value = true; };

// constant-offset field extraction: the inverse of write_bits_raw
// (/root/reference/proj/src/bits.cpp:21-36), little-endian, LSB first
template <int OFF, int W, class Src>
SCION_HOSTDEV uint32_t ext32(const Src& r) {
  static_assert(W >= 1 && W <= 32, "ext32 width");
  if constexpr (is_dynamic_src<Src>::value) return r.template field<OFF, W>();
  else {
  constexpr int i = OFF / 32, s = OFF % 32;
  static_assert(i < Src::kWords, "field outside record");
  if constexpr (s + W <= 32) {
    if constexpr (W == 32) return r.template word<i>();
    else return (r.template word<i>() >> s) & (uint32_t)((1ull << W) - 1ull);
  } else {
    static_assert(i + 1 < Src::kWords, "field outside record");
    return ((r.template word<i>() >> s) | (r.template word<i + 1>() << (32 - s))) & (uint32_t)((1ull << W) - 1ull);
  }
  }
}
template <int OFF, int W, class Src>
SCION_HOSTDEV uint64_t ext64(const Src& r) {
  static_assert(W > 32 && W <= 64, "ext64 width");
  uint64_t lo = ext32<OFF, 32>(r);
  uint64_t hi = ext32<OFF + 32, W - 32>(r);
  return lo | (hi << 32);
}
template <int OFF, class Src>
SCION_HOSTDEV float extf(const Src& r) {
  return u2f(ext32<OFF, 32>(r));
}

// constant-offset field store into a zero-initialised record image: write_bits_raw (/root/reference/proj/src/bits.cpp:21-36)
// specialised to constant offsets — used by the emitted constructors (build_<Variant>, the compiled `build` block)
template <int OFF, int W>
SCION_HOSTDEV void dep32(uint32_t* w, uint32_t v) {
  static_assert(W >= 1 && W <= 32, "dep32 width");
  constexpr int i = OFF / 32, s = OFF % 32;
  const uint32_t m = (uint32_t)((1ull << W) - 1ull);
  v &= m;
  w[i] = (w[i] & ~(m << s)) | (v << s);
  if constexpr (s + W > 32) w[i + 1] = (w[i + 1] & ~(m >> (32 - s))) | (v >> (32 - s));
}
template <int OFF, int W>
SCION_HOSTDEV void dep64(uint32_t* w, uint64_t v) {
  static_assert(W > 32 && W <= 64, "dep64 width");
  dep32<OFF, 32>(w, (uint32_t)v);
  dep32<OFF + 32, W - 32>(w, (uint32_t)(v >> 32));
}

template <class T> SCION_HOSTDEV T glob(const TreeView& T_, int i);
template <> SCION_HOSTDEV float glob<float>(const TreeView& t, int i) { return u2f(t.glob[i][0]); }
template <> SCION_HOSTDEV uint32_t glob<uint32_t>(const TreeView& t, int i) { return t.glob[i][0]; }
template <> SCION_HOSTDEV int32_t glob<int32_t>(const TreeView& t, int i) { return (int32_t)t.glob[i][0]; }
template <> SCION_HOSTDEV uint64_t glob<uint64_t>(const TreeView& t, int i) { return (uint64_t)t.glob[i][0] | ((uint64_t)t.glob[i][1] << 32); }
template <> SCION_HOSTDEV f32x3 glob<f32x3>(const TreeView& t, int i) { return f32x3{u2f(t.glob[i][0]), u2f(t.glob[i][1]), u2f(t.glob[i][2])}; }
template <> SCION_HOSTDEV f32x4 glob<f32x4>(const TreeView& t, int i) {
  return f32x4{u2f(t.glob[i][0]), u2f(t.glob[i][1]), u2f(t.glob[i][2]), u2f(t.glob[i][3])};
}

}  // namespace scion
