// Device restatement of the DSL standard library the traversals call
// (/root/reference/proj/corpus/lib/geometry.scion, corpus/lib/dop.scion), strict binary32:
// compiled with -fmad=false -prec-div=true -prec-sqrt=true -ftz=false, no fast-math, so that
// every + - * / is a separately rounded IEEE operation exactly as in the CPU oracle
// (reference flag -ffp-contract=off, proj/CMakeLists.txt:13-15).
#pragma once
#include "scion_rt.cuh"

#ifndef SCION_TRI_LDG32
#define SCION_TRI_LDG32 0
#endif
#ifndef SCION_TRI_LDG256  /* 1: a triangle is fetched by two 256-bit loads (its two 32-byte sectors) instead of three 128-bit ones */
#define SCION_TRI_LDG256 0
#endif

namespace scion {

#ifndef SCION_SEL_MASK
// 0: near / far plane chosen by FSEL on three predicates re-derived from `neg` in every step (2 LOP3 + 2 ISETP);
// 1: chosen by a bitwise mux — near = lo ^ ((lo ^ hi) & m), ONE LOP3 per plane, no predicates — on per-axis masks
//    m = direction[a] < 0 ? ~0 : 0 kept in registers (2 more than `neg`).  Same values bit for bit.
#define SCION_SEL_MASK 0
#endif
struct RayCtx {
  float ox, oy, oz, tmax;
  float dx, dy, dz;
  float rdx, rdy, rdz;  // 1.0 / direction, hoisted (pure, geometry.scion:13)
#if SCION_SEL_MASK
  uint32_t mx, my, mz;  // all ones iff direction[a] < 0.0 (-0.0 is not negative)
#else
  uint32_t neg;         // bit a set iff direction[a] < 0.0 (-0.0 is not negative); one register instead of three flags
#endif
};

SCION_DEV RayCtx make_ray(float ox, float oy, float oz, float tmax, float dx, float dy, float dz) {
  RayCtx r;
  r.ox = ox; r.oy = oy; r.oz = oz; r.tmax = tmax;
  r.dx = dx; r.dy = dy; r.dz = dz;
  r.rdx = 1.0f / dx; r.rdy = 1.0f / dy; r.rdz = 1.0f / dz;
#if SCION_SEL_MASK
  r.mx = dx < 0.0f ? 0xffffffffu : 0u;
  r.my = dy < 0.0f ? 0xffffffffu : 0u;
  r.mz = dz < 0.0f ? 0xffffffffu : 0u;
#else
  r.neg = (dx < 0.0f ? 1u : 0u) | (dy < 0.0f ? 2u : 0u) | (dz < 0.0f ? 4u : 0u);
#endif
  return r;
}

// intersectsp_ray_aabb, geometry.scion:12-22.  Returns `some`; t_near/t_far are the interval.
SCION_DEV bool ray_aabb(const RayCtx& r, const f32x3& lo, const f32x3& hi, float& t_near, float& t_far) {
#if SCION_SEL_MASK
  auto mux = [](float a, float b, uint32_t m) {  // m ? b : a bit by bit: ONE LOP3 (the C++ form becomes three per axis, the common a ^ b first)
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xD8;" : "=r"(d) : "r"(f2u(a)), "r"(f2u(b)), "r"(m));
    return u2f(d);
  };
  const float nx = mux(lo.x, hi.x, r.mx), fx = mux(hi.x, lo.x, r.mx);
  const float ny = mux(lo.y, hi.y, r.my), fy = mux(hi.y, lo.y, r.my);
  const float nz = mux(lo.z, hi.z, r.mz), fz = mux(hi.z, lo.z, r.mz);
#else
  const bool sx = (r.neg & 1u) != 0u, sy = (r.neg & 2u) != 0u, sz = (r.neg & 4u) != 0u;
  const float nx = sx ? hi.x : lo.x, fx = sx ? lo.x : hi.x;
  const float ny = sy ? hi.y : lo.y, fy = sy ? lo.y : hi.y;
  const float nz = sz ? hi.z : lo.z, fz = sz ? lo.z : hi.z;
#endif
  const float t_nx = (nx - r.ox) * r.rdx, t_fx = (fx - r.ox) * r.rdx;
  const float t_ny = (ny - r.oy) * r.rdy, t_fy = (fy - r.oy) * r.rdy;
  const float t_nz = (nz - r.oz) * r.rdz, t_fz = (fz - r.oz) * r.rdz;
  t_near = fmaxf(0.0f, fmaxf(t_nx, fmaxf(t_ny, t_nz)));
  t_far = fminf(r.tmax, fminf(t_fx, fminf(t_fy, t_fz)));
  return t_near <= t_far;
}
// intersects(Ray, AABB) geometry.scion:61-63 given the interval
SCION_DEV bool interval_intersects(const RayCtx& r, bool some, float t_near, float t_far) {
  return some && (t_near < r.tmax) && (t_far > 0.0f);
}

// intersectsp_ray_tri_mt, geometry.scion:25-38 (sign-masked Moeller-Trumbore); returns hit and t
SCION_DEV bool ray_tri_mt(const RayCtx& ray, const float* p, float& t_out) {
  const f32x3 p0{p[0], p[1], p[2]}, p1{p[3], p[4], p[5]}, p2{p[6], p[7], p[8]};
  const f32x3 e1 = p0 - p1, e2 = p2 - p0;
  const f32x3 ng = cross(e2, e1);
  const f32x3 c = p0 - f32x3{ray.ox, ray.oy, ray.oz};
  const f32x3 d{ray.dx, ray.dy, ray.dz};
  const f32x3 r = cross(c, d);
  const float D = dot(ng, d);
  if (D == 0.0f) return false;
  const float abs_D = scion::abs(D);
  const uint32_t sgn_D = f2u(D) & 2147483648u;
  const float u_raw = u2f(f2u(dot(r, e2)) ^ sgn_D);
  const float v_raw = u2f(f2u(dot(r, e1)) ^ sgn_D);
  if (!(u_raw >= 0.0f && v_raw >= 0.0f && u_raw + v_raw <= abs_D)) return false;
  const float t_raw = u2f(f2u(dot(ng, c)) ^ sgn_D);
  if (!(abs_D * 0.0f < t_raw && t_raw <= abs_D * ray.tmax)) return false;
  const float inv_abs_D = 1.0f / abs_D;
  t_out = t_raw * inv_abs_D;
  return true;
}

// full results of the two ray/triangle tests of geometry.scion (batch entry point scion_ray_triangle):
// intersectsp_ray_tri_mt :25-38 with barycentrics, and the Pluecker-coordinate test intersectsp_ray_tri_pc
// :40-55 (2^-23 tolerance band; `min({..})` folds left to right).  The corpus dispatcher (:57-59) always
// takes MT — the Pluecker test is here for the Appendix F fidelity check (SPEC acceptance criterion 9).
SCION_DEV bool ray_tri_mt_full(const RayCtx& ray, const float* p, float& b0, float& b1, float& b2, float& t_out) {
  const f32x3 p0{p[0], p[1], p[2]}, p1{p[3], p[4], p[5]}, p2{p[6], p[7], p[8]};
  const f32x3 e1 = p0 - p1, e2 = p2 - p0;
  const f32x3 ng = cross(e2, e1);
  const f32x3 c = p0 - f32x3{ray.ox, ray.oy, ray.oz};
  const f32x3 d{ray.dx, ray.dy, ray.dz};
  const f32x3 r = cross(c, d);
  const float D = dot(ng, d);
  if (D == 0.0f) return false;
  const float abs_D = scion::abs(D);
  const uint32_t sgn_D = f2u(D) & 2147483648u;
  const float u_raw = u2f(f2u(dot(r, e2)) ^ sgn_D);
  const float v_raw = u2f(f2u(dot(r, e1)) ^ sgn_D);
  if (!(u_raw >= 0.0f && v_raw >= 0.0f && u_raw + v_raw <= abs_D)) return false;
  const float t_raw = u2f(f2u(dot(ng, c)) ^ sgn_D);
  if (!(abs_D * 0.0f < t_raw && t_raw <= abs_D * ray.tmax)) return false;
  const float inv_abs_D = 1.0f / abs_D;
  t_out = t_raw * inv_abs_D;
  const float u = u_raw * inv_abs_D, v = v_raw * inv_abs_D;
  b0 = 1.0f - u - v;
  b1 = u;
  b2 = v;
  return true;
}
SCION_DEV bool ray_tri_pc_full(const RayCtx& ray, const float* p, float& b0, float& b1, float& b2, float& t_out) {
  const f32x3 o{ray.ox, ray.oy, ray.oz}, d{ray.dx, ray.dy, ray.dz};
  const f32x3 v0 = f32x3{p[0], p[1], p[2]} - o, v1 = f32x3{p[3], p[4], p[5]} - o, v2 = f32x3{p[6], p[7], p[8]} - o;
  const f32x3 e0 = v2 - v0, e1 = v0 - v1, e2 = v1 - v2;
  const float u_raw = dot(cross(e0, v2 + v0), d);
  const float v_raw = dot(cross(e1, v0 + v1), d);
  const float w_raw = dot(cross(e2, v1 + v2), d);
  const float uvw = (u_raw + v_raw) + w_raw;
  const float e = 0.00000011920928955078125f * scion::abs(uvw);
  const float min_uvw = fminf(fminf(u_raw, v_raw), w_raw), max_uvw = fmaxf(fmaxf(u_raw, v_raw), w_raw);
  if (!(min_uvw >= -e || max_uvw <= e)) return false;
  const f32x3 ng = cross(e0, e1);
  const float den = 2.0f * dot(ng, d), t_raw = 2.0f * dot(v0, ng);
  const float t = t_raw / den;
  if (!(t >= 0.0f && t <= ray.tmax)) return false;
  if (den == 0.0f) return false;
  const float inv_uvw = 1.0f / uvw;
  b0 = w_raw * inv_uvw;
  b1 = u_raw * inv_uvw;
  b2 = v_raw * inv_uvw;
  if (b0 < 0.0f || b1 < 0.0f || b2 < 0.0f) return false;
  t_out = t;
  return true;
}

// slab_hit, dop.scion:5-17
SCION_DEV bool slab_hit(float o, float d, float lo, float hi, float& tn, float& tf) {
  if (d == 0.0f) return !(o < lo || o > hi);
  const float inv = 1.0f / d;
  const float ta = (lo - o) * inv, tb = (hi - o) * inv;
  const float t0 = fminf(ta, tb), t1 = fmaxf(ta, tb);
  const float ntn = fmaxf(tn, t0), ntf = fminf(tf, t1);
  if (ntn <= ntf) { tn = ntn; tf = ntf; return true; }
  return false;
}
// the four diagonal slabs of dop_interval, dop.scion:22-43, refining an AABB interval in place
SCION_DEV bool dop_diagonals(const RayCtx& r, const f32x4& lo2, const f32x4& hi2, float& tn, float& tf) {
  const float o0 = r.ox + r.oy + r.oz, d0 = r.dx + r.dy + r.dz;
  const float o1 = r.ox + r.oy - r.oz, d1 = r.dx + r.dy - r.dz;
  const float o2 = r.ox - r.oy + r.oz, d2 = r.dx - r.dy + r.dz;
  const float o3 = r.ox - r.oy - r.oz, d3 = r.dx - r.dy - r.dz;
  if (!slab_hit(o0, d0, lo2.x, hi2.x, tn, tf)) return false;
  if (!slab_hit(o1, d1, lo2.y, hi2.y, tn, tf)) return false;
  if (!slab_hit(o2, d2, lo2.z, hi2.z, tn, tf)) return false;
  return slab_hit(o3, d3, lo2.w, hi2.w, tn, tf);
}

// square_distance_point_aabb, geometry.scion:105-110
SCION_DEV float sqdist_point_aabb(const f32x3& v, const f32x3& lo, const f32x3& hi) {
  const f32x3 dl = lo - v, dh = v - hi;
  const f32x3 sq_low = dl * dl, sq_high = dh * dh;
  const f32x3 low{v.x < lo.x ? sq_low.x : 0.0f, v.y < lo.y ? sq_low.y : 0.0f, v.z < lo.z ? sq_low.z : 0.0f};
  const f32x3 high{v.x > hi.x ? sq_high.x : 0.0f, v.y > hi.y ? sq_high.y : 0.0f, v.z > hi.z ? sq_high.z : 0.0f};
  return sum(low + high);
}
// distmax, geometry.scion:116-118
SCION_DEV float distmax_point_aabb(const f32x3& p, const f32x3& lo, const f32x3& hi) {
  const f32x3 u = lo - p, v = p - hi;
  const f32x3 d{fminf(u.x, v.x), fminf(u.y, v.y), fminf(u.z, v.z)};
  return dot(d, d);
}
// distmin_dop_point, dop.scion:61-77
SCION_DEV float distmin_dop_point(const f32x3& p, const f32x3& lo1, const f32x3& hi1, const f32x4& lo2, const f32x4& hi2) {
  const float base = sqdist_point_aabb(p, lo1, hi1);
  const float s0 = p.x + p.y + p.z, s1 = p.x + p.y - p.z, s2 = p.x - p.y + p.z, s3 = p.x - p.y - p.z;
  const float v0 = fmaxf(lo2.x - s0, fmaxf(s0 - hi2.x, 0.0f));
  const float v1 = fmaxf(lo2.y - s1, fmaxf(s1 - hi2.y, 0.0f));
  const float v2 = fmaxf(lo2.z - s2, fmaxf(s2 - hi2.z, 0.0f));
  const float v3 = fmaxf(lo2.w - s3, fmaxf(s3 - hi2.w, 0.0f));
  const float third = 1.0f / 3.0f;
  const float d0 = v0 * v0 * third, d1 = v1 * v1 * third, d2 = v2 * v2 * third, d3 = v3 * v3 * third;
  return fmaxf(base, fmaxf(fmaxf(d0, d1), fmaxf(d2, d3)));
}
// distmin_point_triangle, geometry.scion:76-100 (closest point only; barycentrics are unused by cpq)
SCION_DEV f32x3 closest_point_triangle(const f32x3& p, const float* t) {
  const f32x3 a{t[0], t[1], t[2]}, b{t[3], t[4], t[5]}, c{t[6], t[7], t[8]};
  const f32x3 ab = b - a, ac = c - a, ap = p - a;
  const float d1 = dot(ab, ap), d2 = dot(ac, ap);
  if (d1 <= 0.0f && d2 <= 0.0f) return a;
  const f32x3 bp = p - b;
  const float d3 = dot(ab, bp), d4 = dot(ac, bp);
  if (d3 >= 0.0f && d4 <= d3) return b;
  const float vc = d1 * d4 - d3 * d2;
  if (vc <= 0.0f && d1 >= 0.0f && d3 <= 0.0f) {
    const float v0 = d1 / (d1 - d3);
    return a + ab * v0;  // a + v0 * ab: multiplication commutes bitwise
  }
  const f32x3 cp = p - c;
  const float d5 = dot(ab, cp), d6 = dot(ac, cp);
  if (d6 >= 0.0f && d5 <= d6) return c;
  const float vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0f && d2 >= 0.0f && d6 <= 0.0f) {
    const float w0 = d2 / (d2 - d6);
    return a + ac * w0;
  }
  const float va = d3 * d6 - d5 * d4;
  if (va <= 0.0f && (d4 - d3) >= 0.0f && (d5 - d6) >= 0.0f) {
    const float w1 = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    return b + (c - b) * w1;
  }
  const float D = 1.0f / (va + vb + vc);
  const float v = vb * D, w = vc * D;
  return (a + ab * v) + ac * w;
}

// Triangle = 3 x f32x3 = 36 B at a 4-byte-aligned address (stride 36, plan.cpp:195-210).  One
// triangle is fetched as the three aligned 16-byte words that cover it — 3 read-only vector
// loads instead of nine 4-byte ones — and re-aligned in registers.  Device buffers carry 16
// bytes of slack so the covering read of the last triangle stays inside the allocation.
SCION_DEV void load_triangle36(const uint8_t* prims, uint64_t index, float (&v)[9]) {
#if defined(__CUDA_ARCH__) && SCION_TRI_LDG32
  const uint32_t* q = reinterpret_cast<const uint32_t*>(prims + index * 36ull);
#pragma unroll
  for (int j = 0; j < 9; j++) v[j] = u2f(__ldg(q + j));
#elif defined(__CUDA_ARCH__) && SCION_TRI_LDG256
  // 36 bytes at a 4-byte aligned address never span more than two 32-byte sectors: two 256-bit loads (one L1 wavefront
  // per lane each) instead of three 128-bit ones, word re-alignment by a three-level select
  const uint64_t addr = (uint64_t)prims + index * 36ull;
  const uint8_t* q = reinterpret_cast<const uint8_t*>(addr & ~31ull);
  const uint32_t s = (uint32_t)(addr >> 2) & 7u;
  uint32_t w[16];
#if SCION_CACHE_HINTS >= 3
  const uint64_t pol = l2_policy_stream();
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]) : "l"(q), "l"(pol));
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
               : "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15]) : "l"(q + 32), "l"(pol));
#else
  ld256(q, w);
  ld256(q + 32, w + 8);
#endif
  const bool s1 = (s & 1u) != 0u, s2 = (s & 2u) != 0u, s4 = (s & 4u) != 0u;
  uint32_t x[12];  // words s4 ? [4, 16) : [0, 12)
#pragma unroll
  for (int j = 0; j < 12; j++) x[j] = s4 ? w[j + 4] : w[j];
#pragma unroll
  for (int j = 0; j < 9; j++) {
    const uint32_t lo = s1 ? x[j + 1] : x[j];
    const uint32_t hi = s1 ? x[j + 3] : x[j + 2];
    v[j] = u2f(s2 ? hi : lo);
  }
#elif defined(__CUDA_ARCH__)
  const uint64_t addr = (uint64_t)prims + index * 36ull;
  const uint4* q = reinterpret_cast<const uint4*>(addr & ~15ull);
  const uint32_t s = (uint32_t)(addr >> 2) & 3u;
#if SCION_CACHE_HINTS >= 3
  uint4 a, b, c;
  const uint64_t pol = l2_policy_stream();
#ifndef SCION_L2_PROMO_TRI
#define SCION_L2_PROMO_TRI 0
#endif
#if SCION_L2_PROMO_TRI > 0
#define SCION_TRI_Q ".L2::" SCION_STR(SCION_L2_PROMO_TRI) "B"
#else
#define SCION_TRI_Q ""
#endif
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint" SCION_TRI_Q ".v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(q), "l"(pol));
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint" SCION_TRI_Q ".v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(q + 1), "l"(pol));
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint" SCION_TRI_Q ".v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "l"(q + 2), "l"(pol));
#elif SCION_CACHE_HINTS >= 2
  uint4 a, b, c;
  const uint64_t pol = l2_policy_stream();
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(q), "l"(pol));
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(q + 1), "l"(pol));
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "l"(q + 2), "l"(pol));
#else
  const uint4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
#endif
  const uint32_t w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
  const bool s1 = (s & 1u) != 0u, s2 = (s & 2u) != 0u;
#pragma unroll
  for (int j = 0; j < 9; j++) {
    const uint32_t lo = s1 ? w[j + 1] : w[j];
    const uint32_t hi = s1 ? w[j + 3] : w[j + 2];
    v[j] = u2f(s2 ? hi : lo);
  }
#else
  memcpy(v, prims + index * 36ull, 36);
#endif
}

}  // namespace scion
