// TEST INFRASTRUCTURE — CPU oracle, not part of the product.  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may use anything under oracle/.
//
// Strict binary32 restatement of the reference's DSL standard library:
//   /root/reference/proj/corpus/lib/geometry.scion  (ray/AABB :12-22, MT :25-38, dispatcher :57-72,
//   closest point on triangle :76-100, point/AABB :105-118)
//   /root/reference/proj/corpus/lib/dop.scion       (slab_hit :5-17, dop_interval :19-46,
//   intersects_dop/distmin_dop :48-57, distmin_dop_point :61-77)
// Typing rules that fix the precision: every float is f32 (src/sema.cpp:498-504, :586-610).
// Compile with -ffp-contract=off (the reference's own flag, proj/CMakeLists.txt:13-15).
//
// PARITY PINNING: the reference ships no executor (src/interp.cpp is a placeholder), so this
// restatement is pinned against the reference's known-answer vectors (SPEC.md:446-448, :455-457,
// :472-474, :490-492, :499-504) in tests/test_oracle_kats.py.  The intrinsic conventions the
// reference leaves open are frozen here (SURVEY §8c "parity unpinned" list): dot/cross/sum
// association ((x+y)+z), min/max = fminf/fmaxf, select(m,a,b) = m ? a : b, abs = clear sign bit,
// TRUE directed rounding.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>

namespace oracle {

struct V3 { float x, y, z; };
struct V4 { float x, y, z, w; };
struct Ray { V3 o, d; float tmax; };
struct Box { V3 lo, hi; };
struct Tri { V3 p0, p1, p2; };

static const float INF = std::numeric_limits<float>::infinity();

inline uint32_t bits_of(float f) { uint32_t u; std::memcpy(&u, &f, 4); return u; }
inline float float_of(uint32_t u) { float f; std::memcpy(&f, &u, 4); return f; }

inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 mul(V3 a, float s) { return {a.x * s, a.y * s, a.z * s}; }
inline float dot(V3 a, V3 b) { return ((a.x * b.x) + (a.y * b.y)) + (a.z * b.z); }
inline V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline float fabs_bits(float a) { return float_of(bits_of(a) & 0x7fffffffu); }

// ------------------------------------------------------------------ directed rounding
// Exact: the product of two binary32 values is exact in binary64; sums use the TwoSum error
// term; quotients of binary32 values never fall within half a binary64 ulp of a binary32
// boundary without being exact.  (Deliberately NOT the fesetround route the product's host
// encoder takes, so the two implementations check each other.)
inline float next_down(float f) { return std::nextafterf(f, -INF); }
inline float next_up(float f) { return std::nextafterf(f, INF); }
inline float round_from_double(double exact, bool up) {
  float f = (float)exact;
  if (std::isnan(exact) || std::isinf(f)) {
    // overflow of a finite exact value: round-down gives FLT_MAX for +, round-up gives -FLT_MAX for -
    if (std::isinf(f) && std::isfinite(exact)) {
      if (!up && f > 0) return std::numeric_limits<float>::max();
      if (up && f < 0) return -std::numeric_limits<float>::max();
    }
    return f;
  }
  if (!up && (double)f > exact) return next_down(f);
  if (up && (double)f < exact) return next_up(f);
  return f;
}
inline float fmul_rd(float a, float b) { return round_from_double((double)a * (double)b, false); }
inline float fadd_dir(float a, float b, bool up) {
  float s = a + b;
  if (!std::isfinite(s) || !std::isfinite(a) || !std::isfinite(b)) return s;
  float bb = s - a;
  float err = (a - (s - bb)) + (b - bb);  // exact error of the RNE sum
  if (s == 0.0f && err == 0.0f) {
    // exact zero: sign depends on the rounding direction (x + (-x) = -0 when rounding down)
    if (bits_of(a) != bits_of(b) || a != 0.0f) return up ? 0.0f : -0.0f;
    return s;
  }
  if (!up && err < 0.0f) return next_down(s);
  if (up && err > 0.0f) return next_up(s);
  return s;
}
inline float fadd_rd(float a, float b) { return fadd_dir(a, b, false); }
inline float fsub_rd(float a, float b) { return fadd_dir(a, -b, false); }
inline float fsub_ru(float a, float b) { return fadd_dir(a, -b, true); }
inline float fdiv_rd(float a, float b) { return round_from_double((double)a / (double)b, false); }
inline float frcp_rd(float a) { return round_from_double(1.0 / (double)a, false); }

// ------------------------------------------------------------------ geometry.scion:12-22
struct Interval { bool some; float low, high; };
inline Interval ray_aabb(const Ray& r, const Box& b) {
  float rdx = 1.0f / r.d.x, rdy = 1.0f / r.d.y, rdz = 1.0f / r.d.z;
  bool nx_ = r.d.x < 0.0f, ny_ = r.d.y < 0.0f, nz_ = r.d.z < 0.0f;
  float nx = nx_ ? b.hi.x : b.lo.x, fx = nx_ ? b.lo.x : b.hi.x;
  float ny = ny_ ? b.hi.y : b.lo.y, fy = ny_ ? b.lo.y : b.hi.y;
  float nz = nz_ ? b.hi.z : b.lo.z, fz = nz_ ? b.lo.z : b.hi.z;
  float t_nx = (nx - r.o.x) * rdx, t_fx = (fx - r.o.x) * rdx;
  float t_ny = (ny - r.o.y) * rdy, t_fy = (fy - r.o.y) * rdy;
  float t_nz = (nz - r.o.z) * rdz, t_fz = (fz - r.o.z) * rdz;
  float t_near = fmaxf(0.0f, fmaxf(t_nx, fmaxf(t_ny, t_nz)));
  float t_far = fminf(r.tmax, fminf(t_fx, fminf(t_fy, t_fz)));
  if (t_near <= t_far) return {true, t_near, t_far};
  return {false, 0.0f, 0.0f};
}
// geometry.scion:61-66
inline bool intersects(const Ray& r, const Box& b) {
  Interval I = ray_aabb(r, b);
  if (I.some) return I.low < r.tmax && I.high > 0;
  return false;
}
inline float distmin(const Ray& r, const Box& b) {
  Interval I = ray_aabb(r, b);
  if (I.some) return I.low;
  return INF;
}

// ------------------------------------------------------------------ geometry.scion:25-38
struct TriHit { bool some; float b0, b1, b2, t; };
inline TriHit ray_tri_mt(const Ray& ray, const Tri& tri) {
  V3 e1 = sub(tri.p0, tri.p1), e2 = sub(tri.p2, tri.p0), ng = cross(e2, e1);
  V3 c = sub(tri.p0, ray.o), r = cross(c, ray.d);
  float D = dot(ng, ray.d);
  if (D == 0.0f) return {false, 0, 0, 0, 0};
  float abs_D = fabs_bits(D);
  uint32_t sgn_D = bits_of(D) & 2147483648u;
  float u_raw = float_of(bits_of(dot(r, e2)) ^ sgn_D), v_raw = float_of(bits_of(dot(r, e1)) ^ sgn_D);
  if (!(u_raw >= 0.0f && v_raw >= 0.0f && u_raw + v_raw <= abs_D)) return {false, 0, 0, 0, 0};
  float t_raw = float_of(bits_of(dot(ng, c)) ^ sgn_D);
  if (!(abs_D * 0.0f < t_raw && t_raw <= abs_D * ray.tmax)) return {false, 0, 0, 0, 0};
  float inv_abs_D = 1.0f / abs_D;
  float t = t_raw * inv_abs_D, u = u_raw * inv_abs_D, v = v_raw * inv_abs_D;
  float b0 = 1.0f - u - v;
  return {true, b0, u, v, t};
}

// ------------------------------------------------------------------ geometry.scion:40-55 (Pluecker-coordinate test)
// 2^-23 edge tolerance band; `min({..})` / `max({..})` fold left to right; the dispatcher
// (geometry.scion:57-59) always selects MT, so no traversal of the corpus calls this one — it exists for the
// Appendix F fidelity check (SPEC acceptance criterion 9: MT vs Pluecker cross-agreement).
inline TriHit ray_tri_pc(const Ray& ray, const Tri& tri) {
  V3 v0 = sub(tri.p0, ray.o), v1 = sub(tri.p1, ray.o), v2 = sub(tri.p2, ray.o);
  V3 e0 = sub(v2, v0), e1 = sub(v0, v1), e2 = sub(v1, v2);
  float u_raw = dot(cross(e0, add(v2, v0)), ray.d);
  float v_raw = dot(cross(e1, add(v0, v1)), ray.d);
  float w_raw = dot(cross(e2, add(v1, v2)), ray.d);
  float uvw = (u_raw + v_raw) + w_raw;
  float e = 0.00000011920928955078125f * fabs_bits(uvw);
  float min_uvw = fminf(fminf(u_raw, v_raw), w_raw), max_uvw = fmaxf(fmaxf(u_raw, v_raw), w_raw);
  if (!(min_uvw >= -e || max_uvw <= e)) return {false, 0, 0, 0, 0};
  V3 ng = cross(e0, e1);
  float den = 2.0f * dot(ng, ray.d), t_raw = 2.0f * dot(v0, ng);
  float t = t_raw / den;
  if (!(t >= 0.0f && t <= ray.tmax)) return {false, 0, 0, 0, 0};
  if (den == 0.0f) return {false, 0, 0, 0, 0};
  float inv_uvw = 1.0f / uvw;
  float b0 = w_raw * inv_uvw, b1 = u_raw * inv_uvw, b2 = v_raw * inv_uvw;
  if (b0 < 0.0f || b1 < 0.0f || b2 < 0.0f) return {false, 0, 0, 0, 0};
  return {true, b0, b1, b2, t};
}

// ------------------------------------------------------------------ geometry.scion:76-100
struct ClosestPt { V3 p; V3 bary; };
inline ClosestPt point_triangle(V3 p, const Tri& tri) {
  V3 a = tri.p0, b = tri.p1, c = tri.p2;
  V3 ab = sub(b, a), ac = sub(c, a), ap = sub(p, a);
  float d1 = dot(ab, ap), d2 = dot(ac, ap);
  if (d1 <= 0.0f && d2 <= 0.0f) return {a, {1.0f, 0.0f, 0.0f}};
  V3 bp = sub(p, b);
  float d3 = dot(ab, bp), d4 = dot(ac, bp);
  if (d3 >= 0.0f && d4 <= d3) return {b, {0.0f, 1.0f, 0.0f}};
  float vc = d1 * d4 - d3 * d2;
  if (vc <= 0.0f && d1 >= 0.0f && d3 <= 0.0f) {
    float v0 = d1 / (d1 - d3);
    return {add(a, mul(ab, v0)), {1.0f - v0, v0, 0.0f}};
  }
  V3 cp = sub(p, c);
  float d5 = dot(ab, cp), d6 = dot(ac, cp);
  if (d6 >= 0.0f && d5 <= d6) return {c, {0.0f, 0.0f, 1.0f}};
  float vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0f && d2 >= 0.0f && d6 <= 0.0f) {
    float w0 = d2 / (d2 - d6);
    return {add(a, mul(ac, w0)), {1.0f - w0, 0.0f, w0}};
  }
  float va = d3 * d6 - d5 * d4;
  if (va <= 0.0f && (d4 - d3) >= 0.0f && (d5 - d6) >= 0.0f) {
    float w1 = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    return {add(b, mul(sub(c, b), w1)), {0.0f, 1.0f - w1, w1}};
  }
  float D = 1.0f / (va + vb + vc);
  float v = vb * D, w = vc * D, u = va * D;
  return {add(add(a, mul(ab, v)), mul(ac, w)), {u, v, w}};
}
// geometry.scion:105-110
inline float sqdist_point_aabb(V3 v, const Box& a) {
  V3 dl = sub(a.lo, v), dh = sub(v, a.hi);
  V3 sq_low = {dl.x * dl.x, dl.y * dl.y, dl.z * dl.z};
  V3 low = {v.x < a.lo.x ? sq_low.x : 0.0f, v.y < a.lo.y ? sq_low.y : 0.0f, v.z < a.lo.z ? sq_low.z : 0.0f};
  V3 sq_high = {dh.x * dh.x, dh.y * dh.y, dh.z * dh.z};
  V3 high = {v.x > a.hi.x ? sq_high.x : 0.0f, v.y > a.hi.y ? sq_high.y : 0.0f, v.z > a.hi.z ? sq_high.z : 0.0f};
  V3 s = add(low, high);
  return (s.x + s.y) + s.z;
}
// geometry.scion:116-118
inline float distmax_point_aabb(V3 p, const Box& a) {
  V3 u = sub(a.lo, p), v = sub(p, a.hi);
  V3 d = {fminf(u.x, v.x), fminf(u.y, v.y), fminf(u.z, v.z)};
  return dot(d, d);
}

// ------------------------------------------------------------------ dop.scion:5-57
inline Interval slab_hit(float o, float d, float lo, float hi, float tn, float tf) {
  if (d == 0.0f) {
    if (o < lo || o > hi) return {false, 0, 0};
    return {true, tn, tf};
  }
  float inv = 1.0f / d;
  float ta = (lo - o) * inv, tb = (hi - o) * inv;
  float t0 = fminf(ta, tb), t1 = fmaxf(ta, tb);
  float ntn = fmaxf(tn, t0), ntf = fminf(tf, t1);
  if (ntn <= ntf) return {true, ntn, ntf};
  return {false, 0, 0};
}
inline Interval dop_interval(const Ray& r, V3 lo1, V3 hi1, V4 lo2, V4 hi2) {
  Interval I = ray_aabb(r, Box{lo1, hi1});
  if (I.some) {
    float o0 = r.o.x + r.o.y + r.o.z, d0 = r.d.x + r.d.y + r.d.z;
    float o1 = r.o.x + r.o.y - r.o.z, d1 = r.d.x + r.d.y - r.d.z;
    float o2 = r.o.x - r.o.y + r.o.z, d2 = r.d.x - r.d.y + r.d.z;
    float o3 = r.o.x - r.o.y - r.o.z, d3 = r.d.x - r.d.y - r.d.z;
    Interval s0 = slab_hit(o0, d0, lo2.x, hi2.x, I.low, I.high);
    if (s0.some) {
      Interval s1 = slab_hit(o1, d1, lo2.y, hi2.y, s0.low, s0.high);
      if (s1.some) {
        Interval s2 = slab_hit(o2, d2, lo2.z, hi2.z, s1.low, s1.high);
        if (s2.some) {
          Interval s3 = slab_hit(o3, d3, lo2.w, hi2.w, s2.low, s2.high);
          if (s3.some) return s3;
        }
      }
    }
  }
  return {false, 0, 0};
}
inline bool intersects_dop(const Ray& r, V3 lo1, V3 hi1, V4 lo2, V4 hi2) {
  Interval I = dop_interval(r, lo1, hi1, lo2, hi2);
  if (I.some) return I.low < r.tmax && I.high > 0;
  return false;
}
inline float distmin_dop(const Ray& r, V3 lo1, V3 hi1, V4 lo2, V4 hi2) {
  Interval I = dop_interval(r, lo1, hi1, lo2, hi2);
  if (I.some) return I.low;
  return INF;
}
// dop.scion:61-77
inline float distmin_dop_point(V3 p, V3 lo1, V3 hi1, V4 lo2, V4 hi2) {
  float base = sqdist_point_aabb(p, Box{lo1, hi1});
  float s0 = p.x + p.y + p.z, s1 = p.x + p.y - p.z, s2 = p.x - p.y + p.z, s3 = p.x - p.y - p.z;
  float v0 = fmaxf(lo2.x - s0, fmaxf(s0 - hi2.x, 0.0f));
  float v1 = fmaxf(lo2.y - s1, fmaxf(s1 - hi2.y, 0.0f));
  float v2 = fmaxf(lo2.z - s2, fmaxf(s2 - hi2.z, 0.0f));
  float v3 = fmaxf(lo2.w - s3, fmaxf(s3 - hi2.w, 0.0f));
  float third = 1.0f / 3.0f;
  float d0 = v0 * v0 * third, d1 = v1 * v1 * third, d2 = v2 * v2 * third, d3 = v3 * v3 * third;
  return fmaxf(base, fmaxf(fmaxf(d0, d1), fmaxf(d2, d3)));
}

// ------------------------------------------------------------------ geometry.scion:112-157 (collision detection)
// project6 (:112-118)
inline int project6(V3 ax, V3 p1, V3 p2, V3 p3, V3 q1, V3 q2, V3 q3) {
  float P1 = dot(ax, p1), P2 = dot(ax, p2), P3 = dot(ax, p3);
  float Q1 = dot(ax, q1), Q2 = dot(ax, q2), Q3 = dot(ax, q3);
  float mn1 = fminf(fminf(P1, P2), P3), mx2 = fmaxf(fmaxf(Q1, Q2), Q3);
  if (mn1 > mx2) return 0;
  float mx1 = fmaxf(fmaxf(P1, P2), P3), mn2 = fminf(fminf(Q1, Q2), Q3);
  if (mn2 > mx1) return 0;
  return 1;
}
// SAT_triangle_intersection over the 17 candidate axes (:120-154)
inline bool sat_triangles(const Tri& A, const Tri& B) {
  V3 p1{0.0f, 0.0f, 0.0f}, p2 = sub(A.p1, A.p0), p3 = sub(A.p2, A.p0);
  V3 q1 = sub(B.p0, A.p0), q2 = sub(B.p1, A.p0), q3 = sub(B.p2, A.p0);
  V3 e1 = sub(p2, p1), e2 = sub(p3, p2), n1 = cross(e1, e2);
  if (project6(n1, p1, p2, p3, q1, q2, q3) == 0) return false;
  V3 f1 = sub(q2, q1), f2 = sub(q3, q2), m1 = cross(f1, f2);
  if (project6(m1, p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(e1, f1), p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(e1, f2), p1, p2, p3, q1, q2, q3) == 0) return false;
  V3 f3 = sub(q1, q3);
  if (project6(cross(e1, f3), p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(e2, f1), p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(e2, f2), p1, p2, p3, q1, q2, q3) == 0) return false;
  if (project6(cross(e2, f3), p1, p2, p3, q1, q2, q3) == 0) return false;
  V3 e3 = sub(p1, p3);
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
// intersects(AABB, AABB) (:158-160)
inline bool aabb_overlap(const Box& a, const Box& b) {
  V3 low{fmaxf(a.lo.x, b.lo.x), fmaxf(a.lo.y, b.lo.y), fmaxf(a.lo.z, b.lo.z)};
  V3 high{fminf(a.hi.x, b.hi.x), fminf(a.hi.y, b.hi.y), fminf(a.hi.z, b.hi.z)};
  return low.x <= high.x && low.y <= high.y && low.z <= high.z;
}
// intersects_dop_dop (dop.scion:81-90)
inline bool dop_overlap(const Box& a, V4 alo2, V4 ahi2, const Box& b, V4 blo2, V4 bhi2) {
  if (!aabb_overlap(a, b)) return false;
  if (alo2.x > bhi2.x || blo2.x > ahi2.x) return false;
  if (alo2.y > bhi2.y || blo2.y > ahi2.y) return false;
  if (alo2.z > bhi2.z || blo2.z > ahi2.z) return false;
  if (alo2.w > bhi2.w || blo2.w > ahi2.w) return false;
  return true;
}

}  // namespace oracle
