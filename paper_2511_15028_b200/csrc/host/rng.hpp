// Seeded stateless PRNG + query generators shared by host code and device code.
//
// Stands in for the reference's src/rng.cpp (a 15-byte placeholder); the contract is
// "named 64-bit seeded PRNG (splitmix-style)", seeded
// generation reproducible byte-for-byte.  Every query is a pure function of
// (seed, global query index), so any number of ranks generates identical inputs.
//
// Only + - * / sqrt and integer ops are used; with -fmad=false (device) and
// -ffp-contract=off (host) the host and device twins are bit-identical.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define SCION_HD __host__ __device__ __forceinline__
#else
#define SCION_HD inline
#endif

#include "scion_b200.h"

namespace scion {

SCION_HD float rng_inf() {
#if defined(__CUDA_ARCH__)
  return __int_as_float(0x7f800000);
#else
  return __builtin_inff();
#endif
}

SCION_HD uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// counter-based stream: draw k of query `index` under `seed`
struct Stream {
  uint64_t key;
  uint64_t ctr;
  SCION_HD Stream(uint64_t seed, uint64_t index) : key(splitmix64(seed ^ 0x5ca1ab1e0ddba11ull) + index * 0xd1342543de82ef95ull), ctr(0) {}
  SCION_HD uint64_t next() { return splitmix64(key + (ctr++) * 0x9e3779b97f4a7c15ull); }
  // uniform in [0,1): 24 random bits, exactly representable
  SCION_HD float uniform() { return (float)(next() >> 40) * (1.0f / 16777216.0f); }
};

SCION_HD float sqrt_rn(float x) {
#if defined(__CUDA_ARCH__)
  return __fsqrt_rn(x);
#else
  return __builtin_sqrtf(x);
#endif
}
SCION_HD float div_rn(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fdiv_rn(a, b);
#else
  return a / b;
#endif
}
SCION_HD float mul_rn(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fmul_rn(a, b);
#else
  return a * b;
#endif
}
SCION_HD float add_rn(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fadd_rn(a, b);
#else
  return a + b;
#endif
}
SCION_HD float sub_rn(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fsub_rn(a, b);
#else
  return a - b;
#endif
}

// Camera basis prepared on the host once (double precision trig stays on the host).
struct CameraBasis {
  float eye[3];
  float fwd[3], right[3], up[3];  // orthonormal-ish basis
  float tan_half_x, tan_half_y;
  uint32_t width, height;
};

// Primary ray for pixel index (row-major), direction normalised with correctly rounded ops.
SCION_HD scion_ray primary_ray(const CameraBasis& c, uint64_t index) {
  uint64_t npix = (uint64_t)c.width * c.height;
  uint64_t p = index % npix;
  uint32_t px = (uint32_t)(p % c.width), py = (uint32_t)(p / c.width);
  // pixel centre in [-1,1]
  float u = sub_rn(mul_rn(div_rn(add_rn((float)px, 0.5f), (float)c.width), 2.0f), 1.0f);
  float v = sub_rn(1.0f, mul_rn(div_rn(add_rn((float)py, 0.5f), (float)c.height), 2.0f));
  float su = mul_rn(u, c.tan_half_x), sv = mul_rn(v, c.tan_half_y);
  float d[3];
  for (int a = 0; a < 3; a++) d[a] = add_rn(add_rn(c.fwd[a], mul_rn(su, c.right[a])), mul_rn(sv, c.up[a]));
  float len = sqrt_rn(add_rn(add_rn(mul_rn(d[0], d[0]), mul_rn(d[1], d[1])), mul_rn(d[2], d[2])));
  scion_ray r;
  r.ox = c.eye[0]; r.oy = c.eye[1]; r.oz = c.eye[2];
  r.dx = div_rn(d[0], len); r.dy = div_rn(d[1], len); r.dz = div_rn(d[2], len);
  r.tmax = rng_inf();
  r.pad = 0.0f;
  return r;
}

// Secondary ray: origin on a hash-chosen triangle (+ eps * normal), direction uniform over
// the hemisphere about the geometric normal (rejection-sampled unit-ball vector, normalised).
SCION_HD scion_ray secondary_ray(const float* tris9, uint64_t ntris, uint64_t seed, uint64_t index) {
  Stream s(seed, index);
  uint64_t t = s.next() % ntris;
  const float* T = tris9 + t * 9;
  float b0 = s.uniform(), b1 = s.uniform();
  if (add_rn(b0, b1) > 1.0f) { b0 = sub_rn(1.0f, b0); b1 = sub_rn(1.0f, b1); }
  float b2 = sub_rn(sub_rn(1.0f, b0), b1);
  float o[3], e1[3], e2[3];
  for (int a = 0; a < 3; a++) {
    o[a] = add_rn(add_rn(mul_rn(b0, T[a]), mul_rn(b1, T[3 + a])), mul_rn(b2, T[6 + a]));
    e1[a] = sub_rn(T[3 + a], T[a]);
    e2[a] = sub_rn(T[6 + a], T[a]);
  }
  float n[3] = {sub_rn(mul_rn(e1[1], e2[2]), mul_rn(e1[2], e2[1])), sub_rn(mul_rn(e1[2], e2[0]), mul_rn(e1[0], e2[2])),
                sub_rn(mul_rn(e1[0], e2[1]), mul_rn(e1[1], e2[0]))};
  float nl = sqrt_rn(add_rn(add_rn(mul_rn(n[0], n[0]), mul_rn(n[1], n[1])), mul_rn(n[2], n[2])));
  if (nl > 0.0f) { n[0] = div_rn(n[0], nl); n[1] = div_rn(n[1], nl); n[2] = div_rn(n[2], nl); }
  else { n[0] = 0.0f; n[1] = 1.0f; n[2] = 0.0f; }
  float d[3], l2;
  int tries = 0;
  do {
    d[0] = sub_rn(mul_rn(s.uniform(), 2.0f), 1.0f);
    d[1] = sub_rn(mul_rn(s.uniform(), 2.0f), 1.0f);
    d[2] = sub_rn(mul_rn(s.uniform(), 2.0f), 1.0f);
    l2 = add_rn(add_rn(mul_rn(d[0], d[0]), mul_rn(d[1], d[1])), mul_rn(d[2], d[2]));
  } while ((l2 > 1.0f || l2 < 1e-6f) && ++tries < 64);
  if (l2 > 1.0f || l2 < 1e-6f) { d[0] = n[0]; d[1] = n[1]; d[2] = n[2]; l2 = 1.0f; }
  float l = sqrt_rn(l2);
  d[0] = div_rn(d[0], l); d[1] = div_rn(d[1], l); d[2] = div_rn(d[2], l);
  float dn = add_rn(add_rn(mul_rn(d[0], n[0]), mul_rn(d[1], n[1])), mul_rn(d[2], n[2]));
  if (dn < 0.0f) { d[0] = -d[0]; d[1] = -d[1]; d[2] = -d[2]; }
  const float eps = 1.0f / 4096.0f;
  scion_ray r;
  r.ox = add_rn(o[0], mul_rn(eps, n[0])); r.oy = add_rn(o[1], mul_rn(eps, n[1])); r.oz = add_rn(o[2], mul_rn(eps, n[2]));
  r.dx = d[0]; r.dy = d[1]; r.dz = d[2];
  r.tmax = rng_inf();
  r.pad = 0.0f;
  return r;
}

SCION_HD void query_point(const float lo[3], const float hi[3], uint64_t seed, uint64_t index, float out[3]) {
  Stream s(seed, index);
  for (int a = 0; a < 3; a++) out[a] = add_rn(lo[a], mul_rn(s.uniform(), sub_rn(hi[a], lo[a])));
}

}  // namespace scion
