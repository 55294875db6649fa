"""Pins the CPU oracle (oracle/) against every known-answer vector the reference holds for this
path (SPEC.md [MODULE] geometry-runtime examples :446-504, layout-model :214-217, specializer
:282-284) and against the properties it states (directed rounding post-conditions, quantisation
enclosure, bit-packing round trips — acceptance criteria 3 and 5)."""
import ctypes as C

import numpy as np
import pytest

F = lambda *v: np.array(v, np.float32)
INF = np.float32(np.inf)


def ray_aabb(orc, o, d, tmax, lo, hi):
    out = np.zeros(2, np.float32)
    o, d, lo, hi = F(*o), F(*d), F(*lo), F(*hi)  # keep the arrays alive across the call
    some = orc.lib.oracle_ray_aabb(o.ctypes.data, d.ctypes.data, tmax, lo.ctypes.data, hi.ctypes.data, out.ctypes.data)
    return some, out


def ray_tri(orc, o, d, tmax, tri):
    out = np.zeros(4, np.float32)
    o, d, tri = F(*o), F(*d), F(*tri)
    some = orc.lib.oracle_ray_tri(o.ctypes.data, d.ctypes.data, tmax, tri.ctypes.data, out.ctypes.data)
    return some, out


def point_tri(orc, p, tri):
    pt, b = np.zeros(3, np.float32), np.zeros(3, np.float32)
    p, tri = F(*p), F(*tri)
    orc.lib.oracle_point_tri(p.ctypes.data, tri.ctypes.data, pt.ctypes.data, b.ctypes.data)
    return pt, b


def box_fn(fn, p, lo, hi):
    p, lo, hi = F(*p), F(*lo), F(*hi)
    return fn(p.ctypes.data, lo.ctypes.data, hi.ctypes.data)


def test_ray_aabb_kats(oracle):
    some, I = ray_aabb(oracle, (0, 0, -2), (0, 0, 1), INF, (-1, -1, -1), (1, 1, 1))
    assert some == 1 and I[0] == 1.0 and I[1] == 3.0
    some, _ = ray_aabb(oracle, (0, 0, -2), (0, 0, 1), 0.5, (-1, -1, -1), (1, 1, 1))
    assert some == 0
    some, I = ray_aabb(oracle, (0.1, 0.2, 0.3), (0, 0, 1), INF, (-1, -1, -1), (1, 1, 1))
    assert some == 1 and I[0] == 0.0


def test_ray_aabb_zero_direction_nan_path(oracle):
    # direction component 0 and origin exactly on a slab plane: 0 * inf = NaN must be absorbed by
    # fmaxf/fminf — the ray grazing the face still reports an interval
    some, I = ray_aabb(oracle, (-1.0, 0, -2), (0, 0, 1), INF, (-1, -1, -1), (1, 1, 1))
    assert some == 1 and I[0] == 1.0
    some, _ = ray_aabb(oracle, (-1.5, 0, -2), (0, 0, 1), INF, (-1, -1, -1), (1, 1, 1))
    assert some == 0


def test_moeller_trumbore_kats(oracle):
    tri = (0, 0, 0, 1, 0, 0, 0, 1, 0)
    some, r = ray_tri(oracle, (0.25, 0.25, -1), (0, 0, 1), INF, tri)
    assert some == 1 and tuple(r) == (0.5, 0.25, 0.25, 1.0)
    some, _ = ray_tri(oracle, (0.25, 0.25, -1), (1, 0, 0), INF, tri)  # parallel to the plane: D == 0
    assert some == 0
    some, _ = ray_tri(oracle, (0.25, 0.25, -1), (0, 0, 1), 0.5, tri)  # beyond tmax
    assert some == 0
    some, r = ray_tri(oracle, (0.25, 0.25, 1), (0, 0, -1), INF, tri)  # back face: sign mask path
    assert some == 1 and r[3] == 1.0


def test_closest_point_triangle_kats(oracle):
    tri = (0, 0, 0, 1, 0, 0, 0, 1, 0)
    pt, b = point_tri(oracle, (-1, -1, 0.5), tri)
    assert tuple(pt) == (0, 0, 0) and tuple(b) == (1, 0, 0)  # vertex region a
    pt, b = point_tri(oracle, (0.25, 0.25, 0), tri)
    assert tuple(pt) == (0.25, 0.25, 0)  # on the triangle: distance 0
    pt, b = point_tri(oracle, (0.25, 0.25, 2), tri)
    assert np.allclose(pt, (0.25, 0.25, 0)) and abs(b.sum() - 1) < 1e-6  # orthogonal projection
    pt, b = point_tri(oracle, (0, 0, 0), (3, 4, 5, 3, 4, 5, 3, 4, 5))  # degenerate triangle = point (BASELINE config 4)
    assert tuple(pt) == (3, 4, 5)


def test_point_aabb(oracle):
    assert box_fn(oracle.lib.oracle_sqdist_point_aabb, (2, 0, 0), (-1, -1, -1), (1, 1, 1)) == 1.0
    assert box_fn(oracle.lib.oracle_sqdist_point_aabb, (0, 0, 0), (-1, -1, -1), (1, 1, 1)) == 0.0
    assert box_fn(oracle.lib.oracle_distmax_point_aabb, (0, 0, 0), (-1, -1, -1), (1, 1, 1)) == 3.0


def test_directed_rounding_kats_and_properties(oracle):
    L = oracle.lib
    third = np.float32(1) / np.float32(3)
    assert L.oracle_fmul_rd(third, 3.0) <= 1.0
    assert L.oracle_fdiv_rd(1023.0, 1.0) == 1023.0
    rng = np.random.default_rng(0xbeefcafe)
    a = (rng.standard_normal(20000) * 10.0 ** rng.integers(-6, 7, 20000)).astype(np.float32)
    b = (rng.standard_normal(20000) * 10.0 ** rng.integers(-6, 7, 20000)).astype(np.float32)
    for x, y in zip(a, b):
        xd, yd = float(x), float(y)  # binary64 holds binary32 sums/products exactly enough for the sign test
        lo, hi = L.oracle_fsub_rd(x, y), L.oracle_fsub_ru(x, y)
        assert float(lo) <= xd - yd <= float(hi)
        assert hi == lo or np.nextafter(np.float32(lo), INF) == np.float32(hi)
        assert float(L.oracle_fadd_rd(x, y)) <= xd + yd
        p = L.oracle_fmul_rd(x, y)
        assert float(p) <= xd * yd and float(np.nextafter(np.float32(p), INF)) > xd * yd
        if y != 0:
            q = L.oracle_fdiv_rd(x, y)
            assert float(q) <= xd / yd or abs(float(q) - xd / yd) < abs(xd / yd) * 2 ** -40
            assert float(np.nextafter(np.float32(q), INF)) >= xd / yd
    assert np.signbit(np.float32(L.oracle_fsub_rd(0.5, 0.5)))  # x - x = -0 when rounding down


def test_read_bits_against_naive_bit_array(oracle):  # acceptance criterion 5 (widths 1-64, offsets 0-255)
    rng = np.random.default_rng(0xbeefcafe)
    buf = rng.integers(0, 256, 64, dtype=np.uint8)
    for _ in range(20000):
        w = int(rng.integers(1, 65))
        off = int(rng.integers(0, 256))
        assert oracle.lib.oracle_read_bits(buf.ctypes.data, off, w) == oracle.lib.oracle_read_bits_naive(buf.ctypes.data, off, w)
    one = np.zeros(8, np.uint8)
    one[0] = 0b10100000  # 0b101 at bit offset 5
    assert oracle.lib.oracle_read_bits(one.ctypes.data, 5, 3) == 0b101


def roundtrip(orc, scheme, wlo, whi, lo, hi):
    codes, box = np.zeros(6, np.uint32), np.zeros(6, np.float32)
    orc.lib.oracle_quantize_roundtrip(scheme, wlo.ctypes.data, whi.ctypes.data, lo.ctypes.data, hi.ctypes.data, codes.ctypes.data, box.ctypes.data)
    return codes, box


def test_quantisation_world_box_codes(oracle):
    wlo, whi = F(-3, 0.5, 10), F(5, 2.5, 11)
    codes, box = roundtrip(oracle, 0, wlo, whi, wlo, whi)  # sg-eq: box == world box -> codes 0 / 0, exact
    assert tuple(codes) == (0,) * 6 and tuple(box[:3]) == tuple(wlo) and tuple(box[3:]) == tuple(whi)
    codes, box = roundtrip(oracle, 1, wlo, whi, wlo, whi)  # q16: lo codes 0, hi codes 65535
    assert tuple(codes) == (0, 0, 0, 65535, 65535, 65535) and tuple(box[:3]) == tuple(wlo)
    codes, _ = roundtrip(oracle, 2, wlo, whi, wlo, whi)
    assert tuple(codes) == (0, 0, 0, 255, 255, 255)


def test_quantisation_enclosure_1e5(oracle):  # acceptance criterion 3
    rng = np.random.default_rng(7)
    n = 100000
    wlo = (rng.standard_normal((n, 3)) * 10).astype(np.float32)
    ext = (rng.random((n, 3)) * 20 + 1e-3).astype(np.float32)
    whi = wlo + ext
    a = (wlo + rng.random((n, 3)).astype(np.float32) * ext).astype(np.float32)
    b = (wlo + rng.random((n, 3)).astype(np.float32) * ext).astype(np.float32)
    lo, hi = np.clip(np.minimum(a, b), wlo, whi), np.clip(np.maximum(a, b), wlo, whi)
    viol = {0: 0, 1: 0, 2: 0}
    worst = {0: 0.0, 1: 0.0, 2: 0.0}
    for i in range(n):
        for scheme in (0, 1, 2):
            _, box = roundtrip(oracle, scheme, wlo[i], whi[i], lo[i], hi[i])
            if not (np.all(box[:3] <= lo[i]) and np.all(box[3:] >= hi[i])):
                viol[scheme] += 1
                gap = max(float(np.max(box[:3] - lo[i])), float(np.max(hi[i] - box[3:])))
                worst[scheme] = max(worst[scheme], gap / float(np.max(np.abs(ext[i]))))
    # sg-eq uses directed rounding end to end: enclosure is exact (0 violations)
    assert viol[0] == 0
    # q16 / q8 dequantise with round-to-nearest (pbrt_q16.scion:6-13): not conservative to the last
    # ulp (SURVEY App. A "L2 parity"); violations stay within a few ulps of the frame extent.
    assert worst[1] < 1e-6 and worst[2] < 1e-6, (viol, worst)
