"""Collision detection: corpus/alg/cd.scion, cd_dop14.scion, SAT triangle/triangle
(geometry.scion:112-157).  Contract: SET equality of the colliding triangle pairs."""
import numpy as np
import pytest

TRI = lambda *v: np.array(v, np.float32)


def test_sat_kats(oracle):
    a = TRI(0, 0, 0, 1, 0, 0, 0, 1, 0)
    assert oracle.sat(a, a)  # coincident triangles
    assert not oracle.sat(a, a + TRI(*([5, 0, 0] * 3)))  # separated along x by a gap
    b = TRI(0.25, 0.25, -1, 0.25, 0.25, 1, 0.75, 0.75, 0)  # perpendicular, interlocking
    assert oracle.sat(a, b) and oracle.sat(b, a)
    rng = np.random.default_rng(5)
    for _ in range(500):  # project6 symmetry: sat(t1, t2) == sat(t2, t1)
        t1, t2 = rng.random(9).astype(np.float32), (rng.random(9) * 1.5).astype(np.float32)
        assert oracle.sat(t1, t2) == oracle.sat(t2, t1)


def two_meshes(sb, g=10):
    a = sb.Scene.terrain(g, 3)
    tb = sb.Scene.terrain(g, 9).triangles().copy()
    tb[:, 1::3] += 0.02  # second scene + rigid transform: a slightly lifted, different terrain
    return a, sb.Scene.from_triangles(tb)


def test_oracle_cd_equals_brute_force(built, oracle):
    sb = built
    sa, sbn = two_meshes(sb)
    la, lb = sa.build_median(1), sbn.build_median(1)  # the paper's CD setup: median split, 1 primitive per leaf (PAPER §8.3.3)
    brute = oracle.brute_collisions(la.triangles(), lb.triangles())
    assert 50 < len(brute) < la.nprims * lb.nprims
    ident, st = oracle.collide(oracle.logical_bytes(la, "@logical2"), oracle.logical_bytes(lb, "@logical2"))
    assert np.array_equal(ident, brute)
    for layout in ("identity", "ptr", "pbrt", "pbrt-q16", "sg-eq", "shared-slab", "dop14", "pbrt-post", "pbrt-soa"):
        got, st2 = oracle.collide(oracle.tree_bytes(la.encode(layout)), oracle.tree_bytes(lb.encode(layout)))
        assert np.array_equal(got, brute), layout
    # two identical 2-triangle meshes -> all 4 pairs; disjoint meshes -> empty set (:616)
    quad = np.array([[0, 0, 0, 1, 0, 0, 1, 1, 0], [0, 0, 0, 1, 1, 0, 0, 1, 0]], np.float32)
    q = sb.Scene.from_triangles(quad).build_median(1)
    four, _ = oracle.collide(oracle.tree_bytes(q.encode("pbrt")), oracle.tree_bytes(q.encode("pbrt")))
    assert len(four) == 4
    far = sb.Scene.from_triangles(quad + np.float32(10)).build_median(1)
    none, _ = oracle.collide(oracle.tree_bytes(q.encode("pbrt")), oracle.tree_bytes(far.encode("pbrt")))
    assert len(none) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["identity", "ptr", "pbrt", "pbrt-align16", "pbrt-soa", "pbrt-post", "pbrt-q16", "sg-eq", "sg-eq-align16", "shared-slab", "dop14",
                                    "pbrt-soaos", "pbrt-soaos-align16", "pbrt-q16-soaos"])
def test_gpu_cd_matches_oracle(built, oracle, layout):
    sb = built
    sa, sbn = two_meshes(sb, 24)
    for builder in ("median", "sah"):
        la = sa.build_median(1) if builder == "median" else sa.build_sah(32, 4)
        lb = sbn.build_median(1) if builder == "median" else sbn.build_sah(32, 4)
        pa, pb = la.encode(layout), lb.encode(layout)
        want, wst = oracle.collide(oracle.tree_bytes(pa), oracle.tree_bytes(pb))
        da, db = pa.upload(0), pb.upload(0)
        got, n, st = da.collide_host(db, capacity=1 << 20)
        assert n == len(want) and np.array_equal(got, want), (layout, builder, n, len(want))
        assert st["node_pairs"] == wst["node_pairs"] and st["tri_tests"] == wst["tri_tests"]  # same recursion, level by level
        # self collision (same tree twice) and the capacity contract: the true count is reported, nothing is lost silently
        self_want, _ = oracle.collide(oracle.tree_bytes(pa), oracle.tree_bytes(pa))
        self_got, n2, _ = da.collide_host(da, capacity=1 << 20)
        assert np.array_equal(self_got, self_want)
        few, n3, _ = da.collide_host(da, capacity=16)
        assert n3 == n2 and len(few) == 16
        da.free()
        db.free()


@pytest.mark.gpu
def test_gpu_cd_rejects_bad_arguments(built):
    sb = built
    lt = sb.Scene.terrain(6, 1).build_sah(32, 4).collapse8()
    wide, flat, q16 = lt.encode("bvh8-q8-ci").upload(0), lt.encode("pbrt").upload(0), lt.encode("pbrt-q16").upload(0)
    with pytest.raises(sb.ScionError):  # "cd requires a binary layout" (corpus.cpp:86)
        wide.collide_host(wide)
    with pytest.raises(sb.ScionError):  # both trees must share the layout
        flat.collide_host(q16)
    for t in (wide, flat, q16):
        t.free()


def test_sat_against_constructed_pairs(oracle):
    """SPEC acceptance criterion 9: SAT vs a construction-based overlap oracle on 10^3 pairs, none inside an
    epsilon-thick boundary band: (a) pairs separated by a gap of at least 0.05 along a random axis, (b) pairs where an
    edge of the second triangle pierces the first one at an interior point, end points >= 0.05 off its plane."""
    rng = np.random.default_rng(17)
    for _ in range(500):
        a = rng.uniform(-1, 1, (3, 3)).astype(np.float32)
        b = rng.uniform(-1, 1, (3, 3)).astype(np.float32)
        axis = rng.normal(size=3)
        axis /= np.linalg.norm(axis)
        gap = (a @ axis).max() - (b @ axis).min() + 0.05 + rng.uniform(0, 1)
        b_far = (b + gap * axis).astype(np.float32)  # every vertex of b_far is beyond every vertex of a along `axis`
        assert (b_far @ axis).min() - (a @ axis).max() > 0.04
        assert not oracle.sat(a.reshape(-1), b_far.reshape(-1)) and not oracle.sat(b_far.reshape(-1), a.reshape(-1))
    for _ in range(500):
        a = rng.uniform(-1, 1, (3, 3))
        w = rng.uniform(0.15, 0.7, 3)
        w /= w.sum()
        p = w @ a  # interior point of a
        n = np.cross(a[1] - a[0], a[2] - a[0])
        if np.linalg.norm(n) < 0.2:
            continue
        n /= np.linalg.norm(n)
        d = n + 0.5 * rng.uniform(-1, 1, 3)
        d /= np.linalg.norm(d)
        q0, q1 = p + d * rng.uniform(0.1, 1.0), p - d * rng.uniform(0.1, 1.0)  # the segment q0-q1 passes through p
        assert abs((q0 - p) @ n) > 0.05 and abs((q1 - p) @ n) > 0.05
        q2 = q0 + rng.uniform(-1, 1, 3)
        b = np.stack([q0, q1, q2]).astype(np.float32)
        a32 = a.astype(np.float32)
        assert oracle.sat(a32.reshape(-1), b.reshape(-1)) and oracle.sat(b.reshape(-1), a32.reshape(-1))
