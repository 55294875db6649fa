"""Scene tools + encoders on the CPU: builder invariants, constructor layout
facts (acceptance criterion 6), and — for every layout — the oracle's
independent decode of the product-encoded bytes agrees with the LogicalTree (decode o encode = id;
quantised layouts reproduce the oracle's own codes)."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def small(built):
    scene = built.Scene.terrain(20, seed=3)
    return scene, scene.build_sah(32, 4).collapse8()


def test_builder_invariants(built, small):
    scene, lt = small
    nodes, tris = lt.nodes(), lt.triangles()
    assert lt.nprims == scene.ntris == 800
    assert sorted(lt.prim_ids().tolist()) == list(range(scene.ntris))  # primitive multiset preserved
    assert np.array_equal(tris, scene.triangles()[lt.prim_ids()])
    interior = nodes["left"] >= 0
    idx = np.arange(len(nodes))
    assert np.all(nodes["left"][interior] == idx[interior] + 1)  # preorder: left child at this+1 for 100%
    assert np.all(nodes["right"][interior] > nodes["left"][interior])
    leaves = nodes[~interior]
    assert leaves["nprims"].min() >= 1 and leaves["nprims"].max() <= 4
    assert np.array_equal(leaves["first_prim"], np.concatenate([[0], np.cumsum(leaves["nprims"])[:-1]]))  # append order == DFS leaf order
    for i in np.nonzero(interior)[0]:  # bounds invariant: exact comparison on stored binary32 values
        for c in (nodes["left"][i], nodes["right"][i]):
            assert np.all(nodes["lo"][i] <= nodes["lo"][c]) and np.all(nodes["hi"][i] >= nodes["hi"][c])
    for l in leaves:
        t = tris[l["first_prim"]:l["first_prim"] + l["nprims"]].reshape(-1, 3)
        assert np.array_equal(l["lo"], t.min(axis=0)) and np.array_equal(l["hi"], t.max(axis=0))
    assert lt.depth < 62


def test_builder_degenerate_inputs(built):
    one = built.Scene.from_triangles(np.array([[0, 0, 0, 1, 0, 0, 0, 1, 0]], np.float32))
    lt = one.build_sah(32, 4).collapse8()
    assert lt.nnodes == 1 and lt.nodes()["nprims"][0] == 1 and lt.wroot == -1  # single leaf
    same = built.Scene.from_triangles(np.tile(np.array([[0, 0, 0, 1, 0, 0, 0, 1, 0]], np.float32), (9, 1)))
    lt = same.build_sah(32, 1)  # coincident centroids -> index halves
    assert lt.nprims == 9 and (lt.nodes()["nprims"] <= 1).all() and lt.depth == 4
    lt2 = built.Scene.from_triangles(np.array([[0, 0, 0, 1, 0, 0, 0, 1, 0], [5, 0, 0, 6, 0, 0, 5, 1, 0]], np.float32)).build_median(1)
    assert lt2.nnodes == 3  # 2 triangles -> 1 interior, 2 leaves
    cloud = built.Scene.cloud(1000, 3)
    t = cloud.triangles()
    assert np.array_equal(t[:, 0:3], t[:, 3:6]) and np.array_equal(t[:, 0:3], t[:, 6:9]) and t.min() >= 0 and t.max() < 1


def test_collapse_to_wide(built, small):
    _, lt = small
    wn, wl = lt.wnodes(), lt.wleaves()
    assert wl["nprims"].sum() == lt.nprims
    assert np.array_equal(wl["first_prim"], np.concatenate([[0], np.cumsum(wl["nprims"])[:-1]]))
    for w in wn:
        used = w["child"] != built.W_SENTINEL
        k = int(used.sum())
        assert k >= 2 and used[:k].all() and not used[k:].any()  # left-packed, SENTINELs after
        assert np.all(np.isposinf(w["lo"][k:])) and np.all(np.isneginf(w["hi"][k:]))  # inverted boxes
    # complete binary tree of depth 3 -> one 8-wide root over 8 leaves
    tri = lambda x: [x, 0, 0, x + 0.5, 0, 0, x, 0.5, 0]
    lt8 = built.Scene.from_triangles(np.array([tri(i) for i in range(8)], np.float32)).build_median(1).collapse8()
    assert len(lt8.wnodes()) == 1 and len(lt8.wleaves()) == 8 and (lt8.wnodes()["child"][0] < 0).all()


def test_constructor_layout_facts(built, oracle):
    # 2-interior / 3-leaf tree -> N = 5, preorder, c_o = right - this, 160-byte node buffer
    tri = lambda x: [x, 0, 0, x + 0.5, 0, 0, x, 0.5, 0]
    lt = built.Scene.from_triangles(np.array([tri(0), tri(1), tri(4)], np.float32)).build_median(1).collapse8()
    assert lt.nnodes == 5
    pt = lt.encode("pbrt")
    nodes = [b for b in pt.buffers() if b["name"] == "nodes"][0]
    prims = [b for b in pt.buffers() if b["name"] == "primitives"][0]
    assert nodes["bytes"] == 160 and prims["bytes"] == 3 * 36
    raw = nodes["data"]
    n = lt.nodes()
    for i in range(5):
        nprims = int.from_bytes(raw[32 * i + 28:32 * i + 30].tobytes(), "little")  # nprims @ bit 224
        word = int.from_bytes(raw[32 * i + 24:32 * i + 28].tobytes(), "little")  # union @ bit 192
        if n["left"][i] >= 0:
            assert nprims == 0 and word == n["right"][i] - i
        else:
            assert nprims == n["nprims"][i] and word == n["first_prim"][i]
        assert np.array_equal(np.frombuffer(raw[32 * i:32 * i + 24].tobytes(), np.float32), np.concatenate([n["lo"][i], n["hi"][i]]))
    # App. C.2 leaf reference for (poffset = 0, nprims = 3) equals 8 (acceptance criterion 6)
    lt3 = built.Scene.from_triangles(np.array([tri(0), tri(0.1), tri(0.2)], np.float32)).build_sah(32, 4).collapse8()
    assert lt3.encode("bvh8-q8-ci").root()[0] == 8 and lt3.encode("bvh8").root()[0] == 8
    # default root reference of the wide layouts is 1 = interior 0 (bvh8_q8_ci.scion:27)
    assert lt.encode("bvh8-q8-ci").root()[0] == 1
    # footprints
    assert [b for b in lt.encode("bvh8-q8-ci").buffers() if b["name"] == "Interiors"][0]["bytes"] == 104 * len(lt.wnodes())
    d = [b for b in lt.encode("dop14").buffers() if b["name"] == "nodes"][0]
    assert d["seg_bases"] == [0, 160] and d["bytes"] == 320  # two 32-byte segments, base[1] = 160 for N = 5 (test_plan.cpp:179-195)


@pytest.mark.parametrize("scene_kind", ["terrain", "sphere"])
def test_every_layout_decodes_back_to_the_logical_tree(built, oracle, scene_kind):
    scene = built.Scene.terrain(18, 11) if scene_kind == "terrain" else built.Scene.sphere(14, 11)
    lt = scene.build_sah(32, 4).collapse8()
    lo, hi = scene.bounds()
    cam = built.default_camera(lo, hi, scene_kind == "terrain", 48, 48)
    rays = np.concatenate([built.gen_primary_host(cam, 0, 48 * 48), built.gen_secondary_host(lt.triangles(), 3, 0, 1024)])
    pts = built.gen_points_host(lo - 0.3, hi + 0.3, 8, 0, 512)
    ref, _ = oracle.closest_hit(oracle.logical_bytes(lt, "@logical2"), rays)
    ref8, _ = oracle.closest_hit(oracle.logical_bytes(lt, "@logical8"), rays)
    refd, _ = oracle.closest_hit(oracle.logical_bytes(lt, "@logical-dop14"), rays)
    brute = oracle.brute_hit(lt.triangles(), rays)
    refp, _ = oracle.closest_point(oracle.logical_bytes(lt, "@logical2"), pts)
    refpd, _ = oracle.closest_point(oracle.logical_bytes(lt, "@logical-dop14"), pts)
    brutep = oracle.brute_point(lt.triangles(), pts)
    assert (ref["prim"] != built.MISS_PRIM).mean() > 0.15
    # the identity oracle agrees with brute force on which triangle / distance wins
    assert np.array_equal(ref["t"], brute["t"]) and np.array_equal(ref["prim"], brute["prim"])
    assert np.array_equal(ref8["t"], brute["t"]) and np.array_equal(refd["t"], brute["t"])
    assert np.array_equal(refp["d2"], brutep["d2"])
    for l in built.layouts():
        pt = lt.encode(l["name"])
        bad, msg, loose = oracle.check_encoding(pt, lt)
        assert bad == 0, msg
        if l["name"] in ("sg-eq", "sg-eq-align16") or "q" not in l["name"]:
            assert loose == 0, l["name"]  # directed rounding / float32 layouts enclose exactly
        tb = oracle.tree_bytes(pt)
        h, st = oracle.closest_hit(tb, rays)
        assert st.max() == 0
        # reference `verify` contract: identical primitive, bitwise-equal t vs the identity oracle
        assert np.array_equal(h["prim"], ref["prim"]) and np.array_equal(h["t"].view(np.uint32), ref["t"].view(np.uint32)), l["name"]
        if l["has_cpq"]:
            cp, st = oracle.closest_point(tb, pts)
            # cpq_dop14.scion orders children by the DOP distance, so among equal-d2 candidates (shared
            # vertices / edges) it may pick another primitive than cpq.scion: compare like with like
            want = refpd if l["family"] == 1 else refp
            assert np.array_equal(cp["d2"], want["d2"]) and np.array_equal(cp["d2"], brutep["d2"]), l["name"]
            exact_boxes = l["name"] not in ("pbrt-q16", "sg-eq", "sg-eq-align16", "shared-slab")
            if exact_boxes:  # same boxes => same child order => same winner among ties
                assert np.array_equal(cp["prim"], want["prim"]), l["name"]
            else:  # looser boxes reorder the L < R child sort: ties (shared vertices) may resolve differently
                differ = cp["prim"] != want["prim"]
                t = lt.triangles()
                for i in np.nonzero(differ)[0]:  # ... but only ever to another primitive at exactly the same distance
                    alt = oracle.brute_point(t[cp["prim"][i]:cp["prim"][i] + 1], pts[i:i + 1])
                    assert alt["d2"][0] == want["d2"][i], l["name"]


def test_fault_injection_is_detected(built, oracle, small):
    """corrupt one c_o byte => the oracle's structural check and the query results notice"""
    _, lt = small
    pt = lt.encode("pbrt")
    assert oracle.check_encoding(pt, lt)[0] == 0
    pt.corrupt(1, 24, 0x02)  # node 0, union word (c_o) low byte
    assert oracle.check_encoding(pt, lt)[0] > 0


def test_counters_sg_eq_visits_at_least_pbrt(built, oracle, small):
    """coarser bounds never visit fewer nodes"""
    scene, lt = small
    lo, hi = scene.bounds()
    rays = built.gen_primary_host(built.default_camera(lo, hi, True, 32, 32), 0, 1024)
    _, _, c_p = oracle.closest_hit(oracle.tree_bytes(lt.encode("pbrt")), rays, counters=True)
    _, _, c_s = oracle.closest_hit(oracle.tree_bytes(lt.encode("sg-eq")), rays, counters=True)
    assert c_s["node_visits"].sum() >= c_p["node_visits"].sum()


def test_container_file_round_trip(built, oracle, small, tmp_path):
    """PhysicalTree container: save -> load is byte-identical for every layout; foreign or
    truncated files are rejected with a diagnostic, never half-loaded"""
    _, lt = small
    for l in built.layouts():
        pt = lt.encode(l["name"])
        path = str(tmp_path / (l["name"] + ".scionpt"))
        pt.save(path)
        back = built.PhysicalTree.load(path)
        assert back.layout == pt.layout and back.root() == pt.root() and back.total_bytes == pt.total_bytes
        for a, b in zip(pt.buffers(), back.buffers()):
            assert a["name"] == b["name"] and a["count"] == b["count"] and a["seg_bases"] == b["seg_bases"] and np.array_equal(a["data"], b["data"])
        assert [g["raw"] for g in pt.globals()] == [g["raw"] for g in back.globals()]
        assert oracle.check_encoding(back, lt)[0] == 0
    raw = open(path, "rb").read()
    open(path, "wb").write(raw[: len(raw) // 2])
    with pytest.raises(built.ScionError):
        built.PhysicalTree.load(path)
    open(path, "wb").write(b"NOTSCION" + raw[8:])
    with pytest.raises(built.ScionError):
        built.PhysicalTree.load(path)
