"""In-memory PhysicalTree import (scion_ptree_from_buffers / scion_tree_upload): the way a tree built by someone
else's build_physical enters the backend without a file round trip (one descriptor per
BufferDesc / GlobalDesc of the MemoryPlan, /root/reference/proj/include/layoutc/plan.hpp:31-48), and the validation
every foreign tree goes through (sizes == footprint(), /root/reference/proj/src/plan.cpp:333-347)."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def small(built):
    scene = built.Scene.terrain(20, 9)
    return scene, scene.build_sah(32, 4).collapse8()


def test_export_import_is_byte_identical(built, oracle, small):
    _, lt = small
    for l in built.layouts():
        pt = lt.encode(l["name"])
        layout, bufs, globs, root, carried = pt.export()
        back = built.PhysicalTree.from_buffers(layout, list(reversed(bufs)), list(reversed(globs)), root, carried)  # any order: matched by name
        assert back.layout == pt.layout and back.root() == pt.root() and back.total_bytes == pt.total_bytes and back.image_bytes == pt.image_bytes
        for a, b in zip(pt.buffers(), back.buffers()):
            assert a["name"] == b["name"] and a["count"] == b["count"] and a["seg_bases"] == b["seg_bases"] and np.array_equal(a["data"], b["data"]), l["name"]
        assert [g["raw"] for g in pt.globals()] == [g["raw"] for g in back.globals()]
        assert oracle.check_encoding(back, lt)[0] == 0
        # segment bases are optional (derived from the plan) but must be the plan's when given
        nosb = [dict(b, seg_bases=None) for b in bufs]
        again = built.PhysicalTree.from_buffers(layout, nosb, globs, root, carried)
        assert [b["seg_bases"] for b in again.buffers()] == [b["seg_bases"] for b in pt.buffers()]


def test_import_rejects_what_the_plan_does_not_describe(built, small):
    sb = built
    _, lt = small
    pt = lt.encode("dop14")
    layout, bufs, globs, root, carried = pt.export()

    def bad(**kw):
        with pytest.raises(sb.ScionError) as e:
            sb.PhysicalTree.from_buffers(kw.get("layout", layout), kw.get("bufs", bufs), kw.get("globs", globs), kw.get("root", root), carried)
        assert e.value.code == sb.ERR_ARG
        return str(e.value)

    assert "unknown layout" in bad(layout="no-such-layout")
    nodes = [b for b in bufs if b["name"] == "nodes"][0]
    others = [b for b in bufs if b["name"] != "nodes"]
    assert "footprint" in bad(bufs=others + [dict(nodes, data=nodes["data"][:-32])])          # truncated buffer
    assert "footprint" in bad(bufs=others + [dict(nodes, count=nodes["count"] + 1)])           # count that does not match the bytes
    assert "segment bases" in bad(bufs=others + [dict(nodes, seg_bases=[0, nodes["seg_bases"][1] + 32])])  # SoA base moved
    assert "missing buffer" in bad(bufs=others)
    assert "no buffer" in bad(bufs=bufs + [dict(name="extra", data=np.zeros(4, np.uint8), count=1, seg_bases=None)])
    assert "given twice" in bad(bufs=bufs + [nodes])
    assert "missing global" in bad(globs=globs[:-1])
    assert "no global" in bad(globs=globs + [dict(name="bogus", raw=b"")])
    assert "not a node index" in bad(root=nodes["count"])
    # 8-wide tagged root reference and arena root
    p8 = lt.encode("bvh8-q8-ci")
    l8, b8, g8, r8, c8 = p8.export()
    with pytest.raises(sb.ScionError):
        sb.PhysicalTree.from_buffers(l8, b8, g8, (10 ** 6 << 2) | 1, c8)
    pa = lt.encode("ptr")
    la, ba, ga, ra, ca = pa.export()
    with pytest.raises(sb.ScionError):
        sb.PhysicalTree.from_buffers(la, ba, ga, 1 << 40, ca)


def test_container_rejects_inconsistent_tables(built, small, tmp_path):
    """a hostile container must not upload cleanly — sizes, counts, segment tables and the root are validated."""
    sb = built
    _, lt = small
    pt = lt.encode("pbrt-q16")
    path = str(tmp_path / "t.scionpt")
    pt.save(path)
    raw = bytearray(open(path, "rb").read())
    # header: magic 8 | version 4 | name_len 4 | name | nprims 8 | root0 8 | ...
    name_len = int.from_bytes(raw[12:16], "little")
    root_off = 16 + name_len + 8
    bad = bytearray(raw)
    bad[root_off:root_off + 8] = (2 ** 40).to_bytes(8, "little")
    open(path, "wb").write(bad)
    with pytest.raises(sb.ScionError) as e:
        sb.PhysicalTree.load(path)
    assert "root reference" in str(e.value)
    # a buffer size far beyond the file: rejected before any allocation
    idx = raw.find(b"nodes")
    assert idx > 0
    bad = bytearray(raw)
    size_off = idx + 5 + 8  # name | count u64 | bytes u64
    bad[size_off:size_off + 8] = (2 ** 60).to_bytes(8, "little")
    open(path, "wb").write(bad)
    with pytest.raises(sb.ScionError) as e:
        sb.PhysicalTree.load(path)
    assert "exceed the file" in str(e.value) or "footprint" in str(e.value)
    open(path, "wb").write(raw)
    assert sb.PhysicalTree.load(path).total_bytes == pt.total_bytes


@pytest.mark.gpu
def test_imported_tree_answers_like_the_original(built, oracle, small):
    import torch
    sb = built
    scene, lt = small
    lo, hi = scene.bounds()
    cam = sb.default_camera(lo, hi, True, 64, 64)
    rays = np.concatenate([sb.gen_primary_host(cam, 0, 4096), sb.gen_secondary_host(lt.triangles(), 3, 0, 4096)])
    d_rays = torch.from_numpy(rays.view(np.uint8).reshape(-1)).to("cuda:0")
    n = len(rays)
    for name in ("pbrt", "pbrt-q16", "dop14", "ptr", "shared-slab", "bvh8-q8-ci", "bvh8"):
        pt = lt.encode(name)
        ref = pt.upload(0)
        layout, bufs, globs, root, carried = pt.export()
        imp = sb.tree_upload(layout, bufs, globs, root, carried, 0)
        assert np.array_equal(ref.download_image(), imp.download_image()), name  # byte-identical device image
        outs = []
        for dt in (ref, imp):
            d_hits = torch.empty(n * 8, dtype=torch.uint8, device="cuda:0")
            dt.closest_hit(d_rays.data_ptr(), n, d_hits.data_ptr())
            torch.cuda.synchronize()
            outs.append(d_hits.cpu().numpy().view(sb.HIT_DTYPE))
        assert np.array_equal(outs[0].view(np.uint64), outs[1].view(np.uint64)), name
        want, _ = oracle.closest_hit(oracle.tree_bytes(pt), rays)
        assert np.array_equal(outs[1]["prim"], want["prim"]) and np.array_equal(outs[1]["t"].view(np.uint32), want["t"].view(np.uint32)), name
        ref.free()
        imp.free()
