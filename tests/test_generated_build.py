"""Constructor specialisation (SPEC.md:276-284 specialize_constructors, :387-395 build_physical):
the `build` block of every shipped layout, compiled by the layout compiler into gen/<layout>.cuh build_<Variant>() and run
by scion_encode_generated (count pass + recursive emit pass), must produce the SAME PhysicalTree — every buffer byte,
segment bases, element counts, global slots, root reference, tree-carried root components — as the hand-written
per-family encoders behind scion_encode.  Two independent statements of the reference's build semantics that agree byte
for byte, on a machine without a GPU."""
import numpy as np
import pytest


def trees_equal(a, b):
    ba, bb = a.buffers(), b.buffers()
    assert len(ba) == len(bb)
    for x, y in zip(ba, bb):
        assert x["name"] == y["name"]
        assert x["count"] == y["count"], (x["name"], x["count"], y["count"])
        assert list(x["seg_bases"]) == list(y["seg_bases"]), x["name"]
        assert x["bytes"] == y["bytes"], (x["name"], x["bytes"], y["bytes"])
        da, db = x["data"], y["data"]
        bad = np.nonzero(da != db)[0]
        assert bad.size == 0, f"buffer {x['name']}: {bad.size} bytes differ, first at {bad[:8]}"
    ga, gb = a.globals(), b.globals()
    assert [g["name"] for g in ga] == [g["name"] for g in gb]
    for x, y in zip(ga, gb):
        assert bytes(x["raw"]) == bytes(y["raw"]), (x["name"], bytes(x["raw"]).hex(), bytes(y["raw"]).hex())
    ra, rb = a.root(), b.root()
    assert ra[0] == rb[0], (ra, rb)
    assert np.array_equal(np.asarray(ra[1], np.float32).view(np.uint32), np.asarray(rb[1], np.float32).view(np.uint32)), (ra, rb)


@pytest.fixture(scope="module")
def scenes(built):
    out = []
    for name, scene in (("terrain", built.Scene.terrain(23, 11)), ("sphere", built.Scene.sphere(17, 5))):
        out.append((name + "/sah", scene.build_sah(32, 4).collapse8()))
    out.append(("terrain/median", built.Scene.terrain(9, 2).build_median(1).collapse8()))
    return out


def test_every_layout_carries_a_build_block(built):
    for l in built.layouts():
        assert built.lib().scion_layout_has_build(l["name"].encode()) == 1, l["name"]


def test_generated_constructors_match_the_hand_written_encoders(built, scenes):
    for l in built.layouts():
        for what, lt in scenes:
            hand = lt.encode(l["name"])
            gen = lt.encode_generated(l["name"])
            try:
                trees_equal(hand, gen)
            except AssertionError as e:
                raise AssertionError(f"{l['name']} on {what}: {e}") from None


def test_generated_build_faults(built):
    """capacity violations are build faults, never silent"""
    scene = built.Scene.terrain(6, 1)
    lt = scene.build_sah(32, 12)  # leaves of up to 12 primitives
    lt32 = scene.build_sah(32, 40)  # leaves of up to 40 primitives: beyond the u4 / u5 nprims fields
    for layout in ("pbrt-q16", "sg-eq", "shared-slab"):
        with pytest.raises(Exception):
            lt32.encode_generated(layout)
    with pytest.raises(Exception):
        lt.encode_generated("bvh8-q8-ci")  # not collapsed


REF_LAYOUTS = "/root/reference/proj/corpus/layouts"


@pytest.mark.skipif(not __import__("os").path.isdir(REF_LAYOUTS), reason="the reference tree only exists in the build container")
def test_reference_build_blocks_compile_to_the_same_trees(built, scenes, tmp_path):
    """The REFERENCE's own build blocks (its 15 corpus files, read in place, never copied) go through our layout compiler;
    the constructors it emits from them, run against this library's plan of the same-named layout, must produce the very
    trees our encoders produce: the reference's text and our two implementations of it agree byte for byte."""
    import ctypes as C
    import glob
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    csrc = os.path.join(root, "paper_2511_15028_b200", "csrc")
    scionc = os.path.join(root, "paper_2511_15028_b200", "bin", "scionc")
    libdir = os.path.join(root, "paper_2511_15028_b200")
    files = sorted(glob.glob(os.path.join(REF_LAYOUTS, "*.scion")))
    assert len(files) == 15
    from paper_2511_15028_b200 import PhysicalTree
    for f in files:
        ident = os.path.basename(f)[:-6]
        name = ident.replace("_", "-")
        hdr = tmp_path / f"{ident}.cuh"
        r = subprocess.run([scionc, "emit-cuda", name, f], capture_output=True, text=True)
        assert r.returncode == 0, (name, r.stderr[-2000:])
        hdr.write_text(r.stdout.replace('#include "../device/scion_rt.cuh"', '#include "device/scion_rt.cuh"'))
        so = tmp_path / f"ref_build_{ident}.so"
        r = subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", "-fPIC", "-shared", "-ffp-contract=off", "-frounding-math", "-I", csrc, "-I", os.path.join(root, "include"),
                            f'-DGEN_HEADER="{hdr}"', f"-DGEN_STRUCT=L_{ident}", os.path.join(root, "tests", "ref_build_shim.cpp"), "-o", str(so),
                            "-L", libdir, "-lscion_b200", f"-Wl,-rpath,{libdir}"], capture_output=True, text=True)
        assert r.returncode == 0, (name, r.stderr[-3000:])
        shim = C.CDLL(str(so))
        shim.ref_build.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.c_char_p, C.c_int]
        for what, lt in scenes[:2]:
            h, err = C.c_void_p(), C.create_string_buffer(512)
            assert shim.ref_build(lt._h, C.byref(h), err, 512) == 0, (name, err.value)
            try:
                trees_equal(lt.encode(name), PhysicalTree(h))
            except AssertionError as e:
                raise AssertionError(f"{name} on {what}: {e}") from None


def test_reference_check_build_accepts_our_build_blocks(built):
    """the reference's own semantic checker of build blocks (src/sema_build.cpp check_build, linked into
    oracle/_ref/ref_probe) over OUR 24 layout files: no diagnostics"""
    import glob
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    probe = os.path.join(root, "oracle", "_ref", "ref_probe")
    if not os.path.exists(probe):
        pytest.skip("oracle/_ref/ref_probe is only built where /root/reference exists")
    files = sorted(glob.glob(os.path.join(root, "paper_2511_15028_b200", "layouts", "*.scion")))
    assert len(files) == 24
    for f in files:
        r = subprocess.run([probe, f], capture_output=True, text=True)
        assert r.returncode == 0 and "check_build ok" in r.stderr, (f, r.stderr[-1000:])


def test_generated_constructors_at_full_size(built):
    """BASELINE configs[4] scale: 9,999,392 triangles, ~5.8 M binary nodes / ~0.8 M 8-wide interiors — the compiled build
    blocks and the hand-written encoders still agree byte for byte (recursion depth, append cursors and u28 offsets at size)"""
    import paper_2511_15028_b200.workloads as W
    scene = W.make_scene(W.workload("c5"))
    assert scene.ntris == 9999392
    lt = scene.build_sah(32, 4).collapse8()
    for layout in ("pbrt-q16", "sg-eq", "bvh8-q8-ci", "pbrt-post"):
        try:
            trees_equal(lt.encode(layout), lt.encode_generated(layout))
        except AssertionError as e:
            raise AssertionError(f"{layout}: {e}") from None
