"""closest_point pinned against the REFERENCE'S OWN compiled traversal.

tests/golden/ref_ir_cpq.npz holds (d2, closest point) computed by the reference's lowered IR of cpq.scion /
cpq_dop14.scion — its parser, type checker, planner and `specialize_destructors`, executed by oracle/ref_interp.cpp —
on trees produced by this repository's encoders, for the reference's 10 binary corpus layouts on three scenes
(terrain, sphere, point cloud = degenerate triangles).  The unmodified reference corrupts this lowering through a
dangling `Frame&` (src/lower_internal.hpp:1073 held across the push_back of :890); oracle/Makefile patches that ONE
token (std::vector -> std::deque) in a throw-away copy at build time (`ref_interp_fx`), and
test_patched_build_lowers_closest_hit_identically shows the patch changes nothing else.  The CPU oracle and the CUDA
kernel must reproduce the fixture bit for bit: bound refinement by distmax, the `L < R` tie rule, strict `<`
everywhere, visit order, and every decode (cpq.scion:3-33)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BINARY = ["identity", "ptr", "pbrt", "pbrt-align16", "pbrt-post", "pbrt-q16", "sg-eq", "sg-eq-align16", "shared-slab", "dop14"]
# authored here (the paper's table points the corpus does not ship): the reference compiles OUR .scion file (ref_interp "@family:/path")
AUTHORED = ["pbrt-soa", "pbrt-soaos", "pbrt-soaos-align16", "pbrt-q16-soaos"]
REF_HERE = os.path.exists(os.path.join(ROOT, "oracle", "_ref", "ref_interp_fx")) and os.path.isdir("/root/reference/proj/corpus")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(ROOT, "tests", "golden", "ref_ir_cpq.npz"))


def trees(sb, gold):
    for tag in ("terrain", "sphere", "cloud"):
        g, seed = (int(x) for x in gold[f"{tag}:scene"])
        scene = {"terrain": sb.Scene.terrain, "sphere": sb.Scene.sphere, "cloud": sb.Scene.cloud}[tag](g, seed)
        lt = scene.build_median(2) if tag == "sphere" else scene.build_sah(32, 4)
        yield tag, lt, np.ascontiguousarray(gold[f"{tag}:points"], np.float32)


def test_fixture_is_meaningful(built, gold):
    for tag, lt, pts in trees(built, gold):
        d2 = gold[f"{tag}:d2:pbrt"]
        assert len(d2) == len(pts) == 430 and (d2 == 0).sum() >= 10 and np.isfinite(d2).all()
        for layout in BINARY:  # d2 is layout-invariant up to conservative-box ties; exact boxes agree bit for bit
            if layout in ("identity", "ptr", "pbrt-align16", "pbrt-post"):
                assert np.array_equal(gold[f"{tag}:d2:{layout}"], d2), layout
            assert np.allclose(gold[f"{tag}:d2:{layout}"], d2, rtol=1e-6), layout


@pytest.mark.parametrize("layout", BINARY + AUTHORED)
def test_oracle_reproduces_the_reference_ir(built, oracle, gold, layout):
    for tag, lt, pts in trees(built, gold):
        got, st = oracle.closest_point(oracle.tree_bytes(lt.encode(layout)), pts)
        assert not st.any()
        assert np.array_equal(got["d2"].view(np.uint32), gold[f"{tag}:d2:{layout}"].view(np.uint32)), (tag, layout)
        xyz = np.stack([got["x"], got["y"], got["z"]], axis=1)
        assert np.array_equal(xyz.view(np.uint32), gold[f"{tag}:point:{layout}"].view(np.uint32)), (tag, layout)


@pytest.mark.gpu
@pytest.mark.parametrize("layout", BINARY + AUTHORED)
def test_kernel_reproduces_the_reference_ir(built, gold, layout):
    import torch
    sb = built
    for tag, lt, pts in trees(sb, gold):
        n = len(pts)
        d_p = torch.from_numpy(pts.reshape(-1).copy()).cuda()
        for dt in (lt.encode(layout).upload(0), lt.encode_device(layout, 0)):
            d_o = torch.empty(n * 20, dtype=torch.uint8, device="cuda:0")
            d_st = torch.ones(n, dtype=torch.int32, device="cuda:0")
            dt.closest_point(d_p.data_ptr(), n, d_o.data_ptr(), d_st.data_ptr())
            torch.cuda.synchronize()
            got = d_o.cpu().numpy().view(sb.CP_DTYPE)
            assert int(d_st.sum()) == 0
            assert np.array_equal(got["d2"].view(np.uint32), gold[f"{tag}:d2:{layout}"].view(np.uint32)), (tag, layout)
            xyz = np.stack([got["x"], got["y"], got["z"]], axis=1)
            assert np.array_equal(xyz.view(np.uint32), gold[f"{tag}:point:{layout}"].view(np.uint32)), (tag, layout)
            dt.free()


@pytest.mark.skipif(not REF_HERE, reason="reference not present (GPU box): the committed fixture is used")
def test_patched_build_lowers_closest_hit_identically(built):
    """the build-time patch (vector -> deque) must be neutral wherever the unpatched reference works: closest_hit lowers
    to byte-identical IR in both builds for every corpus layout; for closest_point the builds differ (that is the bug)"""
    a, b = os.path.join(ROOT, "oracle", "_ref", "ref_interp"), os.path.join(ROOT, "oracle", "_ref", "ref_interp_fx")
    for layout in BINARY + ["bvh8", "bvh8-q8", "bvh8-q8-ci", "bvh8-q16", "bvh8-q16-ci"]:
        ia = subprocess.run([a, "--print-ir", layout, "chrt"], capture_output=True, text=True)
        ib = subprocess.run([b, "--print-ir", layout, "chrt"], capture_output=True, text=True)
        assert ia.returncode == 0 and ib.returncode == 0 and len(ia.stdout) > 1000
        assert ia.stdout == ib.stdout, layout
    ia = subprocess.run([a, "--print-ir", "pbrt", "cpq"], capture_output=True, text=True).stdout
    ib = subprocess.run([b, "--print-ir", "pbrt", "cpq"], capture_output=True, text=True).stdout
    diff = [(x, y) for x, y in zip(ia.splitlines(), ib.splitlines()) if x != y]
    assert len(ia.splitlines()) == len(ib.splitlines()) and 1 <= len(diff) <= 4
    assert all("__ret_" in y for _, y in diff)  # the patched build writes the inlined callee's result where it belongs


@pytest.mark.skipif(not REF_HERE, reason="reference not present (GPU box): the committed fixture is used")
def test_fixture_is_fresh(built, gold, tmp_path):
    import importlib.util
    spec = importlib.util.spec_from_file_location("gen_ref_ir_golden", os.path.join(ROOT, "tools", "gen_ref_ir_golden.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    for tag, lt, pts in trees(built, gold):
        for layout in ("pbrt-q16", "dop14"):
            fin, fout = str(tmp_path / "in.bin"), str(tmp_path / "out.bin")
            gen.write_input(fin, lt.encode(layout), gen.as_rays(pts))
            r = subprocess.run([gen.INTERP_FX, layout, "cpq", fin, fout], capture_output=True, text=True)
            assert r.returncode == 0, r.stderr
            rec = np.fromfile(fout, np.float32).reshape(-1, 10)
            assert np.array_equal(rec[:, 0].view(np.uint32), gold[f"{tag}:d2:{layout}"].view(np.uint32))
