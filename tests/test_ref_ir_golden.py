"""Pins against the REFERENCE'S OWN compiled traversal.  tests/golden/ref_ir.npz holds closest-hit answers that
were computed by the reference's lowered IR (its parser, type checker, planner and `specialize_destructors`,
executed by oracle/ref_interp.cpp — tools/gen_ref_ir_golden.py) on trees produced by this repository's encoders,
for the reference's 15 corpus layouts on two scenes.  The reference returns (t, Triangle value); the fixture
stores t and the index of that triangle.  Both the CPU oracle and the CUDA kernels must reproduce them
bit-for-bit — which pins, through the reference itself: every slot offset the decoders use, the decode
expressions, the visit order, the strictness of every comparison and the short-circuits."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CORPUS = ["identity", "ptr", "pbrt", "pbrt-align16", "pbrt-post", "pbrt-q16", "sg-eq", "sg-eq-align16", "shared-slab", "dop14",
          "bvh8", "bvh8-q8", "bvh8-q8-ci", "bvh8-q16", "bvh8-q16-ci"]
# authored here (PAPER.md:854-857, :872-880 table points + the SoA point of BASELINE config 2): the reference's own front-end,
# planner and destructor specialiser compile OUR .scion file (ref_interp "@family:/path"), same pin as the corpus
AUTHORED = ["pbrt-soa", "pbrt-soaos", "pbrt-soaos-align16", "pbrt-q16-soaos"] + \
    ["bvh8-align16", "bvh8-q8-align16", "bvh8-q8-ci-align16", "bvh8-q16-align16", "bvh8-q16-ci-align16"]


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(ROOT, "tests", "golden", "ref_ir.npz"))


def trees(sb, gold):
    for tag in ("terrain", "sphere"):
        g, seed = (int(x) for x in gold[f"{tag}:scene"])
        scene = sb.Scene.terrain(g, seed) if tag == "terrain" else sb.Scene.sphere(g, seed)
        lt = (scene.build_sah(32, 4) if tag == "terrain" else scene.build_median(2)).collapse8()
        rays = np.ascontiguousarray(gold[f"{tag}:rays"]).reshape(-1).view(sb.RAY_DTYPE)
        yield tag, lt, rays


def test_fixture_is_meaningful(built, gold):
    sb = built
    for tag, lt, rays in trees(sb, gold):
        t = gold[f"{tag}:t:pbrt"]
        assert len(t) == len(rays) == 487 and 150 < np.isfinite(t).sum() < 300
        # zero direction components, finite tmax, -0.0 and a root miss are all in the set
        assert (rays["dx"] == 0).any() and np.isfinite(rays["tmax"]).any() and (np.signbit(rays["dx"]) & (rays["dx"] == 0)).any()
        # cross-layout invariant of the reference: every layout of the corpus gives the same hit set
        for layout in CORPUS + AUTHORED:
            assert np.array_equal(np.isfinite(gold[f"{tag}:t:{layout}"]), np.isfinite(t)), layout


@pytest.mark.parametrize("layout", CORPUS + AUTHORED)
def test_oracle_reproduces_the_reference_ir(built, oracle, gold, layout):
    sb = built
    for tag, lt, rays in trees(sb, gold):
        pt = lt.encode(layout)
        got, st = oracle.closest_hit(oracle.tree_bytes(pt), rays)
        assert np.array_equal(got["t"].view(np.uint32), gold[f"{tag}:t:{layout}"].view(np.uint32)), (tag, layout)
        assert np.array_equal(got["prim"], gold[f"{tag}:prim:{layout}"]), (tag, layout)
        assert not st.any()


@pytest.mark.gpu
@pytest.mark.parametrize("layout", CORPUS + AUTHORED)
def test_kernels_reproduce_the_reference_ir(built, gold, layout):
    import torch
    sb = built
    for tag, lt, rays in trees(sb, gold):
        n = len(rays)
        d_rays = torch.from_numpy(rays.view(np.uint8).reshape(-1).copy()).cuda()
        for dt in (lt.encode(layout).upload(0), lt.encode_device(layout, 0)):
            hits = torch.empty(n * 8, dtype=torch.uint8, device="cuda:0")
            dt.closest_hit(d_rays.data_ptr(), n, hits.data_ptr())
            torch.cuda.synchronize()
            got = hits.cpu().numpy().view(sb.HIT_DTYPE)
            assert np.array_equal(got["t"].view(np.uint32), gold[f"{tag}:t:{layout}"].view(np.uint32)), (tag, layout)
            assert np.array_equal(got["prim"], gold[f"{tag}:prim:{layout}"]), (tag, layout)
            dt.free()


@pytest.mark.skipif(not (os.path.exists(os.path.join(ROOT, "oracle", "_ref", "ref_interp")) and os.path.isdir("/root/reference/proj/corpus")),
                    reason="reference not present (GPU box): the committed fixture is used")
def test_fixture_is_fresh(built, gold, tmp_path):
    """In the build container: re-run the reference IR for two layouts and compare with the committed fixture."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("gen_ref_ir_golden", os.path.join(ROOT, "tools", "gen_ref_ir_golden.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    sb = built
    for tag, lt, rays in trees(sb, gold):
        for layout in ("pbrt-q16", "bvh8-q8-ci"):
            fin, fout = str(tmp_path / "in.bin"), str(tmp_path / "out.bin")
            gen.write_input(fin, lt.encode(layout), rays)
            r = subprocess.run([gen.INTERP, layout, "chrt", fin, fout], capture_output=True, text=True)
            assert r.returncode == 0, r.stderr
            rec = np.fromfile(fout, np.float32).reshape(-1, 10)
            assert np.array_equal(rec[:, 0].view(np.uint32), gold[f"{tag}:t:{layout}"].view(np.uint32))
