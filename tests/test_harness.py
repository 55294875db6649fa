"""CLI harness: check / footprint / emit-cuda on the CPU; verify (full matrix: every layout x applicable
algorithm x 2 scenes x 4096 queries, acceptance criterion 2 of SPEC.md:657) and bench on the GPU."""
import io
import json
import os
import subprocess
import sys
from contextlib import redirect_stdout

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(argv):
    from paper_2511_15028_b200 import harness
    buf = io.StringIO()
    with redirect_stdout(buf):
        rc = harness.main(argv)
    return rc, buf.getvalue()


def test_check_footprint_emit(built):
    rc, out = run(["check"])
    assert rc == 0 and out.count(" ok ") == len(built.layouts())
    rc, out = run(["footprint", "--layout", "pbrt", "--scene", "terrain:16"])
    rep = json.loads(out)
    assert rc == 0 and rep["node_stride"] == 32 and rep["primitives"] == 512
    nodes = [b for b in rep["buffers"] if b["name"] == "nodes"][0]
    assert nodes["bytes"] == 32 * nodes["count"] and rep["total_bytes"] == nodes["bytes"] + 512 * 36
    rc, out = run(["emit-cuda", "--layout", "bvh8-q8-ci"])
    assert rc == 0 and "static_assert(sizeof(Record_Interiors_s0) == 104" in out
    assert run(["footprint", "--layout", "nope"])[0] == 2  # usage error class
    assert run([])[0] == 2


@pytest.mark.gpu
def test_verify_matrix(built):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from tests import verify_cli
    total = 0
    for scene in ("terrain:24", "sphere:20"):
        for l in built.layouts():
            for alg in (("chrt", "cpq") if l["has_cpq"] else ("chrt",)):
                rep = verify_cli.verify(l["name"], alg, scene, 4096)
                assert rep["mismatches_vs_oracle_same_layout"] == 0, rep
                if alg == "chrt":
                    assert rep["mismatches_vs_identity_oracle"] == 0, rep
                total += 1
    assert total == 2 * (24 + 14)  # 24 layouts (15 corpus + 9 authored), 14 of them binary (closest_point)
    # fault injection: one corrupted c_o byte must be reported
    rep = verify_cli.verify("pbrt", "chrt", "terrain:24", 4096, corrupt=(1, 24, 1))
    assert rep["mismatches_vs_identity_oracle"] >= 1 and len(rep["first_offenders"]) <= 10


@pytest.mark.gpu
def test_bench_csv(built):
    rc, out = run(["bench", "--layout", "pbrt,pbrt-q16", "--scene", "terrain:64", "--queries", "65536", "--rays", "secondary"])
    lines = out.strip().splitlines()
    assert rc == 0 and lines[0].startswith("layout,algorithm,scene,n_gpus") and len(lines) == 3
    assert float(lines[1].split(",")[7]) > 0


def test_native_harness_footprint_equals_python(built):
    """csrc/tools/scion_run.cpp: a C++ caller that uses nothing but include/scion_b200.h (the drop-in boundary)."""
    import json, os, subprocess
    sb = built
    exe = os.path.join(os.path.dirname(sb.__file__), "bin", "scion_run")
    assert os.path.exists(exe), "scion_run is built by csrc/Makefile"
    out = subprocess.run([exe, "layouts"], capture_output=True, text=True)
    assert out.returncode == 0 and len(out.stdout.strip().splitlines()) == len(sb.layouts())
    for layout in ("pbrt-q16", "bvh8-q8-ci", "dop14"):
        r = subprocess.run([exe, "footprint", layout, "terrain:24"], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        rep = json.loads(r.stdout)
        lt = sb.Scene.terrain(24, 1).build_sah(32, 4).collapse8()
        pt = lt.encode(layout)
        assert rep["total_bytes"] == pt.total_bytes and rep["node_bytes"] == pt.node_bytes and rep["primitives"] == lt.nprims
    assert subprocess.run([exe, "footprint", "no-such-layout", "terrain:8"], capture_output=True).returncode == 2  # usage class
    if sb.device_count() == 0:  # the product has no CPU fallback: bench must fail loudly
        r = subprocess.run([exe, "bench", "pbrt-q16", "terrain:8", "256"], capture_output=True, text=True)
        assert r.returncode == 1 and "no CUDA device" in r.stderr


@pytest.mark.gpu
def test_native_harness_bench(built):
    import os, subprocess
    sb = built
    exe = os.path.join(os.path.dirname(sb.__file__), "bin", "scion_run")
    for args in (["pbrt-q16", "terrain:64", "65536", "primary"], ["bvh8-q8-ci", "terrain:64", "65536", "secondary"], ["pbrt-soa", "sphere:32", "4096", "points"],
                 ["sg-eq", "terrain:64", "65536", "secondary", "--host-encode"]):
        r = subprocess.run([exe, "bench"] + args, capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        head, row = r.stdout.strip().splitlines()
        rec = dict(zip(head.split(","), row.split(",")))
        assert rec["layout"] == args[0] and float(rec["mqueries_per_s"]) > 0 and int(rec["query_errors"]) == 0 and float(rec["node_visits"]) > 0


def test_compile_build_tree_build(built, tmp_path):
    """compile / build-tree / build: the host-side sub-commands either side of the traversal path."""
    src = os.path.join(ROOT, "paper_2511_15028_b200", "layouts", "pbrt_q16.scion")
    cuh, plan = str(tmp_path / "q16.cuh"), str(tmp_path / "q16.json")
    rc, out = run(["compile", src, "--plan", plan, "--emit-cuda", cuh])
    rep = json.loads(out)
    assert rc == 0 and rep["node_stride"] == 16
    assert "static_assert(sizeof(Record_" in open(cuh).read() and json.load(open(plan))["node_group"] == rep["node_group"]
    bad = tmp_path / "bad.scion"
    bad.write_text("type BVH(low: f32x3) = Interior(left: BVH) | Leaf(n: u8); layout BVH(I: u32) { group g[align = 3] by I { low: f32x3; }; };")
    assert run(["compile", str(bad)])[0] == 1  # diagnostics class
    assert run(["compile", str(tmp_path / "missing.scion")])[0] == 2
    tree = str(tmp_path / "tree.npz")
    rc, out = run(["build-tree", "--scene", "terrain:16", "-o", tree])
    assert rc == 0 and json.loads(out)["primitives"] == 512
    for layout in ("pbrt-q16", "bvh8-q8-ci", "shared-slab"):
        f1, f2 = str(tmp_path / f"{layout}.a.scionpt"), str(tmp_path / f"{layout}.b.scionpt")
        rc, out = run(["build", "--layout", layout, "--tree", tree, "-o", f1])
        assert rc == 0 and json.loads(out)["primitives"] == 512
        assert run(["build", "--layout", layout, "--scene", "terrain:16", "-o", f2])[0] == 0
        assert open(f1, "rb").read() == open(f2, "rb").read(), layout  # deterministic, and the .npz round trip loses nothing
        pt = built.PhysicalTree.load(f1)
        want = built.Scene.terrain(16, 1).build_sah(32, 4).collapse8().encode(layout)
        assert pt.layout == layout and pt.total_bytes == want.total_bytes
        for b, w in zip(pt.buffers(), want.buffers()):
            assert b["name"] == w["name"] and bytes(b["data"]) == bytes(w["data"]), (layout, b["name"])


@pytest.mark.gpu
def test_run_container_file(built, oracle, tmp_path):
    """run: container file -> results; equal to the oracle on the same generated queries."""
    import numpy as np
    f, out_bin = str(tmp_path / "t.scionpt"), str(tmp_path / "hits.bin")
    assert run(["build", "--layout", "pbrt-q16", "--scene", "terrain:24", "-o", f])[0] == 0
    rc, out = run(["run", f, "--alg", "chrt", "--queries", "4096", "--rays", "secondary", "--seed", "11", "-o", out_bin])
    rep = json.loads(out)
    assert rc == 0 and rep["query_errors"] == 0 and rep["queries"] == 4096 and rep["found"] > 500
    pt = built.PhysicalTree.load(f)
    lt = built.Scene.terrain(24, 1).build_sah(32, 4)
    rays = built.gen_secondary_host(lt.triangles(), 11, 0, 4096)
    want, _ = oracle.closest_hit(oracle.tree_bytes(pt), rays)
    got = np.fromfile(out_bin, built.HIT_DTYPE)
    assert np.array_equal(got["prim"], want["prim"]) and np.array_equal(got["t"].view(np.uint32), want["t"].view(np.uint32))
    rc, out = run(["run", f, "--alg", "cpq", "--queries", "2048"])
    rep = json.loads(out)
    assert rc == 0 and rep["found"] == 2048 and rep["query_errors"] == 0
