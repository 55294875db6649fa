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
    assert total == 2 * (16 + 11)
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
