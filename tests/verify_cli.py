"""`verify` of the reference harness for the B200 backend — TEST INFRASTRUCTURE (uses the
CPU oracle): compile + build the subject layout AND the identity oracle, run the same queries on the GPU and on
the oracle, diff: CHRT identical primitive + bitwise-equal t; CPQ identical primitive, d2 within 1e-6 relative.
Prints the VerifyReport as JSON (total, mismatches: first 10 offenders, footprint, counters); exit 0 / 1 / 2.

  python tests/verify_cli.py --layout pbrt-q16 --alg chrt --scene terrain:64 --queries 4096
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_15028_b200 as sb  # noqa: E402
from paper_2511_15028_b200.harness import parse_scene  # noqa: E402
from tests.oracle_lib import Oracle  # noqa: E402


def verify(layout, alg, scene_spec, n, corrupt=None):
    import torch
    orc = Oracle()
    scene = parse_scene(scene_spec)
    lt = scene.build_sah(32, 4).collapse8()
    lo, hi = scene.bounds()
    pt = lt.encode(layout)
    if corrupt:
        pt.corrupt(*corrupt)
    fam = sb.layout_info(layout)["family"]
    dt = pt.upload(0)
    rep = {"layout": layout, "algorithm": alg, "scene": scene_spec, "total": n, "footprint": {"total_bytes": pt.total_bytes, "node_bytes": pt.node_bytes}}
    if alg == "chrt":
        side = max(1, int(np.sqrt(n // 2)))
        rays = np.concatenate([sb.gen_primary_host(sb.default_camera(lo, hi, scene_spec.startswith("terrain"), side, side), 0, side * side),
                               sb.gen_secondary_host(lt.triangles(), 3, 0, n - side * side)])
        status = np.zeros(n, np.uint32)
        got = dt.closest_hit_host(rays, status=status)
        want, wst, ctr = orc.closest_hit(orc.tree_bytes(pt), rays, counters=True)
        ident, _ = orc.closest_hit(orc.logical_bytes(lt, {0: "@logical2", 1: "@logical-dop14", 2: "@logical8"}[fam]), rays)
        bad = np.nonzero((got["prim"] != want["prim"]) | (got["t"].view(np.uint32) != want["t"].view(np.uint32)) | (status != wst))[0]
        bad_ident = np.nonzero((got["prim"] != ident["prim"]) | (got["t"].view(np.uint32) != ident["t"].view(np.uint32)))[0]
        fmt = lambda a, i: {"t": float(a["t"][i]), "prim": int(a["prim"][i])}
    else:
        pts = sb.gen_points_host(lo - 0.25, hi + 0.25, 5, 0, n)
        status = np.zeros(n, np.uint32)
        got = dt.closest_point_host(pts, status=status)
        want, wst, ctr = orc.closest_point(orc.tree_bytes(pt), pts, counters=True)
        ident, _ = orc.closest_point(orc.logical_bytes(lt, "@logical-dop14" if fam == 1 else "@logical2"), pts)
        rel = np.abs(got["d2"] - want["d2"]) / np.maximum(np.abs(want["d2"]), 1e-30)
        bad = np.nonzero((got["prim"] != want["prim"]) | (rel > 1e-6) | (status != wst))[0]
        reli = np.abs(got["d2"] - ident["d2"]) / np.maximum(np.abs(ident["d2"]), 1e-30)
        bad_ident = np.nonzero(reli > 1e-6)[0]
        fmt = lambda a, i: {"d2": float(a["d2"][i]), "prim": int(a["prim"][i])}
    rep["mismatches_vs_oracle_same_layout"] = int(bad.size)
    rep["mismatches_vs_identity_oracle"] = int(bad_ident.size)
    rep["first_offenders"] = [{"query": int(i), "oracle": fmt(want, i), "subject": fmt(got, i)} for i in bad[:10]]
    rep["counters"] = {"node_visits": float(ctr["node_visits"].mean()), "prim_tests": float(ctr["prim_tests"].mean())}
    dt.free()
    return rep


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--layout", required=True)
    ap.add_argument("--alg", default="chrt", choices=["chrt", "cpq"])
    ap.add_argument("--scene", default="terrain:32")
    ap.add_argument("--queries", type=int, default=4096)
    ap.add_argument("--corrupt", default=None, help="buffer:byte:xor fault injection (SPEC.md:625)")
    try:
        a = ap.parse_args(argv)
    except SystemExit:
        return 2
    corrupt = tuple(int(x, 0) for x in a.corrupt.split(":")) if a.corrupt else None
    rep = verify(a.layout, a.alg, a.scene, a.queries, corrupt)
    print(json.dumps(rep, indent=1))
    return 0 if rep["mismatches_vs_oracle_same_layout"] == 0 and rep["mismatches_vs_identity_oracle"] == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
