"""Regenerates the committed golden fixtures under tests/golden/ (run in the build container,
where /root/reference exists):
  ref_plans.json      — the REFERENCE planner's output (oracle/_ref/ref_probe, i.e. the reference's
                        own parse_corpus -> check_layout -> plan_layout) for its 15 corpus layouts
                        and for our authored layout files.
  ref_ir.npz          — written by tools/gen_ref_ir_golden.py (the reference's own lowered IR, interpreted): see there.
  hits_small.npz      — oracle results (closest_hit / closest_point) on a small seeded scene for
                        every layout: the GPU tests compare against these even where the oracle
                        library is unavailable.
"""
import json, os, subprocess, sys, glob
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2511_15028_b200 as sb
from tests.oracle_lib import Oracle

probe = os.path.join(ROOT, "oracle", "_ref", "ref_probe")
corpus = json.loads(subprocess.run([probe], capture_output=True, text=True, check=True).stdout)
mine = json.loads(subprocess.run([probe] + sorted(glob.glob(os.path.join(ROOT, "paper_2511_15028_b200", "layouts", "*.scion"))), capture_output=True, text=True, check=True).stdout)
json.dump({"reference_corpus": corpus, "authored": mine}, open(os.path.join(ROOT, "tests", "golden", "ref_plans.json"), "w"), indent=1, sort_keys=True)

orc = Oracle()
scene = sb.Scene.terrain(12, seed=5)
lt = scene.build_sah(32, 4).collapse8()
lo, hi = scene.bounds()
cam = sb.default_camera(lo, hi, True, 24, 24)
rays = np.concatenate([sb.gen_primary_host(cam, 0, 24 * 24), sb.gen_secondary_host(lt.triangles(), 9, 0, 448)])
pts = sb.gen_points_host(lo - 0.25, hi + 0.25, 4, 0, 256)
out = {"rays": rays.view(np.float32).reshape(-1, 8), "points": pts, "terrain_grid": np.array([12, 5])}
for l in sb.layouts():
    pt = lt.encode(l["name"])
    tb = orc.tree_bytes(pt)
    h, st, c = orc.closest_hit(tb, rays, counters=True)
    out[f"hit_t:{l['name']}"] = h["t"].copy()
    out[f"hit_prim:{l['name']}"] = h["prim"].copy()
    out[f"hit_visits:{l['name']}"] = c["node_visits"].copy()
    if l["has_cpq"]:
        cp, st, c = orc.closest_point(tb, pts, counters=True)
        out[f"cp:{l['name']}"] = cp.view(np.uint32).reshape(-1, 5).copy()
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "hits_small.npz"), **out)
print("golden fixtures written")
