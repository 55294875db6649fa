"""Layout exploration through the run-time registration (scion_layout_register): variants of shipped layouts are derived
from their .scion text, compiled into plugins and timed on the C5 probe (10 M triangles, 2^24 primary + 2^24 secondary
rays) next to the layouts they derive from.  Every variant must return its parent's hits bit for bit.
usage: python tools/layout_explore.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2511_15028_b200 as sb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
def src(name): return open(os.path.join(ROOT, "paper_2511_15028_b200", "layouts", name + ".scion")).read()

VARIANTS = [
    # (new name, parent layout, parent file, text transformation)
    ("bvh8-q8-ci-align32", "bvh8-q8-ci", "bvh8_q8_ci", lambda t: t.replace("indirect group Interiors[size = interior_count]", "indirect group Interiors[size = interior_count, align = 32]")),
    ("bvh8-q8-ci-align128", "bvh8-q8-ci", "bvh8_q8_ci", lambda t: t.replace("indirect group Interiors[size = interior_count]", "indirect group Interiors[size = interior_count, align = 128]")),
    ("bvh8-q16-ci-align32", "bvh8-q16-ci", "bvh8_q16_ci", lambda t: t.replace("indirect group Interiors[size = interior_count]", "indirect group Interiors[size = interior_count, align = 32]")),
    ("dop14-aos", "dop14", "dop14", lambda t: t.replace("    ---\n", "")),
    ("pbrt-q16-align32", "pbrt-q16", "pbrt_q16", lambda t: t.replace("group nodes[size = node_count, align = 16]", "group nodes[size = node_count, align = 32]")),
]

def main():
    dev = "cuda:0"
    scene = sb.Scene.terrain(2236, seed=1)
    lt = scene.build_sah(32, 4).collapse8()
    lo, hi = scene.bounds()
    nr = 1 << 25
    d_rays = torch.empty(nr * 32, dtype=torch.uint8, device=dev)
    cam = sb.default_camera(lo, hi, True, 4096, 4096)
    ref_hits = {}
    def run(layout):
        pt = lt.encode(layout)
        dt = pt.upload(0)
        sb.gen_primary(cam, 0, 1 << 24, d_rays.data_ptr()); dt.gen_secondary(77, 0, 1 << 24, d_rays.data_ptr() + (32 << 24))
        h = torch.empty(nr * 8, dtype=torch.uint8, device=dev)
        for _ in range(2): dt.closest_hit(d_rays.data_ptr(), nr, h.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4): dt.closest_hit(d_rays.data_ptr(), nr, h.data_ptr())
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 4
        info = sb.layout_info(layout)
        print(f"  {layout:22s} stride {info['node_stride']:4d} B  BVH {pt.node_bytes / lt.nprims:6.2f} B/prim  {nr / ms / 1e3:8.1f} Mrays/s", flush=True)
        dt.free()
        return h
    for name, parent, f, tf in VARIANTS:
        text = tf(src(f))
        assert text != src(f), name
        t0 = time.time()
        sb.register_layout(name, text)
        print(f"registered {name} in {time.time() - t0:.1f} s", flush=True)
        if parent not in ref_hits: ref_hits[parent] = run(parent)
        h = run(name)
        print(f"    identical to {parent}: {bool(torch.equal(h, ref_hits[parent]))}", flush=True)

if __name__ == "__main__":
    main()
