"""Scratch GPU probe: parity of every layout vs the oracle on a small scene + quick timings."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2511_15028_b200 as sb
from tests.oracle_lib import Oracle

orc = Oracle()
dev = "cuda:0"
def dbuf(nbytes): return torch.empty(nbytes, dtype=torch.uint8, device=dev)

def parity(G, W, nsec):
    scene = sb.Scene.terrain(G, seed=3)
    lt = scene.build_sah(32, 4).collapse8()
    lo, hi = scene.bounds()
    cam = sb.default_camera(lo, hi, True, W, W)
    n = W * W
    rays_p = sb.gen_primary_host(cam, 0, n)
    rays_s = sb.gen_secondary_host(lt.triangles(), 11, 0, nsec)
    rays = np.concatenate([rays_p, rays_s])
    pts = sb.gen_points_host(lo - 0.2, hi + 0.2, 5, 0, 8192)
    n = rays.shape[0]
    d_rays = torch.from_numpy(rays.view(np.uint8).reshape(-1)).to(dev)
    d_pts = torch.from_numpy(pts.reshape(-1)).to(dev)
    ok = True
    for l in sb.layouts():
        name = l["name"]
        pt = lt.encode(name)
        tb = orc.tree_bytes(pt)
        dt = pt.upload(0)
        d_hits, d_st, d_ctr = dbuf(n * 8), dbuf(n * 4), dbuf(n * 16)
        dt.closest_hit(d_rays.data_ptr(), n, d_hits.data_ptr(), d_st.data_ptr(), d_ctr.data_ptr())
        torch.cuda.synchronize()
        got = d_hits.cpu().numpy().view(sb.HIT_DTYPE); st = d_st.cpu().numpy().view(np.uint32); ctr = d_ctr.cpu().numpy().view(sb.COUNTERS_DTYPE)
        want, wst, wctr = orc.closest_hit(tb, rays, counters=True)
        bad_p = int((got["prim"] != want["prim"]).sum()); bad_t = int((got["t"].view(np.uint32) != want["t"].view(np.uint32)).sum())
        bad_c = int((ctr != wctr).sum()); bad_s = int((st != wst).sum())
        # counter-free kernel must agree too
        d_hits2 = dbuf(n * 8)
        dt.closest_hit(d_rays.data_ptr(), n, d_hits2.data_ptr())
        torch.cuda.synchronize()
        bad_nc = int((d_hits2.cpu().numpy().view(np.uint32) != d_hits.cpu().numpy().view(np.uint32)).sum())
        msg = f"{name:14s} chrt: prim_mismatch {bad_p} t_mismatch {bad_t} counters {bad_c} status {bad_s} nocount {bad_nc} hits {(got['prim']!=sb.MISS_PRIM).mean():.3f} visits/ray {ctr['node_visits'].mean():.1f} tris/ray {ctr['prim_tests'].mean():.1f} maxstack {ctr['max_stack'].max()}"
        if l["has_cpq"]:
            m = pts.shape[0]
            d_out, d_st2, d_ctr2 = dbuf(m * 20), dbuf(m * 4), dbuf(m * 16)
            dt.closest_point(d_pts.data_ptr(), m, d_out.data_ptr(), d_st2.data_ptr(), d_ctr2.data_ptr())
            torch.cuda.synchronize()
            gc = d_out.cpu().numpy().view(sb.CP_DTYPE); cc = d_ctr2.cpu().numpy().view(sb.COUNTERS_DTYPE)
            wc, wcs, wcc = orc.closest_point(tb, pts, counters=True)
            badc = int((gc.view(np.uint8).reshape(m, 20) != wc.view(np.uint8).reshape(m, 20)).any(axis=1).sum())
            msg += f" | cpq: mismatch {badc} counters {int((cc != wcc).sum())} visits {cc['node_visits'].mean():.1f}"
            ok &= badc == 0
        print(msg, flush=True)
        ok &= (bad_p == 0 and bad_t == 0 and bad_c == 0 and bad_s == 0 and bad_nc == 0)
        dt.free()
    return ok

def timing(G, nrays, layouts):
    t0 = time.time(); scene = sb.Scene.terrain(G, seed=3); t1 = time.time()
    lt = scene.build_sah(32, 4).collapse8(); t2 = time.time()
    print(f"scene {scene.ntris} tris gen {t1-t0:.2f}s build {t2-t1:.2f}s nodes {lt.nnodes} depth {lt.depth}", flush=True)
    lo, hi = scene.bounds()
    cam = sb.default_camera(lo, hi, True, 4096, 4096)
    d_rays = dbuf(nrays * 32); d_hits = dbuf(nrays * 8)
    for name in layouts:
        t3 = time.time(); pt = lt.encode(name); t4 = time.time()
        dt = pt.upload(0)
        for kind in ("primary", "secondary"):
            if kind == "primary": sb.gen_primary(cam, 0, nrays, d_rays.data_ptr())
            else: dt.gen_secondary(77, 0, nrays, d_rays.data_ptr())
            torch.cuda.synchronize()
            for _ in range(2): dt.closest_hit(d_rays.data_ptr(), nrays, d_hits.data_ptr())
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3): dt.closest_hit(d_rays.data_ptr(), nrays, d_hits.data_ptr())
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 3
            print(f"  {name:14s} {kind:9s} {nrays/ms/1e3:9.1f} Mrays/s  ({ms:.2f} ms)  encode {t4-t3:.2f}s bytes/prim {pt.node_bytes/lt.nprims:.1f}", flush=True)
        dt.free()

def tune(G, nrays, layouts):
    scene = sb.Scene.terrain(G, seed=3)
    lt = scene.build_sah(32, 4).collapse8()
    lo, hi = scene.bounds()
    cam = sb.default_camera(lo, hi, True, 4096, 4096)
    d_rays = dbuf(nrays * 32); d_hits = dbuf(nrays * 8)
    for name in layouts:
        dt = lt.encode(name).upload(0)
        for kind in ("primary", "secondary"):
            if kind == "primary": sb.gen_primary(cam, 0, nrays, d_rays.data_ptr())
            else: dt.gen_secondary(77, 0, nrays, d_rays.data_ptr())
            torch.cuda.synchronize()
            res = []
            for refill in (1, 4, 8, 16):
                for prim in (1, 4, 8, 12, 16, 24):
                    v = refill | (prim << 8)
                    dt.closest_hit(d_rays.data_ptr(), nrays, d_hits.data_ptr(), variant=v)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(2): dt.closest_hit(d_rays.data_ptr(), nrays, d_hits.data_ptr(), variant=v)
                    e1.record(); torch.cuda.synchronize()
                    res.append((nrays / (e0.elapsed_time(e1) / 2) / 1e3, refill, prim))
            res.sort(reverse=True)
            print(f"  {name:12s} {kind:9s} best: " + ", ".join(f"{m:.0f}(r{r},p{p})" for m, r, p in res[:5]) + " | worst: " + ", ".join(f"{m:.0f}(r{r},p{p})" for m, r, p in res[-3:]), flush=True)
        dt.free()

if __name__ == "__main__":
    if "--c5" in sys.argv:  # C5-like quick timing: 10M terrain, 2^24 primary + 2^24 secondary, pbrt-q16 and pbrt
        scene = sb.Scene.terrain(2236, seed=1)
        lt = scene.build_sah(32, 4).collapse8()
        lo, hi = scene.bounds()
        nr = 1 << 25
        d_rays = dbuf(nr * 32); d_hits = dbuf(nr * 8)
        cam = sb.default_camera(lo, hi, True, 4096, 4096)
        for layout in (sys.argv[sys.argv.index("--c5") + 1].split(",") if len(sys.argv) > sys.argv.index("--c5") + 1 else ("pbrt-q16", "pbrt")):
            dt = lt.encode(layout).upload(0)
            sb.gen_primary(cam, 0, 1 << 24, d_rays.data_ptr()); dt.gen_secondary(77, 0, 1 << 24, d_rays.data_ptr() + (32 << 24))
            for _ in range(2): dt.closest_hit(d_rays.data_ptr(), nr, d_hits.data_ptr())
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(4): dt.closest_hit(d_rays.data_ptr(), nr, d_hits.data_ptr())
            e1.record(); torch.cuda.synchronize()
            print(f"  {os.environ.get('SCION_B200_LIB','default').split('/')[-1]:16s} {layout:10s} {nr / (e0.elapsed_time(e1) / 4) / 1e3:8.1f} Mrays/s", flush=True)
            dt.free()
        sys.exit(0)
    if "--c5split" in sys.argv:  # primary-only vs secondary-only throughput on the 10M scene
        scene = sb.Scene.terrain(2236, seed=1)
        lt = scene.build_sah(32, 4).collapse8()
        lo, hi = scene.bounds()
        nr = 1 << 25
        d_rays = dbuf(nr * 32); d_hits = dbuf(nr * 8)
        cam = sb.default_camera(lo, hi, True, 4096, 4096)
        for layout in sys.argv[sys.argv.index("--c5split") + 1].split(","):
            dt = lt.encode(layout).upload(0)
            for kind in ("primary", "secondary"):
                if kind == "primary":
                    sb.gen_primary(cam, 0, 1 << 24, d_rays.data_ptr()); sb.gen_primary(cam, 0, 1 << 24, d_rays.data_ptr() + (32 << 24))
                else:
                    dt.gen_secondary(77, 0, nr, d_rays.data_ptr())
                for _ in range(2): dt.closest_hit(d_rays.data_ptr(), nr, d_hits.data_ptr())
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(4): dt.closest_hit(d_rays.data_ptr(), nr, d_hits.data_ptr())
                e1.record(); torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 4
                nc = 1 << 22
                d_ctr = dbuf(nc * 16)
                dt.closest_hit(d_rays.data_ptr(), nc, d_hits.data_ptr(), 0, d_ctr.data_ptr())
                torch.cuda.synchronize()
                ctr = d_ctr.cpu().numpy().view(sb.COUNTERS_DTYPE)
                nv, npt = ctr["node_visits"].mean(), ctr["prim_tests"].mean()
                print(f"  {layout:10s} {kind:9s} {nr / ms / 1e3:8.1f} Mrays/s  visits/ray {nv:.1f} tris/ray {npt:.1f} maxstack {ctr['max_stack'].max()} mean stack {ctr['max_stack'].mean():.1f} -> {nr * nv / ms / 1e6:.1f} Gvisits/s", flush=True)
            dt.free()
        sys.exit(0)
    if "--wide8" in sys.argv:  # 8-wide kernels: register-record (variant 1) vs staged-record (variant 4), C5-like mix
        i = sys.argv.index("--wide8")
        layouts = sys.argv[i + 1].split(",") if len(sys.argv) > i + 1 else ["bvh8", "bvh8-align16", "bvh8-q8-align16", "bvh8-q8-ci-align16", "bvh8-q16-align16", "bvh8-q16-ci-align16"]
        scene = sb.Scene.terrain(2236, seed=1)
        lt = scene.build_sah(32, 4).collapse8()
        lo, hi = scene.bounds()
        nr = 1 << 25
        d_rays = dbuf(nr * 32); outs = {1: dbuf(nr * 8), 4: dbuf(nr * 8)}
        cam = sb.default_camera(lo, hi, True, 4096, 4096)
        for layout in layouts:
            dt = lt.encode(layout).upload(0)
            sb.gen_primary(cam, 0, 1 << 24, d_rays.data_ptr()); dt.gen_secondary(77, 0, 1 << 24, d_rays.data_ptr() + (32 << 24))
            res = {}
            for v in (1, 4):
                for _ in range(2): dt.closest_hit(d_rays.data_ptr(), nr, outs[v].data_ptr(), variant=v)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(4): dt.closest_hit(d_rays.data_ptr(), nr, outs[v].data_ptr(), variant=v)
                e1.record(); torch.cuda.synchronize()
                res[v] = nr / (e0.elapsed_time(e1) / 4) / 1e3
            print(f"  {layout:22s} registers {res[1]:8.1f}  staged {res[4]:8.1f} Mrays/s  ({res[4] / res[1]:.3f}x)  identical={bool(torch.equal(outs[1], outs[4]))}", flush=True)
            dt.free()
        sys.exit(0)
    if "--stage" in sys.argv:  # TMA-staged top-levels treelet (variant 2) vs default: identical results? timing?
        for G in (708, 2236):
            scene = sb.Scene.terrain(G, seed=1)
            lt = scene.build_sah(32, 4)
            lo, hi = scene.bounds()
            nr = 1 << 25
            d_rays = dbuf(nr * 32); d_hits = dbuf(nr * 8); d_hits2 = dbuf(nr * 8)
            cam = sb.default_camera(lo, hi, True, 4096, 4096)
            for layout in ("pbrt-q16", "pbrt"):
                dt = lt.encode(layout).upload(0)
                sb.gen_primary(cam, 0, 1 << 24, d_rays.data_ptr()); dt.gen_secondary(77, 0, 1 << 24, d_rays.data_ptr() + (32 << 24))
                res = {}
                for v, out in ((0, d_hits), (2, d_hits2)):
                    for _ in range(2): dt.closest_hit(d_rays.data_ptr(), nr, out.data_ptr(), variant=v)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(4): dt.closest_hit(d_rays.data_ptr(), nr, out.data_ptr(), variant=v)
                    e1.record(); torch.cuda.synchronize()
                    res[v] = nr / (e0.elapsed_time(e1) / 4) / 1e3
                print(f"  G={G} {layout:10s} default {res[0]:8.1f}  staged {res[2]:8.1f} Mrays/s  identical={bool(torch.equal(d_hits, d_hits2))}", flush=True)
                dt.free()
        sys.exit(0)
    if "--ncu" in sys.argv:
        kind = sys.argv[sys.argv.index("--ncu") + 1]      # primary | secondary
        layout = sys.argv[sys.argv.index("--ncu") + 2]
        G = int(sys.argv[sys.argv.index("--ncu") + 3])
        scene = sb.Scene.terrain(G, seed=1)
        lt = scene.build_sah(32, 4).collapse8()
        lo, hi = scene.bounds()
        nr = 1 << 25
        d_rays = dbuf(nr * 32); d_hits = dbuf(nr * 8)
        dt = lt.encode(layout).upload(0)
        if kind == "primary":
            cam = sb.default_camera(lo, hi, True, 4096, 4096)
            sb.gen_primary(cam, 0, 1 << 24, d_rays.data_ptr()); sb.gen_primary(cam, 0, 1 << 24, d_rays.data_ptr() + (32 << 24))
        else:
            dt.gen_secondary(77, 0, nr, d_rays.data_ptr())
        for _ in range(3):
            dt.closest_hit(d_rays.data_ptr(), nr, d_hits.data_ptr())
        torch.cuda.synchronize()
        sys.exit(0)
    if "--tune" in sys.argv:
        tune(708, 1 << 23, ["pbrt", "pbrt-q16", "bvh8-q8-ci"])
        tune(2236, 1 << 23, ["pbrt-q16"])
        sys.exit(0)
    print(torch.cuda.get_device_name(0))
    ok = parity(40, 128, 8192)
    print("PARITY", "OK" if ok else "FAILED", flush=True)
    if "--time" in sys.argv:
        timing(708, 1 << 24, ["pbrt", "pbrt-soa", "pbrt-q16", "sg-eq", "sg-eq-align16", "dop14", "bvh8", "bvh8-q8-ci", "bvh8-q16-ci"])
