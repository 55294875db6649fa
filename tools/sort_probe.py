"""Scratch GPU probe: how much would re-ordering incoherent rays (legal: results are written by query
index) buy?  Times closest_hit on 2^25 C5 secondary rays as generated, and after a Morton sort of the
ray origins at several key widths (sort cost NOT included: this is the upper bound of the gain)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2511_15028_b200 as sb

dev = "cuda:0"
def dbuf(nbytes): return torch.empty(nbytes, dtype=torch.uint8, device=dev)

def spread3(v):  # 10 bits -> every third bit
    v = v & 0x3FF
    v = (v | (v << 16)) & 0x030000FF
    v = (v | (v << 8)) & 0x0300F00F
    v = (v | (v << 4)) & 0x030C30C3
    v = (v | (v << 2)) & 0x09249249
    return v

def time_hit(dt, rays, n, hits, reps=3):
    for _ in range(2): dt.closest_hit(rays.data_ptr(), n, hits.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): dt.closest_hit(rays.data_ptr(), n, hits.data_ptr())
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

if __name__ == "__main__":
    layouts = sys.argv[1].split(",") if len(sys.argv) > 1 else ["pbrt-q16"]
    scene = sb.Scene.terrain(2236, seed=1)
    lt = scene.build_sah(32, 4).collapse8()
    lo, hi = scene.bounds()
    n = 1 << 25
    d_rays = dbuf(n * 32); d_hits = dbuf(n * 8); d_hits2 = dbuf(n * 8)
    for layout in layouts:
        dt = lt.encode(layout).upload(0)
        dt.gen_secondary(77, 0, n, d_rays.data_ptr())
        torch.cuda.synchronize()
        ms0 = time_hit(dt, d_rays, n, d_hits)
        print(f"{layout:12s} unsorted           {ms0:8.2f} ms  {n / ms0 / 1e3:8.1f} Mrays/s", flush=True)
        r = d_rays.view(torch.float32).view(n, 8)
        lo_t = torch.tensor(lo, device=dev); ext = torch.tensor(hi - lo, device=dev).clamp_min(1e-20)
        q = (((r[:, 0:3] - lo_t) / ext).clamp(0, 1) * 1023.0).to(torch.int64)
        morton = (spread3(q[:, 0]) << 2) | (spread3(q[:, 1]) << 1) | spread3(q[:, 2])
        octant = ((r[:, 4] < 0).to(torch.int64) << 2) | ((r[:, 5] < 0).to(torch.int64) << 1) | (r[:, 6] < 0).to(torch.int64)
        for bits, with_oct in ((30, False), (30, True), (24, False), (18, False), (12, False)):
            key = morton >> (30 - bits)
            if with_oct: key = (key << 3) | octant
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); perm = torch.argsort(key); e1.record(); torch.cuda.synchronize()
            sorted_rays = r[perm].contiguous()
            ms = time_hit(dt, sorted_rays.view(torch.uint8).view(-1), n, d_hits2)
            # same answers, permuted
            same = torch.equal(d_hits.view(torch.int64)[perm], d_hits2.view(torch.int64))
            print(f"{layout:12s} morton{bits:2d}{'+oct' if with_oct else '    '}     {ms:8.2f} ms  {n / ms / 1e3:8.1f} Mrays/s  x{ms0 / ms:.2f}  (torch argsort {e0.elapsed_time(e1):.1f} ms, same={same})", flush=True)
            del sorted_rays, perm, key
        dt.free()
