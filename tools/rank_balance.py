"""How evenly does the contiguous partition split the C5 workload?  Times the slice of every rank of a
world of 2, 4 and 8 on ONE GPU (the ranks of a real run do exactly this work, in parallel)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_15028_b200 as sb
import paper_2511_15028_b200.workloads as W

layout = sys.argv[1] if len(sys.argv) > 1 else "pbrt-q16"
wl0 = W.workload("c5")
scene = W.make_scene(wl0)
lt = scene.build_sah(32, 4).collapse8()
lo, hi = scene.bounds()
wl = W.workload("c5", lo, hi)
dt = lt.encode_device(layout, 0)
for world in (1, 2, 4, 8):
    ms = []
    for r in range(world):
        first, count = sb.partition(wl.total, r, world)
        d_q = torch.empty(count * 32, dtype=torch.uint8, device="cuda:0")
        d_r = torch.empty(count * 8, dtype=torch.uint8, device="cuda:0")
        W.generate_device(wl, dt, lo, hi, first, count, d_q.data_ptr())
        for _ in range(2): dt.closest_hit(d_q.data_ptr(), count, d_r.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): dt.closest_hit(d_q.data_ptr(), count, d_r.data_ptr())
        e1.record(); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1) / 3)
        del d_q, d_r
    print(f"world {world}: per-rank ms {[round(m, 2) for m in ms]}  max {max(ms):.2f}  -> {wl.total / max(ms) / 1e3:.0f} Mrays/s whole job, efficiency vs 1 GPU {ms0 / (world * max(ms)) if world > 1 else 1.0:.3f}" if world > 1 or not globals().update(ms0=ms[0]) else "")
