"""Synthetic workloads of BASELINE.json (`configs[0..4]`) and the multi-GPU query partitioner.

Every query is a pure function of (seed, global query index) (host/rng.hpp), so a rank that owns
the contiguous slice [first, first+count) of the global index space generates exactly the
queries a single GPU would have generated for those indices — no scatter is needed; the encoded
tree is replicated (one ncclBroadcast of the packed device image) and hit records are gathered
back.  Stands in for the harness QueryConfig of the reference.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

import paper_2511_15028_b200 as sb


@dataclass
class Segment:
    kind: str          # "primary" | "secondary" | "points"
    count: int
    camera: object = None   # sb.Camera for primary
    seed: int = 0
    offset: int = 0    # first index of this segment inside its generator stream (a stream may be cut into several segments)


@dataclass
class Workload:
    name: str
    scene: str              # "terrain" | "sphere" | "cloud"
    scene_arg: int
    scene_seed: int
    algorithm: str          # "chrt" | "cpq"
    segments: List[Segment] = field(default_factory=list)
    description: str = ""

    @property
    def total(self) -> int:
        return sum(s.count for s in self.segments)


def make_scene(w: Workload) -> "sb.Scene":
    if w.scene == "terrain":
        return sb.Scene.terrain(w.scene_arg, w.scene_seed)
    if w.scene == "sphere":
        return sb.Scene.sphere(w.scene_arg, w.scene_seed)
    if w.scene == "cloud":
        return sb.Scene.cloud(w.scene_arg, w.scene_seed)
    raise ValueError(w.scene)


def orbit_camera(lo, hi, k: int, ncams: int, width: int, height: int) -> "sb.Camera":
    """Camera k of an orbit of `ncams` positions around (and above) the scene bounds."""
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    c = 0.5 * (lo + hi)
    diag = float(np.linalg.norm(hi - lo))
    a = 2.0 * math.pi * k / max(ncams, 1)
    cam = sb.Camera()
    eye = (c[0] + 0.75 * diag * math.cos(a), hi[1] + (0.45 + 0.05 * (k % 3)) * diag, c[2] + 0.75 * diag * math.sin(a))
    for i in range(3):
        cam.eye[i] = eye[i]
        cam.target[i] = c[i]
        cam.up[i] = (0.0, 1.0, 0.0)[i]
    cam.fov_y_deg = 40.0
    cam.width, cam.height = width, height
    return cam


def workload(name: str, lo=None, hi=None, scale: float = 1.0) -> Workload:
    """BASELINE.json configs. `lo`/`hi` = scene bounds (needed for cameras/points); `scale` < 1
    shrinks query counts (tests)."""
    seed = sb.seed_from_env(0x5C10)

    def cnt(n):
        return max(1, int(n * scale))

    if name in ("c1", "c2"):  # 1024x1024 coherent primary rays, ~100K-triangle terrain
        w = Workload(name, "terrain", 224, 1, "chrt", description="100352-triangle terrain, 1024x1024 pinhole primary rays")
        if lo is not None:
            side = max(1, int(round(1024 * math.sqrt(scale))))
            w.segments = [Segment("primary", side * side, sb.default_camera(lo, hi, True, side, side))]
        return w
    if name == "c3":  # 16M incoherent secondary rays, 1M-triangle terrain
        w = Workload(name, "terrain", 708, 1, "chrt", description="1002528-triangle terrain, 2^24 incoherent secondary rays")
        w.segments = [Segment("secondary", cnt(1 << 24), seed=seed + 3)]
        return w
    if name == "c4":  # 16M closest-point queries, 10M-point cloud
        w = Workload(name, "cloud", 10_000_000, 1, "cpq", description="10M-point cloud (degenerate triangles), 2^24 uniform query points")
        w.segments = [Segment("points", cnt(1 << 24), seed=seed + 4)]
        return w
    if name == "c5":  # 256M primary + secondary rays, 10M-triangle terrain
        w = Workload(name, "terrain", 2236, 1, "chrt", description="9999392-triangle terrain, 2^28 rays = 8 orbit cameras x 4096^2 primary + 2^27 secondary, interleaved in 128 strips")
        if lo is not None:
            side = max(1, int(round(4096 * math.sqrt(scale))))
            # Order of the global index space: 8 rounds; round j holds one eighth (a strip of rows) of every camera's
            # image — strip (j + k) mod 8 of camera k, because the top and the bottom of an image cost very different
            # amounts — each followed by one piece of the secondary stream.  Any contiguous 1/2, 1/4 or 1/8
            # of the index space — the range of one rank — then holds the same mix of cheap coherent and expensive
            # incoherent rays and of all eight viewpoints ("the only risk is cost imbalance of
            # contiguous primary-ray ranges").  The SET of rays does not depend on the order.
            img = side * side
            strip = max(1, img // 8)
            rounds = 8 if img % 8 == 0 else 1
            for j in range(rounds):
                for k in range(8):
                    cnt_p = strip if rounds == 8 else img
                    w.segments.append(Segment("primary", cnt_p, orbit_camera(lo, hi, k, 8, side, side), offset=((j + k) % 8) * strip if rounds == 8 else 0))
                    w.segments.append(Segment("secondary", cnt_p, seed=seed + 5, offset=(j * 8 + k) * cnt_p))
        return w
    raise ValueError(f"unknown workload {name}")


def slices(w: Workload, first: int, count: int) -> List[Tuple[Segment, int, int, int]]:
    """Decompose the global query range [first, first+count) into per-segment pieces:
    (segment, local_first, local_count, offset_in_output)."""
    out = []
    base = 0
    end = first + count
    for seg in w.segments:
        a, b = max(first, base), min(end, base + seg.count)
        if a < b:
            out.append((seg, a - base + seg.offset, b - a, a - first))
        base += seg.count
    return out


def generate_device(w: Workload, dtree: "sb.DeviceTree", lo, hi, first: int, count: int, d_ptr: int, stream: int = 0):
    """Fill device memory at d_ptr with queries [first, first+count) (rays: 32 B each; points: 12 B)."""
    for seg, lf, lc, off in slices(w, first, count):
        if seg.kind == "primary":
            sb.gen_primary(seg.camera, lf, lc, d_ptr + off * 32, stream)
        elif seg.kind == "secondary":
            dtree.gen_secondary(seg.seed, lf, lc, d_ptr + off * 32, stream)
        else:
            sb.gen_points(lo, hi, seg.seed, lf, lc, d_ptr + off * 12, stream)


def generate_host(w: Workload, tris: np.ndarray, lo, hi, first: int, count: int) -> np.ndarray:
    """Host twin of generate_device (bit-identical queries)."""
    parts = []
    for seg, lf, lc, off in slices(w, first, count):
        if seg.kind == "primary":
            parts.append(sb.gen_primary_host(seg.camera, lf, lc))
        elif seg.kind == "secondary":
            parts.append(sb.gen_secondary_host(tris, seg.seed, lf, lc))
        else:
            parts.append(sb.gen_points_host(lo, hi, seg.seed, lf, lc))
    if not parts:
        return np.zeros(0, sb.RAY_DTYPE if w.algorithm == "chrt" else np.float32)
    return np.concatenate(parts)


def sample_indices(w: Workload, n_sample: int) -> List[Tuple[int, int]]:
    """A bounded, representative sample of the workload: equal contiguous prefixes of every segment
    (global (first, count) ranges)."""
    per = max(1, n_sample // max(1, len(w.segments)))
    out, base = [], 0
    for seg in w.segments:
        out.append((base, min(per, seg.count)))
        base += seg.count
    return out


def algorithmic_bytes(layout_info: dict, plan: dict, counters: np.ndarray, algorithm: str) -> float:
    """Mean ALGORITHMIC bytes per query: node decodes x node bytes (hot segment) +
    cold-segment reads x cold bytes + 36 x primitive tests + query read + result write."""
    nb = [b for b in plan["buffers"] if b["name"] == plan["node_group"]][0]
    seg = [s["stride_bytes"] for s in nb["segments"]]
    hot = seg[0] if seg else 0
    cold = sum(seg[1:]) if len(seg) > 1 else 0
    q_in, q_out = (32, 8) if algorithm == "chrt" else (12, 20)
    c = counters
    return float(c["node_visits"].mean() * hot + c["cold_loads"].mean() * cold + c["prim_tests"].mean() * 36 + q_in + q_out)
