"""Multi-GPU host logic on the CPU: the contiguous query partitioner, per-rank generation ==
slices of the global generation (every query is a pure function of (seed, global index)), and the
replicate / gather protocol of bench.py exercised with two gloo processes."""
import os
import socket

import numpy as np
import pytest


def test_slices_and_per_rank_generation(built):
    import paper_2511_15028_b200.workloads as W
    scene = built.Scene.terrain(10, 1)
    lt = scene.build_sah(32, 4)
    lo, hi = scene.bounds()
    wl = W.workload("c5", lo, hi, scale=2.0 ** -16)  # 8 cameras x 16x16 primary + 2048 secondary, interleaved in 8 rounds
    assert wl.total == 8 * 256 + 2048 and len(wl.segments) == 128
    # the secondary segments are consecutive pieces of ONE stream (same seed): together they are its first 2048 rays
    sec = [s for s in wl.segments if s.kind == "secondary"]
    assert [s.offset for s in sec] == [i * 32 for i in range(64)] and len({s.seed for s in sec}) == 1
    # every camera's image is covered exactly once
    for k in range(8):
        strips = sorted((s.offset, s.count) for s in wl.segments if s.kind == "primary")[k::8]
    prim = {}
    for s in wl.segments:
        if s.kind == "primary":
            prim.setdefault(tuple(s.camera.eye), []).append((s.offset, s.count))
    assert len(prim) == 8 and all(sorted(v) == [(j * 32, 32) for j in range(8)] for v in prim.values())
    # every eighth of the index space holds the same mix: what makes contiguous rank ranges balanced
    for r in range(8):
        first, count = built.partition(wl.total, r, 8)
        kinds = sorted((seg.kind, c) for seg, _, c, _ in W.slices(wl, first, count))
        assert kinds == [("primary", 32)] * 8 + [("secondary", 32)] * 8
    full = W.generate_host(wl, lt.triangles(), lo, hi, 0, wl.total)
    assert full.shape[0] == wl.total
    for world in (1, 2, 3, 8):
        parts = []
        for r in range(world):
            first, count = built.partition(wl.total, r, world)
            covered = sum(c for _, _, c, _ in W.slices(wl, first, count))
            assert covered == count
            parts.append(W.generate_host(wl, lt.triangles(), lo, hi, first, count))
        got = np.concatenate(parts)
        assert np.array_equal(got.view(np.uint32), full.view(np.uint32)), f"world={world}"
    # determinism + seed override (LAYOUTC_SEED)
    again = W.generate_host(wl, lt.triangles(), lo, hi, 0, wl.total)
    assert np.array_equal(again.view(np.uint32), full.view(np.uint32))
    os.environ["LAYOUTC_SEED"] = "12345"
    try:
        wl2 = W.workload("c5", lo, hi, scale=2.0 ** -16)
        other = W.generate_host(wl2, lt.triangles(), lo, hi, 0, wl2.total)
        assert not np.array_equal(other.view(np.uint32).reshape(-1, 8)[32:64], full.view(np.uint32).reshape(-1, 8)[32:64])  # first secondary piece
    finally:
        del os.environ["LAYOUTC_SEED"]


def test_workload_shapes(built):
    import paper_2511_15028_b200.workloads as W
    assert W.workload("c3").total == 1 << 24 and W.workload("c4").total == 1 << 24 and W.workload("c4").algorithm == "cpq"
    lo, hi = np.zeros(3, np.float32), np.ones(3, np.float32)
    assert W.workload("c1", lo, hi).total == 1 << 20
    assert W.workload("c5", lo, hi).total == 1 << 28
    assert W.workload("c5").scene_arg == 2236 and 2 * 2236 * 2236 == 9_999_392
    rays = built.gen_secondary_host(built.Scene.terrain(6, 2).triangles(), 5, 0, 2000)
    d = np.stack([rays["dx"], rays["dy"], rays["dz"]], 1)
    assert np.allclose(np.linalg.norm(d, axis=1), 1.0, atol=1e-5) and np.isinf(rays["tmax"]).all()


def _worker(rank, world, port, q):
    """replicate (broadcast of the packed image) + partitioned work + gather, over gloo on CPU tensors"""
    import torch
    import torch.distributed as dist
    import paper_2511_15028_b200 as sb
    import paper_2511_15028_b200.workloads as W
    from tests.oracle_lib import Oracle
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        bounds = torch.zeros(6, dtype=torch.float64)
        image = None
        if rank == 0:
            scene = sb.Scene.terrain(10, 1)
            lt = scene.build_sah(32, 4)
            lo, hi = scene.bounds()
            bounds = torch.tensor(list(lo) + list(hi), dtype=torch.float64)
            pt = lt.encode("pbrt-q16")
            # host stand-in for the device image: the raw buffers, concatenated
            bufs = pt.buffers()
            image = torch.from_numpy(np.concatenate([b["data"] for b in bufs]).copy())
            sizes = torch.tensor([len(b["data"]) for b in bufs] + [0] * (6 - len(bufs)), dtype=torch.int64)
        else:
            sizes = torch.zeros(6, dtype=torch.int64)
        dist.broadcast(bounds, 0)
        dist.broadcast(sizes, 0)
        if rank != 0:
            image = torch.empty(int(sizes.sum()), dtype=torch.uint8)
        dist.broadcast(image, 0)  # one message replicates the tree
        lo, hi = bounds[:3].numpy().astype(np.float32), bounds[3:].numpy().astype(np.float32)
        wl = W.workload("c5", lo, hi, scale=2.0 ** -16)
        first, count = sb.partition(wl.total, rank, world)
        prim_bytes = int(sizes[0])
        tris = image[:prim_bytes].numpy().view(np.float32).reshape(-1, 9)
        rays = W.generate_host(wl, tris, lo, hi, first, count)
        # "traverse": a per-rank checksum stands in for the kernel; the gather reassembles global order
        local = torch.from_numpy(rays.view(np.uint32).reshape(-1, 8).sum(axis=1).astype(np.int64))
        outs = [torch.empty(sb.partition(wl.total, r, world)[1], dtype=torch.int64) for r in range(world)]
        dist.all_gather(outs, local)
        full = torch.cat(outs)
        q.put((rank, int(full.sum()), int(image.to(torch.int64).sum()), full.shape[0]))
    finally:
        dist.destroy_process_group()


def test_two_rank_replicate_partition_gather(built):
    import torch.multiprocessing as mp
    import paper_2511_15028_b200.workloads as W
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # both ranks hold the same replicated image and the same gathered result, equal to the 1-rank answer
    assert res[0][1:] == res[1][1:]
    scene = built.Scene.terrain(10, 1)
    lt = scene.build_sah(32, 4)
    lo, hi = scene.bounds()
    wl = W.workload("c5", lo, hi, scale=2.0 ** -16)
    full = W.generate_host(wl, lt.triangles(), lo, hi, 0, wl.total)
    assert res[0][1] == int(full.view(np.uint32).reshape(-1, 8).sum(axis=1).astype(np.int64).sum()) and res[0][3] == wl.total
