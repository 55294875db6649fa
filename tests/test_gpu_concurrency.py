"""Concurrent queries on one shared immutable tree (include/scion_b200.h: "concurrent launches on
different streams are legal").  Every launch owns its work-fetch counter until the event recorded behind it has
completed (abi.cu CounterPool): many more launches in flight than the pool's first block must still answer exactly
like a single-stream run."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("layout,alg", [("pbrt-q16", "chrt"), ("bvh8-q8-ci", "chrt"), ("pbrt", "cpq")])
def test_many_launches_over_many_streams(built, layout, alg):
    import torch
    sb = built
    scene = sb.Scene.terrain(64, 5)
    lt = scene.build_sah(32, 4).collapse8()
    dt = lt.encode(layout).upload(0)
    lo, hi = scene.bounds()
    n_launch, per = 320, 4096 + 37  # 5x the first counter block, ragged size
    n = n_launch * per
    if alg == "chrt":
        q_sz, r_sz = 32, 8
        d_q = torch.empty(n * q_sz, dtype=torch.uint8, device="cuda:0")
        dt.gen_secondary(17, 0, n, d_q.data_ptr())
        call = dt.closest_hit
    else:
        q_sz, r_sz = 12, 20
        d_q = torch.empty(n * q_sz, dtype=torch.uint8, device="cuda:0")
        sb.gen_points(lo - 0.2, hi + 0.2, 23, 0, n, d_q.data_ptr())
        call = dt.closest_point
    torch.cuda.synchronize()
    want = torch.empty(n * r_sz, dtype=torch.uint8, device="cuda:0")
    call(d_q.data_ptr(), n, want.data_ptr())
    torch.cuda.synchronize()

    streams = [torch.cuda.Stream() for _ in range(8)]
    got = torch.zeros(n * r_sz, dtype=torch.uint8, device="cuda:0")
    st = torch.ones(n, dtype=torch.int32, device="cuda:0")
    torch.cuda.synchronize()
    for i in range(n_launch):  # nothing synchronises between launches: hundreds are in flight at once
        s = streams[i % len(streams)].cuda_stream
        call(d_q.data_ptr() + i * per * q_sz, per, got.data_ptr() + i * per * r_sz, st.data_ptr() + i * per * 4, 0, 0, s)
    torch.cuda.synchronize()
    assert int((st != 0).sum()) == 0
    assert torch.equal(got, want), f"{layout}/{alg}: concurrent launches differ from the single-stream answer"

    # the same from several host threads at once (the pool is shared by every caller of the tree)
    got2 = torch.zeros(n * r_sz, dtype=torch.uint8, device="cuda:0")
    errs = []

    def worker(k):
        try:
            torch.cuda.set_device(0)
            for i in range(k, n_launch, 4):
                call(d_q.data_ptr() + i * per * q_sz, per, got2.data_ptr() + i * per * r_sz, 0, 0, 0, streams[(i + k) % len(streams)].cuda_stream)
        except Exception as ex:  # pragma: no cover
            errs.append(ex)

    th = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    [t.start() for t in th]
    [t.join() for t in th]
    torch.cuda.synchronize()
    assert not errs, errs
    assert torch.equal(got2, want)
    dt.free()
