"""Multi-GPU path: C-ABI communicator, tree replication by one ncclBroadcast of the
packed image, contiguous query partition, gather of result records by query index; bench.py --gpus N starts N ranks.
Only one GPU is ever available to the test boxes, so the NCCL calls are exercised over one-rank communicators
(every collective still goes through libnccl) and the N > 1 tests skip unless the node has the GPUs."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus_n_without_the_gpus_fails_loudly(built):
    """`bench.py --gpus 8` must never silently run one rank."""
    import torch
    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(have + 7), "--steps", "1", "--warmup", "1"], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode != 0
    assert "one process per GPU" in (r.stderr + r.stdout)
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]  # no bench line at all


def test_comm_api_without_device_or_nccl_reports(built):
    sb = built
    if sb.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(sb.ScionError):
        sb.Comm.init_all(1)


@pytest.mark.gpu
def test_one_rank_communicator_replicates_and_gathers(built):
    import torch
    sb = built
    assert sb.nccl_version() >= 22000
    scene = sb.Scene.terrain(40, 3)
    lt = scene.build_sah(32, 4).collapse8()
    n = 10007  # ragged on purpose
    for layout in ("pbrt-q16", "bvh8-q8-ci"):
        dt = lt.encode(layout).upload(0)
        comm = sb.Comm.init_rank(sb.Comm.unique_id(), 1, 0, 0)
        assert (comm.rank, comm.size, comm.device) == (0, 1, 0)
        assert comm.broadcast_tree(dt, 0) is dt  # the root keeps its own tree; two ncclBroadcasts ran
        d_rays = torch.empty(n * 32, dtype=torch.uint8, device="cuda:0")
        dt.gen_secondary(5, 0, n, d_rays.data_ptr())
        d_hits = torch.empty(n * 8, dtype=torch.uint8, device="cuda:0")
        dt.closest_hit(d_rays.data_ptr(), n, d_hits.data_ptr())
        full = torch.zeros(n * 8, dtype=torch.uint8, device="cuda:0")
        comm.gather(d_hits.data_ptr(), n, 8, full.data_ptr())
        torch.cuda.synchronize()
        assert torch.equal(full, d_hits)
        comm.gather(full.data_ptr(), n, 8, full.data_ptr())  # in place
        torch.cuda.synchronize()
        assert torch.equal(full, d_hits)
        comm.free()
        # single-process form over ncclCommInitAll
        comms = sb.Comm.init_all(1)
        trees = sb.broadcast_tree_all(dt, 0, comms)
        assert trees[0] is dt
        full.zero_()
        sb.gather_results_all(comms, [d_hits.data_ptr()], n, 8, [full.data_ptr()])
        torch.cuda.synchronize()
        assert torch.equal(full, d_hits)
        for c in comms:
            c.free()
        dt.free()


@pytest.mark.gpu
def test_broadcast_rejects_misuse(built):
    sb = built
    comm = sb.Comm.init_rank(sb.Comm.unique_id(), 1, 0, 0)
    with pytest.raises(sb.ScionError):  # the root must pass its tree
        comm.broadcast_tree(None, 0)
    with pytest.raises(sb.ScionError):
        sb.Comm.init_all(64)
    comm.free()


def _bench(args, env_extra=None, timeout=1500):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True, env=env, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert lines and lines[-1].startswith("{"), "the JSON line must be the LAST line of stdout:\n" + r.stdout[-2000:] + "\n--- stderr ---\n" + r.stderr[-2000:]
    return json.loads(lines[-1]), r


@pytest.mark.gpu
def test_bench_nccl_path_on_one_rank(built):
    """SCION_FORCE_DIST=1: the whole multi-rank code path of bench.py (unique id, communicator, scion_dtree_broadcast,
    scion_gather_results, barriers) with world size 1."""
    line, r = _bench(["--workload", "c3", "--scale", "0.0625", "--steps", "2", "--warmup", "3", "--sweep", "bvh8-q8-ci", "--no-cpu", "--no-e2e"], {"SCION_FORCE_DIST": "1"})
    assert line["n_gpus"] == 1 and line["gather"]["identical_on_all_ranks"] and line["gather"]["bytes"] == (1 << 20) * 8
    assert line["gpu_launches"] == 2 and set(line["layouts"]) == {"pbrt-q16", "bvh8-q8-ci"}
    assert "NCCL INFO" in r.stdout + r.stderr  # communicator log lines stay on


@pytest.mark.gpu
def test_bench_two_ranks(built):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    line, _ = _bench(["--gpus", "2", "--workload", "c3", "--scale", "0.0625", "--steps", "2", "--warmup", "3", "--sweep", "", "--no-cpu"])
    assert line["n_gpus"] == 2 and line["gather"]["identical_on_all_ranks"]
    one, _ = _bench(["--gpus", "1", "--workload", "c3", "--scale", "0.0625", "--steps", "2", "--warmup", "3", "--sweep", "", "--no-cpu"])
    assert one["n_gpus"] == 1 and one["config"]["queries"] == line["config"]["queries"]


@pytest.mark.gpu
def test_native_harness_multi_gpu_path(built):
    """scion_run bench --gpus G: ncclCommInitAll + broadcast_all + gather_all; on a 1-GPU box the same code runs over a
    one-device communicator (SCION_RUN_FORCE_MULTI), on a multi-GPU box over 2 devices."""
    import torch
    exe = os.path.join(ROOT, "paper_2511_15028_b200", "bin", "scion_run")
    g = 2 if torch.cuda.device_count() >= 2 else 1
    env = dict(os.environ, SCION_RUN_FORCE_MULTI="1")
    r = subprocess.run([exe, "bench", "pbrt-q16", "terrain:96", "200003", "secondary", "--gpus", str(g)], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr + r.stdout
    head, row = [l.split(",") for l in r.stdout.strip().splitlines()[-2:]]
    rec = dict(zip(head, row))
    assert int(rec["n_gpus"]) == g and int(rec["gather_mismatches"]) == 0 and float(rec["mqueries_per_s"]) > 1.0
    r = subprocess.run([exe, "bench", "pbrt-q16", "terrain:96", "1000", "secondary", "--gpus", "64"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 2 and "exposes" in r.stderr
