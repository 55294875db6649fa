"""Device-side build_physical: the per-node encoders
of csrc/host/encode_node.hpp run as CUDA threads.  Contract: the device image is BYTE-identical to the host
encoder's (which tests/test_scene_encode.py pins against the reference planner and the oracle decoders)."""
import numpy as np
import pytest

ALL = ["identity", "ptr", "pbrt", "pbrt-align16", "pbrt-soa", "pbrt-post", "pbrt-q16", "sg-eq", "sg-eq-align16", "shared-slab", "dop14",
       "bvh8", "bvh8-q8", "bvh8-q8-ci", "bvh8-q16", "bvh8-q16-ci", "pbrt-soaos", "pbrt-soaos-align16", "pbrt-q16-soaos", "bvh8-align16", "bvh8-q8-align16",
       "bvh8-q8-ci-align16", "bvh8-q16-align16", "bvh8-q16-ci-align16"]


def test_device_encode_fails_loudly_without_a_device(built):
    sb = built
    if sb.device_count() > 0:
        pytest.skip("a CUDA device is present")
    lt = sb.Scene.terrain(4, 1).build_sah(32, 4)
    with pytest.raises(sb.ScionError) as e:
        lt.encode_device("pbrt-q16", 0)
    assert e.value.code == sb.ERR_NO_DEVICE


def test_device_encode_reports_builder_faults(built):
    sb = built
    lt = sb.Scene.terrain(4, 1).build_sah(32, 4)  # not collapsed
    with pytest.raises(sb.ScionError):
        lt.encode_device("bvh8-q8-ci", 0)
    with pytest.raises(sb.ScionError):
        lt.encode_device("no-such-layout", 0)


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ALL)
def test_device_image_equals_host_image(built, layout):
    sb = built
    for scene, builder in ((sb.Scene.terrain(20, 5), "sah"), (sb.Scene.sphere(12, 2), "median"), (sb.Scene.terrain(1, 1), "sah")):
        lt = scene.build_sah(32, 4) if builder == "sah" else scene.build_median(2)
        lt = lt.collapse8()
        host = lt.encode(layout).upload(0)
        dev = lt.encode_device(layout, 0)
        a, b = host.download_image(), dev.download_image()
        assert a.shape == b.shape and a.shape[0] == host.image()[1]
        diff = np.flatnonzero(a != b)
        assert diff.size == 0, (layout, builder, diff[:8], a[diff[:8]], b[diff[:8]])
        host.free()
        dev.free()


@pytest.mark.gpu
def test_device_encoded_tree_answers_like_the_oracle(built, oracle):
    import torch
    sb = built
    scene = sb.Scene.terrain(24, 7)
    lt = scene.build_sah(32, 4).collapse8()
    lo, hi = scene.bounds()
    cam = sb.default_camera(lo, hi, True, 48, 48)
    n = 48 * 48
    rays = sb.gen_primary_host(cam, 0, n)
    d_rays = torch.from_numpy(rays.view(np.uint8).reshape(-1)).cuda()
    for layout in ("pbrt-q16", "sg-eq", "bvh8-q8-ci", "dop14"):
        dt = lt.encode_device(layout, 0)
        hits = torch.empty(n * 8, dtype=torch.uint8, device="cuda:0")
        dt.closest_hit(d_rays.data_ptr(), n, hits.data_ptr())
        torch.cuda.synchronize()
        got = hits.cpu().numpy().view(sb.HIT_DTYPE)
        want, _ = oracle.closest_hit(oracle.tree_bytes(lt.encode(layout)), rays)
        assert np.array_equal(got["prim"], want["prim"]) and np.array_equal(got["t"].view(np.uint32), want["t"].view(np.uint32)), layout
        dt.free()


@pytest.mark.gpu
def test_device_encode_full_size_c5(built):
    """BASELINE config 5 scale (10 M triangles): image equality for the headline layout + timing of both paths."""
    import time
    sb = built
    lt = sb.Scene.terrain(2236, 1).build_sah(32, 4)
    t0 = time.perf_counter(); host = lt.encode("pbrt-q16").upload(0); t1 = time.perf_counter()
    dev = lt.encode_device("pbrt-q16", 0); t2 = time.perf_counter()
    a, b = host.download_image(), dev.download_image()
    assert np.array_equal(a, b)
    print(f"host encode+upload {t1 - t0:.2f} s, device encode (incl. upload of the logical tree) {t2 - t1:.2f} s")
    host.free(); dev.free()
