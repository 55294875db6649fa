"""Appendix F fidelity (SPEC acceptance criterion 9): the Moeller-Trumbore test every traversal uses
(geometry.scion:25-38) against the Pluecker-coordinate test (geometry.scion:40-55) on random (ray, triangle)
pairs — hit/miss identical, t within 1e-5 relative — and the device implementations of both against the
oracle, bit for bit."""
import numpy as np
import pytest

RAY_F = 8


def random_pairs(sb, n, seed):
    """rays aimed at a random point of a random triangle (hits) or well past it (misses); nothing grazing"""
    rng = np.random.default_rng(seed)
    tris = rng.uniform(-1.0, 1.0, (n, 9)).astype(np.float32)
    w = rng.uniform(0.12, 0.76, (n, 3)).astype(np.float32)
    w /= w.sum(axis=1, keepdims=True)
    inside = (tris.reshape(n, 3, 3) * w[:, :, None]).sum(axis=1)
    c = tris.reshape(n, 3, 3).mean(axis=1)
    miss = rng.random(n) < 0.5
    target = np.where(miss[:, None], c + 3.0 * (inside - c) + rng.uniform(0.5, 1.0, (n, 3)) * np.sign(inside - c), inside).astype(np.float32)
    # approach from within ~55 degrees of the triangle normal: no grazing incidence (where the two tests'
    # rounding errors in t grow like 1 / cos and the 1e-5 contract of the SPEC is not meant to hold)
    t3 = tris.reshape(n, 3, 3).astype(np.float64)
    nrm = np.cross(t3[:, 1] - t3[:, 0], t3[:, 2] - t3[:, 0])
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    side = np.where(rng.random(n) < 0.5, 1.0, -1.0)[:, None]
    off = nrm * side + 0.7 * rng.uniform(-1.0, 1.0, (n, 3))
    off /= np.linalg.norm(off, axis=1, keepdims=True)
    origin = (target + rng.uniform(1.5, 3.0, (n, 1)) * off).astype(np.float32)
    d = target - origin
    d = (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)
    rays = np.zeros(n, sb.RAY_DTYPE)
    rays["ox"], rays["oy"], rays["oz"] = origin.T
    rays["dx"], rays["dy"], rays["dz"] = d.T
    rays["tmax"] = np.inf
    return rays, tris


def test_mt_and_pluecker_agree_on_random_pairs(built, oracle):
    sb = built
    rays, tris = random_pairs(sb, 10_000, 11)
    mt, pc = oracle.ray_tri_batch(rays, tris, 0), oracle.ray_tri_batch(rays, tris, 1)
    hit_mt, hit_pc = mt[:, 4].view(np.uint32) != 0, pc[:, 4].view(np.uint32) != 0
    assert 3000 < hit_mt.sum() < 7000
    assert np.array_equal(hit_mt, hit_pc)
    rel = np.abs(mt[hit_mt, 3] - pc[hit_mt, 3]) / np.abs(mt[hit_mt, 3])
    assert rel.max() < 1e-5
    # barycentrics describe the same point
    assert np.abs(mt[hit_mt, :3] - pc[hit_mt, :3]).max() < 1e-3
    # KAT of SPEC.md:455 through both tests: t = 1, b = (0.5, 0.25, 0.25)
    r = np.zeros(1, sb.RAY_DTYPE)
    r["ox"], r["oy"], r["oz"], r["dz"], r["tmax"] = 0.25, 0.25, -1.0, 1.0, np.inf
    tri = np.array([[0, 0, 0, 1, 0, 0, 0, 1, 0]], np.float32)
    for m in (0, 1):
        out = oracle.ray_tri_batch(r, tri, m)[0]
        assert out[4:].view(np.uint32)[0] == 1 and np.allclose(out[:4], [0.5, 0.25, 0.25, 1.0])


@pytest.mark.gpu
def test_device_triangle_tests_match_the_oracle(built, oracle):
    import torch
    sb = built
    rays, tris = random_pairs(sb, 20_000, 5)
    # plus degenerate inputs: zero-area triangle, ray in the triangle's plane, zero direction component, finite tmax
    rays[:4]["dx"], rays[:4]["dy"], rays[:4]["dz"] = 0.0, 0.0, 1.0
    tris[0] = tris[0, :3].repeat(3).reshape(3, 3).T.reshape(-1)
    rays[4:8]["tmax"] = 0.5
    d_rays = torch.from_numpy(rays.view(np.uint8).reshape(-1).copy()).cuda()
    d_tris = torch.from_numpy(tris.reshape(-1).copy()).cuda()
    n = len(rays)
    for method in (sb.TRI_MT, sb.TRI_PLUECKER):
        d_out = torch.empty(n * 20, dtype=torch.uint8, device="cuda:0")
        sb.ray_triangle(d_rays.data_ptr(), d_tris.data_ptr(), n, method, d_out.data_ptr())
        torch.cuda.synchronize()
        got = d_out.cpu().numpy().view(np.uint32).reshape(n, 5)
        want = oracle.ray_tri_batch(rays, tris, method).view(np.uint32)
        assert np.array_equal(got, want), method
    with pytest.raises(sb.ScionError):
        sb.ray_triangle(d_rays.data_ptr(), d_tris.data_ptr(), n, 7, d_out.data_ptr())
