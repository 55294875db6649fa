"""BASELINE-size parity on the GPU ("parity is checked on the full set for C1/C2 and on >= 2^20-query
samples per layout for C3-C5").  Every config runs at its FULL size on the device — C1 2^20 primary rays / 100 K
triangles, C3 2^24 secondary rays / 1 M triangles, C4 2^24 query points / 10 M-point cloud, C5 2^28 mixed rays /
10 M triangles — for EVERY layout the bench sweeps, and the answers are compared bit for bit (primitive id, t / d2 /
closest point) with the CPU oracle: on all queries for C1, on a 2^20-query sample spread evenly over the workload
(64 contiguous chunks) for C3, C4 and C5.  On top of that the size-independent properties the domain offers:
cross-layout invariance on all queries, replay determinism, brute-force agreement, monotonicity in tmax."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SAMPLE = 1 << 20
BINARY = ["pbrt", "pbrt-align16", "pbrt-soa", "pbrt-soaos", "pbrt-soaos-align16", "pbrt-post", "pbrt-q16", "pbrt-q16-soaos", "sg-eq", "sg-eq-align16", "ptr", "identity", "dop14"]
WIDE = ["bvh8", "bvh8-q8", "bvh8-q8-ci", "bvh8-q16", "bvh8-q16-ci", "bvh8-align16", "bvh8-q8-align16", "bvh8-q8-ci-align16", "bvh8-q16-align16", "bvh8-q16-ci-align16"]
EXACT_BOXES = {"pbrt", "pbrt-align16", "pbrt-soa", "pbrt-soaos", "pbrt-soaos-align16", "pbrt-post", "ptr", "identity"}  # f32 boxes of the logical tree, binary visit order


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


def sweep_layouts(sb, extra=()):
    """every layout bench.py sweeps (all registered layouts except shared-slab), corpus + authored"""
    names = [l["name"] for l in sb.layouts() if l["name"] != "shared-slab"]
    return names + [e for e in extra if e not in names]


def spread_index(torch, total, n_sample, chunks=64):
    """indices of `chunks` equal contiguous pieces spread evenly over [0, total) — bench.py's spread_sample"""
    n_sample = min(n_sample, total)
    per = n_sample // chunks
    starts = (torch.arange(chunks, dtype=torch.float64) * (total / chunks)).to(torch.int64)
    return (starts[:, None] + torch.arange(per, dtype=torch.int64)[None, :]).reshape(-1).to("cuda:0")


def run_hits(torch, dt, d_rays, n, d_hits=None):
    if d_hits is None:
        d_hits = torch.empty(n * 8, dtype=torch.uint8, device="cuda:0")
    d_st = torch.ones(n, dtype=torch.int32, device="cuda:0")
    dt.closest_hit(d_rays.data_ptr(), n, d_hits.data_ptr(), d_st.data_ptr())
    torch.cuda.synchronize()
    assert int((d_st != 0).sum()) == 0
    return d_hits


def check_hits_against_oracle(sb, oracle, pt, d_rays, d_hits, idx, what):
    rays = d_rays.view(-1, 32)[idx].cpu().numpy().reshape(-1).view(sb.RAY_DTYPE)
    got = d_hits.view(-1, 8)[idx].cpu().numpy().reshape(-1).view(sb.HIT_DTYPE)
    want, st = oracle.closest_hit(oracle.tree_bytes(pt), rays)
    assert not st.any(), what
    bad = np.nonzero((got["prim"] != want["prim"]) | (got["t"].view(np.uint32) != want["t"].view(np.uint32)))[0]
    assert bad.size == 0, f"{what}: {bad.size} of {len(rays)} sampled queries differ from the oracle, first at sample {bad[:5]}"
    return rays, got


def test_c1_full_parity(built, oracle, torch_cuda):
    """BASELINE configs[0]/[1]: every one of the 1024x1024 primary rays, EVERY layout incl. shared-slab, bit-exact vs the oracle"""
    sb, torch = built, torch_cuda
    import paper_2511_15028_b200.workloads as W
    scene = W.make_scene(W.workload("c1"))
    assert scene.ntris == 100352
    lt = scene.build_sah(32, 4).collapse8()
    lo, hi = scene.bounds()
    wl = W.workload("c1", lo, hi)
    n = wl.total
    assert n == 1 << 20
    d_rays = torch.empty(n * 32, dtype=torch.uint8, device="cuda:0")
    ref = None
    for layout in sweep_layouts(sb, ["shared-slab"]):
        pt = lt.encode(layout)
        dt = pt.upload(0)
        W.generate_device(wl, dt, lo, hi, 0, n, d_rays.data_ptr())
        torch.cuda.synchronize()
        rays = d_rays.cpu().numpy().view(sb.RAY_DTYPE)
        got = run_hits(torch, dt, d_rays, n).cpu().numpy().view(sb.HIT_DTYPE)
        want, st = oracle.closest_hit(oracle.tree_bytes(pt), rays)
        assert not st.any()
        assert np.array_equal(got["prim"], want["prim"]) and np.array_equal(got["t"].view(np.uint32), want["t"].view(np.uint32)), layout
        assert (got["prim"] != sb.MISS_PRIM).mean() > 0.3
        # cross-layout invariant: same logical tree => same answers for every layout
        if ref is None:
            ref = got.copy()
        else:
            assert np.array_equal(got["prim"], ref["prim"]) and np.array_equal(got["t"], ref["t"]), layout
        dt.free()


def test_c3_full_size(built, oracle, torch_cuda):
    """BASELINE configs[2] at full size: 1,002,528 triangles, all 2^24 incoherent secondary rays on the device for every
    swept layout (+ shared-slab on the sample), 2^20-ray spread sample against the oracle per layout."""
    sb, torch = built, torch_cuda
    import paper_2511_15028_b200.workloads as W
    wl = W.workload("c3")
    scene = W.make_scene(wl)
    assert scene.ntris == 1002528
    lt = scene.build_sah(32, 4).collapse8()
    lo, hi = scene.bounds()
    n = wl.total
    assert n == 1 << 24
    d_rays = torch.empty(n * 32, dtype=torch.uint8, device="cuda:0")
    idx = spread_index(torch, n, SAMPLE)
    assert idx.numel() == SAMPLE
    exact = None
    for layout in sweep_layouts(sb):
        pt = lt.encode(layout)
        dt = pt.upload(0)
        W.generate_device(wl, dt, lo, hi, 0, n, d_rays.data_ptr())
        hits = run_hits(torch, dt, d_rays, n)
        rays, got = check_hits_against_oracle(sb, oracle, pt, d_rays, hits, idx, f"c3/{layout}")
        if layout == "pbrt":
            assert torch.equal(hits, run_hits(torch, dt, d_rays, n))  # replay determinism
            exact = hits
            brute = oracle.brute_hit(lt.triangles(), rays[:256])
            assert np.array_equal(got["t"][:256], brute["t"]) and np.array_equal(got["prim"][:256], brute["prim"])
            # monotonicity: shrinking tmax below the hit distance turns the hit into a miss
            r2 = rays[:65536].copy()
            g0 = got[:65536]
            hit = g0["prim"] != sb.MISS_PRIM
            r2["tmax"] = np.where(hit, g0["t"] * 0.5, 1.0).astype(np.float32)
            d2 = torch.from_numpy(r2.view(np.uint8).reshape(-1)).to("cuda:0")
            g2 = run_hits(torch, dt, d2, len(r2)).cpu().numpy().view(sb.HIT_DTYPE)
            w2, _ = oracle.closest_hit(oracle.tree_bytes(pt), r2)
            assert np.array_equal(g2["prim"], w2["prim"]) and np.all(g2["t"][g2["prim"] != sb.MISS_PRIM] <= r2["tmax"][g2["prim"] != sb.MISS_PRIM])
        elif exact is not None:
            same = (hits.view(-1, 8) == exact.view(-1, 8)).all(dim=1).float().mean().item()
            if layout in EXACT_BOXES:
                assert same == 1.0, f"{layout}: differs from pbrt on the same logical tree"
            else:  # conservative boxes / other visit order: equal up to equal-t ties and ulp-level culls — counted, not hidden
                assert same > 0.9999, (layout, same)
        dt.free()
    # shared-slab (one slab per node, ~2600 visits per ray on a terrain): the sample only, still 2^20 rays
    pt = lt.encode("shared-slab")
    dt = pt.upload(0)
    W.generate_device(wl, dt, lo, hi, 0, n, d_rays.data_ptr())
    d_s = d_rays.view(-1, 32)[idx].contiguous().view(-1)
    hs = run_hits(torch, dt, d_s, SAMPLE)
    check_hits_against_oracle(sb, oracle, pt, d_s, hs, torch.arange(SAMPLE, device="cuda:0"), "c3/shared-slab")
    assert torch.equal(hs.view(-1, 8), exact.view(-1, 8)[idx])
    dt.free()


def test_c4_full_size(built, oracle, torch_cuda):
    """BASELINE configs[3] at FULL size: 10,000,000-point cloud (degenerate triangles), all 2^24 query points on the
    device for every binary layout, 2^20-query spread sample against the oracle (d2, closest point, primitive: bit-exact)."""
    sb, torch = built, torch_cuda
    import paper_2511_15028_b200.workloads as W
    wl0 = W.workload("c4")
    scene = W.make_scene(wl0)
    assert scene.ntris == 10_000_000
    lt = scene.build_sah(32, 4)
    lo, hi = scene.bounds()
    wl = W.workload("c4", lo, hi)
    n = wl.total
    assert n == 1 << 24
    d_p = torch.empty(n * 12, dtype=torch.uint8, device="cuda:0")
    idx = spread_index(torch, n, SAMPLE)
    ref = None
    cpq_layouts = [l["name"] for l in sb.layouts() if l["has_cpq"] and l["name"] != "shared-slab"]
    assert set(BINARY) <= set(cpq_layouts)
    for layout in cpq_layouts:
        pt = lt.encode(layout)
        dt = pt.upload(0)
        W.generate_device(wl, dt, lo, hi, 0, n, d_p.data_ptr())
        d_o = torch.empty(n * 20, dtype=torch.uint8, device="cuda:0")
        d_st = torch.ones(n, dtype=torch.int32, device="cuda:0")
        dt.closest_point(d_p.data_ptr(), n, d_o.data_ptr(), d_st.data_ptr())
        torch.cuda.synchronize()
        assert int((d_st != 0).sum()) == 0
        pts = d_p.view(-1, 12)[idx].cpu().numpy().reshape(-1).view(np.float32).reshape(-1, 3)
        got = d_o.view(-1, 20)[idx].cpu().numpy().reshape(-1).view(sb.CP_DTYPE)
        want, st = oracle.closest_point(oracle.tree_bytes(pt), pts)
        assert not st.any()
        bad = np.nonzero((got.view(np.uint32).reshape(-1, 5) != want.view(np.uint32).reshape(-1, 5)).any(axis=1))[0]
        assert bad.size == 0, f"c4/{layout}: {bad.size} of {SAMPLE} sampled queries differ from the oracle, first {bad[:5]}"
        d2 = d_o.view(torch.float32).view(-1, 5)[:, 0]
        if ref is None:
            brute = oracle.brute_point(lt.triangles(), pts[:16])
            assert np.array_equal(got["d2"][:16], brute["d2"])
            ref = d2.clone()
        else:
            assert torch.equal(d2, ref), layout  # d2 is layout-invariant on ALL 2^24 queries (ties may pick other ids)
        dt.free()
        del d_o


def test_c5_full_size(built, oracle, torch_cuda):
    """BASELINE configs[4] = the bench workload at FULL size: 9,999,392 triangles, all 2^28 rays (8 cameras x 4096^2
    primary + 2^27 secondary) on the device for every layout of the bench sweep; 2^20-ray spread sample against the oracle
    per layout; cross-layout agreement on all 2^28 rays; device-encoded image answers identically; replay determinism."""
    sb, torch = built, torch_cuda
    import paper_2511_15028_b200.workloads as W
    scene = W.make_scene(W.workload("c5"))
    assert scene.ntris == 9999392
    lt = scene.build_sah(32, 4).collapse8()
    lo, hi = scene.bounds()
    wl = W.workload("c5", lo, hi)
    n = wl.total
    assert n == 1 << 28
    d_rays = torch.empty(n * 32, dtype=torch.uint8, device="cuda:0")
    hits = torch.empty(n * 8, dtype=torch.uint8, device="cuda:0")
    exact = torch.empty(n * 8, dtype=torch.uint8, device="cuda:0")
    idx = spread_index(torch, n, SAMPLE)
    have_exact = False
    order = ["pbrt"] + [l for l in sweep_layouts(sb) if l != "pbrt"]
    for layout in order:
        pt = lt.encode(layout)
        dt = pt.upload(0)
        if not have_exact:
            W.generate_device(wl, dt, lo, hi, 0, n, d_rays.data_ptr())  # the rays do not depend on the layout
        out = exact if not have_exact else hits
        run_hits(torch, dt, d_rays, n, out)
        rays, got = check_hits_against_oracle(sb, oracle, pt, d_rays, out, idx, f"c5/{layout}")
        assert 0.3 < (got["prim"] != sb.MISS_PRIM).mean() < 1.0
        if not have_exact:
            have_exact = True
            brute = oracle.brute_hit(lt.triangles(), rays[:16])
            assert np.array_equal(got["t"][:16], brute["t"]) and np.array_equal(got["prim"][:16], brute["prim"])
            run_hits(torch, dt, d_rays, n, hits)
            assert torch.equal(hits, exact)  # replay determinism on all 2^28 rays
        else:
            same = (hits.view(torch.int64) == exact.view(torch.int64)).float().mean().item()
            if layout in EXACT_BOXES:
                assert same == 1.0, f"{layout}: differs from pbrt on the same logical tree"
            else:
                assert same > 0.9999, (layout, same)
        if layout == "pbrt-q16":  # device-side encode of the same tree answers identically on every ray
            mine = hits.clone()
            dev = lt.encode_device(layout, 0)
            run_hits(torch, dev, d_rays, n, hits)
            assert torch.equal(hits, mine)
            dev.free()
            del mine
        dt.free()
