"""Parity tests proper: the CUDA path, called through the C ABI, against the CPU oracle on the
same seeded inputs.  Bar (BASELINE.json north_star): hit primitive ids bit-exact with identical
tie-breaking; t within 1e-6 relative — we require and observe BIT-EXACT t (and d2 / closest point
for CPQ), plus identical interpreter counters (node visits, primitive tests), which only holds if
the visit order is the reference's."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def dev_bytes(torch, arr):
    return torch.from_numpy(np.ascontiguousarray(arr).view(np.uint8).reshape(-1)).to("cuda:0")


def gpu_hits(torch, sb, dt, rays, counters=True):
    n = rays.shape[0]
    d_rays = dev_bytes(torch, rays) if n else torch.empty(0, dtype=torch.uint8, device="cuda:0")
    d_hits = torch.zeros(max(n, 1) * 8, dtype=torch.uint8, device="cuda:0")
    d_st = torch.zeros(max(n, 1) * 4, dtype=torch.uint8, device="cuda:0")
    d_ctr = torch.zeros(max(n, 1) * 16, dtype=torch.uint8, device="cuda:0")
    dt.closest_hit(d_rays.data_ptr(), n, d_hits.data_ptr(), d_st.data_ptr(), d_ctr.data_ptr() if counters else 0)
    torch.cuda.synchronize()
    return (d_hits.cpu().numpy().view(sb.HIT_DTYPE)[:n], d_st.cpu().numpy().view(np.uint32)[:n], d_ctr.cpu().numpy().view(sb.COUNTERS_DTYPE)[:n])


def gpu_points(torch, sb, dt, pts):
    n = pts.shape[0]
    d_p = dev_bytes(torch, pts)
    d_o = torch.zeros(n * 20, dtype=torch.uint8, device="cuda:0")
    d_st = torch.zeros(n * 4, dtype=torch.uint8, device="cuda:0")
    d_ctr = torch.zeros(n * 16, dtype=torch.uint8, device="cuda:0")
    dt.closest_point(d_p.data_ptr(), n, d_o.data_ptr(), d_st.data_ptr(), d_ctr.data_ptr())
    torch.cuda.synchronize()
    return d_o.cpu().numpy().view(sb.CP_DTYPE), d_st.cpu().numpy().view(np.uint32), d_ctr.cpu().numpy().view(sb.COUNTERS_DTYPE)


def assert_hits_equal(got, want, what):
    assert np.array_equal(got["prim"], want["prim"]), f"{what}: primitive ids differ at {np.nonzero(got['prim'] != want['prim'])[0][:10]}"
    assert np.array_equal(got["t"].view(np.uint32), want["t"].view(np.uint32)), f"{what}: t not bit-exact"


SCENES = {"terrain": lambda sb: sb.Scene.terrain(36, 3), "sphere": lambda sb: sb.Scene.sphere(28, 5)}


@pytest.fixture(scope="module", params=["terrain", "sphere"])
def world(request, built, oracle):
    sb = built
    scene = SCENES[request.param](sb)
    lt = scene.build_sah(32, 4).collapse8()
    lo, hi = scene.bounds()
    cam = sb.default_camera(lo, hi, request.param == "terrain", 96, 96)
    rays = np.concatenate([sb.gen_primary_host(cam, 0, 96 * 96), sb.gen_secondary_host(lt.triangles(), 11, 0, 6000 + 13)])
    pts = sb.gen_points_host(lo - 0.3, hi + 0.3, 5, 0, 4099)
    return dict(name=request.param, scene=scene, lt=lt, lo=lo, hi=hi, rays=rays, pts=pts)


def layout_names():
    return ["pbrt", "pbrt-align16", "pbrt-soa", "pbrt-post", "pbrt-q16", "sg-eq", "sg-eq-align16", "ptr", "identity", "shared-slab", "dop14", "bvh8", "bvh8-q8",
            "bvh8-q8-ci", "bvh8-q16", "bvh8-q16-ci", "pbrt-soaos", "pbrt-soaos-align16", "pbrt-q16-soaos", "bvh8-align16", "bvh8-q8-align16",
            "bvh8-q8-ci-align16", "bvh8-q16-align16", "bvh8-q16-ci-align16"]


@pytest.mark.parametrize("layout", layout_names())
def test_closest_hit_matches_oracle(built, oracle, torch_cuda, world, layout):
    sb = built
    pt = world["lt"].encode(layout)
    dt = pt.upload(0)
    got, st, ctr = gpu_hits(torch_cuda, sb, dt, world["rays"])
    want, wst, wctr = oracle.closest_hit(oracle.tree_bytes(pt), world["rays"], counters=True)
    assert (want["prim"] != sb.MISS_PRIM).mean() > 0.1
    assert_hits_equal(got, want, f"{layout}/{world['name']}")
    assert np.array_equal(st, wst) and st.max() == 0
    assert np.array_equal(ctr, wctr), f"{layout}: interpreter counters differ => visit order differs"
    # the counter-free production kernel returns the same records
    got2, _, _ = gpu_hits(torch_cuda, sb, dt, world["rays"], counters=False)
    assert_hits_equal(got2, want, f"{layout} (no counters)")
    # host-buffer entry point (H2D + kernel + D2H inside the call)
    st_h = np.full(world["rays"].shape[0], 7, np.uint32)
    got3 = dt.closest_hit_host(world["rays"], status=st_h)
    assert_hits_equal(got3, want, f"{layout} (host entry)")
    assert st_h.max() == 0
    dt.free()


@pytest.mark.parametrize("layout", [l for l in layout_names() if not l.startswith("bvh8")])
def test_closest_point_matches_oracle(built, oracle, torch_cuda, world, layout):
    sb = built
    pt = world["lt"].encode(layout)
    dt = pt.upload(0)
    got, st, ctr = gpu_points(torch_cuda, sb, dt, world["pts"])
    want, wst, wctr = oracle.closest_point(oracle.tree_bytes(pt), world["pts"], counters=True)
    # north_star tolerance for floating point is 1e-6 relative; we require bit-exact d2, point and primitive
    assert np.array_equal(got.view(np.uint32).reshape(-1, 5), want.view(np.uint32).reshape(-1, 5)), layout
    assert np.array_equal(st, wst) and np.array_equal(ctr, wctr)
    rel = np.abs(got["d2"] - want["d2"]) / np.maximum(want["d2"], 1e-30)
    assert rel.max() <= 1e-6
    got_h = dt.closest_point_host(world["pts"])
    assert np.array_equal(got_h.view(np.uint32), got.view(np.uint32))
    dt.free()


def test_wide_layouts_reject_closest_point(built, torch_cuda, world):
    dt = world["lt"].encode("bvh8-q8-ci").upload(0)
    with pytest.raises(built.ScionError) as e:  # corpus.cpp:83 "cpq requires a binary layout"
        dt.closest_point_host(world["pts"][:8])
    assert e.value.code == built.ERR_ARG
    dt.free()


def test_golden_fixture(built, torch_cuda):
    """committed oracle outputs (tests/golden/hits_small.npz, tools/gen_golden.py)"""
    sb = built
    g = np.load(os.path.join(ROOT, "tests", "golden", "hits_small.npz"))
    grid, seed = [int(x) for x in g["terrain_grid"]]
    lt = sb.Scene.terrain(grid, seed).build_sah(32, 4).collapse8()
    rays = np.ascontiguousarray(g["rays"]).view(sb.RAY_DTYPE).reshape(-1)
    for layout in layout_names():
        dt = lt.encode(layout).upload(0)
        got, st, ctr = gpu_hits(torch_cuda, sb, dt, rays)
        assert np.array_equal(got["prim"], g[f"hit_prim:{layout}"]) and np.array_equal(got["t"].view(np.uint32), g[f"hit_t:{layout}"].view(np.uint32)), layout
        assert np.array_equal(ctr["node_visits"], g[f"hit_visits:{layout}"])
        if f"cp:{layout}" in g:
            cp, _, _ = gpu_points(torch_cuda, sb, dt, np.ascontiguousarray(g["points"]))
            assert np.array_equal(cp.view(np.uint32).reshape(-1, 5), g[f"cp:{layout}"]), layout
        dt.free()


def test_edge_cases(built, oracle, torch_cuda):
    sb = built
    scene = sb.Scene.terrain(8, 9)
    lt = scene.build_sah(32, 4).collapse8()
    lo, hi = scene.bounds()
    r = np.zeros(12, sb.RAY_DTYPE)
    r["tmax"] = np.inf
    c = 0.5 * (lo + hi)
    # 0: straight down through the centre; 1: axis-aligned with two zero direction components from a slab plane
    r[0] = (c[0], hi[1] + 1, c[2], np.inf, 0, -1, 0, 0)
    r[1] = (lo[0], hi[1] + 1, c[2], np.inf, 0, -1, 0, 0)  # origin x exactly on the world slab plane: 0 * inf = NaN path
    r[2] = (c[0], hi[1] + 1, c[2], 0.25, 0, -1, 0, 0)  # finite tmax: miss
    r[3] = (c[0], c[1] + 10, c[2], np.inf, 0, 1, 0, 0)  # pointing away
    r[4] = (c[0], lo[1] - 1, c[2], np.inf, 0, 1, 0, 0)  # from below (back faces)
    r[5] = (c[0], c[1], c[2], np.inf, 0.6, 0.0, 0.8, 0)  # origin inside the root box
    r[6] = (c[0], hi[1] + 1, c[2], np.inf, -0.0, -1, -0.0, 0)  # negative zeros are not "negative" (geometry.scion:13)
    r[7] = (lo[0] - 1, c[1], lo[2] - 1, np.inf, 0.70710678, 0, 0.70710678, 0)  # diagonal grazing
    r[8] = (c[0], hi[1] + 1, c[2], np.inf, 0, 0, 0, 0)  # null direction: rdir = inf everywhere
    r[9] = (np.nan, 0, 0, np.inf, 0, -1, 0, 0)  # NaN origin
    r[10] = (c[0], hi[1] + 1, c[2], 0.0, 0, -1, 0, 0)  # tmax = 0
    r[11] = (c[0], hi[1] + 1e30, c[2], np.inf, 0, -1, 0, 0)  # far away: precision loss, still deterministic
    pts = np.array([[c[0], c[1], c[2]], [lo[0], lo[1], lo[2]], [1e6, 1e6, 1e6], [np.nan, 0, 0]], np.float32)
    for layout in layout_names():
        pt = lt.encode(layout)
        dt = pt.upload(0)
        tb = oracle.tree_bytes(pt)
        for n in (12, 1, 0):  # ragged / single / empty launches
            got, st, ctr = gpu_hits(torch_cuda, sb, dt, r[:n])
            want, wst, wctr = oracle.closest_hit(tb, r[:n], counters=True)
            assert_hits_equal(got, want, f"{layout} edge n={n}")
            assert np.array_equal(ctr, wctr)
        assert got.shape[0] == 0
        full, _, _ = gpu_hits(torch_cuda, sb, dt, r)
        assert full["prim"][0] != sb.MISS_PRIM and full["prim"][2] == sb.MISS_PRIM and np.isinf(full["t"][2]) and full["prim"][3] == sb.MISS_PRIM
        if not layout.startswith("bvh8"):
            cp, _, _ = gpu_points(torch_cuda, sb, dt, pts)
            wcp, _ = oracle.closest_point(tb, pts)
            assert np.array_equal(cp.view(np.uint32), wcp.view(np.uint32)), layout
        dt.free()
    # single-leaf tree, every layout ("degenerate tree")
    one = sb.Scene.from_triangles(np.array([[0, 0, 0, 1, 0, 0, 0, 1, 0]], np.float32)).build_sah(32, 4).collapse8()
    ray = np.zeros(2, sb.RAY_DTYPE)
    ray[0] = (0.25, 0.25, -1, np.inf, 0, 0, 1, 0)
    ray[1] = (2.0, 2.0, -1, np.inf, 0, 0, 1, 0)
    for layout in layout_names():
        dt = one.encode(layout).upload(0)
        got, _, _ = gpu_hits(torch_cuda, sb, dt, ray)
        assert got["t"][0] == 1.0 and got["prim"][0] == 0 and got["prim"][1] == sb.MISS_PRIM, layout  # MT KAT through the whole stack
        dt.free()


def deep_chain(sb, depth):
    """left-deep chain: every interior's left child is the next interior, its right child a leaf, all boxes
    identical => a ray through the box accumulates one pending right sibling per level"""
    tri = lambda x: [x, 0, 0, x + 0.5, 0, 0, x, 0.5, 0]
    tris = np.array([tri(float(i)) for i in range(depth + 1)], np.float32)
    nodes = np.zeros(2 * depth + 1, sb.LNODE_DTYPE)
    nodes["lo"][:] = (-1.0, -1.0, -1.0)
    nodes["hi"][:] = (depth + 2.0, 1.0, 1.0)
    for i in range(depth):  # interiors 0..depth-1, leaves depth..2*depth
        nodes["left"][i] = i + 1 if i + 1 < depth else 2 * depth
        nodes["right"][i] = depth + i
    for j in range(depth, 2 * depth + 1):
        nodes["left"][j] = nodes["right"][j] = -1
        nodes["first_prim"][j] = j - depth
        nodes["nprims"][j] = 1
    return sb.LogicalTree.from_arrays(nodes, tris)


@pytest.mark.parametrize("layout", ["pbrt", "pbrt-q16", "sg-eq", "dop14", "ptr", "bvh8-q8-ci"])
def test_stack_overflow_is_a_query_error(built, oracle, torch_cuda, layout):
    """a tree deeper than the 64-entry stack: overflow is reported per query, never silent (SPEC.md:289-292,
    "tree of depth 70 with depth-64 stack -> overflow error"); shallower trees and rays that miss are fine"""
    sb = built
    ray = np.zeros(2, sb.RAY_DTYPE)
    ray[0] = (0.1, 0.1, -1, np.inf, 0, 0, 1, 0)  # through the common box: descends the whole chain
    ray[1] = (0.1, 5.0, -1, np.inf, 0, 0, 1, 0)  # misses the root
    pts = np.array([[0.1, 0.1, 0.0]], np.float32)
    for depth, expect in ((40, 0), (70, 1)):
        lt = deep_chain(sb, depth).collapse8()
        assert lt.depth == depth and lt.nnodes == 2 * depth + 1
        pt = lt.encode(layout)
        dt = pt.upload(0)
        got, st, ctr = gpu_hits(torch_cuda, sb, dt, ray)
        want, wst, wctr = oracle.closest_hit(oracle.tree_bytes(pt), ray, counters=True)
        assert np.array_equal(st, wst), (layout, depth, st, wst)
        assert st[1] == 0
        if layout in ("pbrt", "pbrt-q16", "sg-eq", "ptr"):  # AABB chains: the ray passes every box (dop14's diagonal slabs prune it)
            assert st[0] == expect
        ok = st == 0
        assert np.array_equal(got["prim"][ok], want["prim"][ok]) and np.array_equal(got["t"][ok].view(np.uint32), want["t"][ok].view(np.uint32))
        if not layout.startswith("bvh8"):
            cp, cst, _ = gpu_points(torch_cuda, sb, dt, pts)
            wcp, wcst = oracle.closest_point(oracle.tree_bytes(pt), pts)
            assert np.array_equal(cst, wcst)
            if cst[0] == 0:
                assert np.array_equal(cp.view(np.uint32), wcp.view(np.uint32))
        dt.free()


def test_treelet_variant_is_identical(built, torch_cuda, world):
    """kernel variant 2 (north_star: the top levels of the tree staged in shared memory by one TMA bulk copy per CTA — a
    side treelet in heap order built once per tree, device/treelet.cuh — and served by LDS) must return exactly the
    default kernel's records and per-query status, for every layout that supports it, on host- and device-encoded trees"""
    sb, torch = built, torch_cuda
    n = world["rays"].shape[0]
    d_rays = dev_bytes(torch, world["rays"])
    for layout in ("pbrt", "pbrt-align16", "pbrt-q16", "sg-eq-align16"):
        for dt in (world["lt"].encode(layout).upload(0), world["lt"].encode_device(layout, 0)):
            a = torch.zeros(n * 8, dtype=torch.uint8, device="cuda:0")
            b = torch.full((n * 8,), 0x5A, dtype=torch.uint8, device="cuda:0")
            sa = torch.full((n,), 7, dtype=torch.int32, device="cuda:0")
            sb_ = torch.full((n,), 9, dtype=torch.int32, device="cuda:0")
            dt.closest_hit(d_rays.data_ptr(), n, a.data_ptr(), sa.data_ptr())
            dt.closest_hit(d_rays.data_ptr(), n, b.data_ptr(), sb_.data_ptr(), variant=2)
            torch.cuda.synchronize()
            assert torch.equal(a, b), layout
            assert torch.equal(sa, sb_), layout
            dt.free()


def test_treelet_variant_on_a_tiny_tree(built, torch_cuda):
    """trees shallower than the staged levels (empty treelet slots) and a single-leaf tree"""
    sb, torch = built, torch_cuda
    for grid in (1, 2, 5):
        scene = sb.Scene.terrain(grid, 3)
        lt = scene.build_sah(32, 4)
        lo, hi = scene.bounds()
        cam = sb.default_camera(lo, hi, True, 32, 32)
        rays = sb.gen_primary_host(cam, 0, 1024)
        d_rays = dev_bytes(torch, rays)
        for layout in ("pbrt", "pbrt-q16"):
            dt = lt.encode(layout).upload(0)
            a = torch.zeros(1024 * 8, dtype=torch.uint8, device="cuda:0")
            b = torch.full((1024 * 8,), 0x5A, dtype=torch.uint8, device="cuda:0")
            dt.closest_hit(d_rays.data_ptr(), 1024, a.data_ptr())
            dt.closest_hit(d_rays.data_ptr(), 1024, b.data_ptr(), variant=2)
            torch.cuda.synchronize()
            assert torch.equal(a, b), (grid, layout)
            dt.free()


STAGED8 = ["bvh8", "bvh8-align16", "bvh8-q8-align16", "bvh8-q8-ci-align16", "bvh8-q16-align16", "bvh8-q16-ci-align16"]


@pytest.mark.parametrize("layout", STAGED8)
def test_staged_record_8wide_kernel_is_identical(built, torch_cuda, world, layout):
    """chrt8s_kernel (interior record staged in shared memory by 16-byte cp.async copies, one child slot decoded at a time
    by the emitted decode_slot<K>()) against chrt8_kernel (whole record in registers): hit records, per-query status and
    the interpreter counters (node visits, primitive tests, peak stack) must be equal bit for bit — variants 4 and 1
    select the two kernels explicitly, whichever is the default"""
    sb, torch = built, torch_cuda
    n = world["rays"].shape[0]
    d_rays = dev_bytes(torch, world["rays"])
    dt = world["lt"].encode(layout).upload(0)
    out = {}
    for v in (1, 4):
        h = torch.full((n * 8,), 0x5A, dtype=torch.uint8, device="cuda:0")
        st = torch.full((n,), 7, dtype=torch.int32, device="cuda:0")
        c = torch.zeros(n * 16, dtype=torch.uint8, device="cuda:0")
        dt.closest_hit(d_rays.data_ptr(), n, h.data_ptr(), st.data_ptr(), c.data_ptr(), variant=v)
        h2 = torch.full((n * 8,), 0x5A, dtype=torch.uint8, device="cuda:0")
        dt.closest_hit(d_rays.data_ptr(), n, h2.data_ptr(), variant=v)  # the counter-free build
        torch.cuda.synchronize()
        assert torch.equal(h, h2), (layout, v)
        out[v] = (h, st, c)
    for a, b in zip(out[1], out[4]):
        assert torch.equal(a, b), layout
    dt.free()


COOP8 = ["bvh8", "bvh8-align16", "bvh8-q8", "bvh8-q8-align16", "bvh8-q8-ci", "bvh8-q8-ci-align16", "bvh8-q16", "bvh8-q16-align16", "bvh8-q16-ci",
         "bvh8-q16-ci-align16"]


@pytest.mark.parametrize("layout", COOP8)
def test_lane_cooperative_8wide_kernel_is_identical(built, torch_cuda, world, oracle, layout):
    """chrt8c_kernel (kernel variant 5: a group of 8 lanes owns one ray, lane k decodes and tests child slot k through the
    per-child record view scion::LaneRecord, the group's 8 lanes test 8 triangles of a leaf at a time) against chrt8_kernel
    (variant 1, one ray per lane) AND against the oracle: hit records, per-query status and the interpreter counters
    (node visits, primitive tests, peak stack) must be equal bit for bit, with and without the counter instrumentation"""
    sb, torch = built, torch_cuda
    n = world["rays"].shape[0]
    d_rays = dev_bytes(torch, world["rays"])
    pt = world["lt"].encode(layout)
    dt = pt.upload(0)
    out = {}
    for v in (1, 5):
        h = torch.full((n * 8,), 0x5A, dtype=torch.uint8, device="cuda:0")
        st = torch.full((n,), 7, dtype=torch.int32, device="cuda:0")
        c = torch.zeros(n * 16, dtype=torch.uint8, device="cuda:0")
        dt.closest_hit(d_rays.data_ptr(), n, h.data_ptr(), st.data_ptr(), c.data_ptr(), variant=v)
        h2 = torch.full((n * 8,), 0x5A, dtype=torch.uint8, device="cuda:0")
        dt.closest_hit(d_rays.data_ptr(), n, h2.data_ptr(), variant=v)  # the counter-free build
        torch.cuda.synchronize()
        assert torch.equal(h, h2), (layout, v)
        out[v] = (h, st, c)
    for a, b in zip(out[1], out[5]):
        assert torch.equal(a, b), layout
    got = out[5][0].cpu().numpy().view(sb.HIT_DTYPE)
    want, _ = oracle.closest_hit(oracle.tree_bytes(pt), world["rays"])
    assert np.array_equal(got["prim"], want["prim"]) and np.array_equal(got["t"].view(np.uint32), want["t"].view(np.uint32))
    dt.free()


def test_two_rays_per_lane_variant_is_identical(built, torch_cuda, world):
    """experimental kernel variant 3 (two rays per lane, the next record's load of one ray in flight while the other
    ray's step executes; emitted fetch() / decode_fetched()) must return exactly the default kernel's records and
    per-query status"""
    sb, torch = built, torch_cuda
    n = world["rays"].shape[0]
    d_rays = dev_bytes(torch, world["rays"])
    for layout in ("pbrt", "pbrt-q16"):
        dt = world["lt"].encode(layout).upload(0)
        a = torch.zeros(n * 8, dtype=torch.uint8, device="cuda:0")
        b = torch.full((n * 8,), 0x5A, dtype=torch.uint8, device="cuda:0")
        sa = torch.full((n,), 7, dtype=torch.int32, device="cuda:0")
        sb_ = torch.full((n,), 9, dtype=torch.int32, device="cuda:0")
        dt.closest_hit(d_rays.data_ptr(), n, a.data_ptr(), sa.data_ptr())
        dt.closest_hit(d_rays.data_ptr(), n, b.data_ptr(), sb_.data_ptr(), variant=3)
        torch.cuda.synchronize()
        assert torch.equal(a, b), layout
        assert torch.equal(sa, sb_), layout
        dt.free()


def test_packed_ray_host_entry_is_identical(built, torch_cuda, world):
    """scion_closest_hit_host_packed (host rays in the reference's packed 28-byte Ray record: origin, direction, tmax —
    geometry.scion:4) must return exactly what scion_closest_hit_host returns for the same rays as 32-byte scion_ray
    records, records and per-query status, over several staging chunks and for an empty call; scion_rays_unpack on its own
    must reproduce the scion_ray array (pad = 0)"""
    sb, torch = built, torch_cuda
    rays = np.concatenate([world["rays"]] * 3)  # a few thousand rays; the chunking is exercised through SCION_HOST_CHUNK_LOG2 in the fullsize tests
    rays["pad"] = 0.0
    packed = sb.pack_rays(rays)
    assert packed.shape == (rays.shape[0], 7) and packed.dtype == np.float32
    for layout in ("pbrt-q16", "bvh8-q8-ci", "dop14"):
        dt = world["lt"].encode(layout).upload(0)
        sa, sb_ = np.full(rays.shape[0], 7, np.uint32), np.full(rays.shape[0], 9, np.uint32)
        a = dt.closest_hit_host(rays, status=sa)
        b = dt.closest_hit_host_packed(packed, status=sb_)
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), layout
        assert np.array_equal(sa, sb_), layout
        assert dt.closest_hit_host_packed(packed[:0]).shape[0] == 0
        # origin + direction only (the DSL's default tmax = inf): equal to the padded call on rays whose tmax is inf
        inf_rays = rays.copy()
        inf_rays["tmax"] = np.inf
        c = dt.closest_hit_host(inf_rays)
        d = dt.closest_hit_host_od(np.ascontiguousarray(sb.pack_rays(inf_rays)[:, :6]))
        assert np.array_equal(c.view(np.uint8), d.view(np.uint8)), layout
        dt.free()
    d_p = torch.from_numpy(packed.reshape(-1)).to("cuda:0")
    d_r = torch.full((rays.shape[0] * 8,), 5.0, dtype=torch.float32, device="cuda:0")
    from paper_2511_15028_b200 import lib, _check
    _check(lib().scion_rays_unpack(d_p.data_ptr(), rays.shape[0], d_r.data_ptr(), None))
    torch.cuda.synchronize()
    assert np.array_equal(d_r.cpu().numpy().view(np.uint32), rays.view(np.uint32).reshape(-1))


def test_fault_injection_changes_results(built, oracle, torch_cuda, world):
    """corrupting one c_o byte must surface as >= 1 mismatch against the oracle of the intact tree"""
    sb = built
    pt = world["lt"].encode("pbrt")
    want, _ = oracle.closest_hit(oracle.tree_bytes(pt), world["rays"])
    pt.corrupt(1, 24, 0x01)  # root node: c_o ^= 1 -> right child off by one
    dt = pt.upload(0)
    got, st, _ = gpu_hits(torch_cuda, sb, dt, world["rays"])
    assert (got["prim"] != want["prim"]).sum() + (st != 0).sum() >= 1
    dt.free()


def test_replication_paths_agree(built, oracle, torch_cuda, world):
    """upload / upload_into a caller tensor / from_image of a copied image give identical results"""
    sb, torch = built, torch_cuda
    pt = world["lt"].encode("pbrt-q16")
    a = pt.upload(0)
    ref, _, _ = gpu_hits(torch, sb, a, world["rays"], counters=False)
    img = torch.empty(pt.image_bytes + 256, dtype=torch.uint8, device="cuda:0")
    off = (-img.data_ptr()) % 256
    b = pt.upload_into(0, img.data_ptr() + off, pt.image_bytes)
    gb, _, _ = gpu_hits(torch, sb, b, world["rays"], counters=False)
    copy = img.clone()  # what a broadcast receiver holds
    off2 = (-copy.data_ptr()) % 256
    if off2 != off:
        copy2 = torch.empty(pt.image_bytes + 512, dtype=torch.uint8, device="cuda:0")
        off2 = (-copy2.data_ptr()) % 256
        copy2[off2:off2 + pt.image_bytes] = img[off:off + pt.image_bytes]
        copy = copy2
    c = sb.DeviceTree.from_image(copy.data_ptr() + off2, pt.image_bytes, 0, "pbrt-q16")
    gc, _, _ = gpu_hits(torch, sb, c, world["rays"], counters=False)
    assert_hits_equal(gb, ref, "upload_into")
    assert_hits_equal(gc, ref, "from_image")
    with pytest.raises(sb.ScionError):
        sb.DeviceTree.from_image(copy.data_ptr() + off2, pt.image_bytes, 0, "pbrt")  # wrong layout name is rejected
    for t in (a, b, c):
        t.free()


def test_device_generators_match_host_twins(built, torch_cuda, world):
    sb, torch = built, torch_cuda
    lo, hi = world["lo"], world["hi"]
    cam = sb.default_camera(lo, hi, True, 64, 64)
    n = 64 * 64
    d = torch.empty(n * 32, dtype=torch.uint8, device="cuda:0")
    sb.gen_primary(cam, 5, n - 5, d.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy()[:(n - 5) * 32].view(np.uint32), sb.gen_primary_host(cam, 5, n - 5).view(np.uint32))
    dt = world["lt"].encode("pbrt").upload(0)
    dt.gen_secondary(77, 100, n, d.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy().view(np.uint32), sb.gen_secondary_host(world["lt"].triangles(), 77, 100, n).view(np.uint32))
    p = torch.empty(n * 12, dtype=torch.uint8, device="cuda:0")
    sb.gen_points(lo, hi, 9, 3, n, p.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(p.cpu().numpy().view(np.uint32), sb.gen_points_host(lo, hi, 9, 3, n).view(np.uint32).reshape(-1))
    dt.free()
