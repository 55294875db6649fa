"""Command-line harness of the B200 backend — the reference CLI's sub-commands (`check`, `compile`, `build-tree`,
`build`, `run`, `verify`, `footprint`, `bench`) for the traversal path.

  python -m paper_2511_15028_b200.harness check                      # every registered layout plans + emits
  python -m paper_2511_15028_b200.harness footprint --layout L --scene terrain:224
  python -m paper_2511_15028_b200.harness emit-cuda --layout L [-o file]
  python -m paper_2511_15028_b200.harness compile file.scion [--plan plan.json] [--emit-cuda out.cuh]   # a user-written layout
  python -m paper_2511_15028_b200.harness build-tree --scene terrain:224 [--builder sah|median] -o tree.npz  # Scene -> LogicalTree
  python -m paper_2511_15028_b200.harness build --layout L (--tree tree.npz | --scene terrain:224) -o tree.scionpt   # -> PhysicalTree container
  python -m paper_2511_15028_b200.harness run tree.scionpt --alg chrt|cpq --queries N --rays primary|secondary [-o results.bin]  # container -> results
  python -m paper_2511_15028_b200.harness bench --layout L[,L2..] --alg chrt|cpq --scene terrain:708 --queries 4194304 --rays secondary
  python -m paper_2511_15028_b200.harness bench --layout L[,L2..] --alg cd --scene terrain:224 [--builder median|sah]   # --queries = output capacity

`bench` follows the paper's protocol: 1 warm-up + 9 runs, drop the 2 lowest
and 2 highest, report the mean of the remaining 5, one CSV row per (layout, algorithm, scene, nGPU).
Exit codes as the reference CLI: 0 pass, 1 diagnostics/mismatch, 2 usage.  `verify` (which needs the CPU
oracle) lives in tests/verify_cli.py because only test infrastructure may touch oracle/.
"""
import argparse
import os
import json
import sys

import numpy as np

import paper_2511_15028_b200 as sb


def parse_scene(spec: str) -> "sb.Scene":
    kind, _, arg = spec.partition(":")
    n = int(arg or 64)
    if kind == "terrain":
        return sb.Scene.terrain(n, sb.seed_from_env(1))
    if kind == "sphere":
        return sb.Scene.sphere(n, sb.seed_from_env(1))
    if kind == "cloud":
        return sb.Scene.cloud(n, sb.seed_from_env(1))
    raise SystemExit(2)


def cmd_check(_):
    ok = True
    for l in sb.layouts():
        try:
            plan = sb.layout_plan(l["name"])
            text = sb.emit_cuda(l["name"])
            assert "static void decode(" in text
            has_build = bool(sb.lib().scion_layout_has_build(l["name"].encode()))
            assert has_build == ("static uint64_t build_node(" in text)
            print(f"{l['name']:22s} ok   family={('bvh2', 'dop14', 'bvh8')[l['family']]} node_stride={l['node_stride']} segments={l['n_segments']} slots={len(plan['slots'])} "
                  f"constructors={'compiled' if has_build else 'none'}")
        except Exception as e:  # noqa: BLE001
            ok = False
            print(f"{l['name']:14s} FAILED {e}", file=sys.stderr)
    return 0 if ok else 1


def cmd_footprint(a):
    scene = parse_scene(a.scene)
    lt = scene.build_sah(32, a.max_leaf).collapse8()
    pt = lt.encode(a.layout)
    rep = {"layout": a.layout, "scene": a.scene, "primitives": lt.nprims, "total_bytes": pt.total_bytes, "node_bytes": pt.node_bytes,
           "bvh_bytes_per_prim": pt.node_bytes / lt.nprims,
           "buffers": [{"name": b["name"], "bytes": b["bytes"], "count": b["count"], "segment_bases": b["seg_bases"]} for b in pt.buffers()],
           "node_stride": sb.layout_info(a.layout)["node_stride"]}
    print(json.dumps(rep, indent=1))
    return 0


def cmd_emit(a):
    if getattr(a, "dump_stats", False):  # the reference CLI's --dump-stats: op-count JSON of the decode
        print(json.dumps(sb.layout_stats(a.layout), indent=1))
        return 0
    text = sb.emit_c(a.layout) if a.cmd == "emit-c" else sb.emit_cuda(a.layout)
    if a.output:
        open(a.output, "w").write(text)
    else:
        sys.stdout.write(text)
    return 0


def cmd_bench_cd(a):
    """Collision detection (cd.scion): the scene against a lifted copy of a second scene of the same kind
    (SPEC.md:599 'second scene + rigid transform'), median split with one primitive per leaf as in the
    paper's CD experiment (§8.3.3) unless --builder sah."""
    import torch
    sa = parse_scene(a.scene)
    kind, _, arg = a.scene.partition(":")
    other = {"terrain": sb.Scene.terrain, "sphere": sb.Scene.sphere}.get(kind)
    if other is None:
        print("cd needs a triangle scene (terrain:N or sphere:N)", file=sys.stderr)
        return 2
    tb = other(int(arg or 64), sb.seed_from_env(1) + 8).triangles().copy()
    tb[:, 1::3] += np.float32(0.02)
    sb_scene = sb.Scene.from_triangles(tb)
    build = (lambda s: s.build_median(1)) if a.builder == "median" else (lambda s: s.build_sah(32, a.max_leaf))
    la, lb = build(sa), build(sb_scene)
    cap = a.queries
    d_out = torch.empty(cap * 8, dtype=torch.uint8, device="cuda:0")
    print("layout,algorithm,scene,n_gpus,primitives,builder,mean_ms,pairs,mpairs_tested_per_s,node_pairs,tri_tests,levels,max_frontier,bytes_per_launch,achieved_gbs")
    for layout in a.layout.split(","):
        da, db = la.encode(layout).upload(0), lb.encode(layout).upload(0)
        times, n, st = [], 0, {}
        for i in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            n, st = da.collide(db, d_out.data_ptr(), cap)
            e1.record()
            torch.cuda.synchronize()
            if i:
                times.append(e0.elapsed_time(e1))
        ms = float(np.mean(sorted(times)[2:-2]))
        plan = sb.layout_plan(layout)
        stride = sum(s["stride_bytes"] for b in plan["buffers"] if b["name"] == plan["node_group"] for s in b["segments"])
        nbytes = st["node_pairs"] * (2 * stride + 2 * 4) + st["tri_tests"] * 72 + n * 8  # both records + the pair entry; both triangles; output
        print(f"{layout},cd,{a.scene},1,{la.nprims}+{lb.nprims},{a.builder},{ms:.4f},{n},{(st['node_pairs'] + st['tri_tests']) / ms / 1e3:.2f},{st['node_pairs']},{st['tri_tests']},{st['levels']},{st['max_frontier']},{nbytes},{nbytes / ms / 1e6:.1f}")
        if n > cap:
            print(f"{layout}: output capacity {cap} < {n} colliding pairs (count is exact, list truncated)", file=sys.stderr)
        da.free()
        db.free()
    return 0


def cmd_compile(a):
    """`compile`: a .scion layout file -> memory plan (JSON) + the CUDA device header emit_cuda produces for it."""
    try:
        src = open(a.file).read()
    except OSError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    plan, cuda = sb.compile_layout_text(src)  # diagnostics surface as ScionError -> exit code 1
    if a.plan:
        json.dump(plan, open(a.plan, "w"), indent=1)
    if a.emit_cuda:
        open(a.emit_cuda, "w").write(cuda)
    node = [b for b in plan["buffers"] if b["name"] == plan["node_group"]]
    print(json.dumps({"layout": plan.get("layout"), "node_group": plan["node_group"], "node_stride": sum(x["stride_bytes"] for x in node[0]["segments"]) if node else 0,
                      "buffers": len(plan["buffers"]), "slots": len(plan["slots"]), "cuda_bytes": len(cuda)}))
    return 0


def build_logical(a):
    scene = parse_scene(a.scene)
    lt = scene.build_median(a.max_leaf) if a.builder == "median" else scene.build_sah(32, a.max_leaf)
    return lt


def cmd_build_tree(a):
    """`build-tree`: Scene -> LogicalTree, stored as the two arrays scion_ltree_from_arrays takes back."""
    lt = build_logical(a)
    np.savez(a.output, nodes=lt.nodes(), triangles=lt.triangles())
    print(json.dumps({"scene": a.scene, "builder": a.builder, "nodes": lt.nnodes, "primitives": lt.nprims, "depth": lt.depth}))
    return 0


def cmd_build(a):
    """`build`: LogicalTree -> PhysicalTree in the chosen layout, written as the versioned container file
    (header with magic, version, layout name, global slots + raw little-endian buffers)."""
    if a.tree:
        z = np.load(a.tree)
        lt = sb.LogicalTree.from_arrays(z["nodes"], z["triangles"])
    else:
        lt = build_logical(a)
    if sb.layout_info(a.layout)["family"] == 2:
        lt.collapse8()
    pt = lt.encode(a.layout)
    pt.save(a.output)
    print(json.dumps({"layout": a.layout, "primitives": lt.nprims, "total_bytes": pt.total_bytes, "node_bytes": pt.node_bytes, "file": a.output}))
    return 0


def cmd_run(a):
    """`run`: reads a PhysicalTree container file, uploads it, generates the queries on the device from (seed, index),
    runs them and writes the raw result records (scion_hit / scion_cp, query order) plus a JSON report."""
    import torch
    if not torch.cuda.is_available():
        print("run needs a CUDA device (no CPU fallback)", file=sys.stderr)
        return 1
    pt = sb.PhysicalTree.load(a.file)
    prim = [b for b in pt.buffers() if b["name"] == "primitives"][0]
    tris = np.asarray(prim["data"]).view(np.float32).reshape(-1, 3)
    lo, hi = tris.min(axis=0), tris.max(axis=0)
    dt = pt.upload(0)
    n, dev = a.queries, "cuda:0"
    seed = sb.seed_from_env(a.seed)
    d_st = torch.zeros(n, dtype=torch.int32, device=dev)
    d_ctr = torch.zeros(n * 4, dtype=torch.int32, device=dev)
    if a.alg == "chrt":
        d_q = torch.empty(n * 32, dtype=torch.uint8, device=dev)
        d_r = torch.empty(n * 8, dtype=torch.uint8, device=dev)
        if a.rays == "primary":
            side = int(np.sqrt(n))
            n = side * side
            sb.gen_primary(sb.default_camera(lo, hi, a.look_down_y, side, side), 0, n, d_q.data_ptr())
        else:
            dt.gen_secondary(seed, 0, n, d_q.data_ptr())
        dt.closest_hit(d_q.data_ptr(), n, d_r.data_ptr(), d_st.data_ptr(), d_ctr.data_ptr())
        torch.cuda.synchronize()
        res = d_r.cpu().numpy()[:n * 8].view(sb.HIT_DTYPE)
        found = int((res["prim"] != sb.MISS_PRIM).sum())
    else:
        d_q = torch.empty(n * 12, dtype=torch.uint8, device=dev)
        d_r = torch.empty(n * 20, dtype=torch.uint8, device=dev)
        sb.gen_points(lo, hi, seed, 0, n, d_q.data_ptr())
        dt.closest_point(d_q.data_ptr(), n, d_r.data_ptr(), d_st.data_ptr(), d_ctr.data_ptr())
        torch.cuda.synchronize()
        res = d_r.cpu().numpy().view(sb.CP_DTYPE)
        found = int((res["prim"] != sb.MISS_PRIM).sum())
    errors = int((d_st[:n] != 0).sum())
    c = d_ctr.view(-1, 4)[:n].sum(dim=0, dtype=torch.int64).cpu().numpy()
    if a.output:
        res.tofile(a.output)
    import zlib
    print(json.dumps({"layout": pt.layout, "algorithm": a.alg, "queries": n, "kind": a.rays if a.alg == "chrt" else "points", "seed": seed, "found": found,
                      "query_errors": errors, "node_visits": int(c[0]), "prim_tests": int(c[1]), "crc32": zlib.crc32(res.tobytes()), "results": a.output}))
    dt.free()
    return 1 if errors else 0


def cmd_bench(a):
    import torch
    if not torch.cuda.is_available():
        print("bench needs a CUDA device (no CPU fallback)", file=sys.stderr)
        return 1
    if a.alg == "cd":
        return cmd_bench_cd(a)
    scene = parse_scene(a.scene)
    lt = scene.build_sah(32, a.max_leaf).collapse8()
    lo, hi = scene.bounds()
    n = a.queries
    dev = "cuda:0"
    print("layout,algorithm,scene,n_gpus,queries,kind,mean_ms,mqueries_per_s,bvh_bytes_per_prim,node_visits,prim_tests,bytes_per_query,achieved_gbs")
    for layout in a.layout.split(","):
        pt = lt.encode(layout)
        dt = pt.upload(0)
        if a.alg == "chrt":
            d_q = torch.empty(n * 32, dtype=torch.uint8, device=dev)
            d_r = torch.empty(n * 8, dtype=torch.uint8, device=dev)
            if a.rays == "primary":
                side = int(np.sqrt(n))
                cam = sb.default_camera(lo, hi, scene_is_terrain(a.scene), side, side)
                sb.gen_primary(cam, 0, n, d_q.data_ptr())
            else:
                dt.gen_secondary(sb.seed_from_env(7), 0, n, d_q.data_ptr())
            run = lambda ctr=0, st=0: dt.closest_hit(d_q.data_ptr(), n, d_r.data_ptr(), st, ctr)
        else:
            d_q = torch.empty(n * 12, dtype=torch.uint8, device=dev)
            d_r = torch.empty(n * 20, dtype=torch.uint8, device=dev)
            sb.gen_points(lo, hi, sb.seed_from_env(7), 0, n, d_q.data_ptr())
            run = lambda ctr=0, st=0: dt.closest_point(d_q.data_ptr(), n, d_r.data_ptr(), st, ctr)
        times = []
        for i in range(10):  # 1 warm-up + 9 runs
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            if i:
                times.append(e0.elapsed_time(e1))
        ms = float(np.mean(sorted(times)[2:-2]))  # drop 2 lowest + 2 highest, mean of 5
        d_ctr = torch.zeros(n * 4, dtype=torch.int32, device=dev)
        d_st = torch.zeros(n, dtype=torch.int32, device=dev)
        run(d_ctr.data_ptr(), d_st.data_ptr())
        torch.cuda.synchronize()
        c = d_ctr.view(-1, 4).sum(dim=0, dtype=torch.int64).cpu().numpy() / n
        plan = sb.layout_plan(layout)
        seg = [s["stride_bytes"] for b in plan["buffers"] if b["name"] == plan["node_group"] for s in b["segments"]]
        q_io = 40 if a.alg == "chrt" else 32
        bpq = c[0] * (seg[0] if seg else 0) + c[2] * sum(seg[1:]) + c[1] * 36 + q_io
        print(f"{layout},{a.alg},{a.scene},1,{n},{a.rays if a.alg == 'chrt' else 'points'},{ms:.4f},{n / ms / 1e3:.2f},{pt.node_bytes / lt.nprims:.3f},{c[0]:.2f},{c[1]:.2f},{bpq:.1f},{bpq * n / ms / 1e6:.1f}")
        if int((d_st != 0).sum()) != 0:
            print(f"{layout}: query errors reported", file=sys.stderr)
            return 1
        dt.free()
    return 0


def scene_is_terrain(spec):
    return spec.startswith("terrain")


def main(argv=None):
    ap = argparse.ArgumentParser(prog="paper_2511_15028_b200.harness")
    ap.add_argument("--layout-file", action="append", default=[], metavar="FILE.scion",
                    help="compile and register this layout (layout + build block) at run time under the name of the file "
                         "(my_layout.scion -> my-layout) before the command runs; needs nvcc; repeatable")
    sub = ap.add_subparsers(dest="cmd")
    sub.add_parser("check")
    p = sub.add_parser("footprint")
    p.add_argument("--layout", required=True)
    p.add_argument("--scene", default="terrain:64")
    p.add_argument("--max-leaf", type=int, default=4)
    for name in ("emit-cuda", "emit-c"):  # emit-c: the record half of the reference's emit_c (typed packed records + assertions)
        p = sub.add_parser(name)
        p.add_argument("--layout", required=True)
        p.add_argument("-o", "--output")
        p.add_argument("--dump-stats", action="store_true")
    p = sub.add_parser("compile")
    p.add_argument("file")
    p.add_argument("--plan")
    p.add_argument("--emit-cuda")
    for name in ("build-tree", "build"):
        p = sub.add_parser(name)
        p.add_argument("--scene", default="terrain:64")
        p.add_argument("--builder", default="sah", choices=["sah", "median"])
        p.add_argument("--max-leaf", type=int, default=4)
        p.add_argument("-o", "--output", required=True)
        if name == "build":
            p.add_argument("--layout", required=True)
            p.add_argument("--tree", help="LogicalTree written by build-tree (otherwise built from --scene)")
    p = sub.add_parser("run")
    p.add_argument("file")
    p.add_argument("--alg", default="chrt", choices=["chrt", "cpq"])
    p.add_argument("--queries", type=int, default=1 << 16)
    p.add_argument("--rays", default="primary", choices=["primary", "secondary"])
    p.add_argument("--look-down-y", action="store_true", help="primary camera above the +y face (terrains) instead of the +z face")
    p.add_argument("--seed", type=int, default=7)
    p.add_argument("-o", "--output")
    p = sub.add_parser("bench")
    p.add_argument("--layout", required=True)
    p.add_argument("--alg", default="chrt", choices=["chrt", "cpq", "cd"])
    p.add_argument("--builder", default="median", choices=["median", "sah"], help="cd only: median split, 1 primitive per leaf (paper) or binned SAH")
    p.add_argument("--scene", default="terrain:224")
    p.add_argument("--queries", type=int, default=1 << 20)
    p.add_argument("--rays", default="primary", choices=["primary", "secondary"])
    p.add_argument("--max-leaf", type=int, default=4)
    try:
        a = ap.parse_args(argv)
    except SystemExit:
        return 2
    if a.cmd is None:
        ap.print_usage(sys.stderr)
        return 2
    try:
        for f in a.layout_file:  # open-world layouts: front end -> emit_cuda -> nvcc -> plugin (scion_layout_register)
            name = os.path.splitext(os.path.basename(f))[0].replace("_", "-")
            try:
                text = open(f).read()
            except OSError as e:
                print(f"error: {e}", file=sys.stderr)
                return 2
            sb.register_layout(name, text)
            print(f"registered layout '{name}' from {f}", file=sys.stderr)
        return {"check": cmd_check, "footprint": cmd_footprint, "emit-cuda": cmd_emit, "emit-c": cmd_emit, "bench": cmd_bench, "compile": cmd_compile,
                "build-tree": cmd_build_tree, "build": cmd_build, "run": cmd_run}[a.cmd](a)
    except sb.ScionError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2 if e.code == sb.ERR_ARG else 1


if __name__ == "__main__":
    sys.exit(main())
