"""emit_cuda's generated decoders (csrc/gen/*.cuh), compiled in the host mode of scion_rt.cuh, walk
every node of a product-encoded tree and must agree bit-for-bit with the oracle's independent
decoders — bounds (incl. directed-rounding dequantisation), variant, child references, primitive
ranges.  This pins the codegen on a machine without a GPU."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2511_15028_b200", "csrc")
SHIM = os.path.join(ROOT, "tests", "_host_decode_shim.so")


class TreeView(C.Structure):  # mirror of scion::TreeView (device/scion_rt.cuh)
    _fields_ = [("buf", C.c_void_p * 6), ("seg_base", (C.c_uint64 * 4) * 6), ("count", C.c_uint64 * 6), ("glob", (C.c_uint32 * 4) * 12),
                ("root0", C.c_uint64), ("root_carried", C.c_float * 6), ("treelet", C.c_void_p), ("treelet_slots", C.c_uint32)]


@pytest.fixture(scope="module")
def shim(built):
    src = os.path.join(ROOT, "tests", "host_decode_shim.cpp")
    r = subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", "-fPIC", "-shared", "-ffp-contract=off", "-frounding-math", "-I", CSRC, "-I", os.path.join(ROOT, "include"),
                        src, "-o", SHIM], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    lib = C.CDLL(SHIM)
    assert lib.host_treeview_size() == C.sizeof(TreeView)
    return lib


def make_view(pt):
    tv = TreeView()
    for i, b in enumerate(pt.buffers()):
        tv.buf[i] = b["ptr"]
        tv.count[i] = b["count"]
        for s, v in enumerate(b["seg_bases"]):
            tv.seg_base[i][s] = v
    for i, g in enumerate(pt.globals()):
        raw = np.frombuffer(g["raw"], np.uint32)
        for k in range(4):
            tv.glob[i][k] = int(raw[k])
    r0, carried = pt.root()
    tv.root0 = r0
    for k in range(6):
        tv.root_carried[k] = carried[k]
    return tv


def test_generated_decoders_match_oracle(built, oracle, shim):
    from tests.oracle_lib import TreeBytes
    oracle.lib.oracle_decode2.argtypes = [C.POINTER(TreeBytes), C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
    oracle.lib.oracle_decode8.argtypes = [C.POINTER(TreeBytes), C.c_uint64, C.c_void_p, C.c_void_p]
    shim.host_decode2.argtypes = [C.c_char_p, C.POINTER(TreeView), C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
    shim.host_decode8.argtypes = [C.c_char_p, C.POINTER(TreeView), C.c_uint64, C.c_void_p, C.c_void_p]
    shim.host_decode8_lane.argtypes = [C.c_char_p, C.POINTER(TreeView), C.c_uint64, C.c_void_p, C.c_void_p]
    scene = built.Scene.terrain(14, 21)
    lt = scene.build_sah(32, 4).collapse8()
    for l in built.layouts():
        name = l["name"]
        pt = lt.encode(name)
        tb, tv = oracle.tree_bytes(pt), make_view(pt)
        r0, carried = pt.root()
        visited = 0
        if l["family"] != 2:
            stack = [(r0, np.array(carried, np.float32))]
            while stack:
                ref, car = stack.pop()
                f1, f2 = np.zeros(20, np.float32), np.zeros(20, np.float32)
                u1, u2 = np.zeros(5, np.uint64), np.zeros(5, np.uint64)
                assert oracle.lib.oracle_decode2(C.byref(tb), ref, car.ctypes.data, f1.ctypes.data, u1.ctypes.data) == 0
                assert shim.host_decode2(name.encode(), C.byref(tv), ref, car.ctypes.data, f2.ctypes.data, u2.ctypes.data) == 0, name
                assert np.array_equal(u1, u2), (name, ref, u1, u2)
                nf = 14 if l["family"] == 1 else 6
                assert np.array_equal(f1[:nf].view(np.uint32), f2[:nf].view(np.uint32)), (name, ref, f1[:nf], f2[:nf])
                if name == "shared-slab":
                    assert np.array_equal(f1[14:].view(np.uint32), f2[14:].view(np.uint32)), name
                visited += 1
                if not u1[0]:
                    child_car = f1[14:20].copy() if name == "shared-slab" else car
                    stack.append((int(u1[2]), child_car))
                    stack.append((int(u1[1]), child_car))
            assert visited == lt.nnodes, name
        else:
            stack = [r0]
            while stack:
                ref = stack.pop()
                f1, f2 = np.zeros(48, np.float32), np.zeros(48, np.float32)
                u1, u2 = np.zeros(11, np.uint64), np.zeros(11, np.uint64)
                assert oracle.lib.oracle_decode8(C.byref(tb), ref, f1.ctypes.data, u1.ctypes.data) == 0
                assert shim.host_decode8(name.encode(), C.byref(tv), ref, f2.ctypes.data, u2.ctypes.data) == 0, name
                assert np.array_equal(u1, u2), (name, ref, u1, u2)
                if not u1[0]:  # leaves are encoded in the reference itself: no boxes
                    assert np.array_equal(f1.view(np.uint32), f2.view(np.uint32)), (name, ref)
                # the per-child record view of the lane-cooperative kernel: slot k through decode_slot<0>(LaneRecord{record, k})
                f3, u3 = np.zeros(48, np.float32), np.zeros(11, np.uint64)
                assert shim.host_decode8_lane(name.encode(), C.byref(tv), ref, f3.ctypes.data, u3.ctypes.data) == 0, name
                assert np.array_equal(u1, u3), (name, ref, u1, u3)
                if not u1[0]:
                    assert np.array_equal(f1.view(np.uint32), f3.view(np.uint32)), (name, ref)
                visited += 1
                if not u1[0]:
                    wn = lt.wnodes()[int(ref) >> 2]
                    for k in range(8):
                        if wn["child"][k] != built.W_SENTINEL:
                            stack.append(int(u1[3 + k]))
            assert visited == len(lt.wnodes()) + len(lt.wleaves()), name


def test_emitted_code_differential(built, oracle, shim):
    """SPEC acceptance 8 ("emitted-C differential"), for the CUDA backend: the emitted per-layout
    headers, compiled by the HOST compiler, drive a plain recursive closest_hit (tests/host_decode_shim.cpp) —
    same chosen primitive and bitwise-equal t as the oracle for 1,024 primary + 1,024 incoherent rays, all 16
    layouts (the SPEC asks for 2 layouts and 1 ulp)."""
    shim.host_closest_hit.argtypes = [C.c_char_p, C.POINTER(TreeView), C.c_void_p, C.c_uint64, C.c_void_p]
    scene = built.Scene.terrain(20, 5)
    lt = scene.build_sah(32, 4).collapse8()
    lo, hi = scene.bounds()
    cam = built.default_camera(lo, hi, True, 32, 32)
    rays = np.concatenate([built.gen_primary_host(cam, 0, 1024), built.gen_secondary_host(lt.triangles(), 9, 0, 1024)])
    flat = np.ascontiguousarray(rays).view(np.float32).reshape(-1, 8)
    for l in built.layouts():
        name = l["name"]
        pt = lt.encode(name)
        tb, tv = oracle.tree_bytes(pt), make_view(pt)
        want, _ = oracle.closest_hit(tb, rays)
        got = np.zeros(len(rays), built.HIT_DTYPE)
        assert shim.host_closest_hit(name.encode(), C.byref(tv), flat.ctypes.data, len(rays), got.ctypes.data) == 0, name
        assert np.array_equal(got["prim"], want["prim"]), name
        assert np.array_equal(got["t"].view(np.uint32), want["t"].view(np.uint32)), name
        assert (got["prim"] != built.MISS_PRIM).sum() > 256, name
