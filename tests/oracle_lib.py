"""ctypes binding of the CPU oracle (oracle/liboracle.so) — TEST INFRASTRUCTURE ONLY."""
import ctypes as C
import os

import numpy as np

import paper_2511_15028_b200 as sb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_PATH = os.path.join(ROOT, "oracle", "liboracle.so")


class TreeBytes(C.Structure):
    _fields_ = [("layout", C.c_char_p), ("nbuf", C.c_int), ("buf", C.c_void_p * 6), ("bytes", C.c_uint64 * 6), ("count", C.c_uint64 * 6),
                ("seg_base", (C.c_uint64 * 4) * 6), ("nglob", C.c_int), ("glob", (C.c_uint8 * 16) * 12), ("root0", C.c_uint64), ("carried", C.c_float * 6)]


class Oracle:
    def __init__(self):
        self.lib = C.CDLL(ORACLE_PATH)
        L = self.lib
        vp, u64, u32, i32, f32 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_float
        L.oracle_closest_hit.argtypes = [C.POINTER(TreeBytes), vp, u64, vp, vp, vp, i32]
        L.oracle_closest_point.argtypes = [C.POINTER(TreeBytes), vp, u64, vp, vp, vp, i32]
        L.oracle_brute_hit.argtypes = [vp, u64, vp, u64, vp]
        L.oracle_brute_point.argtypes = [vp, u64, vp, u64, vp]
        L.oracle_check_encoding.argtypes = [C.POINTER(TreeBytes), vp, u64, vp, vp, vp, vp, C.c_int32, C.c_char_p, i32, C.POINTER(u64)]
        L.oracle_check_encoding.restype = u64
        L.oracle_layout_name.restype = C.c_char_p
        L.oracle_layout_stride.argtypes = [C.c_char_p]
        L.oracle_layout_family.argtypes = [C.c_char_p]
        for n in ("fmul_rd", "fadd_rd", "fsub_rd", "fsub_ru", "fdiv_rd"):
            f = getattr(L, "oracle_" + n)
            f.argtypes = [f32, f32]
            f.restype = f32
        L.oracle_frcp_rd.argtypes = [f32]
        L.oracle_frcp_rd.restype = f32
        L.oracle_read_bits.argtypes = [vp, u64, u32]
        L.oracle_read_bits.restype = u64
        L.oracle_read_bits_naive.argtypes = [vp, u64, u32]
        L.oracle_read_bits_naive.restype = u64
        L.oracle_ray_aabb.argtypes = [vp, vp, f32, vp, vp, vp]
        L.oracle_ray_tri.argtypes = [vp, vp, f32, vp, vp]
        L.oracle_point_tri.argtypes = [vp, vp, vp, vp]
        L.oracle_ray_tri_batch.argtypes = [vp, vp, u64, i32, vp]
        L.oracle_ray_tri_batch.restype = None
        L.oracle_sqdist_point_aabb.argtypes = [vp, vp, vp]
        L.oracle_sqdist_point_aabb.restype = f32
        L.oracle_distmax_point_aabb.argtypes = [vp, vp, vp]
        L.oracle_distmax_point_aabb.restype = f32
        L.oracle_quantize_roundtrip.argtypes = [i32, vp, vp, vp, vp, vp, vp]
        L.oracle_collision_detection.argtypes = [C.POINTER(TreeBytes), C.POINTER(TreeBytes), vp, u64, vp]
        L.oracle_collision_detection.restype = C.c_int64
        L.oracle_brute_collisions.argtypes = [vp, u64, vp, u64, vp, u64]
        L.oracle_brute_collisions.restype = C.c_int64
        L.oracle_sat.argtypes = [vp, vp]

    # ------------------------------------------------------------------ tree marshalling
    def tree_bytes(self, ptree: "sb.PhysicalTree"):
        tb = TreeBytes()
        keep = [ptree]
        tb.layout = ptree.layout.encode()
        bufs = ptree.buffers()
        tb.nbuf = len(bufs)
        for i, b in enumerate(bufs):
            tb.buf[i] = b["ptr"]
            tb.bytes[i] = b["bytes"]
            tb.count[i] = b["count"]
            for s, v in enumerate(b["seg_bases"]):
                tb.seg_base[i][s] = v
        gl = ptree.globals()
        tb.nglob = len(gl)
        for i, g in enumerate(gl):
            for k in range(16):
                tb.glob[i][k] = g["raw"][k]
        r0, carried = ptree.root()
        tb.root0 = r0
        for k in range(6):
            tb.carried[k] = carried[k]
        tb._keep = keep
        return tb

    def logical_bytes(self, ltree: "sb.LogicalTree", kind: str):
        """kind: '@logical2' | '@logical-dop14' | '@logical8' — the reference's identity-oracle view."""
        tb = TreeBytes()
        tb.layout = kind.encode()
        tris = ltree.triangles()
        nodes = ltree.nodes()
        lo2, hi2 = ltree.dop()
        keep = [ltree, tris, nodes, lo2, hi2]
        tb.nbuf = 6
        tb.buf[0] = tris.ctypes.data
        tb.buf[1] = nodes.ctypes.data
        tb.buf[2] = lo2.ctypes.data
        tb.buf[3] = hi2.ctypes.data
        tb.root0 = 0
        if kind == "@logical8":
            wn, wl = ltree.wnodes(), ltree.wleaves()
            keep += [wn, wl]
            tb.buf[4] = wn.ctypes.data if wn.size else None
            tb.buf[5] = wl.ctypes.data if wl.size else None
            tb.root0 = ltree.wroot & 0xFFFFFFFF
        tb._keep = keep
        return tb

    # ------------------------------------------------------------------ queries
    def closest_hit(self, tb, rays, counters=False, nthreads=0):
        n = rays.shape[0]
        hits = np.empty(n, sb.HIT_DTYPE)
        status = np.zeros(n, np.uint32)
        ctr = np.zeros(n, sb.COUNTERS_DTYPE) if counters else None
        rc = self.lib.oracle_closest_hit(C.byref(tb), rays.ctypes.data, n, hits.ctypes.data, status.ctypes.data, ctr.ctypes.data if counters else None, nthreads)
        assert rc == 0, f"oracle_closest_hit rc={rc}"
        return (hits, status, ctr) if counters else (hits, status)

    def closest_point(self, tb, pts, counters=False, nthreads=0):
        pts = np.ascontiguousarray(pts, np.float32).reshape(-1, 3)
        n = pts.shape[0]
        out = np.empty(n, sb.CP_DTYPE)
        status = np.zeros(n, np.uint32)
        ctr = np.zeros(n, sb.COUNTERS_DTYPE) if counters else None
        rc = self.lib.oracle_closest_point(C.byref(tb), pts.ctypes.data, n, out.ctypes.data, status.ctypes.data, ctr.ctypes.data if counters else None, nthreads)
        assert rc == 0, f"oracle_closest_point rc={rc}"
        return (out, status, ctr) if counters else (out, status)

    def brute_hit(self, tris, rays):
        tris = np.ascontiguousarray(tris, np.float32).reshape(-1, 9)
        hits = np.empty(rays.shape[0], sb.HIT_DTYPE)
        self.lib.oracle_brute_hit(tris.ctypes.data, tris.shape[0], rays.ctypes.data, rays.shape[0], hits.ctypes.data)
        return hits

    def brute_point(self, tris, pts):
        tris = np.ascontiguousarray(tris, np.float32).reshape(-1, 9)
        pts = np.ascontiguousarray(pts, np.float32).reshape(-1, 3)
        out = np.empty(pts.shape[0], sb.CP_DTYPE)
        self.lib.oracle_brute_point(tris.ctypes.data, tris.shape[0], pts.ctypes.data, pts.shape[0], out.ctypes.data)
        return out

    def check_encoding(self, ptree, ltree):
        tb = self.tree_bytes(ptree)
        nodes = ltree.nodes()
        lo2, hi2 = ltree.dop()
        wn, wl = ltree.wnodes(), ltree.wleaves()
        msg = C.create_string_buffer(256)
        loose = C.c_uint64(0)
        bad = self.lib.oracle_check_encoding(C.byref(tb), nodes.ctypes.data, nodes.shape[0], lo2.ctypes.data, hi2.ctypes.data,
                                             wn.ctypes.data if wn.size else None, wl.ctypes.data if wl.size else None, ltree.wroot, msg, 256, C.byref(loose))
        return bad, msg.value.decode(), loose.value

    # ------------------------------------------------------------------ collision detection
    def collide(self, tb_a, tb_b, capacity=1 << 22):
        out = np.empty(capacity, np.uint64)
        stats = np.zeros(3, np.uint64)
        n = self.lib.oracle_collision_detection(C.byref(tb_a), C.byref(tb_b), out.ctypes.data, capacity, stats.ctypes.data)
        assert 0 <= n <= capacity, n
        return out[:n].copy(), dict(node_pairs=int(stats[0]), tri_tests=int(stats[1]))

    def brute_collisions(self, tris_a, tris_b, capacity=1 << 22):
        a = np.ascontiguousarray(tris_a, np.float32).reshape(-1, 9)
        b = np.ascontiguousarray(tris_b, np.float32).reshape(-1, 9)
        out = np.empty(capacity, np.uint64)
        n = self.lib.oracle_brute_collisions(a.ctypes.data, a.shape[0], b.ctypes.data, b.shape[0], out.ctypes.data, capacity)
        assert 0 <= n <= capacity
        return out[:n].copy()

    def ray_tri_batch(self, rays, tris9, method):
        """(b0, b1, b2, t, hit) per (ray, triangle) pair; method 0 = Moeller-Trumbore, 1 = Pluecker"""
        rays = np.ascontiguousarray(rays)
        tris = np.ascontiguousarray(tris9, np.float32)
        out = np.zeros((rays.shape[0], 5), np.float32)
        self.lib.oracle_ray_tri_batch(rays.ctypes.data, tris.ctypes.data, rays.shape[0], method, out.ctypes.data)
        return out

    def sat(self, a9, b9):
        a, b = np.ascontiguousarray(a9, np.float32), np.ascontiguousarray(b9, np.float32)
        return bool(self.lib.oracle_sat(a.ctypes.data, b.ctypes.data))
