"""scion-b200: B200-native traversal backend for Scion BVH layouts.

Thin ctypes binding over the C ABI in ``include/scion_b200.h`` (``libscion_b200.so``).  The
Python layer mirrors the operations the reference's harness/pybind module would expose for
this path (SPEC.md:367-423 exec-backend, :593-652 cli-harness; python/layoutc_module.cpp is a
placeholder in the reference) and adds nothing to the data path: every query runs in the CUDA
kernels of the shared library.  There is NO CPU fallback — if the library is missing, or no
CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ENV_HIT_VARIANT = int(os.environ.get("SCION_HIT_VARIANT", "0"))
LIB_PATH = os.environ.get("SCION_B200_LIB", os.path.join(_HERE, "libscion_b200.so"))  # env override: kernel-variant experiments


class ScionError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"scion error {code}: {message}")
        self.code = code


# status codes (scion_status)
OK, ERR_ARG, ERR_LAYOUT, ERR_BUILD, ERR_CUDA, ERR_NO_DEVICE, ERR_QUERY = range(7)
MISS_PRIM = 0xFFFFFFFF
FAMILY_BVH2, FAMILY_DOP14, FAMILY_BVH8 = 0, 1, 2
W_SENTINEL = -(2 ** 31)

def pack_rays(rays: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
    """scion_ray records -> the reference's packed Ray record, float32 [n, 7] = origin, direction, tmax (geometry.scion:4)"""
    v = rays.view(np.float32).reshape(-1, 8)
    if out is None:
        out = np.empty((v.shape[0], 7), np.float32)
    out[:, 0:3] = v[:, 0:3]
    out[:, 3:6] = v[:, 4:7]
    out[:, 6] = v[:, 3]
    return out


RAY_DTYPE = np.dtype([("ox", "f4"), ("oy", "f4"), ("oz", "f4"), ("tmax", "f4"), ("dx", "f4"), ("dy", "f4"), ("dz", "f4"), ("pad", "f4")])
HIT_DTYPE = np.dtype([("t", "f4"), ("prim", "u4")])
CP_DTYPE = np.dtype([("d2", "f4"), ("x", "f4"), ("y", "f4"), ("z", "f4"), ("prim", "u4")])
COUNTERS_DTYPE = np.dtype([("node_visits", "u4"), ("prim_tests", "u4"), ("cold_loads", "u4"), ("max_stack", "u4")])
LNODE_DTYPE = np.dtype([("lo", "f4", 3), ("hi", "f4", 3), ("left", "i4"), ("right", "i4"), ("first_prim", "u4"), ("nprims", "u4")])
WNODE_DTYPE = np.dtype([("lo", "f4", (8, 3)), ("hi", "f4", (8, 3)), ("child", "i4", 8)])
WLEAF_DTYPE = np.dtype([("first_prim", "u4"), ("nprims", "u4")])


class LayoutInfo(C.Structure):
    _fields_ = [("name", C.c_char_p), ("family", C.c_int), ("arity", C.c_int), ("node_stride", C.c_uint32), ("node_align", C.c_uint32),
                ("n_segments", C.c_uint32), ("ref_bits", C.c_uint32), ("max_leaf", C.c_uint32), ("has_cpq", C.c_int)]


class BufferDesc(C.Structure):
    _fields_ = [("name", C.c_char_p), ("data", C.c_void_p), ("bytes", C.c_uint64), ("count", C.c_uint64), ("seg_bases", C.POINTER(C.c_uint64)), ("n_seg_bases", C.c_uint32)]


class GlobalDesc(C.Structure):
    _fields_ = [("name", C.c_char_p), ("raw", C.c_uint8 * 16)]


class TreeDesc(C.Structure):
    _fields_ = [("layout", C.c_char_p), ("buffers", C.POINTER(BufferDesc)), ("nbuffers", C.c_uint32), ("globals", C.POINTER(GlobalDesc)), ("nglobals", C.c_uint32),
                ("root_ref", C.c_uint64), ("carried", C.c_float * 6), ("nprims", C.c_uint64)]


class CdStats(C.Structure):
    _fields_ = [("node_pairs", C.c_uint64), ("tri_tests", C.c_uint64), ("levels", C.c_uint64), ("max_frontier", C.c_uint64)]


PAIR_DTYPE = np.dtype([("a", "u4"), ("b", "u4")])


class Camera(C.Structure):
    _fields_ = [("eye", C.c_float * 3), ("target", C.c_float * 3), ("up", C.c_float * 3), ("fov_y_deg", C.c_float), ("width", C.c_uint32), ("height", C.c_uint32)]


_lib = None


def lib() -> C.CDLL:
    """Load the product library; fails loudly when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` (make -C paper_2511_15028_b200/csrc). "
                          "The B200 backend has no CPU fallback.")
    L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    vp, u64, u32, i32, cp = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_char_p
    P = C.POINTER
    sigs = {
        "scion_last_error": (cp, []),
        "scion_abi_version": (i32, []),
        "scion_free": (None, [vp]),
        "scion_kernel_launches": (u64, []),
        "scion_layout_count": (i32, []),
        "scion_layout_info_at": (i32, [i32, P(LayoutInfo)]),
        "scion_layout_registered_count": (i32, []),
        "scion_layout_registered_at": (i32, [i32, P(LayoutInfo)]),
        "scion_layout_find": (i32, [cp, P(LayoutInfo)]),
        "scion_layout_plan_json": (i32, [cp, P(vp)]),
        "scion_layout_emit_cuda": (i32, [cp, P(vp)]),
        "scion_layout_emit_c": (i32, [cp, P(vp)]),
        "scion_layout_stats_json": (i32, [cp, P(vp)]),
        "scion_compile_layout_text": (i32, [cp, P(vp), P(vp)]),
        "scion_scene_terrain": (i32, [u32, u64, P(vp)]),
        "scion_scene_sphere": (i32, [u32, u64, P(vp)]),
        "scion_scene_cloud": (i32, [u64, u64, P(vp)]),
        "scion_scene_from_triangles": (i32, [vp, u64, P(vp)]),
        "scion_scene_ntris": (u64, [vp]),
        "scion_scene_triangles": (vp, [vp]),
        "scion_scene_bounds": (None, [vp, P(C.c_float * 3), P(C.c_float * 3)]),
        "scion_scene_free": (None, [vp]),
        "scion_build_sah": (i32, [vp, u32, u32, u32, P(vp)]),
        "scion_build_median": (i32, [vp, u32, P(vp)]),
        "scion_ltree_collapse8": (i32, [vp]),
        "scion_ltree_from_arrays": (i32, [vp, u64, vp, u64, P(vp)]),
        "scion_ltree_nnodes": (u64, [vp]),
        "scion_ltree_nodes": (vp, [vp]),
        "scion_ltree_nprims": (u64, [vp]),
        "scion_ltree_triangles": (vp, [vp]),
        "scion_ltree_prim_ids": (vp, [vp]),
        "scion_ltree_dop_lo2": (vp, [vp]),
        "scion_ltree_dop_hi2": (vp, [vp]),
        "scion_ltree_depth": (u32, [vp]),
        "scion_ltree_nwnodes": (u64, [vp]),
        "scion_ltree_wnodes": (vp, [vp]),
        "scion_ltree_nwleaves": (u64, [vp]),
        "scion_ltree_wleaves": (vp, [vp]),
        "scion_ltree_wroot": (C.c_int32, [vp]),
        "scion_ltree_free": (None, [vp]),
        "scion_encode": (i32, [vp, cp, P(vp)]),
        "scion_encode_generated": (i32, [vp, cp, P(vp)]),
        "scion_layout_register": (i32, [cp, cp, cp, P(vp)]),
        "scion_layout_has_build": (i32, [cp]),
        "scion_ptree_layout": (cp, [vp]),
        "scion_ptree_nbuffers": (i32, [vp]),
        "scion_ptree_buffer": (i32, [vp, i32, P(cp), P(vp), P(u64), P(u64)]),
        "scion_ptree_segment_bases": (i32, [vp, i32, P(u64), i32]),
        "scion_ptree_nglobals": (i32, [vp]),
        "scion_ptree_global": (i32, [vp, i32, P(cp), P(C.c_uint8), P(u32)]),
        "scion_ptree_root": (i32, [vp, P(u64), P(C.c_float)]),
        "scion_ptree_total_bytes": (u64, [vp]),
        "scion_ptree_node_bytes": (u64, [vp]),
        "scion_ptree_corrupt": (i32, [vp, i32, u64, C.c_uint8]),
        "scion_ptree_save": (i32, [vp, cp]),
        "scion_ptree_load": (i32, [cp, P(vp)]),
        "scion_ptree_from_buffers": (i32, [P(TreeDesc), P(vp)]),
        "scion_tree_upload": (i32, [P(TreeDesc), i32, P(vp)]),
        "scion_ptree_free": (None, [vp]),
        "scion_device_count": (i32, [P(i32)]),
        "scion_dtree_upload": (i32, [vp, i32, P(vp)]),
        "scion_dtree_alloc_like": (i32, [vp, i32, P(vp)]),
        "scion_ptree_image_bytes": (u64, [vp]),
        "scion_dtree_upload_into": (i32, [vp, i32, vp, u64, P(vp)]),
        "scion_dtree_image": (i32, [vp, P(vp), P(u64)]),
        "scion_dtree_download_image": (i32, [vp, vp, u64]),
        "scion_ray_triangle": (i32, [vp, vp, u64, i32, vp, vp]),
        "scion_encode_device": (i32, [vp, cp, i32, P(vp)]),
        "scion_dtree_from_image": (i32, [cp, vp, u64, i32, i32, P(vp)]),
        "scion_dtree_free": (None, [vp]),
        "scion_closest_hit": (i32, [vp, vp, u64, vp, vp, vp, i32, vp]),
        "scion_closest_point": (i32, [vp, vp, u64, vp, vp, vp, i32, vp]),
        "scion_collision_detection": (i32, [vp, vp, vp, u64, P(u64), P(CdStats), u64, vp]),
        "scion_collision_detection_host": (i32, [vp, vp, vp, u64, P(u64), P(CdStats)]),
        "scion_closest_hit_host": (i32, [vp, vp, u64, vp, vp]),
        "scion_closest_hit_host_packed": (i32, [vp, vp, u64, vp, vp]),
        "scion_closest_hit_host_od": (i32, [vp, vp, u64, vp, vp]),
        "scion_rays_unpack": (i32, [vp, u64, vp, vp]),
        "scion_closest_point_host": (i32, [vp, vp, u64, vp, vp]),
        "scion_camera_default": (None, [P(C.c_float * 3), P(C.c_float * 3), i32, u32, u32, P(Camera)]),
        "scion_gen_primary": (i32, [P(Camera), u64, u64, vp, vp]),
        "scion_gen_secondary": (i32, [vp, u64, u64, u64, vp, vp]),
        "scion_gen_points": (i32, [P(C.c_float * 3), P(C.c_float * 3), u64, u64, u64, vp, vp]),
        "scion_gen_primary_host": (i32, [P(Camera), u64, u64, vp]),
        "scion_gen_secondary_host": (i32, [vp, u64, u64, u64, u64, vp]),
        "scion_gen_points_host": (i32, [P(C.c_float * 3), P(C.c_float * 3), u64, u64, u64, vp]),
        "scion_partition": (None, [u64, i32, i32, P(u64), P(u64)]),
        "scion_nccl_version": (i32, [P(i32)]),
        "scion_comm_unique_id": (i32, [P(C.c_uint8)]),
        "scion_comm_init_rank": (i32, [P(C.c_uint8), i32, i32, i32, P(vp)]),
        "scion_comm_init_all": (i32, [i32, P(i32), P(vp)]),
        "scion_comm_adopt": (i32, [vp, P(vp)]),
        "scion_comm_rank": (i32, [vp]),
        "scion_comm_size": (i32, [vp]),
        "scion_comm_device": (i32, [vp]),
        "scion_comm_free": (None, [vp]),
        "scion_dtree_broadcast": (i32, [vp, i32, vp, vp, P(vp)]),
        "scion_dtree_broadcast_all": (i32, [vp, i32, P(vp), i32, P(vp), P(vp)]),
        "scion_gather_results": (i32, [vp, vp, u64, u32, vp, vp]),
        "scion_gather_results_all": (i32, [P(vp), i32, P(vp), u64, u32, P(vp), P(vp)]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)  # AttributeError here == the library does not export a declared symbol
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


ABI_SYMBOLS = None  # filled lazily by abi_symbols()


def abi_symbols():
    """Every function name declared in include/scion_b200.h (parsed from the header text)."""
    import re
    hdr = os.path.join(os.path.dirname(_HERE), "include", "scion_b200.h")
    text = open(hdr).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(scion_[a-z0-9_]+)\s*\(", text)))


def _check(rc: int):
    if rc != 0:
        raise ScionError(rc, lib().scion_last_error().decode())


def _take_string(p: C.c_void_p) -> str:
    s = C.string_at(p).decode()
    lib().scion_free(p)
    return s


def _f3(v):
    return (C.c_float * 3)(*[float(x) for x in v])


def _np_view(ptr, count, dtype, owner=None):
    """Zero-copy numpy view of library-owned memory; the view keeps `owner` (the Python handle object) alive."""
    if not ptr or count == 0:
        return np.zeros(0, dtype=dtype)
    nbytes = int(count) * np.dtype(dtype).itemsize
    buf = (C.c_uint8 * nbytes).from_address(ptr)
    buf._owner = owner  # numpy array -> ctypes buffer -> owner
    return np.frombuffer(buf, dtype=dtype)


# --------------------------------------------------------------------------------------- registry
def layouts():
    out = []
    n = lib().scion_layout_count()
    for i in range(n):
        info = LayoutInfo()
        _check(lib().scion_layout_info_at(i, C.byref(info)))
        out.append(dict(name=info.name.decode(), family=info.family, arity=info.arity, node_stride=info.node_stride, node_align=info.node_align,
                        n_segments=info.n_segments, ref_bits=info.ref_bits, max_leaf=info.max_leaf, has_cpq=bool(info.has_cpq)))
    return out


def registered_layouts():
    """layouts compiled and registered at run time (register_layout), in registration order"""
    out = []
    for i in range(lib().scion_layout_registered_count()):
        info = LayoutInfo()
        _check(lib().scion_layout_registered_at(i, C.byref(info)))
        out.append(dict(name=info.name.decode(), family=info.family, arity=info.arity, node_stride=info.node_stride, node_align=info.node_align,
                        n_segments=info.n_segments, ref_bits=info.ref_bits, max_leaf=info.max_leaf, has_cpq=bool(info.has_cpq)))
    return out


def layout_info(name: str) -> dict:
    for l in layouts() + registered_layouts():
        if l["name"] == name:
            return l
    raise ScionError(ERR_ARG, f"unknown layout '{name}'")


def layout_plan(name: str) -> dict:
    p = C.c_void_p()
    _check(lib().scion_layout_plan_json(name.encode(), C.byref(p)))
    return json.loads(_take_string(p))


def emit_cuda(name: str) -> str:
    p = C.c_void_p()
    _check(lib().scion_layout_emit_cuda(name.encode(), C.byref(p)))
    return _take_string(p)


def emit_c(name: str) -> str:
    """C11 header with the typed packed node records of the layout, their static assertions and the slot table."""
    p = C.c_void_p()
    _check(lib().scion_layout_emit_c(name.encode(), C.byref(p)))
    return _take_string(p)


def layout_stats(name: str) -> dict:
    """op counts of the layout's decode per variant (loads, arithmetic, casts, ...): the --dump-stats report"""
    p = C.c_void_p()
    _check(lib().scion_layout_stats_json(name.encode(), C.byref(p)))
    return json.loads(_take_string(p))


def compile_layout_text(source: str):
    """Layout compiler front door: .scion text -> (plan dict, CUDA header text)."""
    pj, pc = C.c_void_p(), C.c_void_p()
    _check(lib().scion_compile_layout_text(source.encode(), C.byref(pj), C.byref(pc)))
    return json.loads(_take_string(pj)), _take_string(pc)


def register_layout(name: str, source: str, work_dir: Optional[str] = None) -> str:
    """Open-world layouts: compile `source` (.scion text with a layout and its build block) at run time — front end,
    emit_cuda, nvcc, g++ — and register it under `name`; returns the build log.  About a minute; needs nvcc."""
    log = C.c_void_p()
    rc = lib().scion_layout_register(name.encode(), source.encode(), work_dir.encode() if work_dir else None, C.byref(log))
    text = _take_string(log) if log.value else ""
    if rc != 0:
        _check(rc)
    return text


# --------------------------------------------------------------------------------------- scene tools
class Scene:
    def __init__(self, handle):
        self._h = handle

    @staticmethod
    def terrain(grid: int, seed: int = 1) -> "Scene":
        h = C.c_void_p()
        _check(lib().scion_scene_terrain(grid, seed, C.byref(h)))
        return Scene(h)

    @staticmethod
    def sphere(grid: int, seed: int = 1) -> "Scene":
        h = C.c_void_p()
        _check(lib().scion_scene_sphere(grid, seed, C.byref(h)))
        return Scene(h)

    @staticmethod
    def cloud(npoints: int, seed: int = 1) -> "Scene":
        h = C.c_void_p()
        _check(lib().scion_scene_cloud(npoints, seed, C.byref(h)))
        return Scene(h)

    @staticmethod
    def from_triangles(tris) -> "Scene":
        a = np.ascontiguousarray(tris, dtype=np.float32).reshape(-1, 9)
        h = C.c_void_p()
        _check(lib().scion_scene_from_triangles(a.ctypes.data, a.shape[0], C.byref(h)))
        return Scene(h)

    @property
    def ntris(self) -> int:
        return lib().scion_scene_ntris(self._h)

    def triangles(self) -> np.ndarray:
        return _np_view(lib().scion_scene_triangles(self._h), self.ntris * 9, np.float32, self).reshape(-1, 9)

    def bounds(self):
        lo, hi = (C.c_float * 3)(), (C.c_float * 3)()
        lib().scion_scene_bounds(self._h, C.byref(lo), C.byref(hi))
        return np.array(lo[:], np.float32), np.array(hi[:], np.float32)

    def build_sah(self, bins: int = 32, max_leaf: int = 4, max_depth: int = 0) -> "LogicalTree":
        h = C.c_void_p()
        _check(lib().scion_build_sah(self._h, bins, max_leaf, max_depth, C.byref(h)))
        return LogicalTree(h)

    def build_median(self, max_leaf: int = 1) -> "LogicalTree":
        h = C.c_void_p()
        _check(lib().scion_build_median(self._h, max_leaf, C.byref(h)))
        return LogicalTree(h)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.scion_scene_free(self._h)
            self._h = None


class LogicalTree:
    def __init__(self, handle):
        self._h = handle

    @staticmethod
    def from_arrays(nodes: np.ndarray, tris) -> "LogicalTree":
        """Import an externally built binary LogicalTree (nodes: LNODE_DTYPE, root = node 0)."""
        n = np.ascontiguousarray(nodes, dtype=LNODE_DTYPE)
        t = np.ascontiguousarray(tris, dtype=np.float32).reshape(-1, 9)
        h = C.c_void_p()
        _check(lib().scion_ltree_from_arrays(n.ctypes.data, n.shape[0], t.ctypes.data, t.shape[0], C.byref(h)))
        return LogicalTree(h)

    def collapse8(self) -> "LogicalTree":
        _check(lib().scion_ltree_collapse8(self._h))
        return self

    @property
    def nnodes(self) -> int:
        return lib().scion_ltree_nnodes(self._h)

    @property
    def nprims(self) -> int:
        return lib().scion_ltree_nprims(self._h)

    @property
    def depth(self) -> int:
        return lib().scion_ltree_depth(self._h)

    def nodes(self) -> np.ndarray:
        return _np_view(lib().scion_ltree_nodes(self._h), self.nnodes, LNODE_DTYPE, self)

    def triangles(self) -> np.ndarray:
        return _np_view(lib().scion_ltree_triangles(self._h), self.nprims * 9, np.float32, self).reshape(-1, 9)

    def prim_ids(self) -> np.ndarray:
        return _np_view(lib().scion_ltree_prim_ids(self._h), self.nprims, np.uint32, self)

    def dop(self):
        n = self.nnodes
        return (_np_view(lib().scion_ltree_dop_lo2(self._h), n * 4, np.float32, self).reshape(-1, 4),
                _np_view(lib().scion_ltree_dop_hi2(self._h), n * 4, np.float32, self).reshape(-1, 4))

    def wnodes(self) -> np.ndarray:
        return _np_view(lib().scion_ltree_wnodes(self._h), lib().scion_ltree_nwnodes(self._h), WNODE_DTYPE, self)

    def wleaves(self) -> np.ndarray:
        return _np_view(lib().scion_ltree_wleaves(self._h), lib().scion_ltree_nwleaves(self._h), WLEAF_DTYPE, self)

    @property
    def wroot(self) -> int:
        return lib().scion_ltree_wroot(self._h)

    def encode(self, layout: str) -> "PhysicalTree":
        h = C.c_void_p()
        _check(lib().scion_encode(self._h, layout.encode(), C.byref(h)))
        return PhysicalTree(h)

    def encode_generated(self, layout: str) -> "PhysicalTree":
        """build_physical through the layout's own `build` block, compiled by the layout compiler (constructor
        specialisation); must be byte-identical to encode(layout)."""
        h = C.c_void_p()
        _check(lib().scion_encode_generated(self._h, layout.encode(), C.byref(h)))
        return PhysicalTree(h)

    def encode_device(self, layout: str, device: int = 0) -> "DeviceTree":
        """build_physical on the GPU: byte-identical to encode(layout).upload(device)."""
        h = C.c_void_p()
        _check(lib().scion_encode_device(self._h, layout.encode(), device, C.byref(h)))
        return DeviceTree(h, device)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.scion_ltree_free(self._h)
            self._h = None


class PhysicalTree:
    """Host PhysicalTree: buffer id -> bytes, globals, root reference."""

    def __init__(self, handle):
        self._h = handle

    @property
    def layout(self) -> str:
        return lib().scion_ptree_layout(self._h).decode()

    def buffers(self):
        out = []
        for i in range(lib().scion_ptree_nbuffers(self._h)):
            name, data, nbytes, count = C.c_char_p(), C.c_void_p(), C.c_uint64(), C.c_uint64()
            _check(lib().scion_ptree_buffer(self._h, i, C.byref(name), C.byref(data), C.byref(nbytes), C.byref(count)))
            bases = (C.c_uint64 * 4)()
            ns = lib().scion_ptree_segment_bases(self._h, i, bases, 4)
            out.append(dict(name=name.value.decode(), data=_np_view(data.value, nbytes.value, np.uint8, self), ptr=data.value, bytes=nbytes.value,
                            count=count.value, seg_bases=list(bases[:ns])))
        return out

    def globals(self):
        out = []
        for i in range(lib().scion_ptree_nglobals(self._h)):
            name, raw, nb = C.c_char_p(), (C.c_uint8 * 16)(), C.c_uint32()
            _check(lib().scion_ptree_global(self._h, i, C.byref(name), raw, C.byref(nb)))
            out.append(dict(name=name.value.decode(), raw=bytes(raw), nbytes=nb.value))
        return out

    def root(self):
        r, carried = C.c_uint64(), (C.c_float * 6)()
        _check(lib().scion_ptree_root(self._h, C.byref(r), carried))
        return r.value, list(carried)

    @property
    def total_bytes(self) -> int:
        return lib().scion_ptree_total_bytes(self._h)

    @property
    def node_bytes(self) -> int:
        return lib().scion_ptree_node_bytes(self._h)

    def save(self, path: str):
        """Write the PhysicalTree container file."""
        _check(lib().scion_ptree_save(self._h, path.encode()))

    @staticmethod
    def load(path: str) -> "PhysicalTree":
        h = C.c_void_p()
        _check(lib().scion_ptree_load(path.encode(), C.byref(h)))
        return PhysicalTree(h)

    @staticmethod
    def _desc(layout: str, buffers, globals_, root_ref: int, carried=None, nprims: int = 0):
        """TreeDesc for scion_ptree_from_buffers: buffers = [{name, data (uint8 array), count, seg_bases?}], globals_ = [{name, raw}]."""
        keep = []
        bd = (BufferDesc * max(1, len(buffers)))()
        for i, b in enumerate(buffers):
            data = np.ascontiguousarray(b["data"], dtype=np.uint8)
            keep.append(data)
            bd[i].name = b["name"].encode()
            bd[i].data = data.ctypes.data if data.size else None
            bd[i].bytes = b.get("bytes", data.size)
            bd[i].count = b.get("count", 0)
            sb_ = b.get("seg_bases")
            if sb_ is not None:
                arr = (C.c_uint64 * max(1, len(sb_)))(*sb_)
                keep.append(arr)
                bd[i].seg_bases = arr
                bd[i].n_seg_bases = len(sb_)
        gd = (GlobalDesc * max(1, len(globals_)))()
        for i, g in enumerate(globals_):
            gd[i].name = g["name"].encode()
            raw = bytes(g["raw"])[:16].ljust(16, b"\0")
            for k in range(16):
                gd[i].raw[k] = raw[k]
        d = TreeDesc()
        d.layout = layout.encode()
        d.buffers, d.nbuffers = bd, len(buffers)
        d.globals, d.nglobals = gd, len(globals_)
        d.root_ref = root_ref
        for k in range(6):
            d.carried[k] = float(carried[k]) if carried is not None else 0.0
        d.nprims = nprims
        d._keep = (keep, bd, gd)
        return d

    @staticmethod
    def from_buffers(layout: str, buffers, globals_, root_ref: int, carried=None, nprims: int = 0) -> "PhysicalTree":
        """In-memory import of a PhysicalTree built elsewhere (validated against the plan; the library copies)."""
        d = PhysicalTree._desc(layout, buffers, globals_, root_ref, carried, nprims)
        h = C.c_void_p()
        _check(lib().scion_ptree_from_buffers(C.byref(d), C.byref(h)))
        return PhysicalTree(h)

    def export(self):
        """(layout, buffers, globals, root_ref, carried) — the arguments from_buffers() takes."""
        r0, carried = self.root()
        return self.layout, [dict(name=b["name"], data=b["data"], count=b["count"], seg_bases=b["seg_bases"]) for b in self.buffers()], self.globals(), r0, carried

    def corrupt(self, buffer: int, byte_offset: int, xor_mask: int = 0xFF):
        _check(lib().scion_ptree_corrupt(self._h, buffer, byte_offset, xor_mask))

    def upload(self, device: int = 0) -> "DeviceTree":
        h = C.c_void_p()
        _check(lib().scion_dtree_upload(self._h, device, C.byref(h)))
        return DeviceTree(h, device)

    @property
    def image_bytes(self) -> int:
        return lib().scion_ptree_image_bytes(self._h)

    def upload_into(self, device: int, d_image: int, nbytes: int) -> "DeviceTree":
        """Upload into caller-owned device memory (e.g. a torch tensor that is then broadcast)."""
        h = C.c_void_p()
        _check(lib().scion_dtree_upload_into(self._h, device, d_image, nbytes, C.byref(h)))
        return DeviceTree(h, device)

    def alloc_like(self, device: int = 0) -> "DeviceTree":
        h = C.c_void_p()
        _check(lib().scion_dtree_alloc_like(self._h, device, C.byref(h)))
        return DeviceTree(h, device)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.scion_ptree_free(self._h)
            self._h = None


def tree_upload(layout: str, buffers, globals_, root_ref: int, carried=None, device: int = 0) -> "DeviceTree":
    """scion_tree_upload: in-memory import + upload in one call."""
    d = PhysicalTree._desc(layout, buffers, globals_, root_ref, carried)
    h = C.c_void_p()
    _check(lib().scion_tree_upload(C.byref(d), device, C.byref(h)))
    return DeviceTree(h, device)


def device_count() -> int:
    n = C.c_int()
    rc = lib().scion_device_count(C.byref(n))
    return n.value if rc == 0 else 0


class DeviceTree:
    """PhysicalTree resident on one GPU; immutable, safe to query from several streams."""

    def __init__(self, handle, device):
        self._h = handle
        self.device = device

    def image(self):
        p, n = C.c_void_p(), C.c_uint64()
        _check(lib().scion_dtree_image(self._h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def download_image(self) -> np.ndarray:
        """The whole device image (1 KB header + every plan buffer) as host bytes."""
        _, n = self.image()
        out = np.empty(n, np.uint8)
        _check(lib().scion_dtree_download_image(self._h, out.ctypes.data, n))
        return out

    @staticmethod
    def from_image(d_ptr: int, nbytes: int, device: int, layout: Optional[str] = None, adopt: bool = False) -> "DeviceTree":
        h = C.c_void_p()
        _check(lib().scion_dtree_from_image(layout.encode() if layout else None, d_ptr, nbytes, device, 1 if adopt else 0, C.byref(h)))
        return DeviceTree(h, device)

    # device-pointer entry points (asynchronous on `stream`)
    def closest_hit(self, d_rays: int, n: int, d_hits: int, d_status: int = 0, d_counters: int = 0, variant: int = 0, stream: int = 0):
        if variant == 0 and _ENV_HIT_VARIANT:  # experiments: run a whole bench / profile on a selectable kernel variant
            variant = _ENV_HIT_VARIANT
        _check(lib().scion_closest_hit(self._h, d_rays, n, d_hits, d_status or None, d_counters or None, variant, stream or None))

    def closest_point(self, d_points: int, n: int, d_out: int, d_status: int = 0, d_counters: int = 0, variant: int = 0, stream: int = 0):
        _check(lib().scion_closest_point(self._h, d_points, n, d_out, d_status or None, d_counters or None, variant, stream or None))

    # host-buffer entry points (H2D + kernel + D2H inside the call)
    def closest_hit_host(self, rays: np.ndarray, hits: Optional[np.ndarray] = None, status: Optional[np.ndarray] = None):
        assert rays.dtype == RAY_DTYPE and rays.flags.c_contiguous
        n = rays.shape[0]
        if hits is None:
            hits = np.empty(n, HIT_DTYPE)
        _check(lib().scion_closest_hit_host(self._h, rays.ctypes.data, n, hits.ctypes.data, status.ctypes.data if status is not None else None))
        return hits

    def closest_hit_host_packed(self, rays7: np.ndarray, hits: Optional[np.ndarray] = None, status: Optional[np.ndarray] = None):
        """rays as the reference's packed Ray record: float32 [n, 7] = origin, direction, tmax (geometry.scion:4)"""
        assert rays7.dtype == np.float32 and rays7.flags.c_contiguous and rays7.ndim == 2 and rays7.shape[1] == 7
        n = rays7.shape[0]
        if hits is None:
            hits = np.empty(n, HIT_DTYPE)
        _check(lib().scion_closest_hit_host_packed(self._h, rays7.ctypes.data, n, hits.ctypes.data, status.ctypes.data if status is not None else None))
        return hits

    def closest_hit_host_od(self, rays6: np.ndarray, hits: Optional[np.ndarray] = None, status: Optional[np.ndarray] = None):
        """rays with the DSL's default tmax = inf: float32 [n, 6] = origin, direction"""
        assert rays6.dtype == np.float32 and rays6.flags.c_contiguous and rays6.ndim == 2 and rays6.shape[1] == 6
        n = rays6.shape[0]
        if hits is None:
            hits = np.empty(n, HIT_DTYPE)
        _check(lib().scion_closest_hit_host_od(self._h, rays6.ctypes.data, n, hits.ctypes.data, status.ctypes.data if status is not None else None))
        return hits

    def closest_point_host(self, points: np.ndarray, out: Optional[np.ndarray] = None, status: Optional[np.ndarray] = None):
        pts = np.ascontiguousarray(points, np.float32).reshape(-1, 3)
        n = pts.shape[0]
        if out is None:
            out = np.empty(n, CP_DTYPE)
        _check(lib().scion_closest_point_host(self._h, pts.ctypes.data, n, out.ctypes.data, status.ctypes.data if status is not None else None))
        return out

    def collide_host(self, other: "DeviceTree", capacity: int = 1 << 20):
        """collision_detection(self, other): returns (pairs sorted as a set, true count, stats dict)."""
        out = np.empty(capacity, PAIR_DTYPE)
        n, st = C.c_uint64(), CdStats()
        _check(lib().scion_collision_detection_host(self._h, other._h, out.ctypes.data, capacity, C.byref(n), C.byref(st)))
        m = min(n.value, capacity)
        keys = np.sort((out["a"][:m].astype(np.uint64) << np.uint64(32)) | out["b"][:m].astype(np.uint64))
        return keys, n.value, dict(node_pairs=st.node_pairs, tri_tests=st.tri_tests, levels=st.levels, max_frontier=st.max_frontier)

    def collide(self, other: "DeviceTree", d_out: int, capacity: int, frontier_capacity: int = 0, stream: int = 0):
        n, st = C.c_uint64(), CdStats()
        _check(lib().scion_collision_detection(self._h, other._h, d_out, capacity, C.byref(n), C.byref(st), frontier_capacity, stream or None))
        return n.value, dict(node_pairs=st.node_pairs, tri_tests=st.tri_tests, levels=st.levels, max_frontier=st.max_frontier)

    def gen_secondary(self, seed: int, first: int, n: int, d_rays: int, stream: int = 0):
        _check(lib().scion_gen_secondary(self._h, seed, first, n, d_rays, stream or None))

    def free(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.scion_dtree_free(self._h)
            self._h = None

    def __del__(self):
        self.free()


TRIHIT_DTYPE = np.dtype([("b0", np.float32), ("b1", np.float32), ("b2", np.float32), ("t", np.float32), ("hit", np.uint32)])
TRI_MT, TRI_PLUECKER = 0, 1


def ray_triangle(d_rays: int, d_tris9: int, n: int, method: int, d_out: int, stream: int = 0):
    """Batch ray/triangle test on the device: Moeller-Trumbore (0) or Pluecker coordinates (1), geometry.scion:25-55."""
    _check(lib().scion_ray_triangle(d_rays, d_tris9, n, method, d_out, stream or None))


# --------------------------------------------------------------------------------------- generators
def default_camera(lo, hi, look_down_y: bool, width: int, height: int) -> Camera:
    cam = Camera()
    lib().scion_camera_default(C.byref(_f3(lo)), C.byref(_f3(hi)), 1 if look_down_y else 0, width, height, C.byref(cam))
    return cam


def gen_primary(cam: Camera, first: int, n: int, d_rays: int, stream: int = 0):
    _check(lib().scion_gen_primary(C.byref(cam), first, n, d_rays, stream or None))


def gen_points(lo, hi, seed: int, first: int, n: int, d_points: int, stream: int = 0):
    _check(lib().scion_gen_points(C.byref(_f3(lo)), C.byref(_f3(hi)), seed, first, n, d_points, stream or None))


def gen_primary_host(cam: Camera, first: int, n: int) -> np.ndarray:
    rays = np.empty(n, RAY_DTYPE)
    _check(lib().scion_gen_primary_host(C.byref(cam), first, n, rays.ctypes.data))
    return rays


def gen_secondary_host(tris: np.ndarray, seed: int, first: int, n: int) -> np.ndarray:
    t = np.ascontiguousarray(tris, np.float32).reshape(-1, 9)
    rays = np.empty(n, RAY_DTYPE)
    _check(lib().scion_gen_secondary_host(t.ctypes.data, t.shape[0], seed, first, n, rays.ctypes.data))
    return rays


def gen_points_host(lo, hi, seed: int, first: int, n: int) -> np.ndarray:
    pts = np.empty((n, 3), np.float32)
    _check(lib().scion_gen_points_host(C.byref(_f3(lo)), C.byref(_f3(hi)), seed, first, n, pts.ctypes.data))
    return pts


def partition(n: int, rank: int, nranks: int):
    """Contiguous query partition [first, first+count) of rank `rank`."""
    a, b = C.c_uint64(), C.c_uint64()
    lib().scion_partition(n, rank, nranks, C.byref(a), C.byref(b))
    return a.value, b.value


# --------------------------------------------------------------------------------------- multi-GPU
NCCL_UNIQUE_ID_BYTES = 128


def nccl_version() -> int:
    v = C.c_int()
    _check(lib().scion_nccl_version(C.byref(v)))
    return v.value


class Comm:
    """One NCCL communicator bound to one device (scion_comm): tree replication and result gather of the C ABI."""

    def __init__(self, handle):
        self._h = handle

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * NCCL_UNIQUE_ID_BYTES)()
        _check(lib().scion_comm_unique_id(buf))
        return bytes(buf)

    @staticmethod
    def init_rank(unique_id: bytes, nranks: int, rank: int, device: int) -> "Comm":
        assert len(unique_id) == NCCL_UNIQUE_ID_BYTES
        buf = (C.c_uint8 * NCCL_UNIQUE_ID_BYTES)(*unique_id)
        h = C.c_void_p()
        _check(lib().scion_comm_init_rank(buf, nranks, rank, device, C.byref(h)))
        return Comm(h)

    @staticmethod
    def init_all(ndev: int, devices=None):
        out = (C.c_void_p * ndev)()
        devs = (C.c_int * ndev)(*devices) if devices is not None else None
        _check(lib().scion_comm_init_all(ndev, devs, out))
        return [Comm(C.c_void_p(out[i])) for i in range(ndev)]

    @property
    def rank(self) -> int:
        return lib().scion_comm_rank(self._h)

    @property
    def size(self) -> int:
        return lib().scion_comm_size(self._h)

    @property
    def device(self) -> int:
        return lib().scion_comm_device(self._h)

    def broadcast_tree(self, tree: Optional["DeviceTree"], root: int = 0, stream: int = 0) -> "DeviceTree":
        """Collective.  The root passes its resident tree, every other rank None; all ranks get a tree."""
        h = C.c_void_p()
        _check(lib().scion_dtree_broadcast(tree._h if tree is not None else None, root, self._h, stream or None, C.byref(h)))
        if tree is not None:
            return tree
        return DeviceTree(h, self.device)

    def gather(self, d_part: int, n_total: int, record_bytes: int, d_full: int, stream: int = 0):
        _check(lib().scion_gather_results(self._h, d_part, n_total, record_bytes, d_full, stream or None))

    def free(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.scion_comm_free(self._h)
            self._h = None

    def __del__(self):
        self.free()


def broadcast_tree_all(tree: "DeviceTree", root: int, comms) -> list:
    """single-process form (Comm.init_all): returns one DeviceTree per communicator, trees[root] is `tree`"""
    n = len(comms)
    arr = (C.c_void_p * n)(*[c._h for c in comms])
    out = (C.c_void_p * n)()
    _check(lib().scion_dtree_broadcast_all(tree._h, root, arr, n, None, out))
    return [tree if i == root else DeviceTree(C.c_void_p(out[i]), comms[i].device) for i in range(n)]


def gather_results_all(comms, d_parts, n_total: int, record_bytes: int, d_fulls):
    n = len(comms)
    arr = (C.c_void_p * n)(*[c._h for c in comms])
    parts = (C.c_void_p * n)(*d_parts)
    fulls = (C.c_void_p * n)(*d_fulls)
    _check(lib().scion_gather_results_all(arr, n, parts, n_total, record_bytes, fulls, None))


def kernel_launches() -> int:
    return lib().scion_kernel_launches()


def seed_from_env(default: int) -> int:
    """LAYOUTC_SEED overrides the configured seed."""
    v = os.environ.get("LAYOUTC_SEED")
    return int(v, 0) if v else default
