"""The C-ABI boundary: the library loads, exports every symbol include/scion_b200.h declares, the
registry carries the reference's layout names/families/strides (corpus.cpp:11-25),
and — on a machine without a GPU — the query path fails loudly instead of falling back."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest


def test_library_exports_every_declared_symbol(built):
    sb = built
    L = sb.lib()
    names = sb.abi_symbols()
    assert len(names) >= 60
    exported = subprocess.run(["nm", "-D", "--defined-only", sb.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert hasattr(L, n), f"{n} declared in scion_b200.h but not exported"
        assert re.search(rf"\sT {n}$", exported, re.M), f"{n} is not a defined text symbol"
    assert L.scion_abi_version() == 1


def test_header_has_no_torch_or_cxx_types(built):
    hdr = open(os.path.join(os.path.dirname(built.LIB_PATH), "..", "include", "scion_b200.h")).read()
    code = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)  # declarations only, comments stripped
    assert "torch" not in code and "std::" not in code and "at::" not in code and "Tensor" not in code
    assert 'extern "C"' in hdr


# paper Table == corpus.cpp:11-25 == tests/test_plan.cpp:155-164
PAPER_STRIDES = {"ptr": 48, "pbrt": 32, "pbrt-align16": 32, "pbrt-q16": 16, "sg-eq": 12, "sg-eq-align16": 16, "bvh8": 256, "bvh8-q8": 136,
                 "bvh8-q8-ci": 104, "bvh8-q16": 184, "bvh8-q16-ci": 152,
                 # the table points authored here (not in the corpus)
                 "pbrt-soaos": 32, "pbrt-soaos-align16": 32, "pbrt-q16-soaos": 16, "bvh8-align16": 256, "bvh8-q8-align16": 144, "bvh8-q8-ci-align16": 112,
                 "bvh8-q16-align16": 192, "bvh8-q16-ci-align16": 160}
FAMILIES = {"dop14": 1, "bvh8": 2, "bvh8-q8": 2, "bvh8-q8-ci": 2, "bvh8-q16": 2, "bvh8-q16-ci": 2, "bvh8-align16": 2, "bvh8-q8-align16": 2, "bvh8-q8-ci-align16": 2,
            "bvh8-q16-align16": 2, "bvh8-q16-ci-align16": 2}


def test_registry_matches_reference_corpus(built):
    reg = {l["name"]: l for l in built.layouts()}
    corpus = ["identity", "ptr", "pbrt", "pbrt-align16", "pbrt-post", "pbrt-q16", "sg-eq", "sg-eq-align16", "shared-slab", "dop14", "bvh8", "bvh8-q8",
              "bvh8-q8-ci", "bvh8-q16", "bvh8-q16-ci"]
    for n in corpus:
        assert n in reg, f"corpus layout {n} missing from the registry"
    assert "pbrt-soa" in reg  # authored SoA point of BASELINE config 2
    for n, s in PAPER_STRIDES.items():
        assert reg[n]["node_stride"] == s, n
    for n, l in reg.items():
        assert l["family"] == FAMILIES.get(n, 0), n
        assert l["arity"] == (8 if l["family"] == 2 else 2)
        assert l["has_cpq"] == (l["family"] != 2)  # corpus.cpp:83
    assert reg["pbrt-q16"]["max_leaf"] == 15 and reg["shared-slab"]["max_leaf"] == 31 and reg["pbrt"]["max_leaf"] == 65535
    assert reg["bvh8-q8-ci"]["ref_bits"] == 32 and reg["bvh8"]["ref_bits"] == 64


def test_error_reporting(built):
    sb = built
    with pytest.raises(sb.ScionError) as e:
        sb.layout_plan("no-such-layout")
    assert e.value.code == sb.ERR_ARG
    with pytest.raises(sb.ScionError):
        sb.Scene.terrain(0)
    scene = sb.Scene.terrain(4, 1)
    lt = scene.build_sah(32, 4)
    with pytest.raises(sb.ScionError) as e:  # 8-wide layouts need the collapsed tree
        lt.encode("bvh8")
    assert e.value.code == sb.ERR_BUILD
    lt32 = scene.build_sah(32, 32)
    with pytest.raises(sb.ScionError) as e:  # u4 nprims cannot hold 32-primitive leaves
        lt32.encode("pbrt-q16")
    assert e.value.code == sb.ERR_BUILD and "capacity" in str(e.value)


def test_no_cpu_fallback_without_device(built):
    sb = built
    if sb.device_count() > 0:
        pytest.skip("a CUDA device is present")
    pt = sb.Scene.terrain(4, 1).build_sah(32, 4).encode("pbrt")
    with pytest.raises(sb.ScionError) as e:
        pt.upload(0)
    assert e.value.code == sb.ERR_NO_DEVICE


def test_partition_covers_range(built):
    sb = built
    for n in (0, 1, 7, 1 << 20, (1 << 28) + 3):
        for world in (1, 2, 3, 8):
            pos = 0
            for r in range(world):
                first, count = sb.partition(n, r, world)
                assert first == pos
                pos += count
            assert pos == n
