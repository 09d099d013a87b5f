"""The C-ABI library builds, loads without a GPU and exports every symbol include/nbt.h
declares; host-only helpers agree with the oracle's independent versions."""
import math
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import paper_2503_22588_b200 as nbt
from paper_2503_22588_b200 import _build
from nbt_inputs import FOV_H, FOV_V

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return nbt.lib()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "nbt.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nbt_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_binding_exports():
    assert declared_functions() == sorted(nbt.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", nbt.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (nbt_[a-z_0-9]+)", out))
    missing = set(declared_functions()) - exported
    assert not missing, missing
    for name in declared_functions():
        assert hasattr(lib, name)


def test_library_is_sm100a_only(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", nbt.LIB_PATH],
                         capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_no_oracle_in_product():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2503_22588_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text and "orc_" not in text, f
    deps = subprocess.run(["ldd", nbt.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in deps and "libcudart.so" not in deps      # static cudart, no oracle


def test_status_strings(lib):
    assert nbt.nbt_abi_version() == 2
    assert lib.nbt_status_string(2) == b"NBT_ERR_DEGENERATE"


def test_no_gpu_fails_loudly(lib):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(nbt.NbtError):
        nbt.Ctx(0)


@pytest.mark.parametrize("w,h", [(1, 1), (32, 24), (64, 48), (640, 480), (5, 1)])
def test_camera_from_fov_matches_oracle(lib, w, h):
    a = nbt.camera_from_fov(FOV_H, FOV_V, w, h)
    b = oracle.camera_from_fov(FOV_H, FOV_V, w, h)
    for f in ("width", "height", "fx", "fy", "cx", "cy", "add_corners", "tan_half_fov_h", "tan_half_fov_v"):
        assert getattr(a, f) == getattr(b, f), f


@pytest.mark.parametrize("s_g", [5, 50, 100, 200])
def test_camera_grid_scaling_matches_oracle(lib, s_g):
    a = nbt.camera_from_grid_scaling(FOV_H, FOV_V, 3.86, 0.01, s_g)
    b = oracle.camera_from_grid_scaling(FOV_H, FOV_V, 3.86, 0.01, s_g)
    assert (a.width, a.height, a.add_corners, a.fx) == (b.width, b.height, b.add_corners, b.fx)
    assert a.num_rays == oracle.num_rays(b)


def test_camera_rejects_bad_args(lib):
    with pytest.raises(nbt.NbtError):
        nbt.camera_from_fov(0.0, 1.0, 4, 4)
    with pytest.raises(nbt.NbtError):
        nbt.camera_from_fov(1.0, 1.0, 0, 4)
    with pytest.raises(nbt.NbtError):
        nbt.camera_from_grid_scaling(1.0, 1.0, 1.0, 0.01, 0.5)


def test_header_constants_match_the_binding():
    """Sizes the binding hard-codes equal the header's (#define / enum values)."""
    src = open(os.path.join(ROOT, "include", "nbt.h")).read()
    defs = dict(re.findall(r"#define\s+(NBT_[A-Z_]+)\s+(\d+)", src))
    assert int(defs["NBT_ID_TOTALS"]) == nbt.ID_TOTALS
    assert int(defs["NBT_PEER_HANDLE_BYTES"]) == nbt.PEER_HANDLE_BYTES
    kernels = dict((k, int(v)) for k, v in re.findall(r"(NBT_KERNEL_[A-Z_]+)\s*=\s*(\d+)", src))
    assert kernels["NBT_KERNEL_TRACE"] == nbt.KERNEL_TRACE
    assert kernels["NBT_KERNEL_MAP_UPDATE"] == nbt.KERNEL_MAP_UPDATE
    assert kernels["NBT_KERNEL_INTEGRATE"] == nbt.KERNEL_INTEGRATE


def test_missing_library_fails_loudly():
    """No CPU fallback: without libnbt.so the binding raises on first use."""
    code = ("import paper_2503_22588_b200 as nbt\n"
            "try:\n    nbt.lib()\nexcept ImportError as e:\n    print('raised', e)\n")
    env = dict(os.environ, NBT_LIB=os.path.join(ROOT, "no_such_libnbt.so"))
    r = subprocess.run(["python", "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "raised" in r.stdout, r.stdout + r.stderr
