"""CPU-side checks of the C ABI boundary (no compute calls; no GPU needed):
libvrs.so loads, exports every function include/vrs.h declares, and the
ctypes structures of the binding match the C layout of the header."""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vrs.h")


@pytest.fixture(scope="module")
def vrsmod():
    from paper_2505_10144_b200 import build
    build.build()
    import paper_2505_10144_b200.vrs as v
    return v


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^VRS_API\s+[\w\s\*]+?\b(vrs_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("vrs_create", "vrs_upload_gaussians", "vrs_render_views", "vrs_get_frame_stats", "vrs_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol(vrsmod):
    L = vrsmod.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", vrsmod.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (vrs_\w+)", out))
    for name in declared_functions():
        assert name in exported, name
        assert hasattr(L, name)
    assert set(vrsmod.EXPORTS) == set(declared_functions())
    assert L.vrs_abi_version() == 1


def test_library_exports_only_the_abi(vrsmod):
    out = subprocess.run(["nm", "-D", "--defined-only", vrsmod.LIB_PATH], capture_output=True, text=True).stdout
    text_syms = re.findall(r" T (\S+)", out)
    own = [s for s in text_syms if s.startswith("vrs_") or "vrs" in s]
    assert all(s.startswith("vrs_") for s in own), own


def test_struct_layout_matches_header(vrsmod, tmp_path):
    prog = tmp_path / "layout.c"
    prog.write_text(f'''
#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu\\n", sizeof(vrs_config), sizeof(vrs_camera), sizeof(vrs_fovea), sizeof(vrs_frame_stats));
  printf("%zu %zu %zu\\n", offsetof(vrs_config, near_plane), offsetof(vrs_camera, mask_slot), offsetof(vrs_frame_stats, stage_ms));
  return 0; }}
''')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(prog)], check=True)
    lines = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    sizes = [int(x) for x in lines[0].split()]
    offs = [int(x) for x in lines[1].split()]
    assert sizes == [C.sizeof(vrsmod.vrs_config), C.sizeof(vrsmod.vrs_camera), C.sizeof(vrsmod.vrs_fovea),
                     C.sizeof(vrsmod.vrs_frame_stats)]
    assert offs == [vrsmod.vrs_config.near_plane.offset, vrsmod.vrs_camera.mask_slot.offset,
                    vrsmod.vrs_frame_stats.stage_ms.offset]


def test_create_without_gpu_fails_cleanly(vrsmod):
    """No GPU here: vrs_create must return an error status, never crash."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = vrsmod.vrs_config()
    cfg.max_views, cfg.max_gaussians, cfg.max_pairs, cfg.max_width, cfg.max_height = 1, 10, 100, 16, 16
    cfg.window_k, cfg.assign_tile, cfg.near_plane = 16, 16, 0.2
    h = C.c_void_p()
    st = vrsmod.lib().vrs_create(C.byref(cfg), C.byref(h))
    assert st != 0


def test_invalid_config_rejected(vrsmod):
    cfg = vrsmod.vrs_config()
    cfg.max_views = 0  # invalid
    h = C.c_void_p()
    assert vrsmod.lib().vrs_create(C.byref(cfg), C.byref(h)) == vrsmod.VRS_E_INVALID_ARG


def test_product_has_no_oracle_dependency():
    """The product package never imports or links the oracle (DESIGN "Oracle")."""
    pkg = os.path.join(ROOT, "paper_2505_10144_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "oracle.h" not in txt and "liboracle" not in txt, f


def test_binding_validates_buffers_before_the_abi(vrsmod):
    """the binding rejects mismatched output buffers (element count,
    dtype of the output format, device) before calling into libvrs."""
    import numpy as np
    import torch

    class Fake:
        device = 0
        out_fmt = 0

    chk = vrsmod.Renderer._check_buffers
    px = 16
    # CPU tensors are not device buffers
    with pytest.raises(ValueError, match="cuda"):
        chk(Fake(), px, torch.zeros((px, 4)), torch.zeros(px))
    # wrong element count / dtype (host path, where CPU buffers are right)
    with pytest.raises(ValueError, match="need 64"):
        chk(Fake(), px, torch.zeros((px - 1, 4)), torch.zeros(px), host=True)
    with pytest.raises(ValueError, match="float16"):
        f = Fake()
        f.out_fmt = 1
        chk(f, px, torch.zeros((px, 4), dtype=torch.uint8), torch.zeros(px), host=True)
    chk(Fake(), px, np.zeros((px, 4), np.float32), np.zeros(px, np.float32), host=True)
    with pytest.raises(ValueError, match="device tensor"):
        chk(Fake(), px, np.zeros((px, 4), np.float32), np.zeros(px, np.float32))
