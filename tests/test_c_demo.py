"""The C ABI used from plain C (examples/vrs_demo.c): it compiles and links
against the in-tree libvrs.so with gcc (CPU), and renders a foveated stereo
frame through vrs_render_views_host on the GPU."""
from __future__ import annotations

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2505_10144_b200")


def _build(tmp_path):
    from paper_2505_10144_b200 import build
    build.build()
    exe = str(tmp_path / "vrs_demo")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "vrs_demo.c"), "-L", LIBDIR, "-lvrs", f"-Wl,-rpath,{LIBDIR}", "-lm",
           "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_demo_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_c_demo_renders(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    m = re.search(r"status=(\d+) rejected=(\d+) pairs=(\d+) samples=(\d+) mean_rgb=([\d.,]+) mean_alpha=([\d.]+)",
                  r.stdout)
    assert m, r.stdout
    status, rejected, pairs, samples = (int(m.group(i)) for i in range(1, 5))
    alpha = float(m.group(6))
    assert status == 0 and rejected == 0 and pairs > 1000 and samples > 0
    assert 0.0 < alpha < 1.0
