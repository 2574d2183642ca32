"""CPU checks of the evaluation protocol helpers (SPEC psnr / large_fov_protocol
examples) against naive definitions."""
from __future__ import annotations

import math

import numpy as np
import pytest

from helpers import identity_camera
from paper_2505_10144_b200.protocol import centre_crop, psnr, wide_camera


def test_psnr_spec_examples():
    a = np.random.default_rng(0).random((7, 5, 3))
    assert psnr(a, a) == math.inf
    assert psnr(np.zeros((4, 4, 3)), np.full((4, 4, 3), 0.1)) == pytest.approx(20.0, abs=1e-9)
    b = np.random.default_rng(1).random((7, 5, 3))
    s = 0.0
    for i in range(7):
        for j in range(5):
            for c in range(3):
                s += (a[i, j, c] - b[i, j, c]) ** 2
    assert psnr(a, b) == pytest.approx(10 * math.log10(1.0 / (s / a.size)), abs=1e-9)
    with pytest.raises(ValueError):
        psnr(a, b[:3])


def test_wide_camera_crop_casts_original_rays():
    cam = identity_camera(64, 48, 40.0)
    wide = wide_camera(cam)
    assert (wide.width, wide.height) == (192, 144) and wide.fx == cam.fx
    rng = np.random.default_rng(2)
    i, j = rng.integers(0, 64, 50), rng.integers(0, 48, 50)
    # crop pixel (i, j) is wide pixel (64 + i, 48 + j)
    assert np.array_equal((64 + i + 0.5 - wide.cx) / wide.fx, (i + 0.5 - cam.cx) / cam.fx)
    assert np.array_equal((48 + j + 0.5 - wide.cy) / wide.fy, (j + 0.5 - cam.cy) / cam.fy)
    img = np.arange(192 * 144).reshape(144, 192)
    assert centre_crop(img, cam)[0, 0] == img[48, 64] and centre_crop(img, cam).shape == (48, 64)
