"""Seeded synthetic inputs shared by tests, bench.py and the oracle tests.

Holds no arithmetic of the rendering method.
"""
from .rng import Stream  # noqa: F401
from .scenes import (RawScene, Camera, Fovea, random_scene, vr_room, look_camera, stereo_pair,  # noqa: F401
                     trajectory_pose, ellipse_mask, quest_fovea, focal_for_hfov, QUEST_W, QUEST_H)
