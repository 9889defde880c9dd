"""GPU sim::render_depth (proj/src/sim/render.cpp:8-58):
frames bit-identical to the reference renderer for its own scenes, rotated
and translated poses, several camera shapes, host and device outputs."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2112_13169_b200 import voxmap as vm
from tests import scenes

pytestmark = pytest.mark.gpu
ref = pytest.importorskip("oracle.ref")
if not ref.available():
    pytest.skip("oracle/_ref not built", allow_module_level=True)

DEG = math.pi / 180.0


def _yawed(pos, yaw, pitch=0.0):
    R0 = vm.look_along_x((0, 0, 0))[0]
    cy, sy, cp, sp = math.cos(yaw), math.sin(yaw), math.cos(pitch), math.sin(pitch)
    Ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
    Rx = np.array([[1, 0, 0], [0, cp, -sp], [0, sp, cp]])
    return R0 @ Ry @ Rx, np.asarray(pos, dtype=float)


@pytest.mark.parametrize("shape", [(640, 480), (160, 120), (97, 61)])
def test_render_matches_reference(gpu_lib, shape):
    W, H = shape
    cam = vm.CameraModel(85 * DEG, 101 * DEG, W, H, 6.5)
    rng = np.random.default_rng(W)
    worlds = [scenes.box_field_boxes(1), scenes.box_field_boxes(7), scenes.wall_boxes(),
              scenes.corridor_boxes(-10.0, 10.0)]
    for boxes in worlds:
        poses = [vm.look_along_x((0.0, 0.1001 * k - 0.8, 0.0)) for k in range(3)]
        poses += [_yawed(rng.uniform(-1, 1, 3) * [0.5, 1.0, 0.3], rng.uniform(-0.6, 0.6), rng.uniform(-0.3, 0.3))
                  for _ in range(3)]
        got = vm.render_depth(cam, poses, boxes)
        for k, pose in enumerate(poses):
            want = ref.render_depth(cam.to_c(), pose, boxes=boxes, parallel=False)
            assert np.array_equal(got[k], want), (k, int((got[k] != want).sum()))


def test_render_device_output_and_empty_scene(gpu_lib):
    import torch

    cam = vm.CameraModel(85 * DEG, 101 * DEG, 128, 96, 5.0)
    boxes = scenes.box_field_boxes(3)
    poses = [vm.look_along_x((0.0, 0.05 * k, 0.0)) for k in range(5)]
    dev = torch.empty((5, 96, 128), dtype=torch.float32, device="cuda")
    vm.render_depth(cam, poses, boxes, out_ptr=dev.data_ptr())
    host = vm.render_depth(cam, poses, boxes)
    assert np.array_equal(dev.cpu().numpy(), host)
    assert not vm.render_depth(cam, poses[:1], np.zeros((0, 6))).any()  # nothing to hit: all invalid


def test_render_rejects_bad_boxes(gpu_lib):
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 32, 24, 5.0)
    with pytest.raises(ValueError, match="Aabb"):
        vm.render_depth(cam, [vm.look_along_x((0, 0, 0))], np.array([[1.0, 0, 0, 1.0, 1, 1]]))
