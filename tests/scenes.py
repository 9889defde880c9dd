"""Synthetic depth frames for tests and the benchmark (host-side, numpy).

A vectorised restatement of sim::render_depth / ray_box_hit
(proj/src/sim/render.cpp:8-58) with the same fp64 operation order, so the
frames equal the reference generator's (checked in tests/test_cpu_oracle.py
when the reference build is present). The box-field layouts come from the
reference's own Scene::box_field(seed) (proj/src/sim/scene.cpp:32-71),
captured once into tests/golden/box_field_scenes.json by
tests/golden/make_golden.py.
"""
from __future__ import annotations

import json
import math
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def box_field_boxes(seed: int = 1) -> np.ndarray:
    data = json.loads((GOLDEN / "box_field_scenes.json").read_text())
    return np.array(data[str(seed)], dtype=np.float64)


def wall_boxes(distance: float = 5.5) -> np.ndarray:
    """Scene::wall (scene.cpp:25-30)."""
    return np.array([[distance, -12.0, -12.0, distance + 0.3, 12.0, 12.0]])


def corridor_boxes(y_min=-60.0, y_max=60.0, spacing=1.5, seed=7) -> np.ndarray:
    """cfg4's corridor: a backdrop at x in [6.0, 6.3] spanning
    y_min..y_max plus seeded pillars every `spacing` metres."""
    rng = np.random.default_rng(seed)
    boxes = [[6.0, y_min, -8.0, 6.3, y_max, 8.0]]
    y = y_min
    while y < y_max:
        x0 = 2.0 + 2.5 * rng.random()
        w = 0.2 + 0.4 * rng.random()
        z_lo = -1.6 if rng.random() < 0.5 else 0.1 + rng.random()
        z_hi = z_lo + 0.8 + 1.2 * rng.random()
        boxes.append([x0, y, z_lo, x0 + 0.3, y + w, z_hi])
        y += spacing
    return np.array(boxes, dtype=np.float64)


def render(cam, pose, boxes) -> np.ndarray:
    """Depth image (H, W) float32 of an AABB world; 0 = no return within
    cam.max_depth. pose = (R, t) camera->world."""
    R, t = pose
    R = np.asarray(R, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    W, H = cam.width, cam.height
    fx = (W / 2.0) / math.tan(cam.fov_x / 2.0)
    fy = (H / 2.0) / math.tan(cam.fov_y / 2.0)
    cx, cy = W / 2.0, H / 2.0
    u = np.arange(W, dtype=np.float64)[None, :]
    v = np.arange(H, dtype=np.float64)[:, None]
    dc = [np.broadcast_to(((u + 0.5) - cx) / fx, (H, W)), np.broadcast_to(((v + 0.5) - cy) / fy, (H, W)),
          np.ones((H, W))]
    # dir = R * dir_cam, each row a left-to-right dot product
    d = [(R[a, 0] * dc[0] + R[a, 1] * dc[1]) + R[a, 2] * dc[2] for a in range(3)]
    best = np.full((H, W), np.inf)
    with np.errstate(divide="ignore", invalid="ignore"):
        for box in boxes:
            lo, hi = box[:3], box[3:]
            t_near = np.full((H, W), -np.inf)
            t_far = np.full((H, W), np.inf)
            miss = np.zeros((H, W), dtype=bool)
            for a in range(3):
                zero = d[a] == 0.0
                miss |= zero & ((t[a] < lo[a]) | (t[a] > hi[a]))
                ta = (lo[a] - t[a]) / d[a]
                tb = (hi[a] - t[a]) / d[a]
                sw = ta > tb
                ta, tb = np.where(sw, tb, ta), np.where(sw, ta, tb)
                t_near = np.where(zero, t_near, np.where(t_near < ta, ta, t_near))
                t_far = np.where(zero, t_far, np.where(tb < t_far, tb, t_far))
            hit = ~miss & ~((t_near > t_far) | (t_far <= 0.0))
            s = np.where(t_near > 0.0, t_near, t_far)
            take = hit & (s > 0.0) & (s < best)
            best = np.where(take, s, best)
    img = np.where(best <= cam.max_depth, best, 0.0).astype(np.float32)
    return img


def stress_depth(cam, seed=1, invalid=0.05, lo=0.3) -> np.ndarray:
    """S2 stress frame: U(lo, max_depth) depth with a fraction of
    invalid (0) pixels."""
    rng = np.random.default_rng(seed)
    d = rng.uniform(lo, cam.max_depth, size=(cam.height, cam.width)).astype(np.float32)
    d[rng.random((cam.height, cam.width)) < invalid] = 0.0
    return d
