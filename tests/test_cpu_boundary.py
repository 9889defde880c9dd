"""CPU-only checks: the C-ABI library loads and exports every symbol
include/vxm.h declares; host-side arithmetic (grid specs, bundle sizes)
matches the reference; the synthetic frame generator equals the reference's
render_depth. No GPU compute is called here."""
from __future__ import annotations

import math
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2112_13169_b200 import _native as N
from paper_2112_13169_b200 import voxmap as vm
from tests import scenes
from tests.oracle_api import have_ref

ROOT = Path(__file__).resolve().parent.parent
DEG = math.pi / 180.0


def declared_symbols():
    text = (ROOT / "include" / "vxm.h").read_text()
    return sorted(set(re.findall(r"\b(vxm_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(N.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = N.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.vxm_kernel_isa() == b"cuda-sm100a"


def test_no_device_is_reported_not_faked():
    # Without a GPU the runtime must refuse, not fall back to the CPU.
    lib = N.load()
    if lib.vxm_device_count() > 0:
        pytest.skip("GPU present")
    cam = vm.CameraModel(width=64, height=48)
    grid = vm.GridSpec.create_centered(6.0, 6.0, 3.0, 0.15, (0, 0, 0))
    with pytest.raises(N.VxmError):
        vm.MappingPipeline(vm.PipelineConfig(grid, cam, vox_inf=0, depth=4.0))


def test_grid_spec_matches_reference_formulas():
    # proj/tests/test_grid_core.cpp:16-40: 15x15x3 m at 0.15 -> 100x100x20, origin -7.5,-7.5,-1.5
    g = vm.GridSpec.create_centered(15.0, 15.0, 3.0, 0.15, (0, 0, 0))
    assert g.dims == (100, 100, 20)
    assert g.cell_count() == 200000
    assert np.allclose(g.origin, [-7.5, -7.5, -1.5])
    odd = vm.GridSpec.create_centered(0.45, 0.45, 0.45, 0.15, (1.0, 1.0, 1.0))
    assert odd.dims == (3, 3, 3)
    assert odd.origin[0] == pytest.approx(1.0 - 0.15)
    with pytest.raises(ValueError):
        vm.GridSpec.create(0.0, 1.0, 1.0, 0.1)
    with pytest.raises(ValueError):
        vm.GridSpec.create(1.0, 1.0, 1.0, -0.1)


@pytest.mark.parametrize("w,h,depth,vs,expect", [
    (320, 240, 6.5, 0.15, (43, 79, 105)),   # test_raytracer.cpp:35-45 -> 8295 rays
    (640, 480, 6.5, 0.1, (65, 121, 159)),   # cfg1
    (640, 480, 5.0, 0.1, (50, 93, 123)),    # cfg2
    (1280, 720, 6.5, 0.05, (130, 239, 317)),  # cfg3
])
def test_bundle_dimensions(w, h, depth, vs, expect):
    cam = vm.CameraModel(85 * DEG, 101 * DEG, w, h, depth)
    assert vm.bundle_dimensions(cam, depth, vs) == expect
    if expect[0] == 43:
        assert expect[1] * expect[2] == 8295


def test_bundle_dimensions_rejects_bad_input():
    cam = vm.CameraModel(85 * DEG, 101 * DEG, 320, 240, 6.5)
    with pytest.raises(ValueError):
        vm.bundle_dimensions(cam, 0.0, 0.15)
    with pytest.raises(ValueError):
        vm.bundle_dimensions(vm.CameraModel(math.pi, 1.0, 320, 240, 6.5), 6.5, 0.15)


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
def test_scene_renderer_equals_reference_render_depth():
    from oracle import ref

    cam = vm.CameraModel(85 * DEG, 101 * DEG, 160, 120, 6.5)
    for seed, pos in ((1, (0.0, 0.0, 0.0)), (2, (0.3, -0.4, 0.1)), (3, (0.0, 0.6, -0.2))):
        pose = vm.look_along_x(pos)
        got = scenes.render(cam, pose, scenes.box_field_boxes(seed))
        want = ref.render_depth(cam.to_c(), pose, "boxes", seed=seed)
        assert np.array_equal(got, want)
        assert np.array_equal(scenes.render(cam, pose, scenes.wall_boxes()),
                              ref.render_depth(cam.to_c(), pose, "wall"))
