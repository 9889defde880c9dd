"""VOXGRID1 snapshot files (proj/include/voxmap/grid_io.hpp,
proj/src/grid_io.cpp:14-69): the C-ABI writer produces the reference
writer's bytes exactly, each side reads the other's files, and both reject
the same malformed files. Host only — runs without a GPU."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2112_13169_b200 import _native as N
from paper_2112_13169_b200 import voxmap as vm

ref = pytest.importorskip("oracle.ref")
if not ref.available():
    pytest.skip("oracle/_ref not built", allow_module_level=True)

GRIDS = [((15.0, 15.0, 3.0), 0.15, (0.0, 0.0, 0.0)), ((10.0, 10.0, 5.0), 0.1, (0.1001, -50.0, 2.25)),
         ((2.0, 1.0, 0.5), 0.05, (-1.0 / 3.0, 1e-12, 123456.789)), ((0.45, 0.3, 0.15), 0.15, (7.0, -7.0, 0.0))]


def _cells(g, seed):
    return np.random.default_rng(seed).integers(0, 4, g.cell_count()).astype(np.uint8)


@pytest.mark.parametrize("i", range(len(GRIDS)))
def test_writer_bytes_equal_reference(tmp_path, i):
    size, vs, center = GRIDS[i]
    g = vm.GridSpec.create_centered(*size, vs, center)
    cells = _cells(g, i)
    ours, theirs = tmp_path / "ours.vox", tmp_path / "ref.vox"
    vm.write_grid(g, cells, ours)
    ref.write_grid(g.c, cells, theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    assert ours.read_bytes().startswith(b"VOXGRID1\n")


@pytest.mark.parametrize("i", range(len(GRIDS)))
def test_each_side_reads_the_other(tmp_path, i):
    size, vs, center = GRIDS[i]
    g = vm.GridSpec.create_centered(*size, vs, center)
    cells = _cells(g, 10 + i)
    ref.write_grid(g.c, cells, tmp_path / "a.vox")
    g2, c2 = vm.read_grid(tmp_path / "a.vox")
    assert np.array_equal(c2, cells)
    assert g2.dims == g.dims and g2.vox_size == g.vox_size and np.array_equal(g2.origin, g.origin)
    vm.write_grid(g, cells, tmp_path / "b.vox")
    g3, c3 = ref.read_grid(tmp_path / "b.vox")
    assert np.array_equal(c3, cells)
    assert tuple(g3.dims) == g.dims and list(g3.origin) == list(g.origin)
    assert list(g3.size) == list(g2.c.size)  # grid_size = dims * vox_size on both sides


def test_malformed_files_rejected_like_the_reference(tmp_path):
    g = vm.GridSpec.create(0.3, 0.3, 0.3, 0.1)
    good = tmp_path / "good.vox"
    vm.write_grid(g, np.zeros(27, np.uint8), good)
    data = good.read_bytes()
    cases = {
        "magic": data.replace(b"VOXGRID1", b"VOXGRID2"),
        "truncated": data[:-1],
        "state": data[:-1] + b"\x04",
        "dims": data.replace(b"3 3 3", b"3 0 3", 1),
        "voxsize": data.replace(b"0.10000000000000001", b"-0.1", 1),
        "empty": b"",
    }
    for name, blob in cases.items():
        p = tmp_path / f"{name}.vox"
        p.write_bytes(blob)
        with pytest.raises(Exception):
            ref.read_grid(p)
        with pytest.raises(N.VxmError):
            vm.read_grid(p)
    with pytest.raises(N.VxmError):
        vm.read_grid(tmp_path / "missing.vox")
