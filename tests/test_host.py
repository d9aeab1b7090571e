"""Host-side logic of the drop-in API (no GPU)."""

import numpy as np
import pytest

from paper_1903_03406_b200 import PLC, RefineConfig, synth, unit_cube, validate
from paper_1903_03406_b200.errors import InvalidPLC
from paper_1903_03406_b200.plc import augment_with_box, hull_axis_aligned, hull_covered, hull_simplices
from paper_1903_03406_b200.prepare import facet_keep, prepare, shuffle_order


def test_unit_cube_matches_reference_layout():
    c = unit_cube()
    assert len(c.points) == 8 and len(c.segments) == 12 and len(c.polygons) == 6
    assert c.points[5] == (1.0, 0.0, 1.0)            # index = x + 2y + 4z (plc.py:386-408)
    assert c.polygons[0] == (0, 1, 3, 2)
    assert validate(c) == []


def test_validate_reports_violations():
    assert ("polygon-bad-index", 0) in validate(PLC(points=unit_cube().points, segments=[], polygons=[(0, 1, 99)]))
    bad = validate(PLC(points=[(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)], segments=[(0, 1), (1, 2), (2, 3), (0, 3)],
                       polygons=[(0, 1, 2, 3)]))
    assert ("polygon-non-planar", 0) in bad
    assert ("duplicate-point", (0, 1)) in validate(PLC(points=[(0, 0, 0), (0, 0, 0)]))
    crossing = PLC(points=[(0, 0, 0), (1, 1, 0), (1, 0, 0), (0, 1, 0)], segments=[(0, 1), (2, 3)])
    assert ("segment-segment-intersection", (0, 1)) in validate(crossing)


def test_refine_config_validation():
    with pytest.raises(ValueError):
        RefineConfig(B=0)
    with pytest.raises(ValueError):
        RefineConfig(max_rounds=0)
    assert RefineConfig().B == 2.0


def test_box_closure():
    cube = synth.cube_points(10, 0)
    assert hull_covered(cube)
    assert augment_with_box(cube) is cube
    seg = synth.segments_cloud(50, 2, 0)
    aug = augment_with_box(seg)
    assert len(aug.points) == len(seg.points) + 8 and len(aug.polygons) == 6 and len(aug.segments) == 2 + 12


def test_box_for_oblique_hull():
    """A hull tiled by oblique polygons (a sphere) is boxed too (plc.py
    augment_with_box docstring); an axis-aligned tiled hull is not."""
    plc = synth.nested_surfaces(200, level=3, torus=(8, 4))
    hs = hull_simplices(plc)
    assert hull_covered(plc, hs) and not hull_axis_aligned(plc, hs)
    aug = augment_with_box(plc)
    assert len(aug.points) == len(plc.points) + 8 and len(aug.polygons) == len(plc.polygons) + 6
    cube = synth.cube_points(10, 0)
    assert hull_axis_aligned(cube, hull_simplices(cube))


def test_prepare_and_order():
    p = prepare(synth.cube_points(20, 0), seed=0)
    assert p.points.shape == (28, 3) and p.order.dtype == np.int32
    o = list(range(28))
    np.random.default_rng(0).shuffle(o)
    assert p.order.tolist() == o == shuffle_order(28, 0).tolist()
    with pytest.raises(InvalidPLC):
        prepare(PLC(points=[(0, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]))


def test_facet_keep_orientation():
    k = facet_keep(unit_cube())
    assert k.shape == (6, 2)
    for i, j in k:
        assert i != j


def test_generators_deterministic():
    a = synth.config_plc("C2", scale=0.01, seed=3)
    b = synth.config_plc("C2", scale=0.01, seed=3)
    assert a.points == b.points and a.segments == b.segments
    t = synth.triangles_cloud(200, 4, 0)
    assert validate(t) == [] and len(t.polygons) == 4
    g = synth.generate(synth.SynthSpec(100, 0.05, "cube", 0))
    assert len(g.polygons) == 5 and validate(g) == []


def test_shuffle_order_matches_list_shuffle():
    """prepare.shuffle_order shuffles an array; the reference shuffles a list
    (mesh.py:878-880).  Same permutation for every size."""
    for n in (4, 5, 28, 1000, 20011):
        o = list(range(n))
        np.random.default_rng(3).shuffle(o)
        assert shuffle_order(n, 3).tolist() == o
