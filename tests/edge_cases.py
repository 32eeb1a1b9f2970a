"""Diffraction radio-map (edge estimator) cases shared by the golden generator and tests.

Reference: compute_radio_map with D enabled (radiomap.py:985-1023) =
bounce map + compute_radio_map_diffraction over collect_wedges_near_source.
"""

import numpy as np

from cir_cases import CONCRETE, CONCRETE_BENCH, screen_mesh
from paper_2504_21719_b200 import scenes

LAM = 299792458.0 / 3.5e9

EDGE_CASES = {
    "screen_edge": dict(scene="screen", mat=CONCRETE,
                        grid=((0.0, 2.5, 1.7), (1, 0, 0), (0, 1, 0), (0.5, 0.5), (10, 6)),
                        cfg=dict(num_samples=40_000, wedge_samples=100_000, max_depth=2,
                                 seed=3),
                        src=(0.0, -3.0, 2.0), radius=None),
    "cfg1_edge": dict(scene="cfg1", mat=dict(CONCRETE_BENCH, scattering=0.2),
                      grid=((20.0, 0.0, 1.5), (1, 0, 0), (0, 1, 0), (2.0, 2.0), (12, 20)),
                      cfg=dict(num_samples=60_000, wedge_samples=20_000, max_depth=2, seed=1),
                      src=(0.0, 0.0, 10.0), radius=45.0),
    "blocks_edge": dict(scene="blocks", mat=dict(CONCRETE, scattering=0.3),
                        grid=((4.0, 2.0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (16, 14)),
                        cfg=dict(num_samples=40_000, wedge_samples=30_000, max_depth=2,
                                 seed=4),
                        src=(-6.0, -5.0, 3.0), radius=None,
                        pattern=("tr38901", (0.5, 0.0, 0.0)),
                        array=[[0.0, 0.0, 0.0], [0.0, LAM / 2, 0.0], [0.0, LAM, 0.0]],
                        precoder=[0.6, 0.3 + 0.4j, -0.5j]),
}


def edge_geometry(name):
    c = EDGE_CASES[name]
    if c["scene"] == "screen":
        meshes = [screen_mesh()]
    elif c["scene"] == "cfg1":
        meshes = scenes.config1_scene()
    else:
        meshes = [scenes.quad_mesh(half=20.0, z=0.0, object_id=0),
                  scenes.subdivided_box((-2.0, -2.0, 0.0), (2.0, 2.0, 6.0), 2, 1),
                  scenes.box_mesh((3.0, -6.0, 0.0), (5.0, -1.0, 4.0), object_id=2)]
    return meshes, {m.object_id: dict(c["mat"]) for m in meshes}
