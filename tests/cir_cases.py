"""Path-solver (CIR) parity cases shared by the golden generator and the tests.

Geometry is built with the product's deterministic scene helpers; the golden
generator converts the meshes to emtrace meshes, so both sides trace the
same float64 triangles (digest checked).  Materials are plain dicts of
RadioMaterial kwargs (pattern as a tuple) so the reference and the product
construct them independently.
"""

import hashlib

import numpy as np

from paper_2504_21719_b200 import scenes
from paper_2504_21719_b200.geometry import Mesh

BOX_LO = np.array([-3.0, -4.0, 0.0])
BOX_HI = np.array([3.0, 4.0, 3.0])
TX_POS = [-1.0, -2.0, 1.5]
RX_POS = [1.5, 2.0, 1.5]
LAM = 299792458.0 / 3.5e9

CONCRETE = dict(eps_r=5.24, sigma=0.1, thickness=0.3)
CONCRETE_BENCH = dict(eps_r=5.24, sigma=0.0462, thickness=0.1)


def _panel(nv, nh, spacing, plane="yz"):
    """Planar array offsets centred on the origin (rows along z, columns along y)."""
    off = []
    for i in range(nv):
        for j in range(nh):
            a = (i - 0.5 * (nv - 1)) * spacing
            b = (j - 0.5 * (nh - 1)) * spacing
            off.append([0.0, b, a] if plane == "yz" else [b, a, 0.0])
    return off


def _box_targets(n, seed):
    rng = np.random.default_rng(seed)
    return [dict(pos=list(p)) for p in rng.uniform(BOX_LO + 0.5, BOX_HI - 0.5, size=(n, 3))]


def _canyon_targets(n, seed=5):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        p = rng.uniform(-95.0, 95.0, size=2)
        c = (np.floor((p + 100.0) / 20.0) + 0.5) * 20.0 - 100.0
        if np.all(np.abs(p - c) < 6.5):
            continue
        out.append(dict(pos=[float(p[0]), float(p[1]), 1.5]))
    return out


CIR_CASES = {
    "cfg1": dict(scene="cfg1", mat=CONCRETE_BENCH, kinds="R",
                 cfg=dict(num_samples=100_000, max_depth=3, q_diffraction=0.0, seed=0),
                 tx=[dict(pos=[0.0, 0.0, 10.0])], rx=[dict(pos=[5.0, 8.0, 1.5])]),
    "box_r": dict(scene="box", mat=CONCRETE, kinds="R",
                  cfg=dict(num_samples=20_000, max_depth=3, q_diffraction=0.0, seed=0),
                  tx=[dict(pos=TX_POS)], rx=[dict(pos=RX_POS)] + _box_targets(3, 11)),
    "box_rst": dict(scene="box", mat=dict(CONCRETE, scattering=0.4, xpd_kx=0.2,
                                          random_phases=True,
                                          pattern=("backscattering", 3, 2, 0.7)),
                    kinds="RST", velocities={0: [0.5, 0.0, -0.2]},
                    cfg=dict(num_samples=6_000, max_depth=3, q_diffraction=0.2, seed=5),
                    tx=[dict(pos=TX_POS, pattern=("tr38901", (0.3, -0.1, 0.05)),
                             velocity=[1.0, 2.0, 0.0])],
                    rx=[dict(pos=RX_POS, velocity=[0.0, -1.0, 0.5]),
                        dict(pos=[2.0, -3.0, 0.7])]),
    "box_collide": dict(scene="box", mat=dict(CONCRETE, scattering=0.3), kinds="RS",
                        cfg=dict(num_samples=4_000, max_depth=3, q_diffraction=0.0, seed=2,
                                 hash_capacity=997),
                        tx=[dict(pos=TX_POS)], rx=_box_targets(40, 12)),
    "box_trunc": dict(scene="box", mat=dict(CONCRETE, scattering=0.3), kinds="RS",
                      cfg=dict(num_samples=4_000, max_depth=3, q_diffraction=0.0, seed=2,
                               buffer_capacity=3_000),
                      tx=[dict(pos=TX_POS)], rx=_box_targets(40, 12)),
    "screen_rt": dict(scene="screen", mat=CONCRETE, kinds="RT",
                      cfg=dict(num_samples=30_000, max_depth=2, q_diffraction=0.0, seed=0),
                      tx=[dict(pos=[0.0, -3.0, 2.0])],
                      rx=[dict(pos=[0.0, 3.0, 2.5]), dict(pos=[1.0, -2.0, 1.0])]),
    "canyon_r": dict(scene="canyon", mat=CONCRETE_BENCH, kinds="R",
                     cfg=dict(num_samples=20_000, max_depth=4, q_diffraction=0.0, seed=0),
                     tx=[dict(pos=[0.0, 5.0, 20.0])], rx=_canyon_targets(16)),
    "arrays_cfr": dict(scene="cfg1", mat=CONCRETE_BENCH, kinds="R",
                       cfg=dict(num_samples=50_000, max_depth=2, q_diffraction=0.0, seed=0),
                       tx=[dict(pos=[0.0, 0.0, 10.0], pattern=("tr38901", (0.2, 0.0, 0.0)),
                                array=_panel(4, 4, LAM / 2))],
                       rx=[dict(pos=[5.0, 8.0, 1.5], array=_panel(2, 2, LAM / 2))],
                       freqs=3.5e9 + (np.arange(64) - 32) * 30e3),
    "elements": dict(scene="box", mat=CONCRETE, kinds="R",
                     cfg=dict(num_samples=5_000, max_depth=2, q_diffraction=0.0, seed=1,
                              synthetic_arrays=False),
                     tx=[dict(pos=TX_POS, array=[[0.0, 0.0, 0.0], [0.0, 0.0, 0.2]])],
                     rx=[dict(pos=RX_POS, array=[[0.0, 0.0, 0.0], [0.1, 0.0, 0.0]])],
                     freqs=np.array([3.4e9, 3.5e9, 3.6e9])),
    "multi_tx": dict(scene="box", mat=CONCRETE, kinds="R",
                     cfg=dict(num_samples=5_000, max_depth=2, q_diffraction=0.0, seed=3),
                     tx=[dict(pos=TX_POS), dict(pos=[2.0, 1.0, 2.0])],
                     rx=[dict(pos=RX_POS), dict(pos=[-2.0, 3.0, 1.0])]),
}


# first-order diffraction (SURVEY §8f "next" #1), reference defaults for D
D_CASES = {
    "screen_d": dict(scene="screen", mat=CONCRETE, kinds="RSTD",
                     cfg=dict(num_samples=150_000, max_depth=1, q_diffraction=0.3, seed=0),
                     tx=[dict(pos=[0.0, -3.0, 2.0])], rx=[dict(pos=[0.0, 3.0, 2.5])]),
    # no T here: a transmitted ray crossing the wall box reaches z = 0 where the
    # box bottom and the ground overlap coplanar -- an exact t-tie decided at
    # the last ulp of the launch direction (CUDA vs glibc sin/cos), i.e. inside
    # the north star's epsilon exclusion; blocks_rtd covers T with D
    "cfg1_default": dict(scene="cfg1", mat=dict(CONCRETE_BENCH, scattering=0.2), kinds="RSD",
                         cfg=dict(num_samples=60_000, max_depth=3, q_diffraction=0.2, seed=1),
                         tx=[dict(pos=[0.0, 0.0, 10.0])],
                         rx=[dict(pos=[5.0, 8.0, 1.5]), dict(pos=[20.0, 3.0, 2.0])]),
    "canyon_rd": dict(scene="canyon", mat=CONCRETE_BENCH, kinds="RD",
                      cfg=dict(num_samples=20_000, max_depth=3, q_diffraction=0.2, seed=0),
                      tx=[dict(pos=[0.0, 5.0, 20.0])], rx=_canyon_targets(8)),
    "blocks_rtd": dict(scene="blocks", mat=dict(CONCRETE, scattering=0.3, random_phases=True),
                       kinds="RSTD",
                       cfg=dict(num_samples=20_000, max_depth=2, q_diffraction=0.25, seed=4),
                       tx=[dict(pos=[-6.0, -5.0, 3.0], pattern=("tr38901", (0.5, 0.0, 0.0)))],
                       rx=[dict(pos=[6.0, 5.0, 1.5]), dict(pos=[0.0, 7.0, 4.0])]),
}
CIR_CASES.update(D_CASES)


def screen_mesh(half=2.0, center_z=2.0, object_id=5):
    quad = scenes.quad_mesh(half=half, z=0.0, object_id=object_id)
    swap = np.array([[1.0, 0, 0], [0, 0, 1.0], [0, 1.0, 0]])
    verts = quad.vertices @ swap + np.array([0.0, 0.0, center_z])
    return Mesh(verts, quad.triangles, object_id=object_id)


def case_geometry(name):
    """(meshes, {object_id: material kwargs}, velocities or None) of a case."""
    c = CIR_CASES[name]
    if c["scene"] == "box":
        meshes = [scenes.box_mesh(BOX_LO, BOX_HI, object_id=0, inward=True)]
    elif c["scene"] == "cfg1":
        meshes = scenes.config1_scene()
    elif c["scene"] == "screen":
        meshes = [screen_mesh()]
    elif c["scene"] == "canyon":
        meshes = scenes.street_canyon()
    elif c["scene"] == "blocks":
        meshes = [scenes.quad_mesh(half=20.0, z=0.0, object_id=0),
                  scenes.subdivided_box((-2.0, -2.0, 0.0), (2.0, 2.0, 6.0), 2, 1),
                  scenes.box_mesh((3.0, -6.0, 0.0), (5.0, -1.0, 4.0), object_id=2)]
    else:
        raise KeyError(c["scene"])
    mats = {m.object_id: dict(c["mat"]) for m in meshes}
    return meshes, mats, c.get("velocities")


def mesh_digest(meshes):
    h = hashlib.sha256()
    for m in meshes:
        h.update(np.ascontiguousarray(m.vertices, dtype=np.float64).tobytes())
        h.update(np.ascontiguousarray(m.triangles, dtype=np.int64).tobytes())
        h.update(str(int(m.object_id)).encode())
    return h.hexdigest()
