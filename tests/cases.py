"""Radio-map parity cases shared by the oracle (CPU) and GPU tests.

Each case mirrors one entry of tests/golden/make_golden.py, expressed with the
product's host types so both the oracle and the CUDA path consume it.
"""

import numpy as np

from paper_2504_21719_b200 import scenes
from paper_2504_21719_b200.em import ArrayGeometry, make_pattern
from paper_2504_21719_b200.materials import RadioMaterial, ScatteringPattern
from paper_2504_21719_b200.radiomap import MeasurementGrid, RadioMapConfig
from paper_2504_21719_b200.sampling import Interaction

KINDS = {"R": Interaction.REFLECTION, "S": Interaction.SCATTERING,
         "T": Interaction.TRANSMISSION}

MAP_CASES = {
    "box_rs": dict(scene="box", mat=dict(eps_r=5.24, sigma=0.1, thickness=0.3),
                   grid=((0.5, 1.0, 1.2), (1, 0, 0), (0, 1, 0), (0.5, 0.5), (2, 2)),
                   cfg=dict(num_samples=100_000, max_depth=3, seed=1), kinds="RS",
                   src=(-1.0, -2.0, 1.5)),
    "box_rst_rr": dict(scene="box", mat=dict(eps_r=5.24, sigma=0.1, thickness=0.3,
                                             scattering=0.4),
                       grid=((0.5, 1.0, 1.2), (1, 0, 0), (0, 1, 0), (0.5, 0.5), (8, 8)),
                       cfg=dict(num_samples=60_000, max_depth=3, seed=1, rr_depth=1,
                                rr_max=0.9), kinds="RST", src=(-1.0, -2.0, 1.5)),
    "box_thr_patterns": dict(scene="box",
                             mat=dict(eps_r=4.0, sigma=0.05, thickness=0.2, scattering=0.6,
                                      xpd_kx=0.3, random_phases=True,
                                      pattern=("backscattering", 3, 2, 0.7)),
                             grid=((0.0, 0.0, 1.0), (0, 1, 0), (0, 0, 1), (0.7, 0.4), (6, 5)),
                             cfg=dict(num_samples=50_000, max_depth=4, seed=4,
                                      gain_threshold=1e-4), kinds="RST", src=(1.0, 2.0, 2.0)),
    "box_directive_array": dict(scene="box",
                                mat=dict(eps_r=5.24, sigma=0.1, thickness=0.3, scattering=0.5,
                                         pattern=("directive", 4, 1, 1.0)),
                                grid=((0.5, 1.0, 1.2), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (4, 6)),
                                cfg=dict(num_samples=40_000, max_depth=3, seed=2), kinds="RS",
                                src=(-1.0, -2.0, 1.5), pattern=("tr38901", (0.4, -0.2, 0.1)),
                                array=True),
    "canyon_rs": dict(scene="canyon",
                      mat=dict(eps_r=5.24, sigma=0.0462, thickness=0.1, scattering=0.3),
                      grid=((0.0, 0.0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (200, 200)),
                      cfg=dict(num_samples=30_000, max_depth=5, seed=0), kinds="RS",
                      src=(0.0, 5.0, 20.0)),
}

_SCENES = {}


def case_meshes(name):
    c = MAP_CASES[name]
    if c["scene"] not in _SCENES:
        _SCENES[c["scene"]] = (scenes.box_room_walls() if c["scene"] == "box"
                               else scenes.street_canyon())
    return _SCENES[c["scene"]]


def build_case(name):
    """(meshes, materials, source, grid, cfg, kwargs) of a golden radio-map case."""
    c = MAP_CASES[name]
    meshes = case_meshes(name)
    md = dict(c["mat"])
    pat = md.pop("pattern", None)
    if pat is not None:
        md["pattern"] = ScatteringPattern(kind=pat[0], alpha_r=pat[1], alpha_i=pat[2],
                                          lambda_mix=pat[3])
    mat = RadioMaterial("m", **md)
    mats = {m.object_id: mat for m in meshes}
    grid = MeasurementGrid(*c["grid"])
    cfg = RadioMapConfig(enabled=frozenset(KINDS[k] for k in c["kinds"]), **c["cfg"])
    kw = {}
    if "pattern" in c:
        kw["pattern"] = make_pattern(c["pattern"][0], orientation=c["pattern"][1])
    if c.get("array"):
        off = np.zeros((4, 3))
        off[:, 1] = np.arange(4) * cfg.wavelength / 2.0
        kw["array"] = ArrayGeometry(off)
        kw["precoder"] = np.array([0.5, 0.5j, -0.5, 0.1 + 0.3j])
    return meshes, mats, np.array(c["src"]), grid, cfg, kw


def golden_map(g, name):
    vals = g[f"{name}__values"]
    diag = {k.split("__diag__")[1]: int(g[k]) for k in g.files
            if k.startswith(f"{name}__diag__")}
    return vals, diag


COUNTER_KEYS = ("deposits", "escaped", "respawns", "threshold_killed", "roulette_killed",
                "terminated", "direct_visible")
