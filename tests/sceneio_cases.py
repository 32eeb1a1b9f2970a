"""Scene-file / OBJ / writer cases shared by the golden generator and the tests."""

import types

import numpy as np

GOOD = """format_version 1
frequency 3.5e9   # carrier

material concrete
  eps_r 5.24
  sigma 0.1
  thickness 0.3
  scattering 0.3
  xpd 0.1
  scattering_pattern backscattering 3 2 0.7
  random_phases on

material glass
  eps_r 6.27
  sigma 0.0043
  scattering_pattern directive 4

object floor
  mesh floor.obj
  material concrete
  velocity 0 0.5 0

object wall
  mesh sub dir/wall.obj
  material glass

transmitter tx0
  position 0 0 2
  orientation_deg 30 10 0
  pattern tr38901
  array 2 4 0.0428 0.0428
  power 2.0
  velocity 1 0 0

receiver rx0
  position 5 0 1.5

receiver rx1
  position -3 2 1.5
  orientation 0.1 0.2 0.3

grid
  center 0 0 1.5
  axis_u 1 0 0
  axis_v 0 1 0
  cell_size 0.5 0.25
  shape 20 10
"""

MINIMAL = "format_version 1\nfrequency 28e9\n"

BAD = {
    "no_version": "frequency 1e9\n",
    "bad_version": "format_version 2\nfrequency 1e9\n",
    "no_frequency": "format_version 1\n",
    "neg_frequency": "format_version 1\nfrequency -1\n",
    "prop_outside": "format_version 1\nfrequency 1e9\n  eps_r 3\n",
    "dup_key": "format_version 1\nfrequency 1e9\nmaterial m\n  eps_r 3\n  eps_r 4\n",
    "unknown_directive": "format_version 1\nfrequency 1e9\nlight l0\n",
    "block_two_names": "format_version 1\nfrequency 1e9\nmaterial a b\n",
    "mat_redefined": "format_version 1\nfrequency 1e9\nmaterial m\n  eps_r 3\nmaterial m\n  eps_r 4\n",
    "mat_unknown_key": "format_version 1\nfrequency 1e9\nmaterial m\n  color red\n",
    "mat_bad_number": "format_version 1\nfrequency 1e9\nmaterial m\n  eps_r abc\n",
    "mat_two_numbers": "format_version 1\nfrequency 1e9\nmaterial m\n  sigma 1 2\n",
    "mat_bad_bool": "format_version 1\nfrequency 1e9\nmaterial m\n  random_phases maybe\n",
    "mat_bad_pattern": "format_version 1\nfrequency 1e9\nmaterial m\n  scattering_pattern spiky\n",
    "mat_bad_pattern_args": "format_version 1\nfrequency 1e9\nmaterial m\n  scattering_pattern directive x\n",
    "mat_invalid_value": "format_version 1\nfrequency 1e9\nmaterial m\n  scattering 1.5\n",
    "obj_no_mesh": "format_version 1\nfrequency 1e9\nobject o\n  material m\n",
    "obj_no_material": "format_version 1\nfrequency 1e9\nobject o\n  mesh a.obj\n",
    "obj_unknown_key": "format_version 1\nfrequency 1e9\nobject o\n  mesh a.obj\n  material m\n  scale 2\n",
    "dev_no_position": "format_version 1\nfrequency 1e9\ntransmitter t\n  power 1\n",
    "dev_bad_array": "format_version 1\nfrequency 1e9\nreceiver r\n  position 0 0 0\n  array 1.5 2 0.1 0.1\n",
    "dev_zero_power": "format_version 1\nfrequency 1e9\ntransmitter t\n  position 0 0 0\n  power 0\n",
    "dev_unknown_key": "format_version 1\nfrequency 1e9\nreceiver r\n  position 0 0 0\n  gain 3\n",
    "dev_short_vec": "format_version 1\nfrequency 1e9\nreceiver r\n  position 0 0\n",
    "grid_missing": "format_version 1\nfrequency 1e9\ngrid\n  center 0 0 0\n  shape 3 3\n",
    "grid_unknown": "format_version 1\nfrequency 1e9\ngrid\n  center 0 0 0\n  cell_size 1 1\n  shape 3 3\n  tilt 1\n",
    "grid_invalid": "format_version 1\nfrequency 1e9\ngrid\n  center 0 0 0\n  axis_u 1 0 0\n  axis_v 1 0 0\n  cell_size 1 1\n  shape 3 3\n",
    "grid_redefined": "format_version 1\nfrequency 1e9\ngrid\n  center 0 0 0\n  cell_size 1 1\n  shape 3 3\ngrid\n  center 0 0 0\n  cell_size 1 1\n  shape 3 3\n",
}

OBJ = {
    # quad + pentagon (fan-triangulated), negative index, v/vt/vn tokens, comments
    "poly": "# test\nv 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nvn 0 0 1\nf 1/1/1 2//1 3 4\n"
            "v 2 0 0\nv 3 0 0\nv 3.5 1 0\nv 2.5 2 0\nv 2 1 0\nf -5 -4 -3 -2 -1\ng x\ns off\n",
    # one degenerate (collinear) triangle dropped with a warning
    "degenerate": "v 0 0 0\nv 1 0 0\nv 2 0 0\nv 0 1 0\nf 1 2 3\nf 1 2 4\n",
    # an edge shared by three faces
    "nonmanifold": "v 0 0 0\nv 1 0 0\nv 0 1 0\nv 0 -1 0\nv 0 0 1\nf 1 2 3\nf 1 2 4\nf 1 2 5\n",
}

OBJ_BAD = {
    "zero_index": "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 0 1 2\n",
    "out_of_range": "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 4\n",
    "short_vertex": "v 0 0\n",
    "bad_vertex": "v 0 a 0\n",
    "short_face": "v 0 0 0\nv 1 0 0\nf 1 2\n",
    "bad_index": "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 x 3\n",
}


def describe(desc):
    mats = {k: dict(eps_r=m.eps_r, sigma=m.sigma, thickness=m.thickness,
                    scattering=m.scattering, xpd_kx=m.xpd_kx, random_phases=bool(m.random_phases),
                    pattern=[m.pattern.kind, m.pattern.alpha_r, m.pattern.alpha_i,
                             m.pattern.lambda_mix]) for k, m in desc.materials.items()}
    dev = lambda s: dict(name=s.name, position=list(map(float, s.position)),  # noqa: E731
                         orientation=list(map(float, s.orientation)), pattern=s.pattern,
                         array=[s.array[0], s.array[1], float(s.array[2]), float(s.array[3])],
                         power=float(s.power), velocity=list(map(float, s.velocity)))
    g = desc.grid
    return dict(frequency=desc.frequency, materials=mats,
                objects=[dict(name=o.name, mesh_path=o.mesh_path, material=o.material,
                              velocity=list(map(float, o.velocity))) for o in desc.objects],
                transmitters=[dev(s) for s in desc.transmitters],
                receivers=[dev(s) for s in desc.receivers],
                grid=None if g is None else dict(center=g.center.tolist(), u_hat=g.u_hat.tolist(),
                                                 v_hat=g.v_hat.tolist(),
                                                 cell_size=list(g.cell_size),
                                                 shape=list(g.shape)))


def fake_paths():
    rng = np.random.default_rng(3)
    out = []
    for i in range(4):
        d = rng.normal(size=3); d /= np.linalg.norm(d)
        a = rng.normal(size=3); a /= np.linalg.norm(a)
        out.append(dict(tx_index=i % 2, rx_index=i // 2, depth=i % 3,
                        kinds=["R", "S", "T"][:i % 3 + 0] if i % 3 else [],
                        gain=complex(rng.normal() * 1e-5, rng.normal() * 1e-5),
                        delay=float(rng.uniform(1e-8, 1e-6)), doppler=float(rng.normal()),
                        departure=d.tolist(), arrival=a.tolist(),
                        vertices=rng.normal(size=(i % 3 + 2, 3)).tolist()))
    return out


def as_objects(recs):
    objs = []
    for r in recs:
        o = types.SimpleNamespace(**r)
        o.gain = complex(r["gain"][0], r["gain"][1]) if isinstance(r["gain"], list) else r["gain"]
        o.departure, o.arrival = np.array(r["departure"]), np.array(r["arrival"])
        o.vertices = np.array(r["vertices"])
        objs.append(o)
    return types.SimpleNamespace(paths=objs)
