"""Generate golden vectors from the REAL reference (emtrace) for the parity tests.

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py [--ref /tmp/refpkg/src]

The reference is imported from a built copy (Cython kernel compiled with
`python setup.py build_ext --inplace` in a /tmp copy of /root/reference/pkg),
or straight from /root/reference/pkg/src (bit-identical numpy kernel) when no
built copy is given.  Outputs are small .npz fixtures next to this script;
they travel to the GPU box, /root/reference does not.
"""

import argparse
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def _import_reference(path):
    sys.path.insert(0, path)
    import emtrace  # noqa: F401
    return emtrace


def mesh_digest(meshes):
    h = hashlib.sha256()
    for m in meshes:
        h.update(np.ascontiguousarray(m.vertices, dtype=np.float64).tobytes())
        h.update(np.ascontiguousarray(m.triangles, dtype=np.int64).tobytes())
        h.update(str(int(m.object_id)).encode())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    default = "/tmp/refpkg/src" if os.path.isdir("/tmp/refpkg/src") else "/root/reference/pkg/src"
    ap.add_argument("--ref", default=default)
    args = ap.parse_args()
    _import_reference(args.ref)
    sys.path.insert(0, ROOT)

    from emtrace import _kernels
    from emtrace.em import ArrayGeometry, make_pattern as ref_pattern
    from emtrace.geometry import Mesh as RMesh, build_scene_accel
    from emtrace.materials import RadioMaterial as RMat, ScatteringPattern as RSP, slab_fresnel
    from emtrace.paths import SceneModel as RScene, _plane_hash_rows
    from emtrace.radiomap import MeasurementGrid as RGrid, RadioMapConfig as RCfg
    from emtrace.radiomap import compute_radio_map_sbr
    from emtrace.sampling import Interaction as RI, RngStream, fibonacci_directions

    from paper_2504_21719_b200 import scenes

    print("reference kernel backend:", _kernels.backend_name())
    conv = lambda ms: [RMesh(m.vertices, m.triangles, object_id=m.object_id) for m in ms]  # noqa

    # -- RNG streams -----------------------------------------------------------
    streams = [(0, 0, 1, "interaction"), (0, 3, 2, "map-interaction"), (7, 1, 0, "map-respawn"),
               (2**40 + 3, 2**33, 5, "map-roulette"), (1, 0, 3, "phase-2")]
    draws = np.array([RngStream(s, sample=k, depth=d, purpose=p).generator().random(67)
                      for s, k, d, p in streams])
    np.savez_compressed(os.path.join(HERE, "rng.npz"), draws=draws,
                        seeds=np.array([s[0] for s in streams], dtype=np.uint64),
                        samples=np.array([s[1] for s in streams], dtype=np.uint64),
                        depths=np.array([s[2] for s in streams], dtype=np.uint64),
                        purposes=np.array([s[3] for s in streams]))

    # -- Fibonacci lattice ------------------------------------------------------
    fib = {f"full_{n}": fibonacci_directions(n) for n in (1, 2, 7, 1000)}
    big = fibonacci_directions(10_000_000)
    for lo in (0, 4_999_968, 9_999_936):
        fib[f"big_{lo}"] = big[lo:lo + 64]
    del big
    np.savez_compressed(os.path.join(HERE, "fibonacci.npz"), **fib)

    # -- slab Fresnel -------------------------------------------------------------
    mats = [RMat("concrete", eps_r=5.24, sigma=0.0462, thickness=0.1),
            RMat("c2", eps_r=5.24, sigma=0.1, thickness=0.3),
            RMat("glass", eps_r=6.31, sigma=0.0236, thickness=0.003),
            RMat("metal", eps_r=1.0, sigma=1e7, thickness=0.1),
            RMat("vacuum"),
            RMat("lossless", eps_r=3.0, sigma=0.0, thickness=0.05)]
    cos = np.concatenate([np.linspace(0.0, 1.0, 101), [1e-9, 0.5 + 1e-12]])
    fres = []
    for m in mats:
        lam = 299792458.0 / 3.5e9
        f = slab_fresnel(cos, m.complex_permittivity(3.5e9), m.thickness, lam)
        fres.append(np.stack([f.r_perp, f.r_par, f.t_perp, f.t_par], axis=1))
    np.savez_compressed(os.path.join(HERE, "fresnel.npz"), cos=cos, coeff=np.array(fres),
                        eps_r=[m.eps_r for m in mats], sigma=[m.sigma for m in mats],
                        thickness=[m.thickness for m in mats])

    # -- traversal ----------------------------------------------------------------
    rng = np.random.default_rng(0xC0FFEE)
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(args.ref)), "tests"))
    from conftest import random_soup, box_mesh  # reference test fixtures
    meshes = [random_soup(rng, 400, span=2.0, object_id=i) for i in range(3)]
    meshes.append(box_mesh([-1, -1, -1], [1, 1, 1], object_id=9))
    acc = build_scene_accel(meshes)
    n = 4000
    o = rng.normal(size=(n, 3)) * 3.0
    d = rng.uniform(-1, 1, size=(n, 3)) - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t, tri, u, v = acc.trace_batch(o, d)
    obj = np.where(tri >= 0, acc.tri_object_id[tri], -1)
    prim = np.where(tri >= 0, acc.tri_primitive_id[tri], -1)
    tmax = rng.uniform(0.5, 6.0, size=n)
    anyhit = _kernels.active().trace_any(*acc._args(), o, d, 1e-4, tmax)
    a = rng.uniform(-1.5, 1.5, (2000, 3))
    b = rng.uniform(-1.5, 1.5, (2000, 3))
    occ = acc.occluded_batch(a, b)
    soup = {}
    for i, m in enumerate(meshes):
        soup[f"verts_{i}"] = m.vertices
        soup[f"tris_{i}"] = m.triangles
        soup[f"oid_{i}"] = np.array(m.object_id)
    np.savez_compressed(os.path.join(HERE, "trace.npz"), origins=o, dirs=d, t=t, obj=obj,
                        prim=prim, u=u, v=v, tmax=tmax, anyhit=anyhit, seg_a=a, seg_b=b,
                        occluded=occ, nmesh=len(meshes), **soup)

    # -- plane hashes ----------------------------------------------------------------
    hn = rng.normal(size=(300, 3))
    hp = rng.uniform(-50, 50, size=(300, 3))
    hn[:10] = [1, 0, 0]
    hn[10:20] = [0, 0, -1]
    hr, hf = _plane_hash_rows(hn, hp)
    np.savez_compressed(os.path.join(HERE, "hashes.npz"), normals=hn, points=hp, hash_r=hr,
                        hash_f=hf)

    # -- radio maps --------------------------------------------------------------------
    R, S, T = RI.REFLECTION, RI.SCATTERING, RI.TRANSMISSION
    box = scenes.box_room_walls()
    canyon = scenes.street_canyon()
    cases = {
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
                                 grid=((0.0, 0.0, 1.0), (0, 1, 0), (0, 0, 1), (0.7, 0.4),
                                       (6, 5)),
                                 cfg=dict(num_samples=50_000, max_depth=4, seed=4,
                                          gain_threshold=1e-4), kinds="RST",
                                 src=(1.0, 2.0, 2.0)),
        "box_directive_array": dict(scene="box",
                                    mat=dict(eps_r=5.24, sigma=0.1, thickness=0.3,
                                             scattering=0.5, pattern=("directive", 4, 1, 1.0)),
                                    grid=((0.5, 1.0, 1.2), (1, 0, 0), (0, 1, 0), (1.0, 1.0),
                                          (4, 6)),
                                    cfg=dict(num_samples=40_000, max_depth=3, seed=2),
                                    kinds="RS", src=(-1.0, -2.0, 1.5),
                                    pattern=("tr38901", (0.4, -0.2, 0.1)), array=True),
        "canyon_rs": dict(scene="canyon",
                          mat=dict(eps_r=5.24, sigma=0.0462, thickness=0.1, scattering=0.3),
                          grid=((0.0, 0.0, 1.5), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (200, 200)),
                          cfg=dict(num_samples=30_000, max_depth=5, seed=0), kinds="RS",
                          src=(0.0, 5.0, 20.0)),
    }
    kindmap = {"R": R, "S": S, "T": T}
    out = {}
    for name, c in cases.items():
        meshes = box if c["scene"] == "box" else canyon
        md = dict(c["mat"])
        pat = md.pop("pattern", None)
        if pat is not None:
            md["pattern"] = RSP(kind=pat[0], alpha_r=pat[1], alpha_i=pat[2], lambda_mix=pat[3])
        mat = RMat("m", **md)
        rs = RScene(conv(meshes), {m.object_id: mat for m in meshes})
        grid = RGrid(*c["grid"])
        cfg = RCfg(enabled=frozenset(kindmap[k] for k in c["kinds"]), **c["cfg"])
        kw = {}
        if "pattern" in c:
            kw["pattern"] = ref_pattern(c["pattern"][0], orientation=c["pattern"][1])
        if c.get("array"):
            lam = cfg.wavelength
            off = np.zeros((4, 3))
            off[:, 1] = np.arange(4) * lam / 2.0
            kw["array"] = ArrayGeometry(off)
            kw["precoder"] = np.array([0.5, 0.5j, -0.5, 0.1 + 0.3j])
        vals, diag = compute_radio_map_sbr(rs, np.array(c["src"]), grid, cfg, **kw)
        out[f"{name}__values"] = vals
        for k, val in diag.items():
            out[f"{name}__diag__{k}"] = np.array(val)
        print(name, {k: v for k, v in diag.items()})
    out["canyon_digest"] = np.array(mesh_digest(canyon))
    out["box_digest"] = np.array(mesh_digest(box))
    np.savez_compressed(os.path.join(HERE, "radiomap.npz"), **out)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
