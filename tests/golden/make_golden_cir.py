"""Golden CIR / path-solver vectors from the REAL reference (emtrace), for parity tests.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_cir.py [--ref /tmp/refpkg/src]

Cases are defined in tests/cir_cases.py (shared with the tests).  For every
case this records, from emtrace's own entry points:
  * generate_candidates(...) for the first source: the record list
    (sample, target, depth, suffix_start, diffuse flag, chain hash, prefix
    probability, anchor, per-step kind/object/primitive/vertex/normal) and
    the generation diagnostics;
  * compute_paths(...): every ValidPath (indices, gain, delay, doppler,
    departure, arrival, vertices, steps, chain hash, sample) and the
    diagnostics incl. refinement rejections;
  * frequency_response / baseband_gains for cases that ask for them.
Outputs: tests/golden/cir.npz (small).  /root/reference never travels to the
GPU box; these fixtures do.
"""

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
KIND = {"R": 0, "S": 1, "T": 2, "D": 3}


def main():
    ap = argparse.ArgumentParser()
    default = "/tmp/refpkg/src" if os.path.isdir("/tmp/refpkg/src") else "/root/reference/pkg/src"
    ap.add_argument("--ref", default=default)
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import emtrace
    from emtrace import _kernels
    from emtrace.em import ArrayGeometry, make_pattern
    from emtrace.geometry import Mesh as RMesh
    from emtrace.materials import RadioMaterial as RMat, ScatteringPattern as RSP
    from emtrace.paths import (PathConfig, RadioDevice, SceneModel, baseband_gains,
                               compute_paths, frequency_response, generate_candidates)
    from emtrace.sampling import Interaction as RI

    from cir_cases import CIR_CASES, case_geometry, mesh_digest

    print("reference backend:", _kernels.backend_name())
    kinds = {"R": RI.REFLECTION, "S": RI.SCATTERING, "T": RI.TRANSMISSION, "D": RI.DIFFRACTION}

    out_path = os.path.join(HERE, "cir.npz")
    out = dict(np.load(out_path)) if (args.only and os.path.exists(out_path)) else {}
    for name, c in CIR_CASES.items():
        if args.only and name != args.only:
            continue
        meshes, mats, velocities = case_geometry(name)
        rmeshes = [RMesh(m.vertices, m.triangles, object_id=m.object_id) for m in meshes]
        rmats = {}
        for oid, md in mats.items():
            md = dict(md)
            pat = md.pop("pattern", None)
            if pat is not None:
                md["pattern"] = RSP(kind=pat[0], alpha_r=pat[1], alpha_i=pat[2],
                                    lambda_mix=pat[3])
            rmats[oid] = RMat("m%d" % oid, **md)
        scene = SceneModel(rmeshes, rmats, velocities=velocities)
        cfg_kw = dict(c["cfg"])
        cfg_kw["enabled"] = frozenset(kinds[k] for k in c["kinds"])
        cfg = PathConfig(**cfg_kw)

        def device(d):
            kw = {}
            if d.get("pattern"):
                kw["pattern"] = make_pattern(d["pattern"][0], orientation=d["pattern"][1])
            if d.get("array"):
                kw["array"] = ArrayGeometry(np.asarray(d["array"], dtype=np.float64))
            if d.get("velocity") is not None:
                kw["velocity"] = np.asarray(d["velocity"], dtype=np.float64)
            return RadioDevice(position=np.asarray(d["pos"], dtype=np.float64), **kw)

        txs = [device(d) for d in c["tx"]]
        rxs = [device(d) for d in c["rx"]]
        p = f"{name}__"
        out[p + "digest"] = np.array(mesh_digest(meshes))
        W = scene.wedges
        out[p + "wedge_origin"] = np.array([w.origin for w in W]).reshape(-1, 3)
        out[p + "wedge_ehat"] = np.array([w.e_hat for w in W]).reshape(-1, 3)
        out[p + "wedge_length"] = np.array([w.length for w in W])
        out[p + "wedge_n0"] = np.array([w.n0_hat for w in W]).reshape(-1, 3)
        out[p + "wedge_nn"] = np.array([w.nn_hat for w in W]).reshape(-1, 3)
        out[p + "wedge_t0"] = np.array([w.t0_hat for w in W]).reshape(-1, 3)
        out[p + "wedge_n"] = np.array([w.n for w in W])
        own = [(wi, side, o, m, le) for wi, w in enumerate(W)
               for side, lst in ((0, w.face0), (1, w.facen)) for (o, m, le) in lst]
        out[p + "wedge_owners"] = np.array(own, dtype=np.int64).reshape(-1, 5)
        out[p + "wedge_hash_r"] = np.asarray(scene.wedge_hash_round, dtype=np.uint64)
        out[p + "wedge_hash_f"] = np.asarray(scene.wedge_hash_floor, dtype=np.uint64)

        # -- generation (first source, synthetic reference position) -----------
        t0 = time.perf_counter()
        targets = np.array([r.position for r in rxs]) if cfg.synthetic_arrays else \
            np.concatenate([r.element_positions() for r in rxs])
        gen = generate_candidates(scene, txs[0].position if cfg.synthetic_arrays
                                  else txs[0].element_positions()[0], targets, cfg)
        recs = gen.records
        L = max([len(r.steps) for r in recs] + [1])
        n = len(recs)
        g = {
            "sample": np.array([r.sample_id for r in recs], np.int64),
            "target": np.array([r.target_id for r in recs], np.int64),
            "depth": np.array([len(r.steps) for r in recs], np.int64),
            "suffix_start": np.array([r.suffix_start for r in recs], np.int64),
            "diffuse": np.array([r.diffuse_terminal for r in recs], bool),
            "chain_hash": np.array([r.chain_hash for r in recs], np.uint64),
            "prefix_prob": np.array([r.prefix_probability for r in recs]),
            "anchor": np.array([r.anchor for r in recs]).reshape(n, 3),
            "kind": np.full((n, L), -1, np.int64),
            "obj": np.full((n, L), -1, np.int64),
            "prim": np.full((n, L), -1, np.int64),
            "wedge": np.full((n, L), -1, np.int64),
            "vertex": np.zeros((n, L, 3)),
            "normal": np.zeros((n, L, 3)),
        }
        for i, r in enumerate(recs):
            for j, st in enumerate(r.steps):
                g["wedge"][i, j] = st.wedge_index
                g["kind"][i, j] = KIND[st.kind.value]
                g["obj"][i, j] = st.object_id
                g["prim"][i, j] = st.primitive_id
                g["vertex"][i, j] = st.vertex
                g["normal"][i, j] = st.normal
        for k, v in g.items():
            out[p + "gen_" + k] = v
        for k, v in gen.diagnostics.items():
            out[p + "gendiag__" + k] = np.array(v)
        t_gen = time.perf_counter() - t0

        # -- full solver ----------------------------------------------------------
        t0 = time.perf_counter()
        ps = compute_paths(scene, txs, rxs, cfg)
        t_paths = time.perf_counter() - t0
        paths = ps.paths
        n = len(paths)
        L = max([p_.depth for p_ in paths] + [1])
        r = {
            "tx": np.array([q.tx_index for q in paths], np.int64),
            "tx_el": np.array([q.tx_element for q in paths], np.int64),
            "rx": np.array([q.rx_index for q in paths], np.int64),
            "rx_el": np.array([q.rx_element for q in paths], np.int64),
            "gain": np.array([q.gain for q in paths], np.complex128),
            "delay": np.array([q.delay for q in paths]),
            "doppler": np.array([q.doppler for q in paths]),
            "departure": np.array([q.departure for q in paths]).reshape(n, 3),
            "arrival": np.array([q.arrival for q in paths]).reshape(n, 3),
            "depth": np.array([q.depth for q in paths], np.int64),
            "chain_hash": np.array([q.chain_hash for q in paths], np.uint64),
            "sample": np.array([q.sample_id for q in paths], np.int64),
            "kind": np.full((n, L), -1, np.int64),
            "obj": np.full((n, L), -1, np.int64),
            "prim": np.full((n, L), -1, np.int64),
            "wedge": np.full((n, L), -1, np.int64),
            "vertices": np.zeros((n, L + 2, 3)),
        }
        for i, q in enumerate(paths):
            r["vertices"][i, :q.depth + 2] = q.vertices
            for j, st in enumerate(q.steps):
                r["wedge"][i, j] = st.wedge_index
                r["kind"][i, j] = KIND[st.kind.value]
                r["obj"][i, j] = st.object_id
                r["prim"][i, j] = st.primitive_id
        for k, v in r.items():
            out[p + "path_" + k] = v
        for k, v in ps.diagnostics.items():
            if k == "refinement_rejections":
                for kk, vv in v.items():
                    out[p + "diag__rej__" + kk] = np.array(vv)
            else:
                out[p + "diag__" + k] = np.array(v)
        if c.get("freqs") is not None:
            f = np.asarray(c["freqs"], dtype=np.float64)
            out[p + "cfr"] = frequency_response(ps, f, 0, 0)
            gains, delays = baseband_gains(ps, 0, 0)
            out[p + "bb_gain"] = gains
            out[p + "bb_delay"] = delays
        print(f"{name}: {len(gen.records)} records ({t_gen:.2f} s), {len(paths)} paths "
              f"({t_paths:.2f} s); diag {ps.diagnostics}")
    np.savez_compressed(out_path, **out)
    print("written", out_path, os.path.getsize(out_path), "bytes")


if __name__ == "__main__":
    main()
