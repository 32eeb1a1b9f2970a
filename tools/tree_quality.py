"""SAH cost of the device BVH (LBVH / PLOC) vs the reference's binned SAH tree (oracle).

cost = sum_inner SA(node)/SA(root) * C_t + sum_leaf SA(leaf)/SA(root) * n_tris * C_i,
C_t = 1, C_i = 1 (relative comparison only).
"""
import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())


def sa(lo, hi):
    d = np.maximum(hi - lo, 0)
    return 2 * (d[..., 0] * d[..., 1] + d[..., 1] * d[..., 2] + d[..., 2] * d[..., 0])


def device_cost(acc):
    boxes, codes = acc.bvh_nodes()
    lo = boxes[0, :, 0].min(0); hi = boxes[0, :, 1].max(0)
    root = sa(lo, hi)
    child_sa = sa(boxes[:, :, 0], boxes[:, :, 1])        # (M, 2)
    inner = codes >= 0
    cnt = np.where(inner, 0, (~codes & 3) + 1)
    return 1.0 + (child_sa * inner).sum() / root + (child_sa * cnt).sum() / root


def oracle_cost(sc):
    n = sc.num_nodes
    lo, hi = sc.bmin[:n], sc.bmax[:n]
    s = sa(lo, hi)
    inner = sc.count[:n] == 0
    return (s[inner].sum() + (s * sc.count[:n])[~inner].sum()) / s[0]


if __name__ == "__main__":
    import oracle
    from paper_2504_21719_b200 import _native, scenes
    from paper_2504_21719_b200.geometry import build_scene_accel
    for name, meshes in (("canyon", scenes.street_canyon()), ("city", scenes.city())):
        out = [name]
        for b in (0, 1):
            _native.check(_native.lib().sbr_set_bvh_builder(b))
            acc = build_scene_accel(meshes)
            out.append(f"{['lbvh', 'ploc'][b]} {device_cost(acc):.1f} ({acc.num_nodes} inner)")
        osc = oracle.OracleScene(meshes)
        out.append(f"sah(reference) {oracle_cost(osc):.1f} ({osc.num_nodes} nodes)")
        print(" | ".join(out), flush=True)
