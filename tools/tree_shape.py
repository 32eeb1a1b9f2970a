"""Shape of the device BVH for libsbr variants: depth statistics, per-level SAH
share, and the boxes of the top levels (city).  python tools/tree_shape.py v1 v2 ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys; sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tools")
import numpy as np
from tree_quality import sa
from paper_2504_21719_b200 import scenes
from paper_2504_21719_b200.geometry import build_scene_accel
import time
meshes = scenes.city()
build_scene_accel(meshes)
t0 = time.perf_counter(); acc = build_scene_accel(meshes); build_s = time.perf_counter() - t0
boxes, codes = acc.bvh_nodes()
n = len(codes)
depth = np.zeros(n, np.int64); todo = [0]
leaf_depths = []
lvl_sa = {}
root_sa = sa(boxes[0, :, 0].min(0), boxes[0, :, 1].max(0))
while todo:
    i = todo.pop()
    for c in range(2):
        s_ = sa(boxes[i, c, 0], boxes[i, c, 1]) / root_sa
        d = depth[i] + 1
        lvl_sa[d] = lvl_sa.get(d, 0.0) + s_
        if codes[i, c] >= 0:
            depth[codes[i, c]] = d; todo.append(int(codes[i, c]))
        else:
            leaf_depths.append(d)
ld = np.array(leaf_depths)
print("SHAPE build %.3f s nodes %d leaves %d depth mean %.1f p50 %d p99 %d max %d | SA by level 1-12: %s" % (
    build_s, n, len(ld), ld.mean(), np.percentile(ld, 50), np.percentile(ld, 99), ld.max(),
    " ".join("%.2f" % lvl_sa.get(d, 0) for d in range(1, 13))))
'''
for v in ["default"] + sys.argv[1:]:
    env = dict(os.environ)
    if v != "default":
        env["SBR_LIB_PATH"] = os.path.join(ROOT, "paper_2504_21719_b200/_lib/variants/libsbr_%s.so" % v)
    r = subprocess.run([sys.executable, "-c", CHILD.replace("ROOT", repr(ROOT))], env=env,
                       capture_output=True, text=True)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("SHAPE")]
    print(v, line[-1] if line else r.stderr[-500:], flush=True)
