"""SAH cost of the device BVH for libsbr variants (e.g. PLOC radii), city + canyon.

    python tools/tree_sah_variants.py r4 r6 r8 ...   (variants under _lib/variants)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys; sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tools")
from tree_quality import device_cost
from paper_2504_21719_b200 import scenes
from paper_2504_21719_b200.geometry import build_scene_accel
out = []
for name, meshes in (("canyon", scenes.street_canyon()), ("city", scenes.city())):
    acc = build_scene_accel(meshes)
    out.append("%s %.2f" % (name, device_cost(acc)))
print("SAH", " | ".join(out))
'''
for v in ["default"] + sys.argv[1:]:
    env = dict(os.environ)
    if v != "default":
        env["SBR_LIB_PATH"] = os.path.join(ROOT, "paper_2504_21719_b200/_lib/variants/libsbr_%s.so" % v)
    r = subprocess.run([sys.executable, "-c", CHILD.replace("ROOT", repr(ROOT))], env=env,
                       capture_output=True, text=True)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("SAH")]
    print(v, line[-1] if line else r.stderr[-500:], flush=True)
