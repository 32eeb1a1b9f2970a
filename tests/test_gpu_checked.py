"""Every kernel family through the checked build of libsbr (-DSBR_CHECKED).

compute-sanitizer is closed on the GPU pool, so memory-safety evidence comes
from device-side index-range assertions compiled into _lib/checked/libsbr.so
(BVH node and leaf ranges in every traversal, candidate-occluder ids, ray /
scatter queue slots, hit-buffer indices, the visibility kernel's
shared-memory queue): a failed check sets a bit in the scene's error word and
the next sbr_scene_check raises.  The workloads are tools/sanitize_cases.py
(radio maps with {R,S,T}, roulette, threshold, cyclic shards; CIR with heavy
hash collisions, truncation, 64 receivers; PLOC and LBVH builds including a
degenerate deep chain; diffraction CIR and the edge map), each in a fresh
process with SBR_LIB_PATH pointing at the checked library.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2504_21719_b200", "_lib", "checked", "libsbr.so")


@pytest.mark.parametrize("case", ["map", "cir", "build", "edge"])
def test_kernels_pass_device_bounds_checks(cuda, case):
    if not os.path.exists(CHECKED):
        pytest.fail("checked library missing: run __graft_entry__.build()")
    env = dict(os.environ, SBR_LIB_PATH=CHECKED, SBR_REQUIRE_CHECKED="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"), case],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    assert " ok" in r.stdout
