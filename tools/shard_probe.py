"""Per-GPU device time of one rank's config-4 shard at N = 1, 2, 4, 8 (shard 0
of N through sbr_radiomap_bounce_sharded, no collective) on one GPU: the
per-rank time of the strong-scaling run."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2504_21719_b200 import SceneModel, _abi, _native  # noqa: E402
from paper_2504_21719_b200.radiomap import pack_map_params  # noqa: E402

meshes, mats, grid, cfg = bench.c4_workload()
sc = SceneModel(meshes, mats)
sc.bind_frequency(cfg.frequency)
params, _, _ = pack_map_params(sc, np.array(bench.C4_TX), grid, cfg)
nx, ny = grid.shape
dev = torch.device("cuda", 0)
vals = torch.zeros((ny, nx), dtype=torch.float64, device=dev)
cnt = torch.zeros(_abi.SBR_MC_COUNT, dtype=torch.int64, device=dev)
st = torch.cuda.current_stream(dev)
L = _native.lib()
base = None
for n, r in ((1, 0), (2, 0), (2, 1), (4, 0), (4, 3), (8, 0), (8, 5)):
    def step():
        vals.zero_()
        cnt.zero_()
        _native.check(L.sbr_radiomap_bounce_sharded(sc.accel.handle, ctypes.byref(params), r, n,
                                                     _native.ptr(vals), _native.ptr(cnt),
                                                     ctypes.c_void_p(st.cuda_stream)))
    step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        step()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    base = base or ms
    rb = int(cnt[_abi.MAP_COUNTERS.index("ray_bounces")].item())
    print(n, "ms", round(ms, 2), "efficiency vs N=1", round(base / (n * ms), 3), "rb", rb,
          "rb/s", f"{rb / ms * 1e3:.3e}", flush=True)
