import sys, os, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2504_21719_b200 import SceneModel, compute_radio_map_sbr, _native
meshes, mats, grid, cfg = bench.c4_workload()
sc = SceneModel(meshes, mats)
run = bench.MapRunner(sc, grid, cfg, bench.C4_TX, torch.device("cuda", 0), 0, 1)
st = run.stream
def timeit(f, n=4):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); f(); b.record(st); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return np.round(ts, 1)
for ns in (2, 1, 2):
    _native.check(_native.lib().sbr_set_wave_streams(ns))
    print(ns, "runner", timeit(run.step), "api", timeit(lambda: compute_radio_map_sbr(sc, np.array(bench.C4_TX), grid, cfg)),
          "api-tensors", timeit(lambda: compute_radio_map_sbr(sc, np.array(bench.C4_TX), grid, cfg, return_tensors=True)), flush=True)
