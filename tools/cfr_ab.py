"""CFR timing (channel_response = sbr_cfr + host copy) on random path sets:
    SBR_LIB_PATH=... python tools/cfr_ab.py"""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_21719_b200.cir import channel_response
from paper_2504_21719_b200.em import planar_array
lam = 299792458.0 / 3.5e9
txo = planar_array(8, 8, lam / 2, lam / 2).offsets
rxo = planar_array(4, 4, lam / 2, lam / 2).offsets
freqs = 3.5e9 + (np.arange(1024) - 512) * 30e3
out = {"lib": os.path.basename(os.environ.get("SBR_LIB_PATH", "default"))}
for n in (5, 50, 300):
    rng = np.random.default_rng(n)
    d = rng.normal(size=(n, 3)); d /= np.linalg.norm(d, axis=1, keepdims=True)
    a = rng.normal(size=(n, 3)); a /= np.linalg.norm(a, axis=1, keepdims=True)
    g = rng.normal(size=n) + 1j * rng.normal(size=n)
    tau = rng.uniform(1e-8, 3e-6, n)
    args = (g, tau, d, a, freqs, txo, rxo, lam)
    channel_response(*args, return_tensor=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        H = channel_response(*args, return_tensor=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    h = H.cpu().numpy()
    out[f"paths{n}_ms"] = min(ts)
    out[f"paths{n}_sum"] = float(np.abs(h).sum())
print(json.dumps(out))
