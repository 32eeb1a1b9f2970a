"""k_cfr_contract across path counts and array sizes (SURVEY §8f #3 data).

For P paths per link, n_rx x n_tx elements and F subcarriers the contraction
H[(r,t), f] = sum_p W[(r,t), p] E[p, f] does 8 * rows * P * F float64 flops
and writes 16 * rows * F bytes.  Prints ms (CUDA events inside libsbr),
achieved FP64 TFLOP/s and output GB/s per shape; --check compares H with the
oracle's path-by-path sum.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_21719_b200 import _native  # noqa: E402
from paper_2504_21719_b200.cir import channel_response  # noqa: E402
from paper_2504_21719_b200.em import planar_array  # noqa: E402

lam = 299792458.0 / 3.5e9
freqs = 3.5e9 + (np.arange(1024) - 512) * 30e3
rows = []
L = _native.lib()
modes = {"simt": -1, "dmma": 0}
for (ntx, nrx) in ((8, 4), (16, 8)):
    txo = planar_array(ntx, ntx, lam / 2, lam / 2).offsets
    rxo = planar_array(nrx, nrx, lam / 2, lam / 2).offsets
    for n in (5, 20, 50, 100, 300, 1000, 2000):
        rng = np.random.default_rng(n)
        d = rng.normal(size=(n, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        a = rng.normal(size=(n, 3))
        a /= np.linalg.norm(a, axis=1, keepdims=True)
        g = (rng.normal(size=n) + 1j * rng.normal(size=n)) * 1e-6
        tau = rng.uniform(1e-8, 3e-6, n)
        args = (g, tau, d, a, freqs, txo, rxo, lam)
        for mode, mn in modes.items():
            _native.check(L.sbr_set_cfr_dmma_min_paths(mn))
            channel_response(*args, return_tensor=True)
            torch.cuda.synchronize()
            _native.profile_enable(True)
            reps = 5
            for _ in range(reps):
                H = channel_response(*args, return_tensor=True)
            torch.cuda.synchronize()
            ms, nl = _native.profile_kernel_ms("k_cfr_contract")
            _native.profile_enable(False)
            ms /= reps
            R = len(txo) * len(rxo)
            flops = 8.0 * R * n * len(freqs)
            out_b = 16.0 * R * len(freqs)
            h = H.cpu().numpy()
            if mode == "simt":
                ref = h
            rows.append({"mode": mode, "n_tx": len(txo), "n_rx": len(rxo), "paths": n,
                         "F": len(freqs), "ms": round(ms, 4),
                         "fp64_tflops": round(flops / (ms / 1e3) / 1e12, 2),
                         "write_gbs": round(out_b / (ms / 1e3) / 1e9, 1),
                         "max_dev_vs_simt": float(np.abs(h - ref).max() / np.abs(ref).max())})
            print(json.dumps(rows[-1]), flush=True)
_native.check(L.sbr_set_cfr_dmma_min_paths(16))
