"""Count launch directions where CUDA's f64 sin/cos differ from glibc (numpy)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2504_21719_b200.sampling import fibonacci_directions

GOLD = (1.0 + 5.0 ** 0.5) / 2.0
for N in (20000, 100000, 1000000, 10000000):
    g = fibonacci_directions(N, device="cuda:0").cpu().numpy()
    n = np.arange(N, dtype=np.float64) - (N // 2)
    cos_t = 2.0 * n / N
    sin_t = np.sqrt(np.maximum(0.0, 1.0 - cos_t ** 2))
    phi = 2.0 * np.pi * n / GOLD
    ref = np.stack([sin_t * np.cos(phi), sin_t * np.sin(phi), cos_t], axis=1)
    diff = np.any(g != ref, axis=1)
    print(N, "mismatched rows:", int(diff.sum()), "frac", diff.mean(),
          "max abs", float(np.abs(g - ref).max()))
