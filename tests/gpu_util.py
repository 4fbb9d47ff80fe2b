"""Helpers for the -m gpu parity tests (test infrastructure)."""
import numpy as np


def cuda(a):
    import torch
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 2:                     # column-major device copy
        return torch.tensor(np.asfortranarray(a).T.copy(), device="cuda").t()
    return torch.tensor(a, device="cuda")


def host(t):
    return t.detach().cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))
