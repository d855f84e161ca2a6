"""Shared test helpers: tolerances and comparisons (normwise)."""
import numpy as np

# north_star: fp32 outputs within 1e-4, bf16 tensor-core mode within 2e-2, measured
# normwise: max|got - want| / max|want| (element-wise relative error is meaningless
# where outputs cross zero).
TOL_F32 = 1e-4
TOL_BF16 = 2e-2


def normwise(got, want) -> float:
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    den = np.abs(want).max()
    return float(np.abs(got - want).max() / (den if den > 0 else 1.0))


def to_np(t):
    import torch
    return t.detach().float().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def dev(a, dtype=None):
    """numpy (or tensor) -> CUDA tensor of the given dtype (fp32 by default)."""
    import torch
    t = torch.as_tensor(np.ascontiguousarray(a)) if not isinstance(a, torch.Tensor) else a
    return t.to("cuda", dtype or torch.float32)
