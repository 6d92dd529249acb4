"""Helpers shared by the GPU parity tests (comparison rules of DESIGN.md §3, reading R21)."""
import numpy as np
import torch

FP32_TOL = 1e-5   # BASELINE.json north_star: fp32 mode
BF16_TOL = 2e-2   # BASELINE.json north_star: bf16 inputs


def rel_errors(y, y64, scale64):
    """(normwise, componentwise) errors of y against the fp64 oracle y64.

    normwise      = max|y - y64| / max|y64|
    componentwise = max |y - y64| / (|W| |x|)  with |W||x| the oracle's conv of absolute
                    values (the dot-product error scale; elements with zero scale are exact).
    """
    y = np.asarray(y, np.float64)
    d = np.abs(y - y64)
    norm = d.max() / max(np.abs(y64).max(), 1e-300) if d.size else 0.0
    with np.errstate(divide="ignore", invalid="ignore"):
        comp = np.where(scale64 > 0, d / scale64, np.where(d > 0, np.inf, 0.0))
    return float(norm), float(comp.max() if comp.size else 0.0)


def assert_close(y, y64, scale64, tol, what=""):
    norm, comp = rel_errors(y, y64, scale64)
    assert norm <= tol and comp <= tol, f"{what}: normwise {norm:.3e} componentwise {comp:.3e} > {tol}"


def to_np(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy() if t.dtype == torch.bfloat16 else t.detach().cpu().numpy()

