"""Oracle-only expectations for the GPU parity tests.

Every expected value here is computed by ``oracle/`` from the same seeded host inputs the
GPU path receives: coordinates from ``orc.create / quantize / stride``, offsets from
``orc.region``, kernel maps from ``orc.kmap`` and features from ``orc.conv_*``.  Nothing the
GPU produced (its exported map, its region table, its coordinates) is ever fed back into
the oracle, so a defect in any GPU stage shows up as a mismatch instead of cancelling out.
The GPU artefacts are only compared against these expectations (maps and coordinates
byte-identical, features within the tolerances of ``gpu_util``).
"""
from __future__ import annotations

import os

import numpy as np
import torch

from gpu_util import assert_close, to_np


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t if dtype is None else t.to(dtype)


def oracle_threads(orc):
    """All host cores for the oracle's OpenMP loops (results are thread-count independent)."""
    return orc.set_threads(os.cpu_count() or 1)


class Spec:
    """One kernel region, described once and instantiated on both sides independently:
    ``mk.Region`` for the GPU path and ``orc.region`` for the oracle."""

    def __init__(self, kind: int, D: int, size, dilation=1):
        self.kind, self.D = kind, D
        self.size = list(size) if np.ndim(size) else [size] * D
        self.dilation = list(dilation) if np.ndim(dilation) else [dilation] * D

    def mk(self, mk):
        return mk.Region(self.kind, self.D, self.size, self.dilation)

    def orc(self, orc):
        return orc.region(self.kind, self.D, self.size, self.dilation)


def csr_host(m):
    """The GPU map's CSR, on the host (for comparison only)."""
    ptr, ins, outs = m.export()
    return ptr.cpu().numpy(), ins.cpu().numpy(), outs.cpu().numpy()


def assert_map_equal(m, okm, what=""):
    ptr, ins, outs = csr_host(m)
    assert np.array_equal(ptr, okm[0]), f"{what}: CSR offsets differ"
    assert np.array_equal(ins, okm[1]) and np.array_equal(outs, okm[2]), f"{what}: pair lists differ"


def map_pair(mk, orc, ci, co, oc_in, oc_out, spec: Spec, scale, transposed=False, what=""):
    """(GPU map, oracle CSR): the GPU map built from the GPU coordinate handles, the oracle's
    from the oracle's coordinates and offsets; asserts they are byte-identical."""
    m = mk.kmap_build(ci, co, spec.mk(mk), transposed=transposed)
    okm = orc.kmap(oc_in, oc_out, spec.orc(orc), scale, transposed)
    assert_map_equal(m, okm, what)
    return m, okm


def check_features(mk, orc, m, okm, X, W, G, dt, tol, transposed=False, what="", sample_rows=None, repeat=True):
    """fwd, dgrad and wgrad of the GPU path (dt = "f32" | "bf16") against the fp64 oracle on
    the oracle's own map.  bf16 mode rounds the same fp32 samples (R21) and is compared with
    the oracle on the ORIGINAL values.  sample_rows: (out_rows, in_rows) to compare fwd /
    dgrad on sampled rows only (the oracle evaluates them row by row); dW is always full."""
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    Xd, Wd, Gd = dev(X).to(tdt), dev(W).to(tdt), dev(G).to(tdt)
    fwd = mk.conv_transpose_forward if transposed else mk.conv_forward
    bwd = mk.conv_transpose_backward if transposed else mk.conv_backward
    K = W.shape[0]
    n_out, n_in = int(m.n_out), int(m.n_in)
    y = fwd(m, Xd, Wd, out_dtype=torch.float32)
    gin, gw = bwd(m, Gd, Xd, Wd)
    yh, ginh, gwh = to_np(y), to_np(gin), to_np(gw)
    if sample_rows is None:
        assert_close(yh, orc.conv_forward(okm, X, W, n_out), orc.conv_forward(okm, np.abs(X), np.abs(W), n_out), tol,
                     what + " fwd")
        assert_close(ginh, orc.conv_dgrad(okm, G, W, n_in), orc.conv_dgrad(okm, np.abs(G), np.abs(W), n_in), tol,
                     what + " dgrad")
    else:
        ro, ri = sample_rows
        assert_close(yh[ro], orc.conv_forward_rows(okm, X, W, ro), orc.conv_forward_rows(okm, np.abs(X), np.abs(W), ro),
                     tol, what + " fwd (sampled rows)")
        rokm = orc.kmap_reverse(okm, n_in)
        WT = np.ascontiguousarray(np.transpose(W, (0, 2, 1)))
        assert_close(ginh[ri], orc.conv_forward_rows(rokm, G, WT, ri),
                     orc.conv_forward_rows(rokm, np.abs(G), np.abs(WT), ri), tol, what + " dgrad (sampled rows)")
    assert_close(gwh, orc.conv_wgrad(okm, G, X, K), orc.conv_wgrad(okm, np.abs(G), np.abs(X), K), tol,
                 what + " wgrad")
    if repeat:  # determinism: bit-identical on repeat (fixed reduction order, R20)
        y2 = fwd(m, Xd, Wd, out_dtype=torch.float32)
        gin2, gw2 = bwd(m, Gd, Xd, Wd)
        assert torch.equal(y, y2) and torch.equal(gin, gin2) and torch.equal(gw, gw2), what + " not deterministic"
    return y, gin, gw


def sample(n: int, k: int, seed: int) -> np.ndarray:
    """k distinct sampled rows of n plus the first and last row (ragged tail), int32."""
    g = np.random.default_rng(seed)
    r = g.choice(n, min(k, n), replace=False)
    return np.unique(np.concatenate([r, [0, n - 1]])).astype(np.int32)
