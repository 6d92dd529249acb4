"""Pins of the f4 block epilogue of the oracle (reading R26):
act(conv * scale + shift + residual) with BatchNorm in folded inference form."""
import numpy as np

import oracle as orc


def test_identity_epilogue_is_the_conv():
    y = np.random.default_rng(0).normal(size=(7, 5))
    assert np.array_equal(orc.epilogue(y), y)


def test_relu_properties():
    y = np.random.default_rng(1).normal(size=(50, 8))
    z = orc.epilogue(y, relu=True)
    assert (z >= 0).all()
    assert np.array_equal(z[y > 0], y[y > 0]) and (z[y <= 0] == 0).all()
    assert np.array_equal(orc.epilogue(z, relu=True), z)  # idempotent


def test_worked_residual_block_example():
    # 1D, three points, submanifold map with only the centre offset and W = 1: conv(x) = x.
    # Block output relu(2 * conv(x) - 1 + x) = relu(3x - 1): residual added after the affine
    # (not scaled) and before the ReLU.  x = (0.5, -1, 2) -> (0.5, 0, 5), worked by hand.
    x = np.array([[0.5], [-1.0], [2.0]])
    csr = (np.array([0, 3], np.int64), np.array([0, 1, 2], np.int32), np.array([0, 1, 2], np.int32))
    W = np.ones((1, 1, 1))
    y = orc.conv_forward_fused(csr, x, W, 3, scale=[2.0], shift=[-1.0], residual=x, relu=True)
    assert np.allclose(y, [[0.5], [0.0], [5.0]], rtol=0, atol=1e-15)


def test_bn_fold_normalises_with_batch_statistics():
    # With gamma = 1, beta = 0 and the rows' own mean / variance, the folded affine map must
    # produce columns of mean 0 and variance var / (var + eps) (definition of BatchNorm).
    g = np.random.default_rng(2)
    y = g.normal(3.0, 2.0, size=(4000, 6)) * np.arange(1, 7)
    mean, var = y.mean(0), y.var(0)
    scale, shift = orc.bn_fold(np.ones(6), np.zeros(6), mean, var, eps=1e-3)
    z = orc.epilogue(y, scale, shift)
    assert np.allclose(z.mean(0), 0.0, atol=1e-9)
    assert np.allclose(z.var(0), var / (var + 1e-3), rtol=1e-9)
    # gamma / beta then scale and shift the normalised columns
    s2, b2 = orc.bn_fold(np.full(6, 2.0), np.full(6, 0.5), mean, var, eps=1e-3)
    z2 = orc.epilogue(y, s2, b2)
    assert np.allclose(z2, 2.0 * z + 0.5, atol=1e-9)
