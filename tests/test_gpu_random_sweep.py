"""Seeded random sweeps of the integer / copy paths against the CPU oracle — bit-exact
(reference sweep space `verify.py:60-76`): reduce_mask (MAX and AVG), gather (+transpose),
scatter / scatter_add, gather_grad, scatter_grad, downsample_mask; plus the edge cases the
reference tests hold (empty list, zero frames of activity, one-pixel masks, blocks larger
than the image)."""
import numpy as np
import pytest
import torch

import paper_1801_02108_b200 as P
from oracle import sbnet_oracle as O

pytestmark = pytest.mark.gpu


def _cfg(rng):
    n = int(rng.integers(1, 4))
    c = int(rng.integers(1, 17))
    kh = int(rng.choice([1, 2, 3, 5]))
    kw = int(rng.choice([1, 3, 5]))
    sh = int(rng.integers(1, kh + 1))
    sw = int(rng.integers(1, kw + 1))
    h = int(rng.integers(max(kh, 3), 70))
    w = int(rng.integers(max(kw, 3), 70))
    same = bool(rng.random() < 0.5)
    bh = kh + sh * int(rng.integers(1, 12))
    bw = kw + sw * int(rng.integers(1, 12))
    return n, h, w, c, (kh, kw), (sh, sw), same, (bh, bw)


def _mask(rng, n, h, w):
    kind = rng.integers(0, 5)
    if kind == 0:
        return np.zeros((n, h, w), np.uint8)
    if kind == 1:
        m = np.zeros((n, h, w), np.uint8)
        m[:, rng.integers(h), rng.integers(w)] = 1
        return m
    return (rng.random((n, h, w)) < [0.01, 0.05, 0.3][kind - 2]).astype(np.uint8)


@pytest.mark.parametrize("seed", range(4))
def test_random_copy_paths_bit_exact(cuda_device, seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(15):
        n, h, w, c, k, s, same, b = _cfg(rng)
        p = P.ConvParams(k, s, P.Padding.SAME if same else P.Padding.VALID, c)
        try:
            spec = P.compute_block_spec((n, h, w, c), p, b)
        except P.GeometryError:
            continue
        geo = O.geometry(h, w, k, s, same, b)
        m = _mask(rng, n, h, w)
        idx = P.reduce_mask(P.BinaryMask(m), spec)
        ref = O.reduce_mask(m, geo)
        assert np.array_equal(idx.entries, ref)
        thr = float(rng.choice([0.25, 0.5, 1.0]))
        assert np.array_equal(P.reduce_mask(P.BinaryMask(m), spec, P.PoolMode.AVG, thr).entries,
                              O.reduce_mask(m, geo, "avg", thr))
        dt = [np.float32, np.float64][int(rng.integers(2))]
        x = rng.standard_normal((n, h, w, c)).astype(dt)
        g = P.gather(P.Tensor4D(x), idx, spec)
        assert np.array_equal(g.tensor.data.cpu().numpy(), O.gather(x, ref, geo))
        gt = P.gather_transpose(P.Tensor4D(x), idx, spec)
        assert np.array_equal(gt.tensor.data.cpu().numpy(), O.gather_transpose(x, ref, geo))
        obh, obw = spec.out_block_size
        blk = rng.standard_normal((len(ref), obh, obw, c)).astype(dt)
        dst = rng.standard_normal((n, *spec.out_size, c)).astype(dt)
        gb = g.with_tensor(P.Tensor4D(blk))
        assert np.array_equal(P.scatter(gb, spec, P.Tensor4D(dst)).data.cpu().numpy(), O.scatter(blk, ref, geo, dst))
        assert np.array_equal(P.scatter_add(gb, spec, P.Tensor4D(dst)).data.cpu().numpy(),
                              O.scatter(blk, ref, geo, dst, add=True))
        gblk = rng.standard_normal((len(ref), *spec.block_size, c)).astype(dt)
        assert np.array_equal(P.gather_grad(g.with_tensor(P.Tensor4D(gblk)), spec, (n, h, w, c)).data.cpu().numpy(),
                              O.gather_grad(gblk, ref, geo, (n, h, w, c)))
        assert np.array_equal(P.scatter_grad(P.Tensor4D(dst), idx, spec).tensor.data.cpu().numpy(),
                              O.scatter_grad(dst, ref, geo))


@pytest.mark.parametrize("factor", [1, 2, 3, 4, 7])
def test_random_downsample_bit_exact(cuda_device, factor):
    rng = np.random.default_rng(factor)
    m = (rng.random((2, 37, 53)) < 0.1).astype(np.uint8)
    assert np.array_equal(P.downsample_mask(P.BinaryMask(m), factor).data.cpu().numpy(),
                          O.downsample_mask(m, factor))


def test_block_larger_than_image_and_empty_lists(cuda_device):
    x = np.arange(2 * 5 * 6 * 3, dtype=np.float32).reshape(2, 5, 6, 3)
    p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, 3)
    spec = P.compute_block_spec(x.shape, p, (16, 16))  # one block covers everything
    geo = O.geometry(5, 6, (3, 3), (1, 1), True, (16, 16))
    m = np.zeros((2, 5, 6), np.uint8)
    m[1, 4, 5] = 1
    idx = P.reduce_mask(P.BinaryMask(m), spec)
    assert idx.entries.tolist() == [[1, 0, 0]]
    g = P.gather(P.Tensor4D(x), idx, spec)
    assert np.array_equal(g.tensor.data.cpu().numpy(), O.gather(x, O.reduce_mask(m, geo), geo))
    empty = P.reduce_mask(P.BinaryMask(np.zeros((2, 5, 6), np.uint8)), spec)
    assert empty.count == 0
    g0 = P.gather(P.Tensor4D(x), empty, spec)
    assert tuple(g0.tensor.data.shape) == (0, 16, 16, 3)
    out = P.scatter(g0.with_tensor(P.Tensor4D(np.zeros((0, 14, 14, 3), np.float32))), spec, P.Tensor4D(x))
    assert np.array_equal(out.data.cpu().numpy(), x)
    d = P.gather_grad(g0.with_tensor(P.Tensor4D(np.zeros((0, 16, 16, 3), np.float32))), spec, x.shape)
    assert not d.data.any()
