"""Host-side logic of the product package (no GPU needed): geometry, masks generators,
RNG-order of parameter init, FLOP ledger, coverage diagnostic, C-ABI exports, and the
loud failure of the product path without CUDA."""
import os
import re

import numpy as np
import pytest
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200 import _lib
from golden_cases import cases, load
from oracle import sbnet_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _conv(k, s, same, co=1):
    return P.ConvParams(tuple(k), tuple(s), P.Padding.SAME if same else P.Padding.VALID, co)


def test_compute_block_spec_matches_reference_golden():
    g = load("geometry")
    for r in g["rows"]:
        h, w, kh, kw, sh, sw, same, bh, bw = (int(v) for v in r[:9])
        spec = P.compute_block_spec((1, h, w, 1), _conv((kh, kw), (sh, sw), same), (bh, bw))
        got = [*spec.overlap, *spec.in_stride, *spec.out_block_size, *spec.grid_origin,
               *spec.grid_count, *spec.out_size]
        assert got == [int(v) for v in r[9:]]
    for r in g["bad"]:
        with pytest.raises(P.GeometryError):
            P.compute_block_spec((1, int(r[0]), int(r[1]), 1), _conv((r[2], r[3]), (r[4], r[5]), r[6]),
                                 (int(r[7]), int(r[8])))


def test_conv_params_validation_matches_reference():
    with pytest.raises(P.ShapeMismatchError):
        P.ConvParams((3, 3), (4, 1))
    with pytest.raises(P.ShapeMismatchError):
        P.ConvParams((0, 3))
    assert P.ConvParams((2, 2), (1, 1), P.Padding.SAME).out_size(8, 8) == (9, 9)
    with pytest.raises(P.ShapeMismatchError):
        P.ConvParams((5, 5)).out_size(3, 9)


def test_errors_are_value_errors():
    for cls in (P.ShapeMismatchError, P.GeometryError, P.CoverageError, P.UnsupportedConfigError,
                P.EmptyBlockListError, P.FormatError):
        assert issubclass(cls, ValueError) and issubclass(cls, P.BlockConvError)
    assert issubclass(P.CoverageError, P.GeometryError)


def test_synth_masks_match_reference_golden():
    z = load("masks")
    for i in range(5):
        cfg = z[f"tl{i}_cfg"]
        m = P.synth_mask_topleft(tuple(int(v) for v in cfg[:3]), cfg[3] / 1e6)
        assert np.array_equal(m.numpy(), z[f"tl{i}"])
    for i in range(3):
        cfg = z[f"bl{i}_cfg"]
        m = P.synth_mask_blobs(tuple(int(v) for v in cfg[:3]), cfg[3] / 1e6, int(cfg[4]))
        assert np.array_equal(m.numpy(), z[f"bl{i}"])
    m = P.synth_mask_blobs((1, 400, 400), 0.9, 0).numpy()
    assert int(m.sum()) == int(z["cfg2_mask_sum"][0])
    assert np.array_equal(np.packbits(m.reshape(-1)), z["cfg2_mask_packed"])


def test_random_unit_params_rng_order_matches_reference():
    z = load("units")
    for case in cases(z):
        seed, c, m, pre = (int(v) for v in case["cfg"])
        u = P.random_unit_params(np.random.default_rng(seed), c, m, pre_activation=bool(pre))
        for i, (fb, bn) in enumerate(((u.conv1, u.bn1), (u.conv2, u.bn2), (u.conv3, u.bn3)), 1):
            assert np.array_equal(fb.weights, case[f"conv{i}_w"])
            assert np.array_equal(fb.bias, case[f"conv{i}_b"])
            assert np.array_equal(bn.gamma, case[f"bn{i}_gamma"])
            assert np.array_equal(bn.running_var, case[f"bn{i}_var"])
    st = P.build_stage(P.StageConfig(2, (4, 3, 6), (8, 8), 1, 2), np.random.default_rng(5))
    assert np.array_equal(st.projection.weights, z["stage_proj_w"])
    assert np.array_equal(st.units[1].conv2.weights, z["stage_u1_conv2_w"])


def test_bn_fold_is_reference_expression():
    rng = np.random.default_rng(3)
    bn = P.BnParams((0.5 + rng.random(7)).astype(np.float32), rng.standard_normal(7).astype(np.float32),
                    rng.standard_normal(7).astype(np.float32), (0.5 + rng.random(7)).astype(np.float32))
    # reference ops.py:213-216, evaluated with numpy in float32
    scale = (bn.gamma / np.sqrt(bn.running_var + bn.epsilon)).astype(np.float32)
    shift = (bn.beta - bn.running_mean * bn.gamma / np.sqrt(bn.running_var + bn.epsilon)).astype(np.float32)
    g, b, m, v = bn.gamma, bn.beta, bn.running_mean, bn.running_var
    sc = (g / np.sqrt(v + bn.epsilon)).astype(np.float32)
    assert np.array_equal(sc, scale) and shift.dtype == np.float32


def test_flop_ledger_host():
    conv = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, 8)
    spec = P.compute_block_spec((1, 64, 64, 8), conv, (16, 16))
    idx = P.BlockIndexList(O.reduce_mask(P.synth_mask_topleft((1, 64, 64), 0.75).numpy(),
                                         O.geometry(64, 64, (3, 3), (1, 1), True, (16, 16))))
    rep = P.flops_sparse(spec, idx, conv, (8, 8), 1)
    assert rep.sparse_flops == rep.block_count * 2 * 14 * 14 * 9 * 64
    assert P.theoretical_speedup(0.9) == pytest.approx(10.0)
    with pytest.raises(ValueError):
        P.theoretical_speedup(1.0)
    dims = (1, 32, 32, 8)
    spec = P.compute_block_spec(dims, conv, (8, 8))
    idx = P.BlockIndexList(O.reduce_mask(np.ones((1, 32, 32), np.uint8),
                                         O.geometry(32, 32, (3, 3), (1, 1), True, (8, 8))))
    d, s = P.flops_unit_dense(dims, (8, 4)), P.flops_unit_sparse(spec, idx, (8, 4))
    assert d <= s <= 2 * d


def test_coverage_check_host_diagnostic():
    rng = np.random.default_rng(5)
    for _ in range(40):
        h, w = int(rng.integers(6, 30)), int(rng.integers(6, 30))
        k = int(rng.choice([1, 3, 5]))
        same = bool(rng.random() < 0.5)
        b = k + int(rng.integers(1, 8))
        geo = O.geometry(h, w, (k, k), (1, 1), same, (b, b))
        m = (rng.random((1, h, w)) < 0.2).astype(np.uint8)
        idx = P.BlockIndexList(O.reduce_mask(m, geo))
        spec = P.compute_block_spec((1, h, w, 1), _conv((k, k), (1, 1), same), (b, b))
        rep = P.coverage_check(P.BinaryMask(m), spec, idx)
        assert rep.covered_fraction == 1.0
    spec = P.compute_block_spec((1, 8, 8, 1), _conv((1, 1), (1, 1), False), (4, 4))
    with pytest.raises(P.CoverageError):
        P.coverage_check(P.BinaryMask.full(1, 8, 8), spec, P.BlockIndexList([[0, 0, 0]]))
    with pytest.raises(P.CoverageError):
        P.coverage_check(P.BinaryMask.empty(1, 8, 8), spec, P.BlockIndexList([[0, 0, 0], [0, 0, 0]]))


def test_binary_mask_validation():
    with pytest.raises(P.ShapeMismatchError):
        P.BinaryMask(np.full((1, 2, 2), 2, np.uint8))
    with pytest.raises(P.ShapeMismatchError):
        P.BinaryMask(np.zeros((2, 2), np.uint8))
    assert P.BinaryMask.full(1, 3, 4).dims == (1, 3, 4)


def test_tensor4d_contract():
    a = np.arange(2 * 3 * 4 * 5, dtype=np.float32).reshape(2, 3, 4, 5)
    t = P.Tensor4D(a)
    assert t.dims == (2, 3, 4, 5)
    cf = P.transpose_layout(t)
    assert cf.layout is P.Layout.CHANNELS_FIRST and cf.dims == (2, 3, 4, 5)
    assert np.array_equal(P.transpose_layout(cf).numpy(), a)
    assert t.at(1, 2, 3, 4) == a[1, 2, 3, 4] == cf.at(1, 2, 3, 4)
    with pytest.raises(P.ShapeMismatchError):
        P.Tensor4D(np.zeros((2, 2, 2), np.float32))
    with pytest.raises(P.ShapeMismatchError):
        P.Tensor4D(np.zeros((1, 2, 2, 1), np.int32))
    P.Tensor4D(torch.zeros((1, 2, 2, 1), dtype=torch.bfloat16))


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "sbnet.h")).read()
    return sorted(set(re.findall(r"\b(sbn_[a-z0-9_]+)\s*\(", txt)))


def test_c_abi_library_exports_every_header_symbol():
    import ctypes
    assert os.path.exists(_lib.LIB_PATH), "libsbnet.so not built (run __graft_entry__.build())"
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), f"libsbnet.so does not export {s}"
    assert sorted(_lib.exported_symbols()) == syms  # the ctypes prototypes mirror the header
    lib2 = _lib.load(require_cuda=False)
    assert b"sm_100a" in lib2.sbn_version()


def test_c_abi_argument_validation_without_gpu():
    """Status codes for bad arguments are returned before any device work."""
    import ctypes
    lib = _lib.load(require_cuda=False)
    g = _lib.Geometry()
    assert lib.sbn_reduce_mask(None, ctypes.byref(g), 0, 1.0, None, None, None, 0, None) == _lib.SBN_ERR_SHAPE
    assert lib.sbn_downsample_mask(None, 1, 4, 4, 0, None, None) == _lib.SBN_ERR_INVALID
    assert b"factor" in lib.sbn_last_error()
    spec = P.compute_block_spec((1, 64, 64, 16), _conv((3, 3), (1, 1), True, 16), (16, 16))
    cg = spec.c_geometry(1)
    assert lib.sbn_gather(None, 7, 16, ctypes.byref(cg), None, None, 4, 0, None, None) == _lib.SBN_ERR_UNSUPPORTED
    assert lib.sbn_scatter(None, 0, 16, ctypes.byref(cg), None, None, 4, 1, 1, None, None) == _lib.SBN_ERR_UNSUPPORTED
    assert lib.sbn_sparse_conv(None, 0, 16, 16, 3, 3, 4, 1, ctypes.byref(cg), None, None, None, None,
                               None, 4, None, None, 0, 0, None) == _lib.SBN_ERR_INVALID
    with pytest.raises(P.GeometryError):
        _lib.check(_lib.SBN_ERR_INVALID, "x")
    with pytest.raises(P.UnsupportedConfigError):
        _lib.check(_lib.SBN_ERR_UNSUPPORTED, "x")


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_product_path_fails_loudly_without_cuda():
    x = P.Tensor4D(np.zeros((1, 8, 8, 2), np.float32))
    spec = P.compute_block_spec(x.dims, _conv((3, 3), (1, 1), True, 2), (4, 4))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.reduce_mask(P.BinaryMask.full(1, 8, 8), spec)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.sparse_conv2d(x, P.BinaryMask.full(1, 8, 8),
                        P.FilterBank(np.zeros((3, 3, 2, 2), np.float32)), _conv((3, 3), (1, 1), True, 2), (4, 4))


def test_run_stage_rejects_train_stats_bn():
    st = P.build_stage(P.StageConfig(1, (4, 2, 4), (6, 6)), np.random.default_rng(0))
    x = P.Tensor4D(np.zeros((1, 8, 8, 4), np.float32))
    with pytest.raises(P.UnsupportedConfigError):
        P.run_stage(st, x, P.BinaryMask.full(1, 8, 8), bn_mode=P.BnMode.TRAIN_STATS)
