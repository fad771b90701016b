"""GPU parity: every CUDA path vs the reference's golden vectors and the CPU oracle.

Bit-exact for indices and copies; rel_err <= 1e-5 (conv) / 1e-4 (unit) for fp32 as the
reference's own tests; <= 2e-2 for bf16 against the fp32 oracle on bf16-rounded
inputs (north star).  All calls go through the drop-in Python API -> C-ABI -> CUDA.
"""
import numpy as np
import pytest
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200 import _lib
from golden_cases import cases, conv_cfg, load, unit_dict
from oracle import sbnet_oracle as O

NO_RESIDENT = 2048  # SBN_DEBUG_CONV_NO_RESIDENT (include/sbnet.h)

pytestmark = pytest.mark.gpu


def _conv(k, s, same, co=1):
    return P.ConvParams(tuple(k), tuple(s), P.Padding.SAME if same else P.Padding.VALID, co)


def _spec(h, w, k, s, same, b, c=1):
    return P.compute_block_spec((1, h, w, c), _conv(k, s, same, c), b)


def _np(t):
    t = t.data if isinstance(t, P.Tensor4D) else t
    if t.dtype == torch.bfloat16:
        t = t.float()
    return t.detach().cpu().numpy()


def _unit_params(case):
    def fb(i):
        return P.FilterBank(case[f"conv{i}_w"], case[f"conv{i}_b"])

    def bn(i):
        return P.BnParams(case[f"bn{i}_gamma"], case[f"bn{i}_beta"], case[f"bn{i}_mean"],
                          case[f"bn{i}_var"])
    return P.ResidualUnitParams(fb(1), fb(2), fb(3), bn(1), bn(2), bn(3), bool(case["pre"][0]))


# ----------------------------------------------------------------------------- masks

def test_reduce_mask_golden_bit_exact(cuda_device):
    for case in cases(load("reduce_mask"), "c"):
        h, w, k, s, same, b = conv_cfg(case["cfg"])
        avg, thr = int(case["cfg"][9]), int(case["cfg"][10])
        spec = _spec(h, w, k, s, same, b)
        idx = P.reduce_mask(P.BinaryMask(case["mask"]), spec, P.PoolMode.AVG if avg else P.PoolMode.MAX,
                            None if thr < 0 else thr / 1e6)
        assert idx.entries.tolist() == case["idx"].tolist()


def test_downsample_golden_bit_exact(cuda_device):
    for case in cases(load("reduce_mask"), "d"):
        out = P.downsample_mask(P.BinaryMask(case["mask"]), int(case["f"][0]))
        assert np.array_equal(out.numpy(), case["out"])


@pytest.mark.parametrize("block", [8, 16, 32])
@pytest.mark.parametrize("density", [0.05, 0.3, 1.0])
def test_reduce_mask_config3_sizes_vs_oracle(cuda_device, block, density):
    m = P.synth_mask_topleft((2, 800, 700), 1.0 - density)
    spec = _spec(800, 700, (3, 3), (1, 1), True, (block, block), 128)
    idx = P.reduce_mask(m, spec)
    ref = O.reduce_mask(m.numpy(), O.geometry(800, 700, (3, 3), (1, 1), True, (block, block)))
    assert np.array_equal(idx.entries, ref)


def test_reduce_mask_many_frames_ordered_and_repeatable(cuda_device):
    """N=64 blob masks: many tiles exercise the look-back; the self-resetting workspace
    must give identical results call after call (also under CUDA graph replay)."""
    rng = np.random.default_rng(0)
    m = (rng.random((64, 200, 175)) < 0.01).astype(np.uint8)
    spec = _spec(200, 175, (3, 3), (1, 1), True, (10, 10), 8)
    ref = O.reduce_mask(m, O.geometry(200, 175, (3, 3), (1, 1), True, (10, 10)))
    bm = P.BinaryMask(m).cuda()
    for _ in range(3):
        assert np.array_equal(P.reduce_mask(bm, spec).entries, ref)
    # graph capture of the reduce_mask launch (static buffers)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        idx0 = P.reduce_mask(bm, spec)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            idx = P.reduce_mask(bm, spec)
    for _ in range(3):
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(idx.rows[: len(ref)].cpu().numpy(), ref.astype(np.int32))
        assert int(idx.count_dev.item()) == len(ref)
    assert np.array_equal(idx0.entries, ref)


def test_reduce_mask_avg_thresholds_vs_oracle(cuda_device):
    rng = np.random.default_rng(1)
    m = (rng.random((3, 57, 91)) < 0.4).astype(np.uint8)
    for thr in (None, 0.1, 0.4, 0.5, 1.0):
        for blk, same in (((6, 6), True), ((9, 5), False)):
            spec = _spec(57, 91, (3, 3), (1, 1), same, blk)
            got = P.reduce_mask(P.BinaryMask(m), spec, P.PoolMode.AVG, thr).entries
            ref = O.reduce_mask(m, O.geometry(57, 91, (3, 3), (1, 1), same, blk), "avg", thr)
            assert np.array_equal(got, ref)


# ----------------------------------------------------------------------------- gather/scatter

def test_gather_scatter_golden_bit_exact(cuda_device):
    for case in cases(load("gather_scatter")):
        h, w, k, s, same, b = conv_cfg(case["cfg"])
        x = case["x"]
        n, c = x.shape[0], x.shape[3]
        spec = P.compute_block_spec((n, h, w, c), _conv(k, s, same, 1), b)
        idx = P.BlockIndexList(case["idx"])
        g = P.gather(P.Tensor4D(x), idx, spec)
        assert np.array_equal(_np(g.tensor), case["gather"])
        gt = P.gather_transpose(P.Tensor4D(x), idx, spec)
        assert gt.tensor.layout is P.Layout.CHANNELS_FIRST
        assert np.array_equal(_np(gt.tensor), case["gather_t"])
        assert np.array_equal(P.in_bounds_map(idx, spec).cpu().numpy(), case["inb"])
        blk = g.with_tensor(P.Tensor4D(case["blk"]))
        dst = P.Tensor4D(case["dst"])
        assert np.array_equal(_np(P.scatter(blk, spec, dst)), case["scatter"])
        assert np.array_equal(_np(P.scatter_add(blk, spec, dst)), case["scatter_add"])
        blk_t = g.with_tensor(P.transpose_layout(P.Tensor4D(case["blk"])))
        assert np.array_equal(_np(P.scatter_transpose(blk_t, spec, dst)), case["scatter_t"])
        assert np.array_equal(_np(dst), case["dst"])  # functional: dst untouched


def test_gather_scatter_with_device_index_list(cuda_device):
    """reduce_mask's device list feeds gather/scatter directly (count read on device)."""
    rng = np.random.default_rng(2)
    x = rng.standard_normal((2, 40, 50, 24)).astype(np.float32)
    m = (rng.random((2, 40, 50)) < 0.03).astype(np.uint8)
    spec = P.compute_block_spec(x.shape, _conv((3, 3), (1, 1), True, 24), (10, 10))
    geo = O.geometry(40, 50, (3, 3), (1, 1), True, (10, 10))
    idx = P.reduce_mask(P.BinaryMask(m), spec)
    ref_idx = O.reduce_mask(m, geo)
    g = P.gather(P.Tensor4D(x), idx, spec)
    assert np.array_equal(_np(g.tensor), O.gather(x, ref_idx, geo))
    blk = rng.standard_normal((len(ref_idx), 8, 8, 24)).astype(np.float32)
    out = P.scatter_add(g.with_tensor(P.Tensor4D(blk)), spec, P.Tensor4D(x))
    assert np.array_equal(_np(out), O.scatter(blk, ref_idx, geo, x, add=True))


def test_bf16_gather_scatter_bit_exact(cuda_device):
    rng = np.random.default_rng(3)
    x = torch.from_numpy(rng.standard_normal((1, 64, 48, 64)).astype(np.float32)).bfloat16()
    xf = x.float().numpy()
    m = (rng.random((1, 64, 48)) < 0.05).astype(np.uint8)
    spec = P.compute_block_spec(tuple(x.shape), _conv((3, 3), (1, 1), True, 64), (16, 16))
    geo = O.geometry(64, 48, (3, 3), (1, 1), True, (16, 16))
    idx = P.reduce_mask(P.BinaryMask(m), spec)
    ri = O.reduce_mask(m, geo)
    g = P.gather(P.Tensor4D(x), idx, spec)
    assert np.array_equal(_np(g.tensor), O.gather(xf, ri, geo))
    blk = torch.from_numpy(rng.standard_normal((len(ri), 14, 14, 64)).astype(np.float32)).bfloat16()
    out = P.scatter(g.with_tensor(P.Tensor4D(blk)), spec, P.Tensor4D(x))
    assert np.array_equal(_np(out), O.scatter(blk.float().numpy(), ri, geo, xf))


def test_gather_rejects_out_of_grid_index(cuda_device):
    x = P.Tensor4D(np.ones((1, 8, 8, 1), np.float32))
    spec = _spec(8, 8, (1, 1), (1, 1), False, (4, 4))
    with pytest.raises(P.GeometryError):
        P.gather(x, P.BlockIndexList(np.array([[0, 9, 0]])), spec)
    g = P.gather(x, P.BlockIndexList(np.zeros((0, 3))), spec)
    assert g.count == 0 and g.tensor.dims[0] == 0


# ----------------------------------------------------------------------------- sparse conv

def test_sparse_conv_golden_fp32(cuda_device):
    for case in cases(load("sparse_conv")):
        h, w, k, s, same, b = conv_cfg(case["cfg"])
        co = case["w"].shape[3]
        y = P.sparse_conv2d(P.Tensor4D(case["x"]), P.BinaryMask(case["mask"]),
                            P.FilterBank(case["w"], case["b"]), _conv(k, s, same, co), b)
        ref = case["y"]
        assert y.dims == ref.shape
        region = np.abs(ref).sum(-1) != 0
        assert O.rel_err(_np(y), ref) <= 1e-5
        assert np.all(_np(y)[~region] == 0)


def test_config1_golden(cuda_device):
    z = load("config1")
    p = _conv((3, 3), (1, 1), True, 16)
    spec = P.compute_block_spec((1, 64, 64, 16), p, (16, 16))
    idx = P.reduce_mask(P.BinaryMask(z["mask"]), spec)
    assert idx.entries.tolist() == z["idx"].tolist() and idx.count == 12
    y = P.sparse_conv2d(P.Tensor4D(z["x"]), P.BinaryMask(z["mask"]), P.FilterBank(z["w"], z["b"]), p,
                        (16, 16))
    assert O.rel_err(_np(y), z["y"]) <= 1e-5


def test_sparse_conv_random_sweep_vs_oracle(cuda_device):
    """The reference's own sweep space (verify.py:60-76), dense-equivalence on active regions."""
    rng = np.random.default_rng(21)
    kinds = ["full", "empty", "0.25", "0.5", "0.9"]
    for r in range(40):
        n, c, co = int(rng.integers(1, 3)), int(rng.integers(1, 9)), int(rng.integers(1, 9))
        kh, kw = int(rng.choice([1, 3, 5])), int(rng.choice([1, 3, 5]))
        sh = int(rng.choice([1, 2])) if kh > 1 else 1
        sw = int(rng.choice([1, 2])) if kw > 1 else 1
        h, w = int(rng.integers(max(kh, 6), 49)), int(rng.integers(max(kw, 6), 49))
        same = bool(rng.random() < 0.5)
        b = (kh + sh * int(rng.integers(1, 14)), kw + sw * int(rng.integers(1, 14)))
        kind = kinds[r % len(kinds)]
        m = {"full": np.ones((n, h, w), np.uint8), "empty": np.zeros((n, h, w), np.uint8)}.get(
            kind, (rng.random((n, h, w)) < float(kind if kind[0] == "0" else 0)).astype(np.uint8))
        x = rng.standard_normal((n, h, w, c)).astype(np.float32)
        wt = rng.standard_normal((kh, kw, c, co)).astype(np.float32)
        bias = rng.standard_normal(co).astype(np.float32)
        p = _conv((kh, kw), (sh, sw), same, co)
        y = _np(P.sparse_conv2d(P.Tensor4D(x), P.BinaryMask(m), P.FilterBank(wt, bias), p, b))
        geo = O.geometry(h, w, (kh, kw), (sh, sw), same, b)
        idx = O.reduce_mask(m, geo)
        dense = O.dense_conv2d(x, wt, bias, (sh, sw), same)
        reg = O.active_region(geo, idx, n)
        assert O.rel_err(y[reg], dense[reg]) <= 1e-5
        assert np.all(y[~reg] == 0)


def test_sparse_conv_f64_and_dst(cuda_device):
    rng = np.random.default_rng(4)
    x = rng.standard_normal((1, 30, 30, 3))
    wt = rng.standard_normal((3, 3, 3, 5))
    m = (rng.random((1, 30, 30)) < 0.05).astype(np.uint8)
    dst = rng.standard_normal((1, 30, 30, 5))
    p = _conv((3, 3), (1, 1), True, 5)
    y = _np(P.sparse_conv2d(P.Tensor4D(x), P.BinaryMask(m), P.FilterBank(wt), p, (8, 8), dst=P.Tensor4D(dst)))
    ref = O.sparse_conv2d(x, m, wt, None, (1, 1), True, (8, 8), dst=dst)
    assert O.rel_err(y, ref) <= 1e-12


# ----------------------------------------------------------------------------- residual unit

@pytest.mark.parametrize("inplace", [False, True])
def test_residual_unit_golden_fp32(cuda_device, inplace):
    for case in cases(load("residual")):
        n, h, w, c, m, bs, halo, pre = (int(v) for v in case["cfg"])
        u = _unit_params(case)
        x = P.Tensor4D(torch.from_numpy(case["x"]).cuda())
        x_before = x.data.clone()
        y = P.sparse_residual_unit(x, P.BinaryMask(case["mask"]), u, (bs, bs), halo=halo, inplace=inplace)
        assert O.rel_err(_np(y), case["y"]) <= 1e-4
        if inplace:
            assert y.data.data_ptr() == x.data.data_ptr()
        else:
            assert torch.equal(x.data, x_before)


def test_residual_unit_inactive_pixels_bit_identical(cuda_device):
    rng = np.random.default_rng(5)
    x = rng.standard_normal((2, 37, 45, 6)).astype(np.float32)
    mk = (rng.random((2, 37, 45)) < 0.02).astype(np.uint8)
    u = P.random_unit_params(rng, 6, 4)
    y = _np(P.sparse_residual_unit(P.Tensor4D(x), P.BinaryMask(mk), u, (9, 9)))
    geo = O.unit_geometry(37, 45, (9, 9))
    reg = O.active_region(geo, O.reduce_mask(mk, geo), 2)
    assert np.array_equal(y[~reg], x[~reg])
    y0 = _np(P.sparse_residual_unit(P.Tensor4D(x), P.BinaryMask.empty(2, 37, 45), u, (9, 9)))
    assert np.array_equal(y0, x)


def test_residual_unit_halo_accounting(cuda_device):
    """halo 1/2 reproduce the dense unit on active regions; halo 0 does not
    (reference test_layers.py:153-157)."""
    rng = np.random.default_rng(31)
    worst = {0: 0.0, 1: 0.0, 2: 0.0}
    for r in range(8):
        n, c, m = 1, int(rng.integers(2, 9)), int(rng.integers(2, 9))
        h, w = int(rng.integers(8, 41)), int(rng.integers(8, 41))
        x = rng.standard_normal((n, h, w, c)).astype(np.float32)
        mk = (rng.random((n, h, w)) < 0.3).astype(np.uint8)
        u = P.random_unit_params(rng, c, m)
        ud = {"pre": True}
        for i, (fb, bn) in enumerate(((u.conv1, u.bn1), (u.conv2, u.bn2), (u.conv3, u.bn3)), 1):
            ud[f"w{i}"], ud[f"b{i}"] = fb.weights, fb.bias
            ud[f"bn{i}"] = dict(gamma=bn.gamma, beta=bn.beta, mean=bn.running_mean, var=bn.running_var)
        dense = O.dense_residual_unit(x, ud)
        for halo in (0, 1, 2):
            bs = int(rng.integers(max(4, 2 * halo + 1), 17))
            y = _np(P.sparse_residual_unit(P.Tensor4D(x), P.BinaryMask(mk), u, (bs, bs), halo=halo))
            geo = O.unit_geometry(h, w, (bs, bs), halo)
            reg = O.active_region(geo, O.reduce_mask(mk, geo), n)
            if reg.any():
                worst[halo] = max(worst[halo], O.rel_err(y[reg], dense[reg]))
    assert worst[1] <= 1e-4 and worst[2] <= 1e-4
    assert worst[0] > 1e-3


def _bf16_unit_case(seed, h, w, c, m, density, block):
    rng = np.random.default_rng(seed)
    x = torch.from_numpy(rng.standard_normal((1, h, w, c)).astype(np.float32)).bfloat16()
    u = P.random_unit_params(rng, c, m)
    mk = P.synth_mask_blobs((1, h, w), 1.0 - density, seed)
    return x, u, mk


def _oracle_unit_bf16(x_bf16, u, mk, block):
    """fp32 oracle on bf16-rounded inputs and weights (SURVEY §8(c) bf16 policy)."""
    def r(a):
        return torch.from_numpy(np.asarray(a, np.float32)).bfloat16().float().numpy()
    ud = {"pre": u.pre_activation}
    for i, (fb, bn) in enumerate(((u.conv1, u.bn1), (u.conv2, u.bn2), (u.conv3, u.bn3)), 1):
        ud[f"w{i}"], ud[f"b{i}"] = r(fb.weights), r(fb.bias)
        ud[f"bn{i}"] = dict(gamma=bn.gamma, beta=bn.beta, mean=bn.running_mean, var=bn.running_var)
    return O.sparse_residual_unit(x_bf16.float().numpy(), mk.numpy(), ud, block)


@pytest.mark.parametrize("algo", ["auto", "simt"])
def test_residual_unit_bf16_config2_vs_fp32_oracle(cuda_device, algo):
    x, u, mk = _bf16_unit_case(0, 400, 400, 64, 32, 0.1, (16, 16))
    ref = _oracle_unit_bf16(x, u, mk, (16, 16))
    for inplace in (False, True):
        xt = P.Tensor4D(x.clone().cuda())
        y = _np(P.sparse_residual_unit(xt, mk, u, (16, 16), inplace=inplace, algo=algo))
        err = O.rel_err(y, ref)
        assert err <= 2e-2, (algo, inplace, err)


def test_residual_unit_tc_matches_simt_bf16(cuda_device):
    """When the tcgen05 path is built for this config it must agree with the SIMT path."""
    x, u, mk = _bf16_unit_case(1, 160, 144, 64, 32, 0.3, (16, 16))
    spec = P.unit_spec(tuple(x.shape), (16, 16))
    from paper_1801_02108_b200.layers import residual_unit_algo
    if residual_unit_algo(torch.bfloat16, u, spec) != "tcgen05":
        pytest.skip("tcgen05 unit not available for this config")
    a = _np(P.sparse_residual_unit(P.Tensor4D(x.cuda()), mk, u, (16, 16), algo="tcgen05"))
    b = _np(P.sparse_residual_unit(P.Tensor4D(x.cuda()), mk, u, (16, 16), algo="simt"))
    assert O.rel_err(a, b) <= 1e-2


def test_stage_and_backbone_full_mask_match_dense(cuda_device):
    rng = np.random.default_rng(10)
    cfg = P.StageConfig(unit_count=2, channels=(4, 3, 8), block_size=(8, 8), stride=2)
    stage = P.build_stage(cfg, rng)
    x = P.Tensor4D(rng.standard_normal((1, 24, 24, 4)).astype(np.float32))
    mask = P.BinaryMask.full(1, 12, 12)
    sp = P.run_stage(stage, x, mask, sparse=True)
    de = P.run_stage(stage, x, mask, sparse=False)
    assert O.rel_err(_np(sp.output), _np(de.output)) <= 1e-4
    cfgs = [P.StageConfig(1, (2, 2, 4), (6, 6), 1, 1), P.StageConfig(1, (4, 2, 6), (5, 5), 2, 2),
            P.StageConfig(1, (6, 2, 8), (4, 4), 4, 2)]
    bb = P.build_backbone(cfgs, rng)
    xb = P.Tensor4D(rng.standard_normal((1, 32, 48, 2)).astype(np.float32))
    res = P.run_backbone(bb, xb, P.BinaryMask.full(1, 32, 48))
    assert [r.output.dims[1:3] for r in res] == [(32, 48), (16, 24), (8, 12)]
    assert [r.mask.dims[1:] for r in res] == [(32, 48), (16, 24), (8, 12)]


def test_stage_of_one_unit_equals_single_sparse_unit(cuda_device):
    rng = np.random.default_rng(9)
    stage = P.build_stage(P.StageConfig(1, (4, 3, 4), (8, 8)), rng)
    x = P.Tensor4D(rng.standard_normal((1, 16, 16, 4)).astype(np.float32))
    mask = P.BinaryMask((rng.random((1, 16, 16)) < 0.2).astype(np.uint8))
    res = P.run_stage(stage, x, mask)
    direct = P.sparse_residual_unit(x, mask, stage.units[0], (8, 8))
    assert torch.equal(res.output.data, direct.data)


def test_library_kernels_were_launched(cuda_device):
    assert _lib.launch_count() > 0


@pytest.mark.parametrize("shift,pad", [(0, 0), (1, 0), (5, 0), (34, 0), (0, 16), (3, 16), (17, 48)])
def test_umma_plane_descriptor_selftest(cuda_device, shift, pad):
    """tcgen05 descriptors over the plane layout: row-shifted A views and padded plane
    strides (what the fused kernels use for 3x3 taps and bank-conflict-free staging)."""
    import ctypes
    rows = ((128 + shift + 7) // 8) * 8
    g = torch.Generator().manual_seed(shift * 7 + pad)
    a = torch.randn(rows, 32, generator=g).bfloat16().cuda()
    b = torch.randn(32, 32, generator=g).bfloat16().cuda()
    d = torch.empty(128, 32, device="cuda")
    lib = _lib.load()
    st = lib.sbn_selftest_umma(a.data_ptr(), b.data_ptr(), rows, shift, pad, d.data_ptr(),
                               _lib.stream_handle())
    _lib.check(st, "selftest")
    ref = a[shift:shift + 128].float() @ b.float().t()
    torch.cuda.synchronize()
    assert torch.allclose(d, ref, rtol=1e-3, atol=1e-3), (d - ref).abs().max()


@pytest.mark.parametrize("cin,block", [(128, 16), (128, 8), (64, 16), (32, 16)])
def test_sparse_conv_tc_bf16_vs_fp32_oracle(cuda_device, cin, block):
    """tcgen05 implicit-GEMM sparse conv (bf16 in, fp32 accumulate) vs the fp32 oracle on
    bf16-rounded inputs: 2e-2 relative (north star); inactive pixels exactly zero."""
    from paper_1801_02108_b200.layers import sparse_conv_algo
    rng = np.random.default_rng(cin + block)
    h, w = 120, 104
    x = torch.from_numpy(rng.standard_normal((2, h, w, cin)).astype(np.float32)).bfloat16()
    wt = torch.from_numpy((rng.standard_normal((3, 3, cin, cin)) / np.sqrt(9 * cin)).astype(np.float32)).bfloat16()
    bias = torch.from_numpy(rng.standard_normal(cin).astype(np.float32)).bfloat16()
    m = P.synth_mask_blobs((2, h, w), 0.7, 3)
    p = _conv((3, 3), (1, 1), True, cin)
    spec = P.compute_block_spec((2, h, w, cin), p, (block, block))
    fb = P.FilterBank(wt, bias)
    assert sparse_conv_algo(torch.bfloat16, fb, p, spec) == "tcgen05"
    y = _np(P.sparse_conv2d(P.Tensor4D(x), m, fb, p, (block, block)))
    ref = O.sparse_conv2d(x.float().numpy(), m.numpy(), wt.float().numpy(), bias.float().numpy(),
                          (1, 1), True, (block, block))
    assert O.rel_err(y, ref) <= 2e-2
    geo = O.geometry(h, w, (3, 3), (1, 1), True, (block, block))
    reg = O.active_region(geo, O.reduce_mask(m.numpy(), geo), 2)
    assert np.all(y[~reg] == 0)
    y2 = _np(P.sparse_conv2d(P.Tensor4D(x), m, fb, p, (block, block), algo="simt"))
    assert O.rel_err(y, y2) <= 1e-2


@pytest.mark.parametrize("density,nframes", [(0.1, 1), (0.3, 3), (0.9, 2), (0.2, 36)])
def test_fused_mask_unit_bit_identical_to_two_launch_path(cuda_device, density, nframes):
    """The single-kernel sparse_residual_unit (mask reduction fused, unordered block list)
    must equal the ordered reduce_mask + unit path bit for bit (blocks write disjoint
    windows), in place and functional, call after call (self-resetting barriers)."""
    from paper_1801_02108_b200.layers import residual_unit_into
    rng = np.random.default_rng(11)
    x = torch.from_numpy(rng.standard_normal((nframes, 208, 176, 64)).astype(np.float32)).bfloat16().cuda()
    u = P.random_unit_params(rng, 64, 32)
    mk = P.synth_mask_blobs((nframes, 208, 176), 1.0 - density, 5).cuda()
    spec = P.unit_spec(tuple(x.shape), (16, 16))
    ref = x.clone()
    residual_unit_into(ref, x, u, spec, P.reduce_mask(mk, spec))
    for _ in range(3):
        y = P.sparse_residual_unit(P.Tensor4D(x), mk, u, (16, 16))
        assert torch.equal(y.data, ref)
        xi = x.clone()
        P.sparse_residual_unit(P.Tensor4D(xi), mk, u, (16, 16), inplace=True)
        assert torch.equal(xi, ref)


@pytest.mark.parametrize("density,nframes", [(0.1, 1), (0.5, 2), (1.0, 3)])
def test_unit_cta_pair_variant_bit_identical_to_single_cta(cuda_device, density, nframes):
    """The CTA-pair tcgen05 unit (two CTAs per block, DSMEM halo rows) computes exactly what
    the single-CTA kernel computes: fused and two-launch entry points, in place (resident
    and streamed: 3 full frames exceed the co-resident pairs) and functional."""
    from paper_1801_02108_b200.layers import residual_unit_into
    lib = _lib.load()
    rng = np.random.default_rng(12)
    x = torch.from_numpy(rng.standard_normal((nframes, 240, 224, 64)).astype(np.float32)).bfloat16().cuda()
    u = P.random_unit_params(rng, 64, 32)
    mk = (P.synth_mask_blobs((nframes, 240, 224), 1.0 - density, 9) if density < 1 else
          P.BinaryMask.full(nframes, 240, 224)).cuda()
    spec = P.unit_spec(tuple(x.shape), (16, 16))
    outs = []
    for flags in (1, 0):
        old = lib.sbn_debug_set_flags(flags)
        try:
            a = P.sparse_residual_unit(P.Tensor4D(x), mk, u, (16, 16)).data
            b = x.clone()
            P.sparse_residual_unit(P.Tensor4D(b), mk, u, (16, 16), inplace=True)
            c = x.clone()
            residual_unit_into(c, c, u, spec, P.reduce_mask(mk, spec))
            torch.cuda.synchronize()
        finally:
            lib.sbn_debug_set_flags(old)
        assert torch.equal(a, b) and torch.equal(a, c)
        outs.append(a)
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("cin,block,density", [(128, 16, 1.0), (128, 16, 0.3), (64, 8, 0.5), (32, 16, 0.05)])
def test_sparse_conv_double_buffered_bit_identical(cuda_device, cin, block, density):
    """The double-buffered tcgen05 conv (window/accumulator ping-pong, warp-specialised)
    computes exactly what the single-buffered kernel computes, over many blocks per CTA."""
    lib = _lib.load()
    rng = np.random.default_rng(cin * block)
    h, w = 330, 290
    x = torch.from_numpy(rng.standard_normal((2, h, w, cin)).astype(np.float32)).bfloat16()
    wt = torch.from_numpy((rng.standard_normal((3, 3, cin, cin)) / np.sqrt(9 * cin)).astype(np.float32)).bfloat16()
    fb = P.FilterBank(wt, torch.from_numpy(rng.standard_normal(cin).astype(np.float32)).bfloat16())
    m = P.synth_mask_topleft((2, h, w), 1.0 - density)
    p = _conv((3, 3), (1, 1), True, cin)
    outs = []
    for flags in (2, NO_RESIDENT):  # (the resident-weight pair kernel accumulates in another order)
        old = lib.sbn_debug_set_flags(flags)
        try:
            outs.append(P.sparse_conv2d(P.Tensor4D(x), m, fb, p, (block, block)).data)
            torch.cuda.synchronize()
        finally:
            lib.sbn_debug_set_flags(old)
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("c,m,block", [(64, 32, 16), (96, 48, 16), (64, 32, 8)])
def test_residual_unit_host_frame_inplace_bit_identical(cuda_device, c, m, block):
    """inplace=True on a pinned HOST frame (only the active windows cross PCIe) gives the
    device path's result bit for bit, in the caller's host buffer."""
    x, u, mk = _bf16_unit_case(3, 200, 184, c, m, 0.2, (block, block))
    dev_out = P.sparse_residual_unit(P.Tensor4D(x.cuda()), mk, u, (block, block)).data.cpu()
    hx = x.clone().pin_memory()
    hm = P.BinaryMask(mk.data.cpu().pin_memory(), validate=False)
    r = P.sparse_residual_unit(P.Tensor4D(hx), hm, u, (block, block), inplace=True)
    assert r.data.data_ptr() == hx.data_ptr()
    assert torch.equal(hx, dev_out)
    # asynchronous form: same result after a stream sync
    hx2 = x.clone().pin_memory()
    P.sparse_residual_unit(P.Tensor4D(hx2), hm, u, (block, block), inplace=True, blocking=False)
    torch.cuda.synchronize()
    assert torch.equal(hx2, dev_out)


@pytest.mark.parametrize("block,density,n", [(16, 0.1, 1), (16, 0.4, 2), (8, 0.2, 1), (5, 0.3, 1)])
def test_copy_block_regions_union_equals_windows(cuda_device, block, density, n):
    """Region 2 (union of active windows, each pixel copied once) lands exactly the pixels
    region 0 (every window, overlaps copied twice) lands; region 1 the output windows."""
    import ctypes as C
    lib = _lib.load()
    H, W, c = 61, 47, 16
    x = torch.randn(n, H, W, c, device=cuda_device).bfloat16()
    mk = P.synth_mask_blobs((n, H, W), 1 - density, block).cuda()
    spec = P.unit_spec((n, H, W, c), (block, block))
    idx = P.reduce_mask(mk, spec)
    idx.to_device(cuda_device)
    g = spec.c_geometry(n)
    outs = []
    for region in (0, 2, 1):
        d = torch.zeros_like(x)
        _lib.check(lib.sbn_copy_block_regions(x.data_ptr(), d.data_ptr(), 2, c, C.byref(g), idx.rows.data_ptr(),
                                              idx.count_dev.data_ptr(), idx.capacity, region,
                                              _lib.stream_handle(cuda_device)), "copy")
        outs.append(d)
    torch.cuda.synchronize()
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    # region 1 writes exactly the clipped output windows
    sel = torch.zeros(n, H, W, dtype=torch.bool)
    for (fr, by, bx) in idx.rows[:idx.count].cpu().tolist():
        oy, ox = by * spec.out_block_size[0], bx * spec.out_block_size[1]
        sel[fr, oy:oy + spec.out_block_size[0], ox:ox + spec.out_block_size[1]] = True
    o1 = outs[2].cpu()
    assert torch.equal(o1[sel].view(torch.int16), x.cpu()[sel].view(torch.int16))
    assert not o1[~sel].view(torch.int16).any()


def test_fused_unit_alternating_geometries_share_workspace(cuda_device):
    """The mask-fused unit's workspace (launch epoch + tagged block entries) is shared by
    calls with different geometries; whatever one geometry leaves in it (index lists,
    barrier words, rims) must never be taken for another's block entries."""
    from paper_1801_02108_b200.layers import residual_unit_into
    rng = np.random.default_rng(21)
    u = P.random_unit_params(rng, 64, 32)
    shapes = [(1, 96, 112), (4, 208, 176), (2, 150, 90), (6, 208, 176)]
    data = []
    for (n, h, w) in shapes:
        x = torch.from_numpy(rng.standard_normal((n, h, w, 64)).astype(np.float32)).bfloat16().cuda()
        mk = P.synth_mask_blobs((n, h, w), 0.7, n + h).cuda()
        spec = P.unit_spec(tuple(x.shape), (16, 16))
        ref = x.clone()
        residual_unit_into(ref, x, u, spec, P.reduce_mask(mk, spec))
        data.append((x, mk, ref))
    for _ in range(3):
        for x, mk, ref in data + data[::-1]:
            assert torch.equal(P.sparse_residual_unit(P.Tensor4D(x), mk, u, (16, 16)).data, ref)
            xi = x.clone()
            P.sparse_residual_unit(P.Tensor4D(xi), mk, u, (16, 16), inplace=True)
            assert torch.equal(xi, ref)


@pytest.mark.parametrize("cin,density", [(128, 0.3), (64, 1.0), (32, 0.5)])
def test_sparse_conv_cta_pair_bit_identical(cuda_device, cin, density):
    """The CTA-pair (cta_group::2, M = 256, TMA-fed 5-D window boxes, N-split weights)
    sparse conv computes exactly what the single-CTA double-buffered kernel computes."""
    from paper_1801_02108_b200.layers import sparse_conv_into
    lib = _lib.load()
    rng = np.random.default_rng(cin)
    h, w = 150, 136
    x = torch.from_numpy(rng.standard_normal((2, h, w, cin)).astype(np.float32)).bfloat16().cuda()
    fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, cin, cin)) / np.sqrt(9 * cin)).astype(np.float32)).bfloat16(),
                      torch.from_numpy(rng.standard_normal(cin).astype(np.float32)).bfloat16())
    p = _conv((3, 3), (1, 1), True, cin)
    spec = P.compute_block_spec((2, h, w, cin), p, (16, 16))
    mk = P.synth_mask_blobs((2, h, w), 1.0 - density, 4).cuda()
    idx = P.reduce_mask(mk, spec)
    outs = []
    for flag in (32, NO_RESIDENT):  # streamed-weight pair vs the single-CTA double-buffered kernel
        old = lib.sbn_debug_set_flags(flag)
        try:
            o = torch.zeros_like(x)
            sparse_conv_into(x, o, fb, p, spec, idx)
            torch.cuda.synchronize()
        finally:
            lib.sbn_debug_set_flags(old)
        outs.append(o)
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("block,stride", [(16, 1), (9, 1), (17, 2)])
def test_scatter_write_count_matches_oracle(cuda_device, block, stride):
    """Race-freedom of the scatter (reference tests/oracles.py:49-56 write_count_map,
    SPEC.md:270): scatter_add of all-ones blocks onto zeros counts the writes each output
    pixel receives; it must equal the oracle's count map exactly (0 or 1: disjoint
    interiors, no atomics needed)."""
    n, h, w, c = 2, 83, 71, 8
    p = _conv((3, 3), (stride, stride), True, c)
    spec = P.compute_block_spec((n, h, w, c), p, (block, block))
    mk = P.synth_mask_blobs((n, h, w), 0.5, block).cuda()
    idx = P.reduce_mask(mk, spec)
    obh, obw = spec.out_block_size
    ones = P.GatheredBlocks(P.Tensor4D(torch.ones(idx.count, obh, obw, c, device="cuda")), spec, idx)
    oh, ow = spec.out_size
    got = _np(P.scatter_add(ones, spec, P.Tensor4D(torch.zeros(n, oh, ow, c, device="cuda"))))
    want = np.zeros((n, oh, ow), np.int64)
    for i, by, bx in idx.entries:
        want[i, by * obh:min((by + 1) * obh, oh), bx * obw:min((bx + 1) * obw, ow)] += 1
    assert want.max() <= 1
    assert np.array_equal(got, np.repeat(want[..., None], c, axis=-1).astype(np.float32))


def test_fused_unit_empty_and_alternating_masks(cuda_device):
    """The mask-fused tcgen05 unit with an empty mask leaves x bit-identical (in place and
    functional), and launches with no work interleaved with real ones keep the slot /
    epoch protocol consistent (reference layers.py:221-222: empty list returns x)."""
    from paper_1801_02108_b200.layers import residual_unit_into
    rng = np.random.default_rng(31)
    x = torch.from_numpy(rng.standard_normal((1, 160, 144, 64)).astype(np.float32)).bfloat16().cuda()
    u = P.random_unit_params(rng, 64, 32)
    empty = P.BinaryMask(torch.zeros(1, 160, 144, dtype=torch.uint8)).cuda()
    blobs = P.synth_mask_blobs((1, 160, 144), 0.85, 7).cuda()
    spec = P.unit_spec(tuple(x.shape), (16, 16))
    ref = x.clone()
    residual_unit_into(ref, x, u, spec, P.reduce_mask(blobs, spec))
    for _ in range(3):
        y = P.sparse_residual_unit(P.Tensor4D(x), empty, u, (16, 16)).data
        assert torch.equal(y, x)
        xi = x.clone()
        P.sparse_residual_unit(P.Tensor4D(xi), empty, u, (16, 16), inplace=True)
        assert torch.equal(xi, x)
        xi = x.clone()
        P.sparse_residual_unit(P.Tensor4D(xi), blobs, u, (16, 16), inplace=True)
        assert torch.equal(xi, ref)


@pytest.mark.parametrize("cin,block,density,nframes", [(128, 16, 0.1, 1), (64, 8, 0.4, 2), (32, 16, 1.0, 1),
                                                       (128, 16, 0.0, 1), (64, 24, 0.3, 1)])
def test_sparse_conv_mask_fused_bit_identical(cuda_device, cin, block, density, nframes):
    """sparse_conv2d from the mask (one kernel on the tcgen05 double-buffered path: mask
    reduction fused, unordered block list) equals reduce_mask + the conv bit for bit, call
    after call and across geometries sharing the workspaces; empty masks leave zeros."""
    from paper_1801_02108_b200.layers import sparse_conv_into, sparse_conv_masked_into
    rng = np.random.default_rng(cin + block)
    h, w = 131, 117
    x = torch.from_numpy(rng.standard_normal((nframes, h, w, cin)).astype(np.float32)).bfloat16().cuda()
    fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, cin, cin)) / np.sqrt(9 * cin)).astype(np.float32)).bfloat16(),
                      torch.from_numpy(rng.standard_normal(cin).astype(np.float32)).bfloat16())
    p = _conv((3, 3), (1, 1), True, cin)
    spec = P.compute_block_spec((nframes, h, w, cin), p, (block, block))
    mk = (P.synth_mask_blobs((nframes, h, w), 1.0 - density, 5) if density > 0 else
          P.BinaryMask(torch.zeros(nframes, h, w, dtype=torch.uint8))).cuda()
    ref = torch.zeros(nframes, *spec.out_size, cin, dtype=torch.bfloat16, device="cuda")
    sparse_conv_into(x, ref, fb, p, spec, P.reduce_mask(mk, spec))
    for _ in range(3):
        out = torch.zeros_like(ref)
        sparse_conv_masked_into(x, out, mk.data, fb, p, spec)
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
    y = P.sparse_conv2d(P.Tensor4D(x), mk, fb, p, (block, block)).data
    assert torch.equal(y, ref)


@pytest.mark.parametrize("cin,block", [(128, 16), (64, 8), (32, 16)])
def test_sparse_conv_tc_mask_monotonicity(cuda_device, cin, block):
    """Reference test_layers.py:58-70 on the tcgen05 path (bf16): growing the mask never
    changes the output on the smaller mask's active write regions (per-block compute is
    independent of which other blocks are active)."""
    rng = np.random.default_rng(2 + cin)
    n, h, w = 1, 96, 88
    x = P.Tensor4D(torch.from_numpy(rng.standard_normal((n, h, w, cin)).astype(np.float32)).bfloat16().cuda())
    fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, cin, cin)) / np.sqrt(9 * cin)).astype(np.float32)).bfloat16(),
                      torch.from_numpy(rng.standard_normal(cin).astype(np.float32)).bfloat16())
    p = _conv((3, 3), (1, 1), True, cin)
    small = P.BinaryMask((rng.random((n, h, w)) < 0.004).astype(np.uint8))
    grown = P.BinaryMask(np.maximum(small.numpy(), (rng.random((n, h, w)) < 0.004).astype(np.uint8)))
    spec = P.compute_block_spec(x.dims, p, (block, block))
    geo = O.geometry(h, w, (3, 3), (1, 1), True, (block, block))
    region = O.active_region(geo, O.reduce_mask(small.numpy(), geo), n)
    a = _np(P.sparse_conv2d(x, small, fb, p, (block, block)))
    b = _np(P.sparse_conv2d(x, grown, fb, p, (block, block)))
    assert region.any() and np.array_equal(a[region], b[region])


@pytest.mark.parametrize("c,m", [(64, 32), (128, 64)])
def test_tc_residual_unit_zero_weights_is_identity(cuda_device, c, m):
    """Reference test_layers.py:120-133 on the tcgen05 unit (bf16, fused mask, in place and
    functional): zero convolutions with identity BN leave x bit-identical."""
    def fb(kh, kw, ci, co):
        return P.FilterBank(torch.zeros(kh, kw, ci, co, dtype=torch.bfloat16), torch.zeros(co, dtype=torch.bfloat16))
    u = P.ResidualUnitParams(fb(1, 1, c, m), fb(3, 3, m, m), fb(1, 1, m, c),
                             P.BnParams.identity(c), P.BnParams.identity(m), P.BnParams.identity(m))
    rng = np.random.default_rng(5)
    x = torch.from_numpy(rng.standard_normal((1, 64, 80, c)).astype(np.float32)).bfloat16().cuda()
    mask = P.BinaryMask.full(1, 64, 80)
    out = P.sparse_residual_unit(P.Tensor4D(x), mask, u, (16, 16)).data
    assert torch.equal(out, x)
    xi = x.clone()
    P.sparse_residual_unit(P.Tensor4D(xi), mask, u, (16, 16), inplace=True)
    assert torch.equal(xi, x)


@pytest.mark.parametrize("dtype,c,block,w", [(torch.bfloat16, 64, 16, 61), (torch.float32, 16, 8, 61), (torch.bfloat16, 128, 8, 61),
                                             (torch.bfloat16, 64, 16, 62), (torch.bfloat16, 32, 8, 64)])
def test_channels_first_sparse_conv_matches_channels_last(cuda_device, dtype, c, block, w):
    """CHANNELS_FIRST sparse_conv2d (active windows transposed into an NHWC staging frame,
    outputs transposed back) equals the CHANNELS_LAST result bit for bit, and keeps dst
    outside the active write regions."""
    rng = np.random.default_rng(c + block + w)
    n, h = 2, 75  # odd widths take the 2-byte NCHW path, even widths the aligned 4-byte pairs
    x = torch.from_numpy(rng.standard_normal((n, h, w, c)).astype(np.float32)).to(dtype).cuda()
    fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, c, c)) / np.sqrt(9 * c)).astype(np.float32)).to(dtype),
                      torch.from_numpy(rng.standard_normal(c).astype(np.float32)).to(dtype))
    p = _conv((3, 3), (1, 1), True, c)
    mk = P.synth_mask_blobs((n, h, w), 0.8, 3).cuda()
    ref = P.sparse_conv2d(P.Tensor4D(x), mk, fb, p, (block, block)).data
    xcf = P.Tensor4D(x.permute(0, 3, 1, 2).contiguous(), P.Layout.CHANNELS_FIRST)
    ycf = P.sparse_conv2d(xcf, mk, fb, p, (block, block))
    assert ycf.layout is P.Layout.CHANNELS_FIRST
    assert torch.equal(ycf.data.permute(0, 2, 3, 1), ref)
    dst = P.Tensor4D(torch.full((n, c, h, w), 7.0, dtype=dtype, device="cuda"), P.Layout.CHANNELS_FIRST)
    yd = P.sparse_conv2d(xcf, mk, fb, p, (block, block), dst=dst).data.permute(0, 2, 3, 1)
    spec = P.compute_block_spec((n, h, w, c), p, (block, block))
    geo = O.geometry(h, w, (3, 3), (1, 1), True, (block, block))
    reg = torch.from_numpy(O.active_region(geo, O.reduce_mask(mk.numpy(), geo), n)).cuda()
    assert torch.equal(yd[reg], ref[reg]) and bool((yd[~reg] == 7.0).all())


@pytest.mark.parametrize("c,m,inplace,w", [(64, 32, False, 80), (64, 32, True, 80), (128, 64, True, 80), (64, 32, True, 79)])
def test_channels_first_residual_unit_matches_channels_last(cuda_device, c, m, inplace, w):
    """CHANNELS_FIRST sparse_residual_unit (windows through an NHWC staging frame) equals
    the CHANNELS_LAST result bit for bit; inplace updates x's own storage."""
    rng = np.random.default_rng(c)
    x = torch.from_numpy(rng.standard_normal((1, 96, w, c)).astype(np.float32)).bfloat16().cuda()
    u = P.random_unit_params(rng, c, m)
    mk = P.synth_mask_blobs((1, 96, w), 0.8, 4).cuda()
    ref = P.sparse_residual_unit(P.Tensor4D(x), mk, u, (16, 16)).data
    xcf = P.Tensor4D(x.permute(0, 3, 1, 2).contiguous(), P.Layout.CHANNELS_FIRST)
    keep = xcf.data.clone()
    y = P.sparse_residual_unit(xcf, mk, u, (16, 16), inplace=inplace)
    assert y.layout is P.Layout.CHANNELS_FIRST
    assert torch.equal(y.data.permute(0, 2, 3, 1), ref)
    if inplace:
        assert y is xcf and torch.equal(xcf.data.permute(0, 2, 3, 1), ref)
    else:
        assert torch.equal(xcf.data, keep)


def test_backbone_hierarchical_stage_masks_equal_direct_downsample(cuda_device):
    """run_backbone derives each stage's mask from the previous stage's (max-pool composes
    exactly with ceil dims); every stage mask equals downsample_mask(base, scale)."""
    from paper_1801_02108_b200 import perf
    rng = np.random.default_rng(8)
    cfgs = perf.detector_stage_configs()
    bb = P.build_backbone(cfgs, rng)
    n, h, w = 1, 203, 171  # odd sizes: ceil dims at every level
    x = P.Tensor4D(torch.from_numpy(rng.standard_normal((n, h, w, cfgs[0].channels[0])).astype(np.float32)).bfloat16().cuda())
    base = P.BinaryMask((rng.random((n, h, w)) < 0.05).astype(np.uint8)).cuda()
    res = P.run_backbone(bb, x, base)
    for r, c in zip(res, cfgs):
        assert torch.equal(r.mask.data, P.downsample_mask(base, c.mask_scale).data)


@pytest.mark.parametrize("block,density,flags", [(16, 0.1, 0), (16, 0.3, 0), (16, 0.3, 2048), (8, 0.1, 0),
                                                  (32, 0.1, 0)])
def test_sparse_conv_config3_size_vs_fp32_oracle(cuda_device, block, density, flags):
    """BASELINE config 3 at full size (1 x 800 x 700 x 128 bf16, 3x3 SAME, top-left mask) through
    the public sparse_conv2d — the kernels the bench times: the resident-weight CTA pair with
    the one-launch global list (16x16), the single-CTA double-buffered kernel with its
    half-block tail jobs (16x16 at 30 % with the pair disabled: 896 blocks on 148 CTAs),
    mask-fused lists (8x8) and the TMA tap-GEMM (32x32) — against the fp32 oracle on
    bf16-rounded inputs (2e-2, north star); inactive pixels exactly zero."""
    lib = _lib.load()
    old = lib.sbn_debug_set_flags(flags)
    try:
        _config3_case(block, density)
    finally:
        lib.sbn_debug_set_flags(old)


def _config3_case(block, density):
    rng = np.random.default_rng(block * 100 + int(density * 10))
    h, w, c = 800, 700, 128
    x = torch.from_numpy(rng.standard_normal((1, h, w, c), dtype=np.float32)).bfloat16()
    wt = torch.from_numpy((rng.standard_normal((3, 3, c, c)) / np.sqrt(9 * c)).astype(np.float32)).bfloat16()
    bias = torch.from_numpy(rng.standard_normal(c).astype(np.float32)).bfloat16()
    m = P.synth_mask_topleft((1, h, w), 1.0 - density)
    p = _conv((3, 3), (1, 1), True, c)
    y = _np(P.sparse_conv2d(P.Tensor4D(x.cuda()), m.cuda(), P.FilterBank(wt, bias), p, (block, block)))
    ref = O.sparse_conv2d(x.float().numpy(), m.numpy(), wt.float().numpy(), bias.float().numpy(),
                          (1, 1), True, (block, block))
    err = O.rel_err(y, ref)
    print(f"config 3 block {block} density {density}: rel_err {err:.2e}")
    assert err <= 2e-2
    geo = O.geometry(h, w, (3, 3), (1, 1), True, (block, block))
    reg = O.active_region(geo, O.reduce_mask(m.numpy(), geo), 1)
    assert np.all(y[~reg] == 0)


def test_bf16_scatter_add_vs_oracle(cuda_device):
    """bf16 scatter in add mode: one bf16 add per element (x + block, rounded once), i.e. the
    fp32 oracle's sum rounded to bf16; pixels outside the active windows keep dst."""
    rng = np.random.default_rng(11)
    x = torch.from_numpy(rng.standard_normal((2, 70, 58, 64)).astype(np.float32)).bfloat16()
    m = (rng.random((2, 70, 58)) < 0.03).astype(np.uint8)
    spec = P.compute_block_spec(tuple(x.shape), _conv((3, 3), (1, 1), True, 64), (16, 16))
    geo = O.geometry(70, 58, (3, 3), (1, 1), True, (16, 16))
    idx = P.reduce_mask(P.BinaryMask(m), spec)
    ri = O.reduce_mask(m, geo)
    assert len(ri) > 0
    g = P.gather(P.Tensor4D(x), idx, spec)
    blk = torch.from_numpy(rng.standard_normal((len(ri), 14, 14, 64)).astype(np.float32)).bfloat16()
    out = P.scatter_add(g.with_tensor(P.Tensor4D(blk)), spec, P.Tensor4D(x))
    ref = O.scatter(blk.float().numpy(), ri, geo, x.float().numpy(), add=True)
    ref_bf16 = torch.from_numpy(ref).bfloat16().float().numpy()
    assert np.array_equal(_np(out), ref_bf16)


@pytest.mark.parametrize("n,density", [(3, 0.05), (2, 0.5), (1, 1.0), (2, 0.0)])
def test_sparse_conv_resident_pair_modes(cuda_device, n, density):
    """Resident-weight CTA-pair conv (16x16 blocks, 128 -> 128): list mode (reduce_mask list,
    the default from the mask) and the one-launch mask-fused global list give the same output
    bit for bit, call after call and
    interleaved with the single-CTA kernel on the same sync workspace; against the
    double-buffered kernel (another fp32 accumulation order, bf16 outputs) within 2^-7 of the
    largest output; against
    the fp32 oracle within 2e-2; untouched pixels stay zero."""
    from paper_1801_02108_b200.layers import sparse_conv_into, sparse_conv_masked_into
    lib = _lib.load()
    rng = np.random.default_rng(40 + n)
    h, w, c = 190, 230, 128
    x = torch.from_numpy(rng.standard_normal((n, h, w, c)).astype(np.float32)).bfloat16()
    wt = torch.from_numpy((rng.standard_normal((3, 3, c, c)) / np.sqrt(9 * c)).astype(np.float32)).bfloat16()
    bias = torch.from_numpy(rng.standard_normal(c).astype(np.float32)).bfloat16()
    fb = P.FilterBank(wt, bias)
    p = _conv((3, 3), (1, 1), True, c)
    spec = P.compute_block_spec((n, h, w, c), p, (16, 16))
    m = (P.synth_mask_blobs((n, h, w), 1.0 - density, 6) if density < 1 else P.BinaryMask.full(n, h, w))
    mk = m.cuda()
    xd = x.cuda()
    idx = P.reduce_mask(mk, spec)
    res = []
    for _ in range(2):
        # 0: reduce_mask + the pair's list mode; 16384: one launch (mask test + global list in
        # the pair kernel); NO_RESIDENT: the single-CTA double-buffered kernel
        for flags in (0, 16384, NO_RESIDENT):
            old = lib.sbn_debug_set_flags(flags)
            try:
                a = torch.zeros_like(xd)
                sparse_conv_into(xd, a, fb, p, spec, idx)
                b = torch.zeros_like(xd)
                sparse_conv_masked_into(xd, b, mk.data, fb, p, spec)
                torch.cuda.synchronize()
            finally:
                lib.sbn_debug_set_flags(old)
            assert torch.equal(a, b)
            res.append(a)
    assert torch.equal(res[0], res[1]) and torch.equal(res[0], res[3]) and torch.equal(res[2], res[5])
    y, y_db = _np(res[0]), _np(res[2])
    if idx.count == 0:
        assert not y.any()
        return
    assert O.rel_err(y, y_db) <= 2 ** -7  # bf16 outputs: the order may flip a last bit (2^-8 of a value)
    ref = O.sparse_conv2d(x.float().numpy(), m.numpy(), wt.float().numpy(), bias.float().numpy(),
                          (1, 1), True, (16, 16))
    assert O.rel_err(y, ref) <= 2e-2
    geo = O.geometry(h, w, (3, 3), (1, 1), True, (16, 16))
    reg = O.active_region(geo, O.reduce_mask(m.numpy(), geo), n)
    assert np.all(y[~reg] == 0)


@pytest.mark.parametrize("pool,thr", [("max", None), ("avg", 0.3)])
def test_reduce_mask_ranges_kernel_vs_oracle(cuda_device, pool, thr):
    """Large batches (64 frames of 400x400, 16x16 unit windows: 1856 block rows) run the
    ranges kernel (several block rows per CTA, whole-CTA look-back); MAX and AVG pooling,
    vectorised column sums: bit-exact against the oracle and against the one-row-per-CTA
    kernel (SBN_DEBUG_ROW_REDUCE_MASK), call after call."""
    lib = _lib.load()
    m = P.synth_mask_blobs((64, 400, 400), 0.8, 3)
    spec = P.unit_spec((64, 400, 400, 8), (16, 16))
    pm = P.PoolMode.MAX if pool == "max" else P.PoolMode.AVG
    mk = m.cuda()
    got = [P.reduce_mask(mk, spec, pm, thr).entries for _ in range(3)]
    old = lib.sbn_debug_set_flags(8192)
    try:
        row = P.reduce_mask(mk, spec, pm, thr).entries
    finally:
        lib.sbn_debug_set_flags(old)
    geo = O.geometry(400, 400, (3, 3), (1, 1), True, (16, 16))
    ref = O.reduce_mask(m.numpy(), geo, pool, thr)
    assert len(ref) > 0
    for g in got:
        assert np.array_equal(g, ref)
    assert np.array_equal(row, ref)


@pytest.mark.parametrize("h,w,c,block,density", [(400, 704, 24, 32, 0.1), (200, 352, 48, 8, 0.2), (130, 150, 64, 17, 0.5)])
def test_tap_gemm_global_list_mode_bit_identical(cuda_device, h, w, c, block, density):
    """The tap-GEMM conv's one-launch global-list mode (every CTA tests its candidates,
    publishes them, then all stride the list; SBN_DEBUG 65536) computes exactly what
    reduce_mask + the list-mode launch computes (per-tile math identical), call after call."""
    from paper_1801_02108_b200.layers import sparse_conv_algo, sparse_conv_into, sparse_conv_masked_into
    lib = _lib.load()
    rng = np.random.default_rng(h + c)
    x = torch.from_numpy(rng.standard_normal((1, h, w, c)).astype(np.float32)).bfloat16().cuda()
    fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, c, c)) / np.sqrt(9 * c)).astype(np.float32)).bfloat16(),
                      torch.from_numpy(rng.standard_normal(c).astype(np.float32)).bfloat16())
    p = _conv((3, 3), (1, 1), True, c)
    spec = P.compute_block_spec((1, h, w, c), p, (block, block))
    mk = P.synth_mask_topleft((1, h, w), 1.0 - density).cuda()
    idx = P.reduce_mask(mk, spec)
    ref = torch.zeros_like(x)
    sparse_conv_into(x, ref, fb, p, spec, idx)
    old = lib.sbn_debug_set_flags(65536)
    try:
        for _ in range(3):
            o = torch.zeros_like(x)
            sparse_conv_masked_into(x, o, mk.data, fb, p, spec)
            torch.cuda.synchronize()
            assert torch.equal(o, ref)
    finally:
        lib.sbn_debug_set_flags(old)
