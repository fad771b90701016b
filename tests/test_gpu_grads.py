"""GPU parity of the training path against golden vectors from the
reference (`oracle/make_golden.py` gen_grads) and the CPU oracle.

gather_grad / scatter_grad: bit-exact (f32/f64) — the pixel-centric sbn_gather_grad
accumulates in the reference's index order.  Conv / unit gradients: rel_err <= 1e-5
(f32) / 1e-10 (f64), the reference's own finite-difference bar is 1e-5
(`tests/test_grads.py:35-36`).
"""
import numpy as np
import pytest
import torch

import paper_1801_02108_b200 as P
from golden_cases import cases, conv_cfg, load
from oracle import sbnet_oracle as O

pytestmark = pytest.mark.gpu


def _conv(k, s, same, co=1):
    return P.ConvParams(tuple(k), tuple(s), P.Padding.SAME if same else P.Padding.VALID, co)


def _np(t):
    t = t.data if isinstance(t, P.Tensor4D) else t
    return t.detach().cpu().numpy()


def _tol(dt):
    return 1e-10 if dt == np.float64 else 1e-5


def test_gather_grad_and_scatter_grad_golden_bit_exact(cuda_device):
    for cs in cases(load("grads"), "g"):
        h, w, k, s, same, b = conv_cfg(cs["cfg"])
        n, c = int(cs["cfg"][9]), int(cs["cfg"][10])
        spec = P.compute_block_spec((n, h, w, c), _conv(k, s, same, c), b)
        idx = P.BlockIndexList(cs["idx"])
        gb = P.GatheredBlocks(P.Tensor4D(cs["gblk"]), spec, idx)
        dx = P.gather_grad(gb, spec, (n, h, w, c))
        assert np.array_equal(_np(dx), cs["gather_grad"])
        sg = P.scatter_grad(P.Tensor4D(cs["gout"]), idx, spec)
        assert np.array_equal(_np(sg.tensor), cs["scatter_grad"])


def test_gather_grad_with_device_index_list_and_bf16(cuda_device):
    rng = np.random.default_rng(8)
    x = np.zeros((2, 37, 29, 16), np.float32)
    m = (rng.random((2, 37, 29)) < 0.05).astype(np.uint8)
    spec = P.compute_block_spec(x.shape, _conv((3, 3), (1, 1), True, 16), (8, 8))
    geo = O.geometry(37, 29, (3, 3), (1, 1), True, (8, 8))
    idx = P.reduce_mask(P.BinaryMask(m), spec)
    ref_idx = O.reduce_mask(m, geo)
    gblk = rng.standard_normal((len(ref_idx), 8, 8, 16)).astype(np.float32)
    dx = P.gather_grad(P.GatheredBlocks(P.Tensor4D(gblk), spec, idx), spec, x.shape)
    assert np.array_equal(_np(dx), O.gather_grad(gblk, ref_idx, geo, x.shape))
    gb16 = torch.from_numpy(gblk).bfloat16()
    d16 = P.gather_grad(P.GatheredBlocks(P.Tensor4D(gb16), spec, idx), spec, x.shape)
    ref16 = O.gather_grad(gb16.float().numpy(), ref_idx, geo, x.shape)  # fp32 sums of bf16 values
    assert np.array_equal(d16.data.float().cpu().numpy(), torch.from_numpy(ref16).bfloat16().float().numpy())


def test_adjoint_identities_exact(cuda_device):
    """<gather(x), g> == <x, gather_grad(g)> and <scatter(b), y> == <b, scatter_grad(y)>
    exactly on integer-valued float64 data (reference `verify.py:150-177`)."""
    rng = np.random.default_rng(4)
    for r in range(20):
        n, h, w, c = int(rng.integers(1, 3)), int(rng.integers(6, 25)), int(rng.integers(6, 25)), int(rng.integers(1, 5))
        k = int(rng.choice([1, 3, 5]))
        s = int(rng.choice([1, 2])) if k > 1 else 1
        same = bool(r % 2)
        b = k + s * int(rng.integers(1, 6))
        spec = P.compute_block_spec((n, h, w, c), _conv((k, k), (s, s), same, c), (b, b))
        m = (rng.random((n, h, w)) < 0.4).astype(np.uint8)
        idx = P.reduce_mask(P.BinaryMask(m), spec)
        B = idx.count
        x = rng.integers(-8, 9, (n, h, w, c)).astype(np.float64)
        g = rng.integers(-8, 9, (B, b, b, c)).astype(np.float64)
        gat = P.gather(P.Tensor4D(x), idx, spec)
        back = P.gather_grad(gat.with_tensor(P.Tensor4D(g)), spec, x.shape)
        assert float(np.vdot(_np(gat.tensor), g)) == float(np.vdot(x, _np(back)))
        obh, obw = spec.out_block_size
        blk = rng.integers(-8, 9, (B, obh, obw, c)).astype(np.float64)
        gy = rng.integers(-8, 9, (n, *spec.out_size, c)).astype(np.float64)
        sc = P.scatter(gat.with_tensor(P.Tensor4D(blk)), spec, P.Tensor4D(np.zeros((n, *spec.out_size, c))))
        assert float(np.vdot(_np(sc), gy)) == float(np.vdot(blk, _np(P.scatter_grad(P.Tensor4D(gy), idx, spec).tensor)))


def test_sparse_conv2d_grads_golden(cuda_device):
    for cs in cases(load("grads"), "v"):
        h, w, k, s, same, b = conv_cfg(cs["cfg"])
        co = int(cs["cfg"][11])
        p = _conv(k, s, same, co)
        dx, dw, db = P.sparse_conv2d_grads(P.Tensor4D(cs["x"]), P.BinaryMask(cs["mask"]),
                                           P.FilterBank(cs["w"], cs["b"]), p, b, P.Tensor4D(cs["gout"]))
        tol = _tol(cs["x"].dtype)
        assert O.rel_err(_np(dx), cs["dx"]) <= tol
        assert O.rel_err(_np(dw), cs["dw"]) <= tol
        assert O.rel_err(_np(db), cs["db"]) <= tol


def _unit(cs):
    def fb(i):
        return P.FilterBank(cs[f"conv{i}_w"], cs[f"conv{i}_b"])

    def bn(i):
        return P.BnParams(cs[f"bn{i}_gamma"], cs[f"bn{i}_beta"], cs[f"bn{i}_mean"], cs[f"bn{i}_var"])
    return P.ResidualUnitParams(fb(1), fb(2), fb(3), bn(1), bn(2), bn(3), True)


def test_sparse_residual_unit_grads_golden(cuda_device):
    for cs in cases(load("grads"), "u"):
        n, h, w, c, m, bs, halo, _ = (int(v) for v in cs["cfg"])
        dx, dws = P.sparse_residual_unit_grads(P.Tensor4D(cs["x"]), P.BinaryMask(cs["mask"]), _unit(cs),
                                               (bs, bs), P.Tensor4D(cs["gout"]), halo)
        tol = _tol(cs["x"].dtype)
        assert O.rel_err(_np(dx), cs["dx"]) <= tol, (n, h, w, c, m, bs, halo)
        for nm in ("conv1", "conv2", "conv3"):
            assert O.rel_err(_np(dws[nm][0]), cs[f"d{nm}_w"]) <= tol, nm
            assert O.rel_err(_np(dws[nm][1]), cs[f"d{nm}_b"]) <= tol, nm


def test_sparse_batch_norm_train_stats_golden(cuda_device):
    for cs in cases(load("grads"), "b"):
        st = cs["stack"]
        spec = P.compute_block_spec((1, 12, 12, st.shape[3]), _conv((3, 3), (1, 1), True, st.shape[3]), (6, 6))
        gb = P.GatheredBlocks(P.Tensor4D(st), spec, P.BlockIndexList(np.zeros((st.shape[0], 3), np.int64)))
        bn = P.BnParams(cs["gamma"], cs["beta"], np.zeros_like(cs["gamma"]), np.ones_like(cs["gamma"]))
        y, (mean, var) = P.sparse_batch_norm(gb, bn, P.BnMode.TRAIN_STATS)
        assert O.rel_err(_np(y.tensor), cs["y"]) <= 1e-10
        assert O.rel_err(mean.cpu().numpy(), cs["mean"]) <= 1e-10
        assert O.rel_err(var.cpu().numpy(), cs["var"]) <= 1e-10


def test_zero_mask_gives_zero_gradients(cuda_device):
    """reference tests/test_grads.py:24-32"""
    rng = np.random.default_rng(1)
    x = P.Tensor4D(rng.standard_normal((1, 12, 12, 2)))
    f = P.FilterBank(rng.standard_normal((3, 3, 2, 2)), rng.standard_normal(2))
    p = _conv((3, 3), (1, 1), True, 2)
    g_out = P.Tensor4D(rng.standard_normal((1, 12, 12, 2)))
    dx, dw, db = P.sparse_conv2d_grads(x, P.BinaryMask.empty(1, 12, 12), f, p, (6, 6), g_out)
    assert not _np(dx).any() and not _np(dw).any() and not _np(db).any()


@pytest.mark.parametrize("dt,tol", [(torch.float64, 1e-12), (torch.float32, 1e-5)])
def test_native_conv_grads_vs_autograd_and_deterministic(cuda_device, dt, tol):
    """csrc/conv_grad.cu against torch autograd of F.conv2d (same math), at sizes that
    split the weight-gradient reduction into several segments; repeated calls bit-identical."""
    import torch.nn.functional as F

    from paper_1801_02108_b200.ops import conv_grads_nhwc
    g_ = torch.Generator(device="cuda").manual_seed(0)
    for (n, h, w, c, co, k, s, p) in ((4, 40, 36, 16, 12, 3, 1, 1), (2, 33, 29, 8, 20, 5, 2, 2), (3, 17, 19, 6, 7, 1, 1, 0)):
        x = torch.randn(n, h, w, c, device="cuda", dtype=dt, generator=g_)
        wt = torch.randn(k, k, c, co, device="cuda", dtype=dt, generator=g_)
        oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
        go = torch.randn(n, oh, ow, co, device="cuda", dtype=dt, generator=g_)
        dx, dw, db = conv_grads_nhwc(x, wt, (s, s), (p, p), go)
        xr = x.permute(0, 3, 1, 2).clone().requires_grad_()
        wr = wt.permute(3, 2, 0, 1).clone().requires_grad_()
        br = torch.zeros(co, device="cuda", dtype=dt, requires_grad=True)
        torch.backends.cudnn.allow_tf32 = False
        y = F.conv2d(xr, wr, br, stride=s, padding=p)
        y.backward(go.permute(0, 3, 1, 2))
        rel = lambda a, b: float((a - b).abs().max() / b.abs().max())  # noqa: E731
        assert rel(dx, xr.grad.permute(0, 2, 3, 1)) <= tol
        assert rel(dw, wr.grad.permute(2, 3, 1, 0)) <= tol
        assert rel(db, br.grad) <= tol
        dx2, dw2, db2 = conv_grads_nhwc(x, wt, (s, s), (p, p), go)
        assert torch.equal(dx, dx2) and torch.equal(dw, dw2) and torch.equal(db, db2)


@pytest.mark.parametrize("dt,tol", [(torch.float64, 1e-12), (torch.float32, 1e-5)])
def test_native_conv_forward_and_bn_relu(cuda_device, dt, tol):
    """The unit backward's recomputation kernels: sbn_conv_forward against F.conv2d (same
    math, tap order differs), sbn_bn_relu / sbn_bn_relu_grad / sbn_add against the eager torch
    expressions they replace — bit-exact (a rounded multiply, then a rounded add)."""
    import torch.nn.functional as F

    from paper_1801_02108_b200.ops import add_nhwc, bn_relu_grad_nhwc, bn_relu_nhwc, conv_forward_nhwc
    g_ = torch.Generator(device="cuda").manual_seed(1)
    for (n, h, w, c, co, k, s, p) in ((5, 16, 16, 32, 16, 1, 1, 0), (3, 16, 16, 16, 16, 3, 1, 0),
                                      (2, 33, 29, 8, 20, 5, 2, 2)):
        x = torch.randn(n, h, w, c, device="cuda", dtype=dt, generator=g_)
        wt = torch.randn(k, k, c, co, device="cuda", dtype=dt, generator=g_)
        b = torch.randn(co, device="cuda", dtype=dt, generator=g_)
        y = conv_forward_nhwc(x, wt, b, (s, s), (p, p))
        torch.backends.cudnn.allow_tf32 = False
        ref = F.conv2d(x.permute(0, 3, 1, 2), wt.permute(3, 2, 0, 1), b, stride=s, padding=p).permute(0, 2, 3, 1)
        assert float((y - ref).abs().max() / ref.abs().max()) <= tol
    x = torch.randn(4, 16, 16, 24, device="cuda", dtype=dt, generator=g_)
    sc = torch.randn(24, device="cuda", dtype=dt, generator=g_)
    sh = torch.randn(24, device="cuda", dtype=dt, generator=g_)
    valid = (torch.rand(4, 16, 16, 1, device="cuda", generator=g_) > 0.3).to(dt)
    pre, post = bn_relu_nhwc(x, sc, sh, valid)
    assert torch.equal(pre, x * sc + sh) and torch.equal(post, torch.relu(x * sc + sh) * valid)
    g = torch.randn_like(x)
    assert torch.equal(bn_relu_grad_nhwc(g, pre, sc, valid), g * valid * (pre > 0).to(dt) * sc)
    assert torch.equal(bn_relu_grad_nhwc(g, pre, sc), g * (pre > 0).to(dt) * sc)
    assert torch.equal(add_nhwc(x, g), x + g)


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_native_train_stats_bn_vs_torch_and_deterministic(cuda_device, dt):
    """sbn_bn_train (TRAIN_STATS sparse_batch_norm) against the torch expression, at a size
    that splits the statistics into several row segments; repeated calls bit-identical."""
    rng = np.random.default_rng(3)
    t = torch.from_numpy(rng.standard_normal((40, 16, 16, 24)) * 3 + 1).to(dt).cuda()
    idx = P.BlockIndexList(np.zeros((40, 3), np.int32))
    bn = P.BnParams(rng.standard_normal(24), rng.standard_normal(24), np.zeros(24), np.ones(24))
    from paper_1801_02108_b200.blocks import GatheredBlocks
    spec = P.compute_block_spec((1, 64, 64, 24), P.ConvParams((3, 3), (1, 1), P.Padding.SAME, 24), (16, 16))
    blocks = GatheredBlocks(P.Tensor4D(t), spec, idx)
    out, (mean, var) = P.sparse_batch_norm(blocks, bn, P.BnMode.TRAIN_STATS)
    m_ref = t.mean(dim=(0, 1, 2))
    v_ref = t.var(dim=(0, 1, 2), unbiased=False)
    g = torch.as_tensor(np.asarray(bn.gamma), device=t.device, dtype=dt)
    be = torch.as_tensor(np.asarray(bn.beta), device=t.device, dtype=dt)
    ref = (t - m_ref) * (g / torch.sqrt(v_ref + bn.epsilon)) + be
    tol = 1e-12 if dt == torch.float64 else 1e-5
    rel = lambda a, b: float((a - b).abs().max() / b.abs().max())  # noqa: E731
    assert rel(mean, m_ref) <= tol and rel(var, v_ref) <= tol and rel(out.tensor.data, ref) <= tol
    out2, (mean2, var2) = P.sparse_batch_norm(blocks, bn, P.BnMode.TRAIN_STATS)
    assert torch.equal(out.tensor.data, out2.tensor.data) and torch.equal(mean, mean2) and torch.equal(var, var2)
