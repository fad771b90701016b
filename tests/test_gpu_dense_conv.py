"""tcgen05 dense 1x1 / 3x3 / 5x5 conv with fused bias (sbn_dense_conv): the config-4 stage projections
(stride 2) and square stride-1 shapes vs cuDNN in fp32 on the same bf16-rounded inputs;
bf16 output rounding -> rel_err <= 1e-2."""
import numpy as np
import pytest
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200.ops import projection_conv
from oracle import sbnet_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,h,w,cin,cout,stride,same,k", [
    (2, 50, 38, 32, 96, 2, True, 3), (1, 37, 29, 96, 192, 2, True, 3), (2, 22, 19, 192, 256, 2, True, 3),
    (1, 14, 12, 256, 384, 2, True, 3), (1, 40, 33, 64, 64, 1, True, 3), (2, 17, 35, 128, 128, 1, False, 3),
    (1, 24, 24, 32, 32, 3, True, 3), (2, 31, 27, 64, 64, 1, True, 1), (1, 33, 40, 128, 128, 1, False, 1),
    (2, 29, 23, 32, 32, 1, True, 5), (1, 26, 31, 64, 64, 2, False, 5), (1, 19, 22, 32, 32, 3, True, 5),
    # channel counts off the 32 / 64 grid: 16-channel K-chunks (48), K and N padded to 32 (24)
    (2, 33, 41, 24, 24, 1, True, 3), (1, 45, 38, 48, 48, 1, True, 3), (1, 30, 27, 96, 96, 2, True, 3)])
def test_dense_conv_tc_vs_cudnn_fp32(cuda_device, n, h, w, cin, cout, stride, same, k):
    rng = np.random.default_rng(cin + cout + stride + 7 * k)
    x = torch.from_numpy(rng.standard_normal((n, h, w, cin)).astype(np.float32)).bfloat16().cuda()
    wt = (rng.standard_normal((k, k, cin, cout)) / np.sqrt(k * k * cin)).astype(np.float32)
    b = rng.standard_normal(cout).astype(np.float32)
    f = P.FilterBank(torch.from_numpy(wt).bfloat16(), torch.from_numpy(b).bfloat16())
    p = P.ConvParams((k, k), (stride, stride), P.Padding.SAME if same else P.Padding.VALID, cout)
    lib = P._lib.load() if hasattr(P, "_lib") else None
    from paper_1801_02108_b200 import _lib
    assert _lib.load().sbn_dense_conv_supported(2, cin, cout, k, k, stride, stride) == 1
    y = projection_conv(x, f, p).float().cpu().numpy()
    fb32 = P.FilterBank(torch.from_numpy(wt).bfloat16().float(), torch.from_numpy(b).bfloat16().float())
    ref = P.conv2d_direct(P.Tensor4D(x.float()), fb32, p).data.cpu().numpy()
    assert y.shape == ref.shape
    assert O.rel_err(y, ref) <= 1e-2
    del lib


@pytest.mark.parametrize("cin,cout,stride,block,same,k", [
    (64, 64, 2, 17, True, 3), (128, 128, 2, 13, True, 3), (32, 96, 1, 10, True, 3), (64, 64, 3, 24, False, 3),
    (96, 192, 2, 9, True, 3), (64, 64, 1, 10, True, 1), (128, 128, 1, 11, False, 1), (32, 32, 1, 14, True, 5),
    (64, 64, 1, 15, False, 5), (64, 64, 2, 17, True, 5),
    # blocks whose output window exceeds 128 px: several TMA tiles per block
    (128, 128, 1, 32, True, 3), (64, 64, 2, 33, True, 3), (32, 32, 1, 24, False, 5), (64, 64, 1, 19, True, 1),
    # the paper's Table-1 channel counts (24 / 48 / 96)
    (24, 24, 1, 8, True, 3), (24, 24, 1, 16, True, 3), (48, 48, 1, 8, True, 3), (48, 48, 1, 16, True, 3),
    (96, 96, 1, 8, True, 3), (96, 96, 1, 32, True, 3)])
def test_sparse_conv_strided_tc_vs_fp32_oracle(cuda_device, cin, cout, stride, block, same, k):
    """Strided / other-shape sparse 1x1 / 3x3 / 5x5 convs on the TMA tap-GEMM path (kernel
    variant 2) against the fp32 oracle on bf16-rounded inputs."""
    rng = np.random.default_rng(stride * 100 + block + 1000 * k)
    n, h, w = 2, 53, 47
    x = torch.from_numpy(rng.standard_normal((n, h, w, cin)).astype(np.float32)).bfloat16()
    wt = torch.from_numpy((rng.standard_normal((k, k, cin, cout)) / np.sqrt(k * k * cin)).astype(np.float32)).bfloat16()
    b = torch.from_numpy(rng.standard_normal(cout).astype(np.float32)).bfloat16()
    mk = (rng.random((n, h, w)) < 0.03).astype(np.uint8)
    p = P.ConvParams((k, k), (stride, stride), P.Padding.SAME if same else P.Padding.VALID, cout)
    spec = P.compute_block_spec((n, h, w, cin), p, (block, block))
    from paper_1801_02108_b200.layers import sparse_conv_algo
    assert sparse_conv_algo(torch.bfloat16, P.FilterBank(wt, b), p, spec) == "tcgen05"
    y = P.sparse_conv2d(P.Tensor4D(x.cuda()), P.BinaryMask(mk), P.FilterBank(wt, b), p, (block, block))
    ref = O.sparse_conv2d(x.float().numpy(), mk, wt.float().numpy(), b.float().numpy(), (stride, stride), same,
                          (block, block))
    assert O.rel_err(y.data.float().cpu().numpy(), ref) <= 2e-2


@pytest.mark.parametrize("cin,k,stride,block,hw,density", [
    (96, 3, 1, 8, (50, 88), 0.1), (24, 3, 1, 32, (400, 704), 0.1), (48, 3, 1, 16, (61, 77), 0.0),
    (64, 1, 1, 10, (45, 52), 1.0), (32, 5, 2, 17, (70, 66), 0.3), (96, 3, 1, 8, (130, 140), 0.1),
    (96, 3, 1, 8, (200, 200), 0.1)])
def test_mask_fused_tap_gemm_conv_equals_reduce_mask_then_conv(cuda_device, cin, k, stride, block, hw, density):
    """sparse_conv2d's one-launch path on the tap-GEMM kernel (every CTA tests its own <= 4
    (candidate, sub-tile) units; the last case, 1156 units on 148 slots, is above that and
    takes reduce_mask + conv) writes exactly what reduce_mask + the listed conv write, and
    nothing outside the active output blocks."""
    from paper_1801_02108_b200.layers import sparse_conv_algo, sparse_conv_into, sparse_conv_masked_into
    rng = np.random.default_rng(cin + block + hw[0])
    h, w = hw
    x = torch.from_numpy(rng.standard_normal((1, h, w, cin)).astype(np.float32)).bfloat16().cuda()
    f = P.FilterBank(torch.from_numpy((rng.standard_normal((k, k, cin, cin)) / np.sqrt(k * k * cin)).astype(np.float32)).bfloat16(),
                     torch.from_numpy(rng.standard_normal(cin).astype(np.float32)).bfloat16())
    p = P.ConvParams((k, k), (stride, stride), P.Padding.SAME, cin)
    spec = P.compute_block_spec((1, h, w, cin), p, (block, block))
    assert sparse_conv_algo(torch.bfloat16, f, p, spec) == "tcgen05"
    mk = P.synth_mask_topleft((1, h, w), 1.0 - density).cuda()
    oh, ow = spec.out_size
    a = torch.full((1, oh, ow, cin), 3.0, dtype=torch.bfloat16, device="cuda")
    b = a.clone()
    sparse_conv_masked_into(x, a, mk.data, f, p, spec)
    sparse_conv_into(x, b, f, p, spec, P.reduce_mask(mk, spec))
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    if density == 0.0:
        assert bool((a == 3.0).all())


DENSE_SINGLE = 512  # SBN_DEBUG_DENSE_SINGLE: the single-CTA kernel even where the CTA-pair one applies


@pytest.mark.parametrize("n,h,w,cin,cout,stride", [
    (3, 41, 37, 192, 256, 2),   # the config-4 stage-2 projection shape class (streamed halves)
    (2, 27, 23, 256, 384, 2),   # stage 3: streamed halves, two N-slices of 192
    (8, 60, 50, 192, 256, 2),   # many pair tiles per pair (ring wrap-around)
    (1, 9, 15, 192, 256, 2)])   # an odd number of 8 x 16 tiles: the last pair has an empty rank-1 tile
def test_dense_conv_pair_bit_identical_to_single_cta(cuda_device, n, h, w, cin, cout, stride):
    """The CTA-pair (cta_group::2, M = 256, B split along N) projection issues the same k-steps
    per accumulator row as the single-CTA kernel: bit-identical output."""
    from paper_1801_02108_b200 import _lib
    rng = np.random.default_rng(n + h + cin)
    x = torch.from_numpy(rng.standard_normal((n, h, w, cin)).astype(np.float32)).bfloat16().cuda()
    wt = (rng.standard_normal((3, 3, cin, cout)) / np.sqrt(9 * cin)).astype(np.float32)
    b = rng.standard_normal(cout).astype(np.float32)
    f = P.FilterBank(torch.from_numpy(wt).bfloat16(), torch.from_numpy(b).bfloat16())
    p = P.ConvParams((3, 3), (stride, stride), P.Padding.SAME, cout)
    lib = _lib.load()
    pair = projection_conv(x, f, p)
    torch.cuda.synchronize()
    prev = lib.sbn_debug_set_flags(DENSE_SINGLE)
    try:
        single = projection_conv(x, f, p)
        torch.cuda.synchronize()
    finally:
        lib.sbn_debug_set_flags(prev)
    assert torch.equal(pair, single), (pair.float() - single.float()).abs().max().item()
    fb32 = P.FilterBank(torch.from_numpy(wt).bfloat16().float(), torch.from_numpy(b).bfloat16().float())
    ref = P.conv2d_direct(P.Tensor4D(x.float()), fb32, p).data.cpu().numpy()
    assert O.rel_err(pair.float().cpu().numpy(), ref) <= 1e-2
