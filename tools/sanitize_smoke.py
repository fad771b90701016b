"""One small invocation of every hot kernel, for compute-sanitizer (memcheck / racecheck /
synccheck): reduce_mask (ordered + cluster), gather / scatter / scatter_add / transpose,
sparse conv (SIMT fp32, tcgen05 single-CTA, CTA-pair, strided TMA), residual unit (SIMT,
fused mask + CTA pair in place, wide: one launch and three launches), dense conv (single and
CTA pair), host-frame unit copies, the training-path kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200 import _lib
from paper_1801_02108_b200.layers import residual_unit_into, sparse_conv_into

dev = torch.device("cuda", 0)
lib = _lib.load()
rng = np.random.default_rng(0)
n, h, w = 2, 72, 60
mk = P.synth_mask_blobs((n, h, w), 0.6, 1).cuda()

# reduce_mask / gather / scatter
x32 = torch.randn(n, h, w, 16, device=dev)
p3 = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, 16)
spec = P.compute_block_spec((n, h, w, 16), p3, (16, 16))
idx = P.reduce_mask(mk, spec)
P.gather(P.Tensor4D(x32), idx, spec)
spec1 = P.compute_block_spec((n, h, w, 16), P.ConvParams((1, 1), (1, 1), P.Padding.VALID, 16), (8, 8))
idx1 = P.reduce_mask(mk, spec1)
# many block rows: the ranges kernel (several rows per CTA, whole-CTA look-back), vec and not
for (nb, hb, wb) in ((96, 64, 64), (64, 40, 30)):
    mkb = P.synth_mask_blobs((nb, hb, wb), 0.7, 2).cuda()
    P.reduce_mask(mkb, P.compute_block_spec((nb, hb, wb, 8), P.ConvParams((1, 1), (1, 1), P.Padding.VALID, 8), (4, 4)))
g1 = P.gather(P.Tensor4D(x32), idx1, spec1)
P.scatter(g1, spec1, P.Tensor4D(torch.zeros_like(x32)))
P.scatter_add(g1, spec1, P.Tensor4D(torch.zeros_like(x32)))
gt = P.gather_transpose(P.Tensor4D(x32), idx1, spec1)
P.scatter_transpose(gt, spec1, P.Tensor4D(torch.zeros_like(x32)))
# sparse convs
f32 = P.FilterBank(torch.randn(3, 3, 16, 16) * 0.1, torch.randn(16))
P.sparse_conv2d(P.Tensor4D(x32), mk, f32, p3, (16, 16))
for c, blk_, flags in ((128, 16, 0), (128, 16, 16384), (128, 16, 2048), (128, 16, 32), (64, 8, 0)):  # resident pair (two launches / one), single-CTA, streamed pair
    x = torch.randn(n, h, w, c, device=dev).bfloat16()
    fb = P.FilterBank((torch.randn(3, 3, c, c) / (3 * c ** 0.5)).bfloat16(), torch.randn(c).bfloat16())
    pc = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, c)
    old = lib.sbn_debug_set_flags(flags)
    P.sparse_conv2d(P.Tensor4D(x), mk, fb, pc, (blk_, blk_))
    lib.sbn_debug_set_flags(old)
x = torch.randn(n, h, w, 64, device=dev).bfloat16()
fb = P.FilterBank((torch.randn(3, 3, 64, 64) / 24).bfloat16(), torch.randn(64).bfloat16())
P.sparse_conv2d(P.Tensor4D(x), mk, fb, P.ConvParams((3, 3), (2, 2), P.Padding.SAME, 64), (17, 17))
# tap-GEMM conv at the paper's Table-1 channel counts: mask-fused one-launch mode (small
# grids: 135 and 192 units) and list mode (48 channels, 16-channel K-chunks)
for (hh, ww, c, blk_) in ((50, 88, 96, 8), (100, 176, 24, 32), (200, 352, 48, 16)):
    xt = torch.randn(1, hh, ww, c, device=dev).bfloat16()
    ft = P.FilterBank((torch.randn(3, 3, c, c) / (3 * c ** 0.5)).bfloat16(), torch.randn(c).bfloat16())
    P.sparse_conv2d(P.Tensor4D(xt), P.synth_mask_topleft((1, hh, ww), 0.9).cuda(), ft,
                    P.ConvParams((3, 3), (1, 1), P.Padding.SAME, c), (blk_, blk_))
# residual units
u = P.random_unit_params(rng, 64, 32)
P.sparse_residual_unit(P.Tensor4D(x), mk, u, (16, 16))
xi = x.clone()
P.sparse_residual_unit(P.Tensor4D(xi), mk, u, (16, 16), inplace=True)
P.sparse_residual_unit(P.Tensor4D(x.float()), mk, u, (16, 16))
old = lib.sbn_debug_set_flags(4)  # wide three-launch unit
P.sparse_residual_unit(P.Tensor4D(x), mk, u, (16, 16))
lib.sbn_debug_set_flags(old)
# dense projection conv (tcgen05, bias fused)
from paper_1801_02108_b200.ops import projection_conv
xp = torch.randn(1, 50, 38, 32, device=dev).bfloat16()
fp = P.FilterBank((torch.randn(3, 3, 32, 96) / 17).bfloat16(), torch.randn(96).bfloat16())
projection_conv(xp, fp, P.ConvParams((3, 3), (2, 2), P.Padding.SAME, 96))
# host-frame unit (zero-copy copies)
hx = x.cpu().pin_memory()
P.sparse_residual_unit(P.Tensor4D(hx), P.BinaryMask(mk.data.cpu().pin_memory()), u, (16, 16), inplace=True)
# CHANNELS_FIRST paths (transposing window copies)
xcf = P.Tensor4D(x.permute(0, 3, 1, 2).contiguous(), P.Layout.CHANNELS_FIRST)
P.sparse_residual_unit(xcf, mk, u, (16, 16), inplace=True)
P.sparse_conv2d(xcf, mk, fb, P.ConvParams((3, 3), (1, 1), P.Padding.SAME, 64), (16, 16))
# round 2: native conv gradients (segmented weight-gradient reduction), the sliced SIMT conv
# with a staged filter bank (fp32, 12 blocks), the half-block tail jobs of the tcgen05 conv
# (B % grid small: 2*R <= grid), and the backbone's side-stream mask pipeline
from paper_1801_02108_b200.ops import conv_grads_nhwc
xg = torch.randn(3, 40, 36, 8, device=dev, dtype=torch.float64)
wg = torch.randn(3, 3, 8, 6, device=dev, dtype=torch.float64)
conv_grads_nhwc(xg, wg, (1, 1), (1, 1), torch.randn(3, 40, 36, 6, device=dev, dtype=torch.float64))
xs1 = torch.randn(1, 64, 64, 16, device=dev)
P.sparse_conv2d(P.Tensor4D(xs1), P.synth_mask_blobs((1, 64, 64), 0.5, 3).cuda(), f32, p3, (16, 16))
xt3 = torch.randn(1, 180, 200, 128, device=dev).bfloat16()  # 195 blocks on 148 CTAs: 47 split
ft3 = P.FilterBank((torch.randn(3, 3, 128, 128) / 34).bfloat16(), torch.randn(128).bfloat16())
for flags in (0, 2048):  # list mode: resident pair (5 pair rounds) / single-CTA with split tail jobs
    old = lib.sbn_debug_set_flags(flags)
    P.sparse_conv2d(P.Tensor4D(xt3), P.synth_mask_topleft((1, 180, 200), 0.0).cuda(), ft3,
                    P.ConvParams((3, 3), (1, 1), P.Padding.SAME, 128), (16, 16), pool=P.PoolMode.MAX, threshold=1 / 256)
    lib.sbn_debug_set_flags(old)
# tap-GEMM conv, one launch with the global block list (16x16 windows by default; forced for 32x32)
xg2 = torch.randn(1, 120, 150, 24, device=dev).bfloat16()
fg2 = P.FilterBank((torch.randn(3, 3, 24, 24) / 14).bfloat16(), torch.randn(24).bfloat16())
for blk_, flags in ((16, 0), (32, 65536)):
    old = lib.sbn_debug_set_flags(flags)
    P.sparse_conv2d(P.Tensor4D(xg2), P.synth_mask_topleft((1, 120, 150), 0.8).cuda(), fg2,
                    P.ConvParams((3, 3), (1, 1), P.Padding.SAME, 24), (blk_, blk_))
    lib.sbn_debug_set_flags(old)
bb = P.build_backbone([P.StageConfig(1, (8, 12, 24), (16, 16), 1, 1), P.StageConfig(1, (24, 24, 48), (12, 12), 2, 2)],
                      np.random.default_rng(1))
P.run_backbone(bb, P.Tensor4D(torch.randn(1, 60, 52, 8, device=dev)), P.synth_mask_blobs((1, 60, 52), 0.7, 2).cuda())
# round 2, second half: the one-launch wide unit (functional and in place with the rim
# snapshot; c = 64 and the config-4 stage-0 shape c = 96), the three-launch path it
# replaces, the CTA-pair projection, and the native training-path kernels
for c_, m_ in ((64, 32), (96, 48)):
    xw = torch.randn(2, 72, 60, c_, device=dev).bfloat16()
    uw = P.random_unit_params(rng, c_, m_)
    for flags in (4, 4 | 256):
        old = lib.sbn_debug_set_flags(flags)
        P.sparse_residual_unit(P.Tensor4D(xw), mk, uw, (16, 16))
        P.sparse_residual_unit(P.Tensor4D(xw.clone()), mk, uw, (16, 16), inplace=True)
        lib.sbn_debug_set_flags(old)
xq = torch.randn(2, 22, 19, 192, device=dev).bfloat16()
fq = P.FilterBank((torch.randn(3, 3, 192, 256) / 41).bfloat16(), torch.randn(256).bfloat16())
projection_conv(xq, fq, P.ConvParams((3, 3), (2, 2), P.Padding.SAME, 256))
xf = P.Tensor4D(torch.randn(1, 40, 36, 16, device=dev))
uf = P.random_unit_params(rng, 16, 8)
mf = P.synth_mask_blobs((1, 40, 36), 0.5, 4)
P.sparse_residual_unit_grads(xf, mf, uf, (10, 10), P.Tensor4D(torch.randn(1, 40, 36, 16, device=dev)))
specb = P.compute_block_spec((1, 40, 36, 16), P.ConvParams((3, 3), (1, 1), P.Padding.SAME, 16), (10, 10))
gb_ = P.gather(xf, P.reduce_mask(mf, specb), specb)
P.sparse_batch_norm(gb_, P.BnParams.identity(16), P.BnMode.TRAIN_STATS)
torch.cuda.synchronize()
print("sanitize smoke done", flush=True)
