"""GPU parity of the one-launch wide tcgen05 unit (unit_wide.cu, `unit_wide_fused_kernel`:
16x16 blocks; the S1 / S2 rows of a block stay in shared memory, the in-place rims come
from a snapshot taken before the launch).

The fused launch issues the tensor-core k-steps of every accumulator in the same order as
the three-launch path (IN -> S1 stack -> MID -> S2 stack -> OUT) and rounds the same
values, so the unit's output must be BIT-identical to the three-launch path's
(SBN_DEBUG_WIDE_UNFUSED = 256 forces that one), in place and functional.  Both are also
checked against the fp32 oracle (north star: bf16 <= 2e-2).  Cases cover the config-4
stage-0 shape (c = 96) and the config-2 shape (64), ragged frame borders, many blocks per
CTA (ring wrap-around of every buffer), a full mask and an empty one.  The c = 192 / 128
shapes do not fit the one-launch kernel (weights + buffers > shared memory) and must keep
running the three launches.
"""
import numpy as np
import pytest
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200 import _lib
from oracle import sbnet_oracle as O

pytestmark = pytest.mark.gpu

FORCE_WIDE = 4      # SBN_DEBUG_FORCE_WIDE: the wide unit even where the single kernel applies
WIDE_UNFUSED = 256  # SBN_DEBUG_WIDE_UNFUSED: IN and MID as two launches
NO_SPLIT = 1024     # SBN_DEBUG_WIDE_NO_SPLIT: one work item per tile in the three-launch kernels


def _case(seed, n, h, w, c, m, density):
    rng = np.random.default_rng(seed)
    x = torch.from_numpy(rng.standard_normal((n, h, w, c)).astype(np.float32)).bfloat16()
    u = P.random_unit_params(rng, c, m)
    if density >= 1.0:
        mk = np.ones((n, h, w), np.uint8)
    else:
        mk = np.concatenate([P.synth_mask_blobs((1, h, w), 1.0 - density, seed + i).numpy() for i in range(n)])
    return x, u, P.BinaryMask(mk)


def _run(x, mk, u, flags, inplace=False, block=16):
    lib = _lib.load()
    prev = lib.sbn_debug_set_flags(flags)
    try:
        y = P.sparse_residual_unit(P.Tensor4D(x.clone().cuda()), mk, u, (block, block), inplace=inplace)
        torch.cuda.synchronize()
    finally:
        lib.sbn_debug_set_flags(prev)
    return y.data.cpu()


def _oracle(x_bf16, u, mk, block=16):
    def r(a):
        return torch.from_numpy(np.asarray(a, np.float32)).bfloat16().float().numpy()
    ud = {"pre": u.pre_activation}
    for i, (fb, bn) in enumerate(((u.conv1, u.bn1), (u.conv2, u.bn2), (u.conv3, u.bn3)), 1):
        ud[f"w{i}"], ud[f"b{i}"] = r(fb.weights), r(fb.bias)
        ud[f"bn{i}"] = dict(gamma=bn.gamma, beta=bn.beta, mean=bn.running_mean, var=bn.running_var)
    return O.sparse_residual_unit(x_bf16.float().numpy(), mk.numpy(), ud, (block, block))


# (c, m, n, h, w, density)
CASES = [
    (96, 48, 2, 72, 60, 0.3),     # config-4 stage-0 shape, ragged borders
    (192, 96, 2, 60, 44, 0.3),    # stage-1 shape: three launches (does not fit one CTA)
    (64, 32, 2, 96, 80, 0.25),    # config-2 shape
    (32, 16, 1, 50, 47, 0.5),
    (128, 64, 1, 64, 64, 0.4),
    (96, 48, 1, 30, 30, 1.0),     # full mask, one frame of 3x3 blocks
    (192, 96, 1, 16, 16, 1.0),    # 2x2 blocks, three of them clipped by the frame border
]


@pytest.mark.parametrize("c,m,n,h,w,density", CASES)
def test_fused_unit_bit_identical_to_three_launches(cuda_device, c, m, n, h, w, density):
    x, u, mk = _case(c + h, n, h, w, c, m, density)
    fused = _run(x, mk, u, FORCE_WIDE)
    three = _run(x, mk, u, FORCE_WIDE | WIDE_UNFUSED)
    assert torch.equal(fused, three), (c, m, n, h, w, (fused.float() - three.float()).abs().max().item())
    err = O.rel_err(fused.float().numpy(), _oracle(x, u, mk))
    assert err <= 2e-2, err
    # in place (rim snapshot) == functional == three launches in place
    assert torch.equal(_run(x, mk, u, FORCE_WIDE, inplace=True), fused)
    assert torch.equal(_run(x, mk, u, FORCE_WIDE | WIDE_UNFUSED, inplace=True), fused)


@pytest.mark.parametrize("c,m", [(96, 48), (192, 96), (64, 32), (128, 64)])
def test_fused_unit_many_blocks_per_cta(cuda_device, c, m):
    """Several hundred to a few thousand active blocks, in place: every CTA walks many blocks
    (the window ring, both A2 buffers, A3 and the accumulators wrap around many times) while
    other CTAs overwrite the interiors that its windows' rims cover."""
    n, h, w = (12, 200, 176) if c == 192 else (3, 400, 352)
    x, u, mk = _case(7 + c, n, h, w, c, m, 0.35)
    fused = _run(x, mk, u, FORCE_WIDE, inplace=True)
    three = _run(x, mk, u, FORCE_WIDE | WIDE_UNFUSED, inplace=True)
    assert torch.equal(fused, three)
    assert torch.isfinite(fused.float()).all()


def test_fused_unit_empty_mask(cuda_device):
    x, u, _ = _case(3, 2, 40, 36, 96, 48, 0.5)
    empty = P.BinaryMask(np.zeros((2, 40, 36), np.uint8))
    assert torch.equal(_run(x, empty, u, FORCE_WIDE), x)


def test_fused_unit_stage_chain(cuda_device):
    """run_stage on the config-4 stage-0 shape (3 in-place one-launch units sharing one index
    list, each with its own rim snapshot) == the same stage on the three-launch path."""
    rng = np.random.default_rng(9)
    cfg = P.StageConfig(unit_count=3, channels=(96, 48, 96), block_size=(16, 16))
    stage = P.build_stage(cfg, rng)
    x = torch.from_numpy(rng.standard_normal((2, 120, 104, 96)).astype(np.float32)).bfloat16()
    mk = P.BinaryMask(np.concatenate([P.synth_mask_blobs((1, 120, 104), 0.7, s).numpy() for s in (1, 2)]))
    lib = _lib.load()
    outs = []
    for flags in (0, WIDE_UNFUSED):
        prev = lib.sbn_debug_set_flags(flags)
        try:
            outs.append(P.run_stage(stage, P.Tensor4D(x.clone().cuda()), mk).output.data.cpu())
            torch.cuda.synchronize()
        finally:
            lib.sbn_debug_set_flags(prev)
    assert torch.equal(outs[0], outs[1])


# (c, m, block, n, h, w, density): few tiles per launch, so OUT (N >= 128) runs as two
# half-width column slices per tile on different CTAs
SPLIT_CASES = [
    (384, 192, 6, 1, 60, 64, 0.3),    # config-4 stage-3 shape
    (384, 192, 6, 2, 100, 90, 0.5),
    (256, 128, 10, 1, 80, 84, 0.4),   # stage-2 shape
    (192, 96, 16, 1, 64, 64, 0.3),    # stage-1 shape
    (128, 64, 8, 1, 40, 48, 0.5),
]


@pytest.mark.parametrize("c,m,blk,n,h,w,density", SPLIT_CASES)
def test_column_slices_bit_identical(cuda_device, c, m, blk, n, h, w, density):
    """Column slices change which CTA computes which accumulator columns, not the k-step
    order of any column: results are bit-identical to one work item per tile, in place and
    functional, and within the bf16 tolerance of the oracle."""
    x, u, mk = _case(c + blk, n, h, w, c, m, density)
    split = _run(x, mk, u, FORCE_WIDE, block=blk)
    whole = _run(x, mk, u, FORCE_WIDE | NO_SPLIT, block=blk)
    assert torch.equal(split, whole), (c, m, blk, (split.float() - whole.float()).abs().max().item())
    assert torch.equal(_run(x, mk, u, FORCE_WIDE, inplace=True, block=blk), split)
    assert O.rel_err(split.float().numpy(), _oracle(x, u, mk, blk)) <= 2e-2
