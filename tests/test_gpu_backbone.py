"""Configs 4/5 pinned numerically (reference `layers.py:311-353`, its tests
`test_layers.py:168-202`, demo a9 `test_acceptance.py:136-152`).

* fp32: the package's run_backbone against the REFERENCE's own run_backbone output
  (tests/golden/backbone.npz, oracle/make_golden.py gen_backbone) on a partial mask:
  per-stage masks and index lists bit-exact, outputs <= 1e-4 relative.
* bf16: the config-4 detector chain (c = 96/192/256/384, m = c/2, blocks 16/16/10/6,
  stride-2 projections) against the fp32 oracle stage by stage — each stage's oracle
  input is the GPU's bf16 output of the previous stage (bf16 re-rounding at stage
  boundaries), weights bf16-rounded — rel_err <= 2e-2 per stage (north star).  Run at
  the golden's reduced size, at a mid size, and at the exact config-4 frame (800x700).
"""
import numpy as np
import pytest
import torch

import paper_1801_02108_b200 as P
from oracle import sbnet_oracle as O
from golden_cases import backbone_case
from paper_1801_02108_b200.perf import detector_stage_configs

pytestmark = pytest.mark.gpu


def _stage_cfgs(stages):
    return [P.StageConfig(int(u), (int(a), int(b), int(c)), (int(bh), int(bw)), int(sc), int(st))
            for u, a, b, c, bh, bw, sc, st in stages]


def _r(a):
    return torch.from_numpy(np.asarray(a, np.float32)).bfloat16().float().numpy()


def _oracle_stage(stage: "P.Stage", bf16: bool) -> dict:
    """Oracle stage dict from the package's Stage (weights bf16-rounded for the bf16 path,
    as the device sees them)."""
    rr = _r if bf16 else (lambda a: np.asarray(a, np.float32))
    units = []
    for u in stage.units:
        ud = {"pre": u.pre_activation}
        for i, (fb, bn) in enumerate(((u.conv1, u.bn1), (u.conv2, u.bn2), (u.conv3, u.bn3)), 1):
            ud[f"w{i}"], ud[f"b{i}"] = rr(fb.weights), rr(fb.bias)
            ud[f"bn{i}"] = dict(gamma=bn.gamma, beta=bn.beta, mean=bn.running_mean, var=bn.running_var)
        units.append(ud)
    cfg = stage.config
    proj = None if stage.projection is None else (rr(stage.projection.weights), rr(stage.projection.bias))
    return dict(proj=proj, stride=cfg.stride, block=tuple(cfg.block_size), mask_scale=cfg.mask_scale,
                units=units)


@pytest.mark.parametrize("tag", ["det", "demo"])
def test_backbone_fp32_matches_reference_golden(cuda_device, tag):
    cfg, stages, x, mask, ref = backbone_case(tag)
    bb = P.build_backbone(_stage_cfgs(stages), np.random.default_rng(int(cfg[4])))
    res = P.run_backbone(bb, P.Tensor4D(torch.from_numpy(x).cuda()), P.BinaryMask(mask))
    errs = []
    for i, (r, (gy, gm, gidx)) in enumerate(zip(res, ref)):
        assert np.array_equal(r.mask.numpy(), gm), f"stage {i} mask"
        assert r.indices.entries.tolist() == gidx.tolist(), f"stage {i} indices"
        errs.append(O.rel_err(r.output.data.cpu().numpy(), gy))
    print(f"{tag} fp32 per-stage rel_err vs reference:", ["%.2e" % e for e in errs])
    assert max(errs) <= 1e-4, errs


def _bf16_stagewise(stages_cfg, seed, n, h, w, c, density):
    rng = np.random.default_rng(seed)
    bb = P.build_backbone(stages_cfg, rng)
    x = torch.from_numpy(rng.standard_normal((n, h, w, c)).astype(np.float32)).bfloat16().cuda()
    mask = np.concatenate([P.synth_mask_blobs((1, h, w), 1.0 - density, seed + i).numpy() for i in range(n)])
    res = P.run_backbone(bb, P.Tensor4D(x), P.BinaryMask(mask))
    errs, blocks = [], []
    inp = x.float().cpu().numpy()
    for i, (st, r) in enumerate(zip(bb.stages, res)):
        y, m, idx = O.run_stage(_oracle_stage(st, True), inp, mask)
        assert np.array_equal(r.mask.numpy(), m), f"stage {i} mask"
        assert r.indices.entries.tolist() == idx.tolist(), f"stage {i} indices"
        got = r.output.data.float().cpu().numpy()
        assert np.isfinite(got).all()
        errs.append(O.rel_err(got, y))
        blocks.append(len(idx))
        inp = got  # bf16 re-rounding at the stage boundary
    return errs, blocks


@pytest.mark.parametrize("n,h,w,density", [(2, 80, 64, 0.25), (1, 200, 176, 0.2), (2, 256, 224, 0.1)])
def test_backbone_bf16_config4_chain_stagewise(cuda_device, n, h, w, density):
    errs, blocks = _bf16_stagewise(detector_stage_configs(), 11 + h, n, h, w, 32, density)
    print(f"bf16 config-4 chain {n}x{h}x{w} @{density}: blocks {blocks}, per-stage rel_err",
          ["%.2e" % e for e in errs])
    assert max(errs) <= 2e-2, errs


def test_backbone_bf16_config4_full_frame(cuda_device):
    """The exact config-4 frame (800x700x32 -> 4 stages, 18 units), one frame, 20% blobs."""
    errs, blocks = _bf16_stagewise(detector_stage_configs(), 0, 1, 800, 700, 32, 0.2)
    print("bf16 config-4 800x700 per-stage blocks", blocks, "rel_err", ["%.2e" % e for e in errs])
    assert max(errs) <= 2e-2, errs
