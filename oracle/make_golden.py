"""Generate golden vectors by running the REAL reference (``blockconv``) in this container.

TEST INFRASTRUCTURE ONLY.  Imports the reference from ``/root/reference/pkg/src``
(read-only, present only in the build container) and writes small fixtures to
``tests/golden/*.npz``.  The fixtures travel with the repo; ``/root/reference`` does
not, so GPU-box tests compare against these files.

    python oracle/make_golden.py            # regenerate all fixtures

Every case is seeded; inputs are stored alongside outputs so the fixtures are
self-contained (no RNG replay needed on the box).
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("SBNET_REFERENCE_SRC", "/root/reference/pkg/src")
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import blockconv  # noqa: F401  (the reference package)
    return blockconv


def _conv_case(rng):
    """Random conv configuration in the reference's own sweep space (verify.py:60-76)."""
    n = int(rng.integers(1, 3))
    c = int(rng.integers(1, 9))
    co = int(rng.integers(1, 9))
    kh = int(rng.choice([1, 3, 3, 5]))
    kw = int(rng.choice([1, 3, 3, 5]))
    sh = int(rng.choice([1, 1, 1, 2])) if kh > 1 else 1
    sw = int(rng.choice([1, 1, 1, 2])) if kw > 1 else 1
    h = int(rng.integers(max(kh, 6), 49))
    w = int(rng.integers(max(kw, 6), 49))
    same = bool(rng.random() < 0.5)
    bh = min(kh + sh * int(rng.integers(1, 14)), kh + sh * 13)
    bw = min(kw + sw * int(rng.integers(1, 14)), kw + sw * 13)
    return n, h, w, c, co, (kh, kw), (sh, sw), same, (bh, bw)


def _mask(rng, n, h, w, kind):
    if kind == "full":
        return np.ones((n, h, w), np.uint8)
    if kind == "empty":
        return np.zeros((n, h, w), np.uint8)
    if kind == "single":
        m = np.zeros((n, h, w), np.uint8)
        for i in range(n):
            m[i, rng.integers(h), rng.integers(w)] = 1
        return m
    p = float(kind)
    coarse = rng.random((n, -(-h // 4), -(-w // 4))) < p
    return coarse.repeat(4, axis=1).repeat(4, axis=2)[:, :h, :w].astype(np.uint8)


KINDS = ["full", "empty", "single", "0.25", "0.5", "0.75", "0.9"]


def gen_geometry(bc):
    rng = np.random.default_rng(1000)
    rows = []
    for _ in range(300):
        n, h, w, c, co, k, s, same, b = _conv_case(rng)
        pad = bc.Padding.SAME if same else bc.Padding.VALID
        spec = bc.compute_block_spec((n, h, w, c), bc.ConvParams(k, s, pad, co), b)
        rows.append([h, w, *k, *s, int(same), *b, *spec.overlap, *spec.in_stride,
                     *spec.out_block_size, *spec.grid_origin, *spec.grid_count, *spec.out_size])
    # rejection cases: block < kernel, stride not dividing block - kernel
    bad = [[8, 8, 3, 3, 1, 1, 0, 2, 4], [16, 16, 3, 3, 2, 2, 0, 6, 6], [9, 9, 5, 3, 1, 1, 1, 4, 8]]
    for r in bad:
        try:
            bc.compute_block_spec((1, r[0], r[1], 1),
                                  bc.ConvParams((r[2], r[3]), (r[4], r[5]),
                                                bc.Padding.SAME if r[6] else bc.Padding.VALID, 1),
                                  (r[7], r[8]))
            raise AssertionError("reference accepted an invalid geometry")
        except bc.GeometryError:
            pass
    np.savez_compressed(os.path.join(OUT, "geometry.npz"), rows=np.asarray(rows, np.int64),
                        bad=np.asarray(bad, np.int64))


def gen_reduce_mask(bc):
    rng = np.random.default_rng(2000)
    out = {}
    for i in range(60):
        n, h, w, c, co, k, s, same, b = _conv_case(rng)
        pad = bc.Padding.SAME if same else bc.Padding.VALID
        spec = bc.compute_block_spec((n, h, w, c), bc.ConvParams(k, s, pad, co), b)
        m = _mask(rng, n, h, w, KINDS[i % len(KINDS)])
        if i % 5 == 4:  # sparse random pixels
            m = (rng.random((n, h, w)) < 0.05).astype(np.uint8)
        avg = i % 3 == 2
        thr = None
        if avg and i % 2:
            thr = float(rng.choice([0.1, 0.25, 0.5, 0.75, 1.0]))
        idx = bc.reduce_mask(bc.BinaryMask(m), spec, bc.PoolMode.AVG if avg else bc.PoolMode.MAX, thr)
        out[f"c{i}_cfg"] = np.asarray([h, w, *k, *s, int(same), *b, int(avg),
                                       -1 if thr is None else int(round(thr * 1e6))], np.int64)
        out[f"c{i}_mask"] = m
        out[f"c{i}_idx"] = idx.entries
    # downsample cases
    for j in range(10):
        n, h, w = int(rng.integers(1, 3)), int(rng.integers(1, 40)), int(rng.integers(1, 40))
        f = int(rng.integers(1, 6))
        m = (rng.random((n, h, w)) < 0.1).astype(np.uint8)
        out[f"d{j}_f"] = np.asarray([f])
        out[f"d{j}_mask"] = m
        out[f"d{j}_out"] = bc.downsample_mask(bc.BinaryMask(m), f).data
    np.savez_compressed(os.path.join(OUT, "reduce_mask.npz"), **out)


def gen_gather_scatter(bc):
    rng = np.random.default_rng(3000)
    out = {}
    for i in range(30):
        n, h, w, c, co, k, s, same, b = _conv_case(rng)
        pad = bc.Padding.SAME if same else bc.Padding.VALID
        dims = (n, h, w, c)
        spec = bc.compute_block_spec(dims, bc.ConvParams(k, s, pad, co), b)
        m = _mask(rng, n, h, w, KINDS[i % len(KINDS)])
        idx = bc.reduce_mask(bc.BinaryMask(m), spec)
        dt = np.float64 if i % 4 == 3 else np.float32
        x = rng.standard_normal(dims).astype(dt)
        g = bc.gather(bc.Tensor4D(x), idx, spec)
        gt = bc.gather_transpose(bc.Tensor4D(x), idx, spec)
        ib = bc.blocks.in_bounds_map(idx, spec)
        obh, obw = spec.out_block_size
        blk = rng.standard_normal((idx.count, obh, obw, c)).astype(dt)
        dst = rng.standard_normal((n, *spec.out_size, c)).astype(dt)
        gb = g.with_tensor(bc.Tensor4D(blk))
        sw_ = bc.scatter(gb, spec, bc.Tensor4D(dst)).data
        sa_ = bc.scatter_add(gb, spec, bc.Tensor4D(dst)).data
        gbt = g.with_tensor(bc.transpose_layout(bc.Tensor4D(blk)))
        st_ = bc.scatter_transpose(gbt, spec, bc.Tensor4D(dst)).nhwc()
        out[f"c{i}_cfg"] = np.asarray([h, w, *k, *s, int(same), *b], np.int64)
        out[f"c{i}_x"] = x
        out[f"c{i}_idx"] = idx.entries
        out[f"c{i}_gather"] = g.tensor.data
        out[f"c{i}_gather_t"] = gt.tensor.data
        out[f"c{i}_inb"] = ib
        out[f"c{i}_blk"] = blk
        out[f"c{i}_dst"] = dst
        out[f"c{i}_scatter"] = sw_
        out[f"c{i}_scatter_add"] = sa_
        out[f"c{i}_scatter_t"] = np.ascontiguousarray(st_)
    np.savez_compressed(os.path.join(OUT, "gather_scatter.npz"), **out)


def gen_sparse_conv(bc):
    rng = np.random.default_rng(4000)
    out = {}
    for i in range(24):
        n, h, w, c, co, k, s, same, b = _conv_case(rng)
        pad = bc.Padding.SAME if same else bc.Padding.VALID
        p = bc.ConvParams(k, s, pad, co)
        m = _mask(rng, n, h, w, KINDS[i % len(KINDS)])
        x = rng.standard_normal((n, h, w, c)).astype(np.float32)
        wt = rng.standard_normal((*k, c, co)).astype(np.float32)
        bias = rng.standard_normal(co).astype(np.float32)
        y = bc.sparse_conv2d(bc.Tensor4D(x), bc.BinaryMask(m), bc.FilterBank(wt, bias), p, b)
        out[f"c{i}_cfg"] = np.asarray([h, w, *k, *s, int(same), *b], np.int64)
        out[f"c{i}_x"], out[f"c{i}_mask"], out[f"c{i}_w"], out[f"c{i}_b"] = x, m, wt, bias
        out[f"c{i}_y"] = y.data
    np.savez_compressed(os.path.join(OUT, "sparse_conv.npz"), **out)


def _unit_arrays(u):
    d = {"pre": np.asarray([int(u.pre_activation)])}
    for nm in ("conv1", "conv2", "conv3"):
        fb = getattr(u, nm)
        d[nm + "_w"], d[nm + "_b"] = fb.weights, fb.bias
    for nm in ("bn1", "bn2", "bn3"):
        bn = getattr(u, nm)
        d[nm + "_gamma"], d[nm + "_beta"] = bn.gamma, bn.beta
        d[nm + "_mean"], d[nm + "_var"] = bn.running_mean, bn.running_var
    return d


def gen_residual(bc):
    rng = np.random.default_rng(5000)
    out = {}
    for i in range(24):
        n = int(rng.integers(1, 3))
        c = int(rng.integers(2, 9))
        m = int(rng.integers(2, 9))
        h = int(rng.integers(8, 41))
        w = int(rng.integers(8, 41))
        halo = [1, 1, 1, 2, 0][i % 5]
        bs = int(rng.integers(max(4, 2 * halo + 1), 17))
        pre = i % 4 != 3
        mk = _mask(rng, n, h, w, KINDS[i % len(KINDS)])
        x = rng.standard_normal((n, h, w, c)).astype(np.float32)
        u = bc.random_unit_params(rng, c, m, np.float32, pre_activation=pre)
        y = bc.sparse_residual_unit(bc.Tensor4D(x), bc.BinaryMask(mk), u, (bs, bs), halo=halo)
        out[f"c{i}_cfg"] = np.asarray([n, h, w, c, m, bs, halo, int(pre)], np.int64)
        out[f"c{i}_x"], out[f"c{i}_mask"], out[f"c{i}_y"] = x, mk, y.data
        for key, val in _unit_arrays(u).items():
            out[f"c{i}_{key}"] = val
    np.savez_compressed(os.path.join(OUT, "residual.npz"), **out)


def gen_masks(bc):
    out = {}
    for i, (dims, sp) in enumerate([((1, 8, 8), 0.75), ((2, 40, 30), 0.9), ((1, 64, 100), 0.5),
                                    ((1, 7, 13), 0.0), ((1, 9, 9), 1.0)]):
        out[f"tl{i}_cfg"] = np.asarray([*dims, int(round(sp * 1e6))])
        out[f"tl{i}"] = bc.synth_mask_topleft(dims, sp).data
    for i, (dims, sp, seed) in enumerate([((1, 64, 64), 0.9, 0), ((2, 50, 80), 0.75, 3),
                                          ((1, 100, 100), 0.8, 7)]):
        out[f"bl{i}_cfg"] = np.asarray([*dims, int(round(sp * 1e6)), seed])
        out[f"bl{i}"] = bc.synth_mask_blobs(dims, sp, seed).data
    # config-2 mask (400x400, 90% sparsity blob, seed 0): store the active-pixel count + index list
    m = bc.synth_mask_blobs((1, 400, 400), 0.9, 0)
    out["cfg2_mask_sum"] = np.asarray([int(m.data.sum())])
    out["cfg2_mask_packed"] = np.packbits(m.data.reshape(-1))
    np.savez_compressed(os.path.join(OUT, "masks.npz"), **out)


def gen_units(bc):
    """random_unit_params / build_stage draws for fixed seeds (pins the RNG order)."""
    out = {}
    for i, (seed, c, m, pre) in enumerate([(123, 5, 3, True), (7, 8, 4, False), (99, 64, 32, True)]):
        u = bc.random_unit_params(np.random.default_rng(seed), c, m, np.float32, pre_activation=pre)
        out[f"c{i}_cfg"] = np.asarray([seed, c, m, int(pre)])
        for key, val in _unit_arrays(u).items():
            out[f"c{i}_{key}"] = val
    st = bc.build_stage(bc.StageConfig(2, (4, 3, 6), (8, 8), 1, 2), np.random.default_rng(5))
    out["stage_proj_w"], out["stage_proj_b"] = st.projection.weights, st.projection.bias
    out["stage_u1_conv2_w"] = st.units[1].conv2.weights
    np.savez_compressed(os.path.join(OUT, "units.npz"), **out)


def gen_config1(bc):
    """BASELINE config 1: 64x64x16 fp32, 3x3 SAME, block 16, 12 of 25 blocks."""
    rng = np.random.default_rng(0)
    n, h, w, c = 1, 64, 64, 16
    p = bc.ConvParams((3, 3), (1, 1), bc.Padding.SAME, c)
    spec = bc.compute_block_spec((n, h, w, c), p, (16, 16))
    gy, gx = spec.grid_count
    chosen = np.sort(rng.permutation(gy * gx)[: (gy * gx) // 2])
    m = np.zeros((n, h, w), np.uint8)
    obh, obw = spec.out_block_size
    for lin in chosen:
        by, bx = divmod(int(lin), gx)
        m[0, min(by * obh + obh // 2, h - 1), min(bx * obw + obw // 2, w - 1)] = 1
    x = rng.standard_normal((n, h, w, c)).astype(np.float32)
    wt = rng.standard_normal((3, 3, c, c)).astype(np.float32)
    bias = rng.standard_normal(c).astype(np.float32)
    idx = bc.reduce_mask(bc.BinaryMask(m), spec)
    y = bc.sparse_conv2d(bc.Tensor4D(x), bc.BinaryMask(m), bc.FilterBank(wt, bias), p, (16, 16))
    np.savez_compressed(os.path.join(OUT, "config1.npz"), x=x, mask=m, w=wt, b=bias,
                        idx=idx.entries, y=y.data, chosen=chosen)


def gen_grads(bc):
    """Training path: gather_grad / scatter_grad (`blocks.py:162-204`),
    sparse_conv2d_grads (`layers.py:50-65`), sparse_residual_unit_grads (`layers.py:232-270`),
    TRAIN_STATS sparse_batch_norm (`layers.py:68-82`)."""
    rng = np.random.default_rng(6000)
    out = {}
    for i in range(20):  # gather_grad / scatter_grad
        n, h, w, c, co, k, s, same, b = _conv_case(rng)
        pad = bc.Padding.SAME if same else bc.Padding.VALID
        dims = (n, h, w, c)
        spec = bc.compute_block_spec(dims, bc.ConvParams(k, s, pad, co), b)
        m = _mask(rng, n, h, w, KINDS[i % len(KINDS)])
        idx = bc.reduce_mask(bc.BinaryMask(m), spec)
        dt = np.float64 if i % 3 == 2 else np.float32
        g = bc.gather(bc.Tensor4D(np.zeros(dims, dt)), idx, spec)
        gblk = rng.standard_normal((idx.count, *spec.block_size, c)).astype(dt)
        gg = bc.gather_grad(g.with_tensor(bc.Tensor4D(gblk)), spec, dims)
        gout = rng.standard_normal((n, *spec.out_size, c)).astype(dt)
        sg = bc.scatter_grad(bc.Tensor4D(gout), idx, spec)
        out[f"g{i}_cfg"] = np.asarray([h, w, *k, *s, int(same), *b, n, c], np.int64)
        out[f"g{i}_mask"], out[f"g{i}_idx"] = m, idx.entries
        out[f"g{i}_gblk"], out[f"g{i}_gather_grad"] = gblk, gg.data
        out[f"g{i}_gout"], out[f"g{i}_scatter_grad"] = gout, sg.tensor.data
    for i in range(12):  # sparse_conv2d_grads
        n, h, w, c, co, k, s, same, b = _conv_case(rng)
        h, w = min(h, 24), min(w, 24)
        b = (max(min(b[0], h + 4), k[0]), max(min(b[1], w + 4), k[1]))
        b = (k[0] + s[0] * ((b[0] - k[0]) // s[0]), k[1] + s[1] * ((b[1] - k[1]) // s[1]))
        pad = bc.Padding.SAME if same else bc.Padding.VALID
        p = bc.ConvParams(k, s, pad, co)
        m = _mask(rng, n, h, w, KINDS[i % len(KINDS)])
        dt = np.float64 if i % 2 else np.float32
        x = rng.standard_normal((n, h, w, c)).astype(dt)
        wt = rng.standard_normal((*k, c, co)).astype(dt)
        bias = rng.standard_normal(co).astype(dt)
        gout = rng.standard_normal((n, *p.out_size(h, w), co)).astype(dt)
        dx, dw, db = bc.sparse_conv2d_grads(bc.Tensor4D(x), bc.BinaryMask(m), bc.FilterBank(wt, bias), p, b,
                                            bc.Tensor4D(gout))
        out[f"v{i}_cfg"] = np.asarray([h, w, *k, *s, int(same), *b, n, c, co], np.int64)
        out[f"v{i}_x"], out[f"v{i}_mask"], out[f"v{i}_w"], out[f"v{i}_b"] = x, m, wt, bias
        out[f"v{i}_gout"], out[f"v{i}_dx"], out[f"v{i}_dw"], out[f"v{i}_db"] = gout, dx.data, dw, db
    for i in range(10):  # sparse_residual_unit_grads (pre-activation)
        n = int(rng.integers(1, 3))
        c = int(rng.integers(2, 7))
        m_ = int(rng.integers(2, 7))
        h = int(rng.integers(8, 30))
        w = int(rng.integers(8, 30))
        halo = [1, 1, 2][i % 3]
        bs = int(rng.integers(2 * halo + 2, 13))
        mk = _mask(rng, n, h, w, KINDS[i % len(KINDS)])
        dt = np.float64 if i % 2 else np.float32
        x = rng.standard_normal((n, h, w, c)).astype(dt)
        u = bc.random_unit_params(rng, c, m_, dt)
        gout = rng.standard_normal((n, h, w, c)).astype(dt)
        dx, dws = bc.sparse_residual_unit_grads(bc.Tensor4D(x), bc.BinaryMask(mk), u, (bs, bs),
                                                bc.Tensor4D(gout), halo=halo)
        out[f"u{i}_cfg"] = np.asarray([n, h, w, c, m_, bs, halo, 1], np.int64)
        out[f"u{i}_x"], out[f"u{i}_mask"], out[f"u{i}_gout"], out[f"u{i}_dx"] = x, mk, gout, dx.data
        for nm in ("conv1", "conv2", "conv3"):
            out[f"u{i}_d{nm}_w"], out[f"u{i}_d{nm}_b"] = dws[nm]
        for key, val in _unit_arrays(u).items():
            out[f"u{i}_{key}"] = val
    for i in range(4):  # TRAIN_STATS sparse batch norm over gathered blocks
        n, h, w, c = 1, int(rng.integers(10, 30)), int(rng.integers(10, 30)), int(rng.integers(1, 6))
        spec = bc.compute_block_spec((n, h, w, c), bc.ConvParams((3, 3), (1, 1), bc.Padding.SAME, c), (6, 6))
        m = _mask(rng, n, h, w, "0.5")
        idx = bc.reduce_mask(bc.BinaryMask(m), spec)
        x = rng.standard_normal((n, h, w, c))
        blocks = bc.gather(bc.Tensor4D(x), idx, spec)
        gam, bet = rng.random(c) + 0.5, rng.standard_normal(c)
        bn = bc.BnParams(gam, bet, np.zeros(c), np.ones(c))
        if idx.count == 0:
            continue
        y, (mean, var) = bc.sparse_batch_norm(blocks, bn, bc.BnMode.TRAIN_STATS)
        out[f"b{i}_stack"], out[f"b{i}_gamma"], out[f"b{i}_beta"] = blocks.tensor.data, gam, bet
        out[f"b{i}_y"], out[f"b{i}_mean"], out[f"b{i}_var"] = y.tensor.data, mean, var
    np.savez_compressed(os.path.join(OUT, "grads.npz"), **out)


def gen_formats(bc):
    """Reference-written SBT4 / SBMK files and a saved backbone manifest, as raw bytes, so
    the package's readers/writers are pinned to the reference's on-disk formats."""
    import tempfile
    rng = np.random.default_rng(7000)
    out = {}
    with tempfile.TemporaryDirectory() as d:
        t32 = bc.Tensor4D(rng.standard_normal((2, 3, 5, 4)).astype(np.float32))
        t64 = bc.transpose_layout(bc.Tensor4D(rng.standard_normal((1, 4, 3, 6))))
        for nm, t in (("f32", t32), ("f64cf", t64)):
            fp = os.path.join(d, nm + ".sbt4")
            bc.save_sbt4(fp, t)
            out[f"sbt4_{nm}_bytes"] = np.frombuffer(open(fp, "rb").read(), np.uint8)
            out[f"sbt4_{nm}_data"] = t.data
            out[f"sbt4_{nm}_layout"] = np.asarray([t.layout.value])
        m = bc.synth_mask_blobs((2, 20, 30), 0.7, 3)
        fp = os.path.join(d, "m.sbmk")
        bc.save_sbmk(fp, m)
        out["sbmk_bytes"] = np.frombuffer(open(fp, "rb").read(), np.uint8)
        out["sbmk_data"] = m.data
        cfgs = [bc.StageConfig(1, (4, 3, 6), (8, 8), 1, 2), bc.StageConfig(2, (6, 4, 6), (6, 6), 2, 1)]
        bb = bc.build_backbone(cfgs, np.random.default_rng(11))
        bd = os.path.join(d, "bb")
        bc.save_backbone(bd, bb)
        names = sorted(os.listdir(bd))
        out["bb_names"] = np.asarray(names)
        for i, nm in enumerate(names):
            out[f"bb_file{i}"] = np.frombuffer(open(os.path.join(bd, nm), "rb").read(), np.uint8)
    np.savez_compressed(os.path.join(OUT, "formats.npz"), **out)


BACKBONE_SEED = 2024
BACKBONE_DIMS = (2, 80, 64, 32)  # reduced-H*W config 4 (800x700 -> 80x64, N=8 -> 2)
# the package's config-4 detector (paper_1801_02108_b200/perf.py DETECTOR_STAGES): the paper's
# [3, 6, 6, 3] units, [96, 192, 256, 384] channels, m = c/2, blocks (16, 16, 10, 6)
DETECTOR_STAGES = [
    (3, (32, 48, 96), (16, 16), 2, 2),
    (6, (96, 96, 192), (16, 16), 4, 2),
    (6, (192, 128, 256), (10, 10), 8, 2),
    (3, (256, 192, 384), (6, 6), 16, 2),
]


def gen_backbone(bc):
    """Configs 4/5 at reduced H x W: the reference ``run_backbone`` over the detector's
    four stages (``perf.DETECTOR_STAGES`` channel chain, block sizes and mask scales,
    3/6/6/3 units) on a partial blob mask (seed = frame index, as config 5).  Weights are
    re-derived from ``BACKBONE_SEED`` (draw order pinned by units.npz), so only the inputs,
    the masks and the per-stage outputs / index lists are stored."""
    from blockconv.cli import DEMO_INPUT, DEMO_STAGES
    out = {}
    for tag, stages, dims, seed, sp in (("det", DETECTOR_STAGES, BACKBONE_DIMS, BACKBONE_SEED, 0.75),
                                        ("demo", DEMO_STAGES, DEMO_INPUT, 7, 0.8)):
        n, h, w, c = dims
        cfgs = [bc.StageConfig(u, ch, bs, sc, st) for u, ch, bs, sc, st in stages]
        bb = bc.build_backbone(cfgs, np.random.default_rng(seed))
        x = np.random.default_rng(seed + 1).standard_normal((n, h, w, c)).astype(np.float32)
        mask = np.concatenate([bc.synth_mask_blobs((1, h, w), sp, i).data for i in range(n)])
        res = bc.run_backbone(bb, bc.Tensor4D(x), bc.BinaryMask(mask))
        out[f"{tag}_cfg"] = np.asarray([n, h, w, c, seed])
        out[f"{tag}_stages"] = np.asarray([[u, *ch, *bs, sc, st] for u, ch, bs, sc, st in stages])
        out[f"{tag}_x"], out[f"{tag}_mask"] = x, mask
        for i, r in enumerate(res):
            out[f"{tag}_s{i}_y"] = r.output.data
            out[f"{tag}_s{i}_mask"] = r.mask.data
            out[f"{tag}_s{i}_idx"] = r.indices.entries
    np.savez_compressed(os.path.join(OUT, "backbone.npz"), **out)


def main():
    bc = _ref()
    only = set(sys.argv[1:])
    os.makedirs(OUT, exist_ok=True)
    for fn in (gen_geometry, gen_reduce_mask, gen_gather_scatter, gen_sparse_conv, gen_residual,
               gen_masks, gen_units, gen_config1, gen_grads, gen_formats, gen_backbone):
        if only and fn.__name__ not in only:
            continue
        fn(bc)
        print("wrote", fn.__name__)


if __name__ == "__main__":
    main()
