"""Pin the CPU oracle (oracle/sbnet_oracle.py) against the golden vectors produced by the
real reference, and — when /root/reference is present (build container only) — directly
against the reference on extra seeded cases.  CPU-only."""
import os
import sys

import numpy as np
import pytest

from golden_cases import backbone_case, cases, conv_cfg, load, unit_dict
from oracle import sbnet_oracle as O

REF_SRC = "/root/reference/pkg/src"


def test_geometry_matches_reference_rows():
    g = load("geometry")
    for r in g["rows"]:
        h, w, kh, kw, sh, sw, same, bh, bw = (int(v) for v in r[:9])
        geo = O.geometry(h, w, (kh, kw), (sh, sw), bool(same), (bh, bw))
        got = [*geo.overlap, *geo.in_stride, *geo.out_block, *geo.origin, *geo.grid, *geo.out_size]
        assert got == [int(v) for v in r[9:]]
    for r in g["bad"]:
        with pytest.raises(ValueError):
            O.geometry(int(r[0]), int(r[1]), (r[2], r[3]), (r[4], r[5]), bool(r[6]), (r[7], r[8]))


def test_geometry_reference_kats():
    # reference tests/test_tiling.py:12-41
    g = O.geometry(32, 32, (3, 3), (2, 2), False, (5, 5))
    assert (g.overlap, g.in_stride, g.out_block) == ((1, 1), (4, 4), (2, 2))
    g = O.geometry(32, 32, (3, 3), (1, 1), False, (5, 5))
    assert (g.overlap, g.in_stride, g.out_block) == ((2, 2), (3, 3), (3, 3))
    g = O.geometry(8, 8, (3, 3), (1, 1), False, (3, 3))
    assert g.out_block == (1, 1) and g.in_stride == (1, 1)
    g = O.geometry(16, 16, (3, 3), (1, 1), True, (6, 6))
    assert g.origin == (-1, -1)


def test_reduce_mask_matches_reference_golden():
    npz = load("reduce_mask")
    for case in cases(npz, "c"):
        cfg = case["cfg"]
        h, w, k, s, same, b = conv_cfg(cfg)
        avg, thr = int(cfg[9]), int(cfg[10])
        geo = O.geometry(h, w, k, s, same, b)
        pool = "avg" if avg else "max"
        t = None if thr < 0 else thr / 1e6
        got = O.reduce_mask(case["mask"], geo, pool, t)
        assert got.tolist() == case["idx"].tolist()
        assert O.reduce_mask_scan(case["mask"], geo, pool, t).tolist() == case["idx"].tolist()


def test_downsample_matches_reference_golden():
    npz = load("reduce_mask")
    for case in cases(npz, "d"):
        assert np.array_equal(O.downsample_mask(case["mask"], int(case["f"][0])), case["out"])


def test_gather_scatter_match_reference_golden_bit_exact():
    npz = load("gather_scatter")
    for case in cases(npz):
        h, w, k, s, same, b = conv_cfg(case["cfg"])
        geo = O.geometry(h, w, k, s, same, b)
        idx = case["idx"]
        x = case["x"]
        assert np.array_equal(O.gather(x, idx, geo), case["gather"])
        assert np.array_equal(O.gather_transpose(x, idx, geo), case["gather_t"])
        assert np.array_equal(O.in_bounds_map(idx, geo), case["inb"])
        assert np.array_equal(O.scatter(case["blk"], idx, geo, case["dst"]), case["scatter"])
        assert np.array_equal(O.scatter(case["blk"], idx, geo, case["dst"], add=True),
                              case["scatter_add"])
        blk_cf = np.ascontiguousarray(case["blk"].transpose(0, 3, 1, 2))
        assert np.array_equal(O.scatter_transpose(blk_cf, idx, geo, case["dst"]), case["scatter_t"])


def test_sparse_conv_matches_reference_golden():
    npz = load("sparse_conv")
    for case in cases(npz):
        h, w, k, s, same, b = conv_cfg(case["cfg"])
        y = O.sparse_conv2d(case["x"], case["mask"], case["w"], case["b"], s, same, b)
        assert y.shape == case["y"].shape
        assert O.rel_err(y, case["y"]) <= 1e-6


def test_residual_unit_matches_reference_golden():
    npz = load("residual")
    for case in cases(npz):
        n, h, w, c, m, bs, halo, pre = (int(v) for v in case["cfg"])
        y = O.sparse_residual_unit(case["x"], case["mask"], unit_dict(case), (bs, bs), halo)
        assert O.rel_err(y, case["y"]) <= 1e-6


def test_config1_golden():
    z = load("config1")
    geo = O.geometry(64, 64, (3, 3), (1, 1), True, (16, 16))
    idx = O.reduce_mask(z["mask"], geo)
    assert idx.tolist() == z["idx"].tolist()
    assert len(idx) == 12
    y = O.sparse_conv2d(z["x"], z["mask"], z["w"], z["b"], (1, 1), True, (16, 16))
    assert O.rel_err(y, z["y"]) <= 1e-6


@pytest.mark.parametrize("tag", ["det", "demo"])
def test_backbone_matches_reference_golden(tag):
    """Configs 4/5 pinned: the oracle's run_backbone (weights re-drawn from the stored seed
    in the reference's RNG order) reproduces the reference's per-stage outputs, masks and
    index lists on a partial mask."""
    cfg, stages, x, mask, res = backbone_case(tag)
    rng = np.random.default_rng(int(cfg[4]))
    sts = [O.build_stage(rng, int(u), (int(a), int(b), int(c)), (int(bh), int(bw)), int(sc), int(st))
           for u, a, b, c, bh, bw, sc, st in stages]
    out = O.run_backbone(sts, x, mask)
    for (y, m, idx), (gy, gm, gidx) in zip(out, res):
        assert np.array_equal(m, gm)
        assert idx.tolist() == gidx.tolist()
        assert O.rel_err(y, gy) <= 1e-5


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference only in the build container")
def test_oracle_vs_live_reference_random():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import blockconv as bc
    from blockconv.verify import random_mask
    rng = np.random.default_rng(77)
    for r in range(20):
        n, h, w, c = 1, int(rng.integers(10, 40)), int(rng.integers(10, 40)), int(rng.integers(1, 6))
        mk = random_mask(rng, n, h, w, ["0.25", "0.5", "full", "single"][r % 4])
        x = rng.standard_normal((n, h, w, c)).astype(np.float32)
        u = bc.random_unit_params(rng, c, 3)
        bs = int(rng.integers(4, 12))
        ref = bc.sparse_residual_unit(bc.Tensor4D(x), mk, u, (bs, bs)).data
        ud = {"pre": True}
        for i, (cv, bn) in enumerate(((u.conv1, u.bn1), (u.conv2, u.bn2), (u.conv3, u.bn3)), 1):
            ud[f"w{i}"], ud[f"b{i}"] = cv.weights, cv.bias
            ud[f"bn{i}"] = dict(gamma=bn.gamma, beta=bn.beta, mean=bn.running_mean,
                                var=bn.running_var, eps=bn.epsilon)
        got = O.sparse_residual_unit(x, mk.data, ud, (bs, bs))
        assert O.rel_err(got, ref) <= 1e-6


# ----------------------------------------------------------------------------- training path

def _geo(cfg):
    h, w, k, s, same, b = conv_cfg(cfg)
    return O.geometry(h, w, k, s, same, b)


def test_gather_scatter_grad_match_reference_golden():
    z = load("grads")
    for cs in cases(z, "g"):
        g = _geo(cs["cfg"])
        n, c = int(cs["cfg"][9]), int(cs["cfg"][10])
        idx = cs["idx"]
        assert np.array_equal(O.reduce_mask(cs["mask"], g), idx)
        dims = (n, *g.in_size, c)
        gg = O.gather_grad(cs["gblk"], idx, g, dims)
        assert gg.dtype == cs["gather_grad"].dtype and np.array_equal(gg, cs["gather_grad"])
        assert np.array_equal(O.scatter_grad(cs["gout"], idx, g), cs["scatter_grad"])


def test_sparse_conv2d_grads_match_reference_golden():
    z = load("grads")
    for cs in cases(z, "v"):
        h, w, k, s, same, b = conv_cfg(cs["cfg"])
        dx, dw, db = O.sparse_conv2d_grads(cs["x"], cs["mask"], cs["w"], cs["b"], s, same, b, cs["gout"])
        tol = 1e-12 if cs["x"].dtype == np.float64 else 1e-5
        for got, ref in ((dx, cs["dx"]), (dw, cs["dw"]), (db, cs["db"])):
            assert O.rel_err(got, ref) <= tol


def _unit_from(cs):
    u = {"pre": True}
    for i in (1, 2, 3):
        u[f"w{i}"], u[f"b{i}"] = cs[f"conv{i}_w"], cs[f"conv{i}_b"]
        u[f"bn{i}"] = {"gamma": cs[f"bn{i}_gamma"], "beta": cs[f"bn{i}_beta"], "mean": cs[f"bn{i}_mean"],
                       "var": cs[f"bn{i}_var"], "eps": 1e-5}
    return u


def test_sparse_residual_unit_grads_match_reference_golden():
    z = load("grads")
    for cs in cases(z, "u"):
        n, h, w, c, m, bs, halo, _ = (int(v) for v in cs["cfg"])
        dx, dws = O.sparse_residual_unit_grads(cs["x"], cs["mask"], _unit_from(cs), (bs, bs), cs["gout"], halo)
        tol = 1e-12 if cs["x"].dtype == np.float64 else 1e-5
        assert O.rel_err(dx, cs["dx"]) <= tol
        for nm in ("conv1", "conv2", "conv3"):
            assert O.rel_err(dws[nm][0], cs[f"d{nm}_w"]) <= tol
            assert O.rel_err(dws[nm][1], cs[f"d{nm}_b"]) <= tol


def test_sparse_batch_norm_train_matches_reference_golden():
    z = load("grads")
    for cs in cases(z, "b"):
        y, mean, var = O.sparse_batch_norm_train(cs["stack"], cs["gamma"], cs["beta"])
        assert O.rel_err(y, cs["y"]) <= 1e-12
        assert O.rel_err(mean, cs["mean"]) <= 1e-12 and O.rel_err(var, cs["var"]) <= 1e-12
