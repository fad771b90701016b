"""On-disk formats (SBT4, SBMK, weights manifest) pinned byte-for-byte to files written by
the reference (tests/golden/formats.npz, oracle/make_golden.py gen_formats).  CPU-only."""
import json
import os

import numpy as np
import pytest
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200 import formats as F
from golden_cases import load


def _write(path, arr):
    with open(path, "wb") as f:
        f.write(arr.tobytes())


@pytest.mark.parametrize("nm", ["f32", "f64cf"])
def test_sbt4_reads_and_writes_reference_bytes(tmp_path, nm):
    z = load("formats")
    src = tmp_path / "in.sbt4"
    _write(src, z[f"sbt4_{nm}_bytes"])
    t = F.load_sbt4(src)
    assert t.layout.value == int(z[f"sbt4_{nm}_layout"][0])
    assert np.array_equal(t.data.numpy(), z[f"sbt4_{nm}_data"])
    dst = tmp_path / "out.sbt4"
    F.save_sbt4(dst, t)
    assert dst.read_bytes() == src.read_bytes()


def test_sbt4_bf16_round_trip_and_errors(tmp_path):
    t = P.Tensor4D(torch.randn(1, 3, 4, 8).bfloat16())
    F.save_sbt4(tmp_path / "b.sbt4", t)
    back = F.load_sbt4(tmp_path / "b.sbt4")
    assert back.dtype == torch.bfloat16 and torch.equal(back.data, t.data)
    raw = (tmp_path / "b.sbt4").read_bytes()
    for bad, off in ((b"XXXX" + raw[4:], 0), (raw[:4] + b"\x02" + raw[5:], 4), (raw[:10], 10),
                     (raw[:-2], len(raw) - 2)):
        (tmp_path / "bad.sbt4").write_bytes(bad)
        with pytest.raises(P.FormatError) as e:
            F.load_sbt4(tmp_path / "bad.sbt4")
        assert e.value.offset == off


def test_sbmk_reads_and_writes_reference_bytes(tmp_path):
    z = load("formats")
    src = tmp_path / "m.sbmk"
    _write(src, z["sbmk_bytes"])
    m = F.load_sbmk(src)
    assert np.array_equal(m.data.numpy(), z["sbmk_data"])
    F.save_sbmk(tmp_path / "o.sbmk", m)
    assert (tmp_path / "o.sbmk").read_bytes() == src.read_bytes()
    bad = bytearray(src.read_bytes())
    bad[F.SBMK_HEADER.size + 3] = 7
    (tmp_path / "b.sbmk").write_bytes(bytes(bad))
    with pytest.raises(P.FormatError) as e:
        F.load_sbmk(tmp_path / "b.sbmk")
    assert e.value.offset == F.SBMK_HEADER.size + 3


def test_backbone_manifest_interchange(tmp_path):
    z = load("formats")
    ref_dir = tmp_path / "ref"
    ref_dir.mkdir()
    names = [str(n) for n in z["bb_names"]]
    for i, nm in enumerate(names):
        _write(ref_dir / nm, z[f"bb_file{i}"])
    bb = F.load_backbone(ref_dir)
    assert [s.config.channels for s in bb.stages] == [(4, 3, 6), (6, 4, 6)]
    out_dir = tmp_path / "ours"
    F.save_backbone(out_dir, bb)
    assert sorted(os.listdir(out_dir)) == names
    for nm in names:
        a, b = (ref_dir / nm).read_bytes(), (out_dir / nm).read_bytes()
        if nm == "manifest.json":
            assert json.loads(a) == json.loads(b)
        else:
            assert a == b, nm
