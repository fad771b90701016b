"""CLI argument handling and the host-only maskgen command (no GPU needed); the exit-code
contract of the reference CLI (`cli.py:305-317`, tests/test_cli.py)."""
import numpy as np

from paper_1801_02108_b200 import load_sbmk
from paper_1801_02108_b200.cli import COMMANDS, build_parser, main


def test_usage_errors_exit_two(capsys):
    assert main(["bench", "--bogus"]) == 2
    assert main(["bench", "--dims", "1,2"]) == 2
    assert main(["sweep", "--dims", "0,8,8,8"]) == 2
    assert main([]) == 2


def test_commands_and_defaults_match_the_reference():
    assert set(COMMANDS) == {"verify", "bench", "sweep", "maskgen", "demo"}
    a = build_parser().parse_args(["bench"])
    assert (a.dims, a.block, a.sparsity, a.iters, a.warmup, a.op) == ((1, 400, 704, 32), (32, 32), 0.9, 15, 15, "conv")
    s = build_parser().parse_args(["sweep", "--candidates", "8x8;16x32"])
    assert s.candidates == [(8, 8), (16, 32)]
    assert build_parser().parse_args(["sweep", "--candidates", "8,16"]).candidates == [(8, 8), (16, 16)]
    d = build_parser().parse_args(["demo"])
    assert (d.iters, d.warmup, d.check) == (5, 2, False)


def test_maskgen_topleft_and_blob(tmp_path, capsys):
    out = tmp_path / "m.sbmk"
    assert main(["maskgen", "--dims", "1,8,8", "--sparsity", "0.75", "--out", str(out)]) == 0
    assert load_sbmk(out).dims == (1, 8, 8) and int(np.asarray(load_sbmk(out).numpy()).sum()) == 16
    a, b = tmp_path / "a.sbmk", tmp_path / "b.sbmk"
    for p in (a, b):
        main(["maskgen", "--dims", "1,64,64", "--kind", "blob", "--sparsity", "0.8", "--seed", "7", "--out", str(p)])
    assert a.read_bytes() == b.read_bytes()
    assert main(["maskgen", "--dims", "1,8,8", "--out", "/nonexistent/dir/m.sbmk"]) == 2
