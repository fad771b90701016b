"""The CLI commands (reference `tests/test_cli.py`) on the GPU package."""
import numpy as np
import pytest

from paper_1801_02108_b200 import load_sbmk, read_csv
from paper_1801_02108_b200.cli import main

pytestmark = pytest.mark.gpu


def test_verify_small_run_exits_zero(cuda_device, capsys):
    assert main(["verify", "--rounds", "3", "--seed", "2"]) == 0
    out = capsys.readouterr().out
    assert out.count("PASS") == 6 and "FAIL" not in out


def test_verify_broken_halo_exits_one(cuda_device, capsys):
    assert main(["verify", "--rounds", "3", "--seed", "2", "--halo", "0"]) == 1
    assert "dense-equivalence/residual-unit" in capsys.readouterr().err


def test_maskgen_and_bench_csv(cuda_device, tmp_path, capsys):
    mp = tmp_path / "m.sbmk"
    assert main(["maskgen", "--dims", "1,48,48", "--sparsity", "0.75", "--out", str(mp)]) == 0
    assert int(load_sbmk(mp).data.sum()) == 576
    out = tmp_path / "bench.csv"
    assert main(["bench", "--dims", "1,48,48,8", "--block", "8,8", "--mask", str(mp), "--warmup", "2",
                 "--iters", "4", "--out", str(out)]) == 0
    rows = read_csv(out)
    assert [r.config for r in rows] == ["conv-dense", "conv-sparse"] and rows[0].speedup == 1.0
    out2 = tmp_path / "unit.csv"
    assert main(["bench", "--dims", "1,64,64,64", "--block", "16,16", "--op", "unit", "--dtype", "bfloat16",
                 "--warmup", "2", "--iters", "4", "--out", str(out2)]) == 0
    assert [r.config for r in read_csv(out2)] == ["unit-dense", "unit-sparse"]


def test_sweep_and_demo_check(cuda_device, tmp_path, capsys):
    assert main(["sweep", "--dims", "1,64,64,8", "--candidates", "8,16", "--warmup", "1", "--iters", "2"]) == 0
    assert "chosen block size" in capsys.readouterr().out
    assert main(["demo", "--check", "--iters", "1", "--warmup", "1"]) == 0
    assert capsys.readouterr().out.count("PASS") == 4


def test_bad_arguments_exit_codes(capsys):
    assert main(["bench", "--dims", "1,2,3"]) == 2
    assert main(["maskgen", "--dims", "1,8,8", "--out", "/nonexistent/dir/m.sbmk"]) == 2


def test_verify_is_deterministic_per_seed(cuda_device, capsys):
    main(["verify", "--rounds", "3", "--seed", "7"])
    first = capsys.readouterr().out
    main(["verify", "--rounds", "3", "--seed", "7"])
    assert capsys.readouterr().out == first


def test_bench_sparsity_zero_and_missing_mask(cuda_device, tmp_path, capsys):
    out = tmp_path / "b.csv"
    assert main(["bench", "--dims", "1,48,48,8", "--block", "8,8", "--sparsity", "0", "--warmup", "2",
                 "--iters", "4", "--out", str(out)]) == 0
    rows = read_csv(out)
    assert rows[0].speedup == 1.0 and rows[1].flops_sparse >= rows[1].flops_dense  # halo overhead at sparsity 0
    assert main(["bench", "--dims", "1,16,16,2", "--block", "8,8", "--mask", "/nonexistent/m.sbmk",
                 "--warmup", "0", "--iters", "1"]) == 2
    assert "error:" in capsys.readouterr().err
