"""The reference CLI's commands (proj/tools/gridgnn_main.cpp) as the native
`paper_2604_02651_b200/gridgnn` binary: `gen` on the CPU
byte-identical to the reference's writers, option / config-file handling and
usage errors on the CPU; `train`, `verify` and `sample-stats` on a B200."""
import csv
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2604_02651_b200", "gridgnn")


@pytest.fixture(scope="module")
def cli():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2604_02651_b200")], check=True)
    assert os.path.exists(BIN)
    return BIN


def _run(cli, *args, cwd=None, timeout=600):
    return subprocess.run([cli, *map(str, args)], capture_output=True, text=True, cwd=cwd, timeout=timeout)


def test_gen_is_byte_identical_to_reference(cli, ref, tmp_path):
    r = _run(cli, "gen", "--n", 500, "--avg-degree", 7, "--d-in", 9, "--classes", 5, "--data-seed", 3,
             "--out", tmp_path / "mine")
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == f"wrote {tmp_path / 'mine'}.{{edges,sgnf,sgnl,sgns}}: n=500 d_in=9 classes=5"
    theirs = [tmp_path / f"ref.{e}" for e in ("edges", "sgnf", "sgnl", "sgns")]
    ref.save_synthetic(500, 7.0, 9, 5, 3, *theirs)
    for t in theirs:
        assert (tmp_path / f"mine.{t.suffix[1:]}").read_bytes() == t.read_bytes(), t.suffix


def test_config_file_and_command_line_override(cli, tmp_path):
    cfg = tmp_path / "run.cfg"
    cfg.write_text("# gen settings\nn = 64\nd-in = 3\nclasses = 2\nout = " + str(tmp_path / "cfg") + "\n")
    r = _run(cli, "gen", "--config", cfg, "--classes", 6)
    assert r.returncode == 0, r.stderr
    assert "n=64 d_in=3 classes=6" in r.stdout
    assert (tmp_path / "cfg.sgnl").exists()


@pytest.mark.parametrize("args,code,msg", [
    ([], 106, "Subcommands"),
    (["fly"], 109, "not expected: fly"),
    (["train", "--bogus", "1"], 105, "not expected: --bogus"),
    (["gen", "--n", "abc"], 105, "not a number"),
    (["train", "--edges", "/nonexistent/g.edges"], 105, "File does not exist"),
    (["gen", "--draws", "5"], 105, "not expected: --draws"),
    (["train", "--dropout", "1.5"], 105, "[0, 1)"),
    (["train", "--optimizer", "lbfgs"], 105, "adam or sgd"),
])
def test_usage_errors(cli, args, code, msg):
    r = _run(cli, *args)
    assert r.returncode == code, (r.returncode, r.stdout, r.stderr)
    assert msg in r.stdout + r.stderr


@pytest.mark.gpu
def test_train_writes_the_reference_metrics_csv(cli, tmp_path):
    out = tmp_path / "m.csv"
    r = _run(cli, "train", "--n", 600, "--avg-degree", 8, "--d-in", 16, "--classes", 4, "--epochs", 3,
             "--layers", 3, "--hidden-dim", 32, "--prefetch", "--out", out)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == f"wrote {out} (3 epochs)"
    assert lines[1].startswith("final: train_acc=") and lines[2].startswith("comm bytes: x=0 y=0 z=0 d=0")
    rows = list(csv.reader(open(out)))
    assert rows[0] == ["epoch", "step", "loss", "train_acc", "val_acc", "test_acc", "t_sample_ms", "t_fwd_ms",
                       "t_bwd_ms", "t_dpsync_ms", "bytes_x", "bytes_y", "bytes_z", "bytes_d"]
    assert [int(r[0]) for r in rows[1:]] == [1, 2, 3] and [int(r[1]) for r in rows[1:]] == [4, 8, 12]


@pytest.mark.gpu
def test_verify_passes_and_perturb_fails(cli):
    r = _run(cli, "verify")
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") == 3
    r = _run(cli, "verify", "--perturb", 5.0)
    assert r.returncode == 1 and "FAIL" in r.stdout and "1 check(s) failed" in r.stdout, r.stdout


@pytest.mark.gpu
def test_sample_stats_inclusion_and_unbiased_aggregation(cli):
    r = _run(cli, "sample-stats", "--n", 200, "--avg-degree", 6, "--draws", 4000)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == "n=200 B=50 draws=4000"
    freq = float(lines[1].rsplit(" ", 1)[1])
    bias = float(lines[2].split("conditional mean ")[1].split()[0])
    # uniform inclusion at B/N; the 1/p rescaling makes the conditional mean
    # of the aggregation unbiased (Monte Carlo error only)
    assert freq < 0.2 and bias < 0.2, r.stdout


@pytest.mark.gpu
def test_verify_sharded_grid_in_one_process(cli):
    """The reference runs every rank of a grid on threads of one process; so
    does the CLI, one thread per GPU (NCCL between the threads' contexts)."""
    try:
        import torch
        n = torch.cuda.device_count()
    except Exception:
        n = 0
    if n < 2:
        pytest.skip("needs 2 GPUs")
    for grid in ("1x2x1x1", "2x1x1x1"):
        r = _run(cli, "verify", "--grid", grid)
        assert r.returncode == 0, r.stdout + r.stderr
        assert r.stdout.count("PASS") == 3, r.stdout
