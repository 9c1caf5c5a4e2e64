"""CLI and file formats against fixtures produced by
the reference's own CLI (tests/golden/cli/, make_golden.py cli_cases):
formats and exit codes on CPU, `simulate` / `compare` on the GPU."""

import os

import numpy as np
import pytest

from conftest import golden
from paper_2508_03065_b200 import cli, io_formats

HERE = os.path.dirname(os.path.abspath(__file__))
CLI_DIR = os.path.join(HERE, "golden", "cli")


def _config(tmp_path, extra=""):
    text = open(os.path.join(CLI_DIR, "run.cfg")).read().replace("{dir}", CLI_DIR) + extra
    p = tmp_path / "run.cfg"
    p.write_text(text)
    return str(p)


# ------------------------------------------------------------------ CPU
def test_trajectory_and_wav_roundtrip(tmp_path):
    tr = io_formats.read_trajectory(os.path.join(CLI_DIR, "path.txt"))
    assert tr.rate == 16000.0 and tr.positions.shape == (4000, 3)
    io_formats.write_trajectory(tmp_path / "p.txt", tr)
    assert (tmp_path / "p.txt").read_text() == open(os.path.join(CLI_DIR, "path.txt")).read()
    rate, x = io_formats.read_wav(os.path.join(CLI_DIR, "dry.wav"))
    io_formats.write_wav(tmp_path / "x.wav", rate, x)
    assert np.array_equal(io_formats.read_wav(tmp_path / "x.wav")[1], x)
    with pytest.raises(ValueError):
        io_formats.write_wav(tmp_path / "st.wav", rate, np.zeros((10, 2)))
    (tmp_path / "bad.txt").write_text("rate=1\n0 0 0\n")
    with pytest.raises(ValueError):
        io_formats.read_trajectory(tmp_path / "bad.txt")


def test_filter_files_and_default_design(tmp_path):
    f = io_formats.read_filter(io_formats.DEFAULT_FILTER_FILE)
    assert (f.poly_order, f.branch_len, f.passband) == (3, 8, 0.8)
    assert np.array_equal(f.branches, golden("kernels.npz")["design_3_8_08"])  # the reference's design
    io_formats.write_filter(tmp_path / "f.txt", f)
    g = io_formats.read_filter(tmp_path / "f.txt")
    assert np.array_equal(g.branches, f.branches) and g.nominal_delay == 3
    (tmp_path / "short.txt").write_text("3 8 0.8\n1 2 3\n")
    with pytest.raises(ValueError):
        io_formats.read_filter(tmp_path / "short.txt")


def test_config_table_keys(tmp_path):
    t = io_formats.parse_config_text("room.dims = 5 6 4  # comment\nmic.pos = 1 2 1\n"
                                     "synth.tiers = 2:1 5:32 8:256\nfd.kind = hann-sinc\n"
                                     "fd.L = 64\nsynth.precision = fp32\n")
    cfg = io_formats.engine_config_from_table(t)
    assert cfg.synth.tiers == ((2, 1), (5, 32), (8, 256)) and cfg.synth.max_order == 8
    assert cfg.filt.branch_len == 64 and cfg.synth.precision == "fp32"
    assert cfg.room.wall_reflection.tolist() == [0.9] * 6
    for bad in ("mic.pos = 1 2 1\n", "room.dims = 5 6 4\nmic.pos = 1 2 1\nroom.reflection = 1 2\n",
                "room.dims = 5 6 4\nmic.pos = 1 2 1\ntraj.kind = sine\n",
                "room.dims = 5 6 4\nmic.pos = 1 2 1\nfarrow.M = 2\n",
                "room.dims = 5 6 4\nmic.pos = 1 2 1\nfd.kind = lagrange\n", "novalue\n"):
        with pytest.raises(ValueError):
            io_formats.engine_config_from_table(io_formats.parse_config_text(bad))


def test_cli_exit_codes_and_cost(tmp_path, capsys):
    assert cli.main(["design", "--M", "3"]) == cli.EXIT_USAGE
    assert cli.main(["trajectory", "--out", "x"]) == cli.EXIT_USAGE
    assert cli.main(["simulate", "--config", str(tmp_path / "none.cfg"), "--in", "a.wav",
                     "--out", "b.wav"]) == cli.EXIT_IO
    (tmp_path / "bad.cfg").write_text("room.dims = 5 6 4\n")
    assert cli.main(["simulate", "--config", str(tmp_path / "bad.cfg"), "--in", "a.wav",
                     "--out", "b.wav"]) == cli.EXIT_USAGE
    capsys.readouterr()
    assert cli.main(["cost", "--room", "9 10 9", "--t60", "0.6"]) == 0
    lines = dict(l.split("=", 1) for l in capsys.readouterr().out.split())
    # values printed by the reference's `moverb cost --room "9 10 9" --t60 0.6`
    assert lines["images_total"] == "45057" and lines["hierarchical_evals"] == "337250"
    assert float(lines["reduction_ratio"]) == pytest.approx(2137.618977020015, rel=1e-15)


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["hierarchical", "oracle", "splice", "static"])
def test_simulate_matches_reference_cli(tmp_path, mode):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    out = tmp_path / f"{mode}.wav"
    argv = ["simulate", "--config", _config(tmp_path), "--mode", mode,
            "--in", os.path.join(CLI_DIR, "dry.wav"), "--out", str(out)]
    if mode == "splice":
        argv += ["--crossfade", "64"]
    if mode == "hierarchical":
        argv += ["--dump-image", "7", "--dump-csv", str(tmp_path / "image7.csv")]
    assert cli.main(argv) == 0
    _, y = io_formats.read_wav(out)
    _, ref = io_formats.read_wav(os.path.join(CLI_DIR, f"{mode}.wav"))
    assert y.size == ref.size
    # both engines compute in fp64 and write float32 WAVs: equal up to the
    # last float32 rounding
    assert np.max(np.abs(y - ref)) <= 1e-6 * np.max(np.abs(ref))
    if mode == "hierarchical":
        got = np.loadtxt(tmp_path / "image7.csv", delimiter=",", skiprows=1)
        want = np.loadtxt(os.path.join(CLI_DIR, "image7.csv"), delimiter=",", skiprows=1)
        assert got.shape == want.shape
        np.testing.assert_allclose(got, want, rtol=1e-11, atol=0)


@pytest.mark.gpu
def test_compare_matches_reference_cli(tmp_path, capsys):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    rep = tmp_path / "report.txt"
    assert cli.main(["compare", os.path.join(CLI_DIR, "hierarchical.wav"),
                     os.path.join(CLI_DIR, "oracle.wav"), "--report", str(rep),
                     "--csv", str(tmp_path / "c.csv")]) == 0
    got = io_formats.read_report(rep)
    want = io_formats.read_report(os.path.join(CLI_DIR, "report.txt"))
    assert set(got) == set(want)
    for k in want:
        assert float(got[k]) == pytest.approx(float(want[k]), rel=1e-6, abs=1e-6)
    csv = np.loadtxt(tmp_path / "c.csv", delimiter=",", skiprows=1)
    assert csv.shape[0] == io_formats.read_wav(os.path.join(CLI_DIR, "hierarchical.wav"))[1].size
