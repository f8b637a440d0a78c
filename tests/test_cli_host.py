"""CLI harness, file formats and seeded problems on CPU (no solves)."""

import os

import numpy as np
import pytest
from conftest import GOLDEN, golden

from paper_2605_00837_b200 import cli, fileio
from paper_2605_00837_b200.applications import Correspondence
from paper_2605_00837_b200.color import make_rgb_image
from paper_2605_00837_b200.errors import FileFormatError
from paper_2605_00837_b200.problems import generate_grid_problem, normalize_cost


def _rec(**kw):
    base = dict(experiment="bench", variant="log", n=3, m=4, epsilon=0.01, max_cost=None, seed=0, precision="single",
                tolerance=1e-6, max_iterations=10, check_interval=5, status="converged", iterations=5,
                marginal_error=1.2345678e-7, transport_cost=0.1, elapsed_ms=1.5, elapsed_std_ms=0.0, matrix_bytes=48,
                slowdown_vs_full=None, error_trace=((5, 1.2345678e-7),))
    base.update(kw)
    return cli.ExperimentRecord(**base)


def test_csv_and_json_round_trip():
    recs = [_rec(), _rec(variant="standard", max_cost=10.0, slowdown_vs_full=1.25, error_trace=())]
    assert cli.records_from_csv(cli.records_to_csv(recs)) == recs
    assert cli.records_from_json_lines(cli.records_to_json_lines(recs)) == recs
    assert cli.records_to_csv([]).strip().split(",") == cli.CSV_HEADER
    with pytest.raises(ValueError):
        cli.records_from_csv("a,b\n")


def test_reference_jsonl_parses():
    for name in ("cli_bench", "cli_stability", "cli_convergence"):
        with open(os.path.join(GOLDEN, name + ".jsonl")) as fh:
            recs = cli.records_from_json_lines(fh.read())
        assert recs and all(isinstance(r, cli.ExperimentRecord) for r in recs)


@pytest.mark.parametrize("argv", [["bench", "--n", "0"], ["bench", "--m", "0"], ["scale", "--n-list", ""],
                                  ["convergence", "--eps-list", ""], ["bench", "--parallel-experiments", "0"],
                                  ["color-transfer", "--source", "a", "--target", "b", "--out-image", "c",
                                   "--samples", "0"], ["nonsense"]])
def test_usage_errors_exit_2(argv):
    with pytest.raises(SystemExit) as e:
        cli.main(argv)
    assert e.value.code == 2


def test_grid_problems_match_reference():
    G = golden("cli_grid_problems")
    for (n, m, seed) in [(7, 5, 3), (1, 4, 2), (64, 64, 0)]:
        mu, nu, C = generate_grid_problem(n, m, seed)
        np.testing.assert_array_equal(mu.weights, G[f"mu_{n}_{m}_{seed}"])
        np.testing.assert_array_equal(nu.weights, G[f"nu_{n}_{m}_{seed}"])
        np.testing.assert_array_equal(C.values, G[f"C_{n}_{m}_{seed}"])
        np.testing.assert_array_equal(normalize_cost(C, 10.0).values, G[f"Cn_{n}_{m}_{seed}"])


def test_normalize_cost_validation():
    _, _, C = generate_grid_problem(4, 4, 0)
    with pytest.raises(ValueError):
        normalize_cost(C, 0.0)


def test_ppm_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    img = make_rgb_image(5, 3, rng.integers(0, 256, (15, 3)) / 255.0)
    p = tmp_path / "a.ppm"
    fileio.write_ppm(p, img)
    back = fileio.read_ppm(p)
    assert (back.width, back.height) == (5, 3)
    np.testing.assert_array_equal(back.pixels, img.pixels)
    raw = p.read_bytes().replace(b"P6\n", b"P6\n# comment\n", 1)
    q = tmp_path / "b.ppm"
    q.write_bytes(raw)
    np.testing.assert_array_equal(fileio.read_ppm(q).pixels, img.pixels)
    (tmp_path / "c.ppm").write_bytes(b"P5\n1 1\n255\n\x00")
    with pytest.raises(FileFormatError):
        fileio.read_ppm(tmp_path / "c.ppm")
    (tmp_path / "d.ppm").write_bytes(b"P6\n2 2\n255\n\x00\x00")
    with pytest.raises(FileFormatError):
        fileio.read_ppm(tmp_path / "d.ppm")


def test_point_cloud_and_correspondences_round_trip(tmp_path):
    pts = np.random.default_rng(1).standard_normal((6, 3))
    fileio.write_point_cloud(tmp_path / "p.txt", pts)
    np.testing.assert_array_equal(fileio.read_point_cloud(tmp_path / "p.txt"), pts)
    pairs = [Correspondence(0, 2, 0.125), Correspondence(1, 0, 1e-300)]
    fileio.write_correspondences(tmp_path / "c.txt", pairs)
    assert fileio.read_correspondences(tmp_path / "c.txt") == pairs
    (tmp_path / "bad.txt").write_text("1 2\n")
    with pytest.raises(FileFormatError):
        fileio.read_correspondences(tmp_path / "bad.txt")
    (tmp_path / "bad2.txt").write_text("1 2\n3\n")
    with pytest.raises(FileFormatError):
        fileio.read_point_cloud(tmp_path / "bad2.txt")
