"""The CLI harness on the GPU solvers against the reference CLI's own output
(tests/golden/make_golden_cli.py ran the same argv through the reference)."""

import contextlib
import io
import os

import numpy as np
import pytest
from conftest import GOLDEN

from paper_2605_00837_b200 import cli, fileio
from paper_2605_00837_b200.color import make_rgb_image

pytestmark = pytest.mark.gpu

ARGV = {
    "cli_bench": ["bench", "--n", "128", "--eps", "0.01", "--warmup", "0", "--repeats", "1", "--json"],
    "cli_bench_std": ["bench", "--n", "96", "--m", "80", "--eps", "0.05", "--domain", "standard", "--warmup", "0",
                      "--repeats", "1", "--json", "--max-cost", "2.0"],
    "cli_stability": ["stability", "--n", "64", "--eps-grid", "0.1,0.001", "--maxc-grid", "1,100",
                      "--max-iters", "300", "--json"],
    "cli_convergence": ["convergence", "--n-list", "128", "--eps-list", "0.1,0.01", "--max-iters", "2000", "--json"],
}


def run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(argv)
    return rc, cli.records_from_json_lines(buf.getvalue())


@pytest.mark.parametrize("name", sorted(ARGV))
def test_cli_matches_reference(cuda_ok, name):
    rc, got = run(ARGV[name])
    with open(os.path.join(GOLDEN, name + ".jsonl")) as fh:
        want = cli.records_from_json_lines(fh.read())
    assert rc == 0
    assert len(got) == len(want)
    for g, w in zip(got, want):
        for f in ("experiment", "variant", "n", "m", "epsilon", "max_cost", "seed", "precision", "tolerance",
                  "max_iterations", "check_interval", "status", "iterations", "matrix_bytes"):
            assert getattr(g, f) == getattr(w, f), (f, g, w)
        if w.status == "nan":
            assert np.isnan(g.transport_cost)
            continue
        # fp32 errors at eps = 1e-3 sit on the single-precision noise floor (~1e-6),
        # where the summation order moves them by a few 1e-7
        floor = 5e-7 if w.precision == "single" else 1e-12
        assert abs(g.marginal_error - w.marginal_error) <= floor + 0.05 * abs(w.marginal_error)
        assert abs(g.transport_cost - w.transport_cost) <= 1e-5 * abs(w.transport_cost) + 1e-9
        assert [k for k, _ in g.error_trace] == [k for k, _ in w.error_trace]


def test_cli_color_transfer_and_pointcloud(cuda_ok, tmp_path):
    rng = np.random.default_rng(3)
    src = make_rgb_image(16, 16, rng.uniform(0, 1, (256, 3)))
    tgt = make_rgb_image(16, 16, rng.uniform(0, 1, (256, 3)))
    fileio.write_ppm(tmp_path / "s.ppm", src)
    fileio.write_ppm(tmp_path / "t.ppm", tgt)
    rc, recs = run(["color-transfer", "--source", str(tmp_path / "s.ppm"), "--target", str(tmp_path / "t.ppm"),
                    "--out-image", str(tmp_path / "o.ppm"), "--samples", "64", "--eps", "0.05", "--json"])
    assert rc == 0 and recs[0].status == "converged" and recs[0].precision == "double"
    assert fileio.read_ppm(tmp_path / "o.ppm").pixels.shape == (256, 3)
    rc, recs = run(["pointcloud", "--n", "100", "--eps", "0.01", "--out-pairs", str(tmp_path / "p.txt"), "--json"])
    assert rc == 0 and recs[0].status in ("converged", "diverged")
    assert len(fileio.read_correspondences(tmp_path / "p.txt")) == 100


def test_cli_worker_count_invariance(cuda_ok):
    """Reference acceptance criterion 10 / test_cli.py:297-323: records are identical
    (except the two elapsed columns) for --parallel-experiments 1 and 4, and across runs."""
    argv = ["stability", "--n", "48", "--eps-grid", "0.1,0.01", "--maxc-grid", "1,10", "--max-iters", "200",
            "--json"]
    runs = [run(argv + ["--parallel-experiments", str(k)])[1] for k in (1, 4, 1)]
    strip = lambda recs: [{f: getattr(r, f) for f in cli.CSV_HEADER if not f.startswith("elapsed")} for r in recs]
    a, b, c = (strip(r) for r in runs)
    assert a == b == c
