"""Report layer and CLI (pkg/tests/test_bench_cli.py against the B200
backend).  CPU tests cover the named configs, schedules, CSV/JSON identity,
schemas and every usage-error path (they fail before any device work); the
GPU tests run real integrations through run_report / sweep / the CLI."""
import json
import subprocess
import sys

import jsonschema
import pytest

from paper_2408_09229_b200 import bench, cli
from paper_2408_09229_b200.errors import ContractViolationError, IntegrationError
from paper_2408_09229_b200.integrands import lookup


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2408_09229_b200", *args],
                          capture_output=True, text=True, timeout=600)


# ------------------------------------------------------------------- CPU --

def test_named_configs_match_published_table():
    d = bench.NAMED_CONFIGS["def"]
    assert (d["n_intervals"], d["alpha"], d["beta"]) == (1024, 0.5, 0.75)
    v = bench.NAMED_CONFIGS["vf"]
    assert (v["n_intervals"], v["alpha"], v["beta"]) == (50, 1.5, 0.75)
    t = bench.NAMED_CONFIGS["tq"]
    assert t["n_intervals"] is None and t["alpha"] == 0.5
    for c in bench.NAMED_CONFIGS.values():
        assert c["max_it"] == 20 and c["skip"] == 0 and c["batch_size"] == 1_048_576


def test_tq_intervals_computed_from_n_eval():
    n1, n2 = bench.tq_n_intervals(10 ** 6, 2), bench.tq_n_intervals(10 ** 8, 2)
    assert 10 <= n1 < n2 <= 1024


def test_resolve_config_applies_overrides():
    cfg = bench.resolve_config(lookup("linear"), 10_000, "def", seed=5, workers=2, max_it=7,
                               skip=None)
    assert (cfg.seed, cfg.workers, cfg.max_it, cfg.skip, cfg.n_intervals) == (5, 2, 7, 0, 1024)
    with pytest.raises(ContractViolationError):
        bench.resolve_config(lookup("linear"), 10_000, "bogus")
    assert bench.resolve_config(lookup("sinexp"), 10_000, "tq").n_intervals == \
        bench.tq_n_intervals(10_000, 2)


def test_doubling_schedule():
    assert bench.doubling_schedule(1000, 8000) == [1000, 2000, 4000, 8000]
    assert bench.doubling_schedule(1000, 7999) == [1000, 2000, 4000]
    assert bench.doubling_schedule(5, 5) == [5]
    with pytest.raises(ContractViolationError):
        bench.doubling_schedule(0, 100)


def _synthetic_rows():
    rows = []
    for n, w, wall in ((2000, 1, 10.0), (2000, 2, 6.0), (4000, 1, 19.5)):
        rows.append(dict(integrand="sinexp", config="def", dims=2, n_eval=n, workers=w,
                         repeats=1, mean=2.1779795225 + n * 1e-9, sigma=1.0 / n,
                         rel_stderr=0.1 / n, chi2_dof=0.93, wall_ms=wall, fill_fraction=0.71,
                         speedup=None if n == 4000 else 10.0 / wall,
                         efficiency=None if n == 4000 else 10.0 / wall / w))
    return rows


def test_csv_and_json_carry_identical_values():
    rows = _synthetic_rows()
    jsonschema.validate(bench.sweep_report(rows), bench.SWEEP_REPORT_SCHEMA)
    parsed = bench.csv_to_rows(bench.rows_to_csv(rows))
    assert parsed == json.loads(json.dumps(bench.sweep_report(rows)))["rows"] == rows
    with pytest.raises(ContractViolationError):
        bench.csv_to_rows("a,b\n1,2\n")


def test_run_schema_rejects_bad_reports():
    rep = {"schema": 1, "kind": "run", "integrand": "x", "dims": 2, "config": "def",
           "params": {k: 1 for k in ("n_eval", "max_it", "skip", "batch_size", "n_intervals",
                                     "alpha", "beta", "seed", "workers")},
           "iterations": [{"index": 1, "estimate": 1.0, "sigma": 0.1, "included": True}],
           "mean": 1.0, "sigma": 0.1, "chi2_dof": 0.0, "wall_ms": 1.0,
           "phases": {k: 20.0 for k in ("init", "map", "fill", "update", "clear")},
           "fill_fraction": 0.2}
    jsonschema.validate(rep, bench.RUN_REPORT_SCHEMA)
    for key, bad in (("config", "zz"), ("fill_fraction", 1.5), ("sigma", -1.0)):
        with pytest.raises(jsonschema.ValidationError):
            jsonschema.validate(dict(rep, **{key: bad}), bench.RUN_REPORT_SCHEMA)


def test_cli_unknown_integrand_usage_error():
    res = _cli("run", "--integrand", "nope", "--n-eval", "1000")
    assert res.returncode == 2 and "available" in res.stderr


def test_cli_invalid_combination_usage_error():
    res = _cli("run", "--integrand", "sinexp", "--n-eval", "1000", "--iterations", "3",
               "--skip", "9")
    assert res.returncode == 2


def test_cli_usage_errors():
    assert _cli("run", "--n-eval", "1000").returncode == 2            # missing --integrand
    assert _cli("sweep", "--integrand", "sinexp").returncode == 2    # no schedule
    assert _cli("run", "--integrand", "sinexp", "--n-eval", "1.5").returncode == 2
    assert _cli("sweep", "--integrand", "sinexp", "--n-evals", "1e3",
                "--n-eval-min", "1e3", "--n-eval-max", "2e3").returncode == 2


def test_cli_integration_failure_exit_code(monkeypatch, capsys):
    def boom(*a, **k):
        raise IntegrationError("synthetic failure")

    monkeypatch.setattr(bench, "run_report", boom)
    assert cli.main(["run", "--integrand", "sinexp", "--n-eval", "1000"]) == 1
    assert "synthetic failure" in capsys.readouterr().err


# ------------------------------------------------------------------- GPU --

@pytest.mark.gpu
def test_run_report_validates_against_schema():
    rep = bench.run_report("sinexp", 5000, "def", seed=1, max_it=4)
    jsonschema.validate(rep, bench.RUN_REPORT_SCHEMA)
    assert sum(rep["phases"].values()) == pytest.approx(100.0, abs=0.1)
    assert json.loads(json.dumps(rep)) == rep
    assert rep["backend"] == "b200" and rep["evals_per_second"] > 0


@pytest.mark.gpu
def test_run_report_repeats_and_warmup():
    rep = bench.run_report("sinexp", 2000, "def", seed=1, max_it=3, repeats=2, warmup=1)
    assert rep["repeats"] == 2
    with pytest.raises(ContractViolationError):
        bench.run_report("sinexp", 2000, repeats=0)


@pytest.mark.gpu
def test_sweep_rows_schema_and_worker_invariance():
    rows = bench.sweep("sinexp", [2000, 4000], "def", workers=[1, 2], seed=3, max_it=3)
    jsonschema.validate(bench.sweep_report(rows), bench.SWEEP_REPORT_SCHEMA)
    assert len(rows) == 4
    assert rows[0]["speedup"] == 1.0 and rows[0]["efficiency"] == 1.0
    assert rows[0]["mean"] == pytest.approx(rows[1]["mean"], rel=1e-10)
    single = bench.sweep("sinexp", [2000], "def", workers=[1], seed=3, max_it=3)
    assert single[0]["speedup"] is None and single[0]["efficiency"] is None
    parsed = bench.csv_to_rows(bench.rows_to_csv(rows))
    assert parsed == json.loads(json.dumps(bench.sweep_report(rows)))["rows"]


@pytest.mark.gpu
def test_cli_run_json_and_text(tmp_path):
    out_path = tmp_path / "report.json"
    res = _cli("run", "--integrand", "sinexp", "--n-eval", "5e3", "--iterations", "4",
               "--seed", "1", "--format", "json", "--out", str(out_path))
    assert res.returncode == 0, res.stderr
    rep = json.loads(out_path.read_text())
    jsonschema.validate(rep, bench.RUN_REPORT_SCHEMA)
    assert rep["params"]["n_eval"] == 5000
    res = _cli("run", "--integrand", "sinexp", "--n-eval", "2000", "--iterations", "3",
               "--skip", "1", "--seed", "2")
    assert res.returncode == 0 and "mean" in res.stdout and "phases:" in res.stdout
    assert res.stdout.count("\n") >= 6


@pytest.mark.gpu
def test_cli_sweep_csv_and_doubling(tmp_path):
    out_path = tmp_path / "rows.csv"
    res = _cli("sweep", "--integrand", "sinexp", "--n-evals", "2e3,4e3", "--iterations", "3",
               "--seed", "1", "--format", "csv", "--out", str(out_path))
    assert res.returncode == 0, res.stderr
    assert [r["n_eval"] for r in bench.csv_to_rows(out_path.read_text())] == [2000, 4000]
    res = _cli("sweep", "--integrand", "sinexp", "--n-eval-min", "1e3", "--n-eval-max", "4e3",
               "--iterations", "2", "--format", "csv")
    assert res.returncode == 0
    assert [r["n_eval"] for r in bench.csv_to_rows(res.stdout)] == [1000, 2000, 4000]


@pytest.mark.gpu
def test_cli_ablation_linear_and_tq():
    res = _cli("run", "--integrand", "gaussian", "--n-eval", "2e4", "--iterations", "6",
               "--skip", "2", "--beta", "0", "--format", "json")
    assert res.returncode == 0 and json.loads(res.stdout)["params"]["beta"] == 0.0
    res = _cli("run", "--integrand", "linear", "--config", "def", "--n-eval", "1e6", "--seed",
               "1", "--workers", "2", "--format", "json")
    rep = json.loads(res.stdout)
    assert res.returncode == 0 and abs(rep["mean"] - 5.0) <= 5.0 * rep["sigma"]
    res = _cli("run", "--integrand", "sinexp", "--config", "tq", "--n-eval", "1e4",
               "--iterations", "3", "--format", "json")
    assert json.loads(res.stdout)["params"]["n_intervals"] == bench.tq_n_intervals(10_000, 2)
