"""Benchmark report layer on the B200 backend.

Drop-in for the reference's report module (vp/bench.py:1-290): the same
named configurations, schema-1 run and sweep reports, fixed CSV columns
(CSV and JSON decode to identical values), doubling schedules and JSON
schemas -- those are data contracts and are kept verbatim.  The numbers come
from the device backend: ``phases`` are the CUDA-event phase times of the
integration (``PhaseTimes``), ``wall_ms`` the host wall clock around
``integrate`` (device work included).  Run reports carry two extra keys,
``backend`` and ``evals_per_second``, which the reference schema admits.

``workers`` is validated and recorded but the device fill does not depend on
it (the reference guarantees worker-invariant results; here the work is on
the GPU), so worker sweeps report speedups of ~1.  GPU scaling is measured by
``bench.py --gpus N`` at the repository root.
"""

from __future__ import annotations

import csv
import io
import math
import time
from statistics import fmean

from .core import IntegratorConfig, integrate
from .errors import ContractViolationError
from .integrands import IntegrandSpec, lookup

SCHEMA_VERSION = 1
BACKEND = "b200"

_DEFAULT_RUN = dict(max_it=20, skip=0, batch_size=1_048_576)

#: named parameter sets (vp/bench.py:18-28): "def" = library defaults,
#: "vf" / "tq" = the VegasFlow- and TorchQuad-style fixed choices; the tq
#: interval count is computed from n_eval (None here)
NAMED_CONFIGS = {
    "def": {**_DEFAULT_RUN, "n_intervals": 1024, "alpha": 0.5, "beta": 0.75},
    "vf": {**_DEFAULT_RUN, "n_intervals": 50, "alpha": 1.5, "beta": 0.75},
    "tq": {**_DEFAULT_RUN, "n_intervals": None, "alpha": 0.5, "beta": 0.75},
}

# sweep row columns with their CSV decoders (order = CSV header, vp/bench.py:31-33)
_ROW_TYPES = (("integrand", str), ("config", str), ("dims", int), ("n_eval", int),
              ("workers", int), ("repeats", int), ("mean", float), ("sigma", float),
              ("rel_stderr", float), ("chi2_dof", float), ("wall_ms", float),
              ("fill_fraction", float), ("speedup", float), ("efficiency", float))
SWEEP_COLUMNS = tuple(name for name, _ in _ROW_TYPES)


def tq_n_intervals(n_eval: int, dims: int) -> int:
    """Interval count of the tq template: 10 * n_eval^(1/(2d)), clamped to
    [10, 1024] (vp/bench.py:36-39)."""
    guess = math.floor(10 * n_eval ** (1.0 / (2 * dims)))
    return int(max(10, min(1024, guess)))


def resolve_config(spec: IntegrandSpec, n_eval: int, config: str = "def",
                   **overrides) -> IntegratorConfig:
    """IntegratorConfig from a named template; None-valued overrides are
    ignored (vp/bench.py:41-51)."""
    try:
        template = NAMED_CONFIGS[config]
    except KeyError:
        raise ContractViolationError(
            f"unknown config {config!r}; choose from {sorted(NAMED_CONFIGS)}") from None
    fields = {k: v for k, v in template.items()}
    if fields.get("n_intervals") is None:
        fields["n_intervals"] = tq_n_intervals(n_eval, spec.dims)
    for key, val in overrides.items():
        if val is not None:
            fields[key] = val
    return IntegratorConfig(n_eval=int(n_eval), **fields)


def _timed_runs(spec, cfg, repeats, warmup):
    for _ in range(warmup):
        integrate(spec.evaluate_batch, spec.bounds, cfg, batched=True)
    walls, last = [], None
    for _ in range(repeats):
        t0 = time.perf_counter()
        last = integrate(spec.evaluate_batch, spec.bounds, cfg, batched=True)
        walls.append(time.perf_counter() - t0)
    return last, fmean(walls)


def _params_block(cfg: IntegratorConfig, n_strat: int) -> dict:
    keys = ("n_eval", "max_it", "skip", "batch_size", "n_intervals", "alpha", "beta",
            "seed", "workers")
    block = {k: getattr(cfg, k) for k in keys}
    block["n_strat"] = n_strat
    return block


def run_report(name: str, n_eval: int, config: str = "def", dim=None,
               repeats: int = 1, warmup: int = 0, **overrides) -> dict:
    """One timed integration as a schema-1 report (vp/bench.py:54-105): the
    mean wall clock of ``repeats`` measured runs after ``warmup`` unmeasured
    ones; the numbers are the last run's (the seed is fixed)."""
    if repeats < 1:
        raise ContractViolationError(f"repeats must be >= 1, got {repeats}")
    if warmup < 0:
        raise ContractViolationError(f"warmup must be >= 0, got {warmup}")
    spec = lookup(name, dim=dim)
    cfg = resolve_config(spec, n_eval, config, **overrides)
    out, wall = _timed_runs(spec, cfg, repeats, warmup)
    phases = out.timing.percentages()
    evals = [int(e) for e in out.evals_per_iteration]
    rep = dict(schema=SCHEMA_VERSION, kind="run", backend=BACKEND, integrand=spec.name,
               dims=spec.dims, config=config, params=_params_block(cfg, out.n_strat),
               reference_value=spec.reference_value)
    rep["iterations"] = [dict(index=it.index, estimate=it.estimate, sigma=it.sigma,
                              included=it.included) for it in out.iterations]
    rep.update(mean=out.mean, sigma=out.sigma,
               rel_stderr=None if out.mean == 0.0 else out.sigma / abs(out.mean),
               chi2_dof=out.chi2_dof, repeats=repeats, wall_ms=wall * 1e3, phases=phases,
               fill_fraction=phases["fill"] / 100.0, evals_per_iteration=evals,
               evals_per_second=(sum(evals) / wall) if wall > 0 else None)
    return rep


def doubling_schedule(n_eval_min: int, n_eval_max: int) -> list[int]:
    """n_eval_min, 2 n_eval_min, ... up to n_eval_max inclusive."""
    if n_eval_min < 4 or n_eval_max < n_eval_min:
        raise ContractViolationError(f"bad schedule bounds ({n_eval_min}, {n_eval_max})")
    steps = int(math.floor(math.log2(n_eval_max / n_eval_min) + 1e-12))
    vals = [int(n_eval_min) << k for k in range(steps + 1)]
    return [v for v in vals if v <= n_eval_max]


def _row(rep: dict, config: str, n_eval: int, workers: int, repeats: int) -> dict:
    row = dict.fromkeys(SWEEP_COLUMNS)
    row.update(integrand=rep["integrand"], config=config, dims=rep["dims"], n_eval=int(n_eval),
               workers=int(workers), repeats=int(repeats))
    for key in ("mean", "sigma", "rel_stderr", "chi2_dof", "wall_ms", "fill_fraction"):
        row[key] = rep[key]
    return row


def sweep(name: str, n_evals, config: str = "def", workers=(1,), dim=None,
          repeats: int = 1, warmup: int = 0, **overrides) -> list[dict]:
    """Rows for every (n_eval, workers) point; with several worker counts an
    n_eval group gets speedup and efficiency against its smallest count
    (vp/bench.py:121-161)."""
    counts = [int(w) for w in workers]
    rows: list[dict] = []
    for n_eval in n_evals:
        group = [_row(run_report(name, n_eval, config, dim=dim, repeats=repeats, warmup=warmup,
                                 workers=w, **overrides), config, n_eval, w, repeats)
                 for w in counts]
        if len(group) > 1:
            ref = min(group, key=lambda r: r["workers"])
            for row in group:
                row["speedup"] = ref["wall_ms"] / row["wall_ms"]
                row["efficiency"] = row["speedup"] * ref["workers"] / row["workers"]
        rows += group
    return rows


def sweep_report(rows: list[dict]) -> dict:
    return {"schema": SCHEMA_VERSION, "kind": "sweep", "rows": rows}


def _cell(v) -> str:
    if v is None:
        return ""
    return repr(v) if isinstance(v, float) else str(v)


def rows_to_csv(rows: list[dict]) -> str:
    """Fixed-header CSV; floats via repr so the CSV decodes to the JSON values."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(SWEEP_COLUMNS)
    for row in rows:
        w.writerow([_cell(row.get(c)) for c in SWEEP_COLUMNS])
    return buf.getvalue()


def csv_to_rows(text: str) -> list[dict]:
    """Inverse of rows_to_csv (empty fields decode to None)."""
    records = [r for r in csv.reader(io.StringIO(text.strip())) if r]
    if tuple(records[0]) != SWEEP_COLUMNS:
        raise ContractViolationError(f"unexpected CSV header: {records[0]}")
    return [{name: (None if cell == "" else typ(cell))
             for (name, typ), cell in zip(_ROW_TYPES, rec)} for rec in records[1:]]


# --------------------------------------------------------------- schemas --
# JSON schemas of the reports (vp/bench.py:207-290), assembled from tables.

_NUM_OR_NULL = {"type": ["number", "null"]}
_JSON_TYPE = {str: {"type": "string"}, int: {"type": "integer"}, float: {"type": "number"}}
_NULLABLE = {"rel_stderr", "speedup", "efficiency"}


def _obj(required, props=None, **extra):
    d = {"type": "object", "required": list(required)}
    if props:
        d["properties"] = props
    d.update(extra)
    return d


_ITERATION = _obj(("index", "estimate", "sigma", "included"), {
    "index": {"type": "integer", "minimum": 1}, "estimate": {"type": "number"},
    "sigma": {"type": "number", "minimum": 0}, "included": {"type": "boolean"}})

RUN_REPORT_SCHEMA = {
    "$schema": "http://json-schema.org/draft-07/schema#",
    **_obj(("schema", "kind", "integrand", "dims", "config", "params", "iterations", "mean",
            "sigma", "chi2_dof", "wall_ms", "phases", "fill_fraction"), {
        "schema": {"const": SCHEMA_VERSION},
        "kind": {"const": "run"},
        "integrand": {"type": "string"},
        "dims": {"type": "integer", "minimum": 1},
        "config": {"enum": sorted(NAMED_CONFIGS)},
        "params": _obj(("n_eval", "max_it", "skip", "batch_size", "n_intervals", "alpha",
                        "beta", "seed", "workers")),
        "reference_value": _NUM_OR_NULL,
        "iterations": {"type": "array", "minItems": 1, "items": _ITERATION},
        "mean": {"type": "number"},
        "sigma": {"type": "number", "minimum": 0},
        "rel_stderr": _NUM_OR_NULL,
        "chi2_dof": {"type": "number", "minimum": 0},
        "repeats": {"type": "integer", "minimum": 1},
        "wall_ms": {"type": "number", "minimum": 0},
        "phases": _obj(("init", "map", "fill", "update", "clear"),
                       additionalProperties={"type": "number"}),
        "fill_fraction": {"type": "number", "minimum": 0, "maximum": 1},
    }),
}

_ROW_PROPS = {name: (_NUM_OR_NULL if name in _NULLABLE else dict(_JSON_TYPE[typ]))
              for name, typ in _ROW_TYPES}
_ROW_PROPS["config"] = {"enum": sorted(NAMED_CONFIGS)}

SWEEP_REPORT_SCHEMA = {
    "$schema": "http://json-schema.org/draft-07/schema#",
    **_obj(("schema", "kind", "rows"), {
        "schema": {"const": SCHEMA_VERSION},
        "kind": {"const": "sweep"},
        "rows": {"type": "array", "items": _obj(SWEEP_COLUMNS, _ROW_PROPS)},
    }),
}
