"""``vegasplus-bench``-compatible command line on the B200 backend.

Same contract as the reference CLI (vp/cli.py:1-193): subcommands ``run``
(one integration, per-iteration detail and phase breakdown) and ``sweep``
(grids over n_eval and worker counts), the same flags, output formats
text / json / csv, and exit codes 0 success, 1 integration failure, 2 usage
error (unknown integrand, invalid parameter combination, bad flags).

    python -m paper_2408_09229_b200 run --integrand gaussian --n-eval 1e6 --format json
"""

from __future__ import annotations

import argparse
import json
import sys

from . import bench
from .errors import ContractViolationError, VegasError
from .integrands import UnknownIntegrandError

USAGE_EXIT = 2
FAILURE_EXIT = 1
_PHASES = ("init", "map", "fill", "update", "clear")


def _count(text: str) -> int:
    """Non-negative integer given as 1000000, 1e6 or 2.5e5."""
    try:
        value = float(text)
    except ValueError:
        raise argparse.ArgumentTypeError(f"expected a count, got {text!r}") from None
    if value < 0 or value != int(value):
        raise argparse.ArgumentTypeError(f"expected a nonnegative integer, got {text}")
    return int(value)


def _count_list(text: str) -> list[int]:
    return [_count(tok) for tok in text.split(",") if tok]


# (flags, argparse keyword arguments) shared by both subcommands
_COMMON = (
    (("--integrand",), dict(required=True, help="registry name")),
    (("--dim",), dict(type=int, default=None,
                      help="dimension override (variable-size integrands only)")),
    (("--config",), dict(choices=sorted(bench.NAMED_CONFIGS), default="def")),
    (("--iterations",), dict(type=int, default=None, dest="max_it",
                             help="iterations per run (max_it)")),
    (("--skip",), dict(type=int, default=None,
                       help="initial iterations excluded from the combination")),
    (("--alpha",), dict(type=float, default=None, help="map damping exponent")),
    (("--beta",), dict(type=float, default=None,
                       help="stratification damping exponent (0 disables adaptation)")),
    (("--n-intervals",), dict(type=_count, default=None, help="map intervals per axis")),
    (("--n-strat",), dict(type=_count, default=None, help="strata per axis override")),
    (("--batch-size",), dict(type=_count, default=None, help="logical RNG slots")),
    (("--seed",), dict(type=int, default=None)),
    (("--repeats",), dict(type=int, default=1, help="measured repetitions")),
    (("--warmup",), dict(type=int, default=0, help="unmeasured warm-up runs")),
    (("--format",), dict(choices=("text", "json", "csv"), default="text")),
    (("--out",), dict(default=None, help="write the report to this path")),
)
_OVERRIDE_KEYS = ("max_it", "skip", "alpha", "beta", "n_intervals", "n_strat", "batch_size",
                  "seed")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="vegasplus-bench",
                                 description="VEGAS+ benchmark command line (B200 backend)")
    sub = ap.add_subparsers(dest="command", required=True)
    run = sub.add_parser("run", help="single integration with full detail")
    sweep = sub.add_parser("sweep", help="error-vs-time / scaling / ablation grids")
    for p in (run, sweep):
        for flags, kw in _COMMON:
            p.add_argument(*flags, **kw)
    run.add_argument("--n-eval", type=_count, required=True,
                     help="evaluation budget per iteration")
    run.add_argument("--workers", type=int, default=1)
    sweep.add_argument("--n-evals", type=_count_list, default=None,
                       help="comma-separated n_eval list")
    sweep.add_argument("--n-eval-min", type=_count, default=None,
                       help="doubling schedule start (with --n-eval-max)")
    sweep.add_argument("--n-eval-max", type=_count, default=None, help="doubling schedule end")
    sweep.add_argument("--workers", type=_count_list, default=[1],
                       help="comma-separated worker counts")
    return ap


def _write(text: str, path):
    if path is None:
        sys.stdout.write(text)
        return
    with open(path, "w") as fh:
        fh.write(text)


def render_run_text(rep: dict) -> str:
    p = rep["params"]
    out = [f"integrand {rep['integrand']} ({rep['dims']}D)  config {rep['config']}  "
           f"n_eval {p['n_eval']}  seed {p['seed']}  workers {p['workers']}",
           f"{'it':>4} {'estimate':>16} {'sigma':>12}  included"]
    out += [f"{it['index']:>4} {it['estimate']:>16.8g} {it['sigma']:>12.4g}  "
            f"{'yes' if it['included'] else 'no'}" for it in rep["iterations"]]
    tail = f"mean {rep['mean']:.10g}  sigma {rep['sigma']:.4g}  chi2/dof {rep['chi2_dof']:.3g}"
    if rep["reference_value"] is not None:
        tail += f"  reference {rep['reference_value']:.10g}"
    out.append(tail)
    ph = rep["phases"]
    out.append(f"wall {rep['wall_ms']:.1f} ms  phases: " +
               "  ".join(f"{k} {ph[k]:.1f}%" for k in _PHASES))
    return "\n".join(out) + "\n"


def render_sweep_text(rows: list[dict]) -> str:
    width = {c: max(12, len(c)) for c in bench.SWEEP_COLUMNS}

    def fmt(v):
        if v is None:
            return "-"
        return f"{v:.6g}" if isinstance(v, float) else str(v)

    lines = ["  ".join(c.ljust(width[c]) for c in bench.SWEEP_COLUMNS)]
    lines += ["  ".join(fmt(r[c]).ljust(width[c]) for c in bench.SWEEP_COLUMNS) for r in rows]
    return "\n".join(lines) + "\n"


def _do_run(args, overrides) -> str:
    rep = bench.run_report(args.integrand, args.n_eval, args.config, dim=args.dim,
                           repeats=args.repeats, warmup=args.warmup, workers=args.workers,
                           **overrides)
    if args.format == "json":
        return json.dumps(rep, indent=2) + "\n"
    if args.format == "csv":
        row = {c: rep.get(c) for c in bench.SWEEP_COLUMNS}
        row.update(config=rep["config"], n_eval=rep["params"]["n_eval"],
                   workers=rep["params"]["workers"])
        return bench.rows_to_csv([row])
    return render_run_text(rep)


def _schedule(ap, args) -> list[int]:
    have_list = args.n_evals is not None
    have_range = args.n_eval_min is not None or args.n_eval_max is not None
    if have_list and have_range:
        ap.error("--n-evals conflicts with --n-eval-min/--n-eval-max")
    if not have_list:
        if args.n_eval_min is None or args.n_eval_max is None:
            ap.error("sweep needs --n-evals or --n-eval-min/--n-eval-max")
        return bench.doubling_schedule(args.n_eval_min, args.n_eval_max)
    if not args.n_evals:
        ap.error("empty n_eval list")
    return args.n_evals


def _do_sweep(ap, args, overrides) -> str:
    n_evals = _schedule(ap, args)
    rows = bench.sweep(args.integrand, n_evals, args.config, workers=args.workers,
                       dim=args.dim, repeats=args.repeats, warmup=args.warmup, **overrides)
    if args.format == "json":
        return json.dumps(bench.sweep_report(rows), indent=2) + "\n"
    if args.format == "csv":
        return bench.rows_to_csv(rows)
    return render_sweep_text(rows)


def main(argv=None) -> int:
    ap = build_parser()
    args = ap.parse_args(argv)          # usage errors exit 2 from argparse
    overrides = {k: getattr(args, k) for k in _OVERRIDE_KEYS}
    try:
        text = _do_run(args, overrides) if args.command == "run" else \
            _do_sweep(ap, args, overrides)
    except (UnknownIntegrandError, ContractViolationError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return USAGE_EXIT
    except VegasError as exc:
        print(f"integration failed: {exc}", file=sys.stderr)
        return FAILURE_EXIT
    _write(text, args.out)
    return 0


if __name__ == "__main__":
    sys.exit(main())
