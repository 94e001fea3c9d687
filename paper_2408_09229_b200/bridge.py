"""Stdio bridge for foreign runtimes, B200 backend.

Wire-compatible with the reference bridge (vp/bridge.py:1-150; the
TypeScript codec fe/src/frames.ts): every message is a frame = 4-byte
little-endian header length, a UTF-8 JSON header, then ``header["nbytes"]``
bytes of raw payload.

The reference evaluates the integrand on the foreign side, streaming
``eval`` frames out and reading ``values`` frames back for every batch.  A
host callback cannot run inside the fused device fill, and there is no CPU
fallback, so this bridge integrates *registered device integrands*: the init
frame names one, and the only frames exchanged are ``init`` -> ``result`` (or
``error``) -- no per-batch round trips.

    in : {"type": "init", "integrand": "gaussian" | {"name": .., "dim": .., "params": {..}},
          "bounds": [[lo, hi], ...] (optional: the registry bounds),
          "config": {...IntegratorConfig fields...}}
    out: {"type": "result", "mean": .., "sigma": .., "diagnostics": {...}}
    out: {"type": "error", "message": str, "point": [..] | null}

An init frame without ``integrand`` (a callback-driven client) gets an error
frame saying so.  ``python -m paper_2408_09229_b200.bridge`` serves one
integration on stdin/stdout.
"""

from __future__ import annotations

import json
import struct
import sys

from .core import IntegratorConfig, integrate
from .errors import NonFiniteIntegrandError, VegasError
from .integrands import lookup

_HDR = struct.Struct("<I")
CONFIG_FIELDS = frozenset(("n_eval", "max_it", "skip", "batch_size", "n_intervals", "alpha",
                           "beta", "seed", "workers", "cube_cap", "n_strat"))


def _take(stream, n: int) -> bytes:
    buf = bytearray()
    while len(buf) < n:
        part = stream.read(n - len(buf))
        if not part:
            raise EOFError("peer closed the bridge stream")
        buf += part
    return bytes(buf)


def read_frame(stream):
    """One frame -> (header dict, payload bytes)."""
    (hlen,) = _HDR.unpack(_take(stream, 4))
    header = json.loads(_take(stream, hlen).decode("utf-8"))
    size = int(header.get("nbytes") or 0)
    return header, (_take(stream, size) if size else b"")


def write_frame(stream, header: dict, payload: bytes = b""):
    """Send one frame; ``nbytes`` is set from the payload."""
    raw = json.dumps({**header, "nbytes": len(payload)}).encode("utf-8")
    stream.write(_HDR.pack(len(raw)) + raw + payload)
    stream.flush()


def _error(out, message: str, point=None) -> int:
    write_frame(out, {"type": "error", "message": message,
                      "point": None if point is None else [float(v) for v in point]})
    return 1


def _spec_from(desc):
    if isinstance(desc, str):
        return lookup(desc)
    if isinstance(desc, dict) and "name" in desc:
        return lookup(desc["name"], dim=desc.get("dim"), **dict(desc.get("params") or {}))
    raise ValueError("init.integrand must be a registry name or {name, dim?, params?}")


def result_header(out) -> dict:
    """The reference's result frame (vp/bridge.py:126-141) for an IntegralOutcome."""
    return {
        "type": "result",
        "mean": out.mean,
        "sigma": out.sigma,
        "diagnostics": {
            "chi2_dof": out.chi2_dof,
            "n_strat": out.n_strat,
            "n_cubes": out.n_cubes,
            "evals_per_iteration": [int(e) for e in out.evals_per_iteration],
            "iterations": [{"index": r.index, "estimate": r.estimate, "sigma": r.sigma,
                            "included": r.included} for r in out.iterations],
            "timing": out.timing.percentages(),
        },
    }


def serve(inp, out) -> int:
    """Serve one integration: read the init frame, answer result or error."""
    try:
        header, _ = read_frame(inp)
    except (EOFError, ValueError, struct.error) as exc:
        return _error(out, f"bad init frame: {exc}")
    if header.get("type") != "init":
        return _error(out, f"expected init frame, got {header.get('type')!r}")
    if "integrand" not in header:
        return _error(out, "the B200 backend integrates registered device integrands: name one "
                           "in init.integrand (host callbacks over eval/values frames cannot "
                           "run inside the fused device fill)")
    try:
        spec = _spec_from(header["integrand"])
        raw = dict(header.get("config") or {})
        raw.pop("concurrent", None)   # reference flag for host callbacks; moot here
        cfg = IntegratorConfig(**{k: v for k, v in raw.items() if k in CONFIG_FIELDS})
        bounds = header.get("bounds")
        bounds = spec.bounds if bounds is None else [(float(a), float(b)) for a, b in bounds]
        result = integrate(spec.evaluate_batch, bounds, cfg, batched=True)
    except NonFiniteIntegrandError as exc:
        return _error(out, str(exc), exc.point)
    except (VegasError, ValueError, TypeError, KeyError) as exc:
        return _error(out, str(exc))
    write_frame(out, result_header(result))
    return 0


def main() -> int:
    return serve(sys.stdin.buffer, sys.stdout.buffer)


if __name__ == "__main__":
    sys.exit(main())
