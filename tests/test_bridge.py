"""Stdio bridge (pkg/tests/test_bridge.py against the B200 backend): the
reference's frame codec and error frames; integration of registered device
integrands (no per-batch callbacks -- see paper_2408_09229_b200/bridge.py)."""
import io
import subprocess
import sys

import numpy as np
import pytest

from paper_2408_09229_b200 import integrate
from paper_2408_09229_b200.bridge import read_frame, write_frame
from paper_2408_09229_b200.integrands import lookup


def _spawn():
    return subprocess.Popen([sys.executable, "-m", "paper_2408_09229_b200.bridge"],
                            stdin=subprocess.PIPE, stdout=subprocess.PIPE)


def _one_shot(header, timeout=600):
    proc = _spawn()
    try:
        write_frame(proc.stdin, header)
        reply, _ = read_frame(proc.stdout)
    finally:
        proc.stdin.close()
        code = proc.wait(timeout=timeout)
    return reply, code


def test_frame_round_trip():
    buf = io.BytesIO()
    payload = np.arange(6, dtype=np.float64).tobytes()
    write_frame(buf, {"type": "eval", "count": 6}, payload)
    buf.seek(0)
    header, back = read_frame(buf)
    assert header["type"] == "eval" and header["nbytes"] == len(payload)
    assert back == payload
    buf = io.BytesIO()
    write_frame(buf, {"type": "init"})
    buf.seek(0)
    assert read_frame(buf) == ({"type": "init", "nbytes": 0}, b"")


def test_bridge_rejects_garbled_init():
    reply, code = _one_shot({"type": "values"})
    assert reply["type"] == "error" and code == 1


def test_bridge_requires_a_device_integrand():
    # a callback-driven client (the reference protocol's eval frames) is told why
    reply, code = _one_shot({"type": "init", "bounds": [[0.0, 1.0]], "config": {"n_eval": 100}})
    assert reply["type"] == "error" and code == 1
    assert "device integrand" in reply["message"]


def test_bridge_usage_errors_before_device_work():
    reply, code = _one_shot({"type": "init", "integrand": "nope", "config": {"n_eval": 100}})
    assert reply["type"] == "error" and "available" in reply["message"] and code == 1
    reply, code = _one_shot({"type": "init", "integrand": "sinexp",
                             "config": {"n_eval": 100, "max_it": 3, "skip": 5}})
    assert reply["type"] == "error" and code == 1


@pytest.mark.gpu
def test_bridge_constant_integrand_volume():
    reply, code = _one_shot({"type": "init",
                             "integrand": {"name": "constant", "dim": 2, "params": {"value": 1.0}},
                             "bounds": [[0.0, 2.0], [0.0, 1.0]],
                             "config": {"n_eval": 2000, "max_it": 3, "seed": 4}})
    assert code == 0 and reply["type"] == "result"
    assert reply["mean"] == pytest.approx(2.0, rel=1e-12)
    assert reply["sigma"] == pytest.approx(0.0, abs=1e-12)
    assert reply["diagnostics"]["iterations"][0]["index"] == 1


@pytest.mark.gpu
def test_bridge_matches_in_process():
    spec = lookup("linear")
    config = {"n_eval": 20_000, "max_it": 6, "skip": 2, "seed": 123}
    reply, code = _one_shot({"type": "init", "integrand": "linear",
                             "bounds": [list(b) for b in spec.bounds], "config": config})
    native = integrate(spec.evaluate_batch, spec.bounds, batched=True, **config)
    assert code == 0
    # the interval histograms are summed with shared-memory atomics, so two
    # processes agree to rounding, not bitwise (tests/test_gpu_api.py header)
    assert reply["mean"] == pytest.approx(native.mean, rel=1e-12)
    assert reply["sigma"] == pytest.approx(native.sigma, rel=1e-9)
    assert reply["diagnostics"]["evals_per_iteration"] == list(native.evals_per_iteration)


@pytest.mark.gpu
def test_bridge_parametrised_integrand():
    reply, code = _one_shot({"type": "init",
                             "integrand": {"name": "path_integral", "dim": 4},
                             "config": {"n_eval": 100_000, "max_it": 10, "skip": 3, "seed": 4}})
    ref = lookup("path_integral", dim=4).reference_value
    assert code == 0 and abs(reply["mean"] - ref) < 5 * reply["sigma"]
