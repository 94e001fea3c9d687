"""CPU-only checks: the C ABI library builds/loads and exports every symbol the
header declares, host-side logic mirrors the reference, and the multi-rank
merge works over gloo.  No GPU compute is called here."""
import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vegas_b200.h")


@pytest.fixture(scope="module")
def lib_path():
    from paper_2408_09229_b200 import build as B
    return B.build()


def header_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(vpb_\w+)\s*\(", src, re.M)))


def test_header_declares_the_abi():
    syms = header_symbols()
    for s in ("vpb_create", "vpb_iterate", "vpb_history", "vpb_fill_host",
              "vpb_update_evals_host", "vpb_compute_results_host", "vpb_update_grid_host",
              "vpb_attach_nccl", "vpb_iteration_host"):
        assert s in syms


def test_library_exports_every_header_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (vpb_\w+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing


def test_library_is_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_ctypes_binding_matches_header(lib_path):
    from paper_2408_09229_b200 import _native as N
    L = N.load()
    assert L.vpb_abi_version() == N.ABI_VERSION
    assert set(N.SIGNATURES) >= set(header_symbols())


def test_compute_without_gpu_fails_loudly(lib_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2408_09229_b200 as P
    with pytest.raises(P.NativeLibraryError):
        P.lookup("gaussian").evaluate_batch(np.zeros((2, 4)))
    with pytest.raises((P.NativeLibraryError, P.VegasError)):
        P.integrate("gaussian", [(0, 1)] * 4, n_eval=1000, max_it=2)


def _magic(D):
    l = 0
    while l < 32 and (1 << l) < D:
        l += 1
    return (((1 << 32) * ((1 << l) - D)) // D + 1) & 0xFFFFFFFF, l


def test_magic_division():
    # devmath.cuh MagicDiv: q = (umulhi(n, m) + n) >> l for n < 2^31
    g = np.random.default_rng(0)
    for D in list(range(1, 3000)) + [2 ** 20, 2 ** 31, 999, 1000, 1024, 390625]:
        m, l = _magic(D)
        n = np.concatenate([g.integers(0, 2 ** 31, 3000, dtype=np.uint64),
                            np.array([0, 1, D - 1, D, D + 1, 2 ** 31 - 1], dtype=np.uint64)
                            % np.uint64(2 ** 31)])
        q = (((n * np.uint64(m)) >> np.uint64(32)) + n) >> np.uint64(l)
        np.testing.assert_array_equal(q, n // np.uint64(D))


@pytest.mark.parametrize("src", ["markstein_div.c", "markstein_general.c"])
def test_division_proofs(tmp_path, src):
    # The fill kernel's exactly-rounded divisions (devmath.cuh div_exact and
    # the fused uniform/N form of sample_axis) against IEEE division on the
    # host FPU (bounded sample; the tools run the full sweep without args).
    exe = str(tmp_path / "proof")
    subprocess.run(["gcc", "-O2", "-mfma", "-o", exe, os.path.join(ROOT, "tools", "proofs", src),
                    "-lm"], check=True)
    r = subprocess.run([exe, "300"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 mismatches" in r.stdout


def test_device_exp_accuracy(tmp_path):
    # devmath.cuh fast_exp_core restated in C with the same coefficients:
    # < 1 ulp against expl (tools/proofs/exp_accuracy.c)
    exe = str(tmp_path / "expacc")
    subprocess.run(["gcc", "-O2", "-mfma", "-o", exe,
                    os.path.join(ROOT, "tools", "proofs", "exp_accuracy.c"), "-lm"], check=True)
    r = subprocess.run([exe, "1"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_partition_runs_matches_reference_rule():
    from paper_2408_09229_b200.distributed import partition_runs
    assert partition_runs(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert partition_runs(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    for total in (0, 1, 7, 1000, 100_000_003):
        for k in (1, 2, 3, 8):
            r = partition_runs(total, k)
            assert r[0][0] == 0 and r[-1][1] == total
            sizes = [b - a for a, b in r]
            assert max(sizes) - min(sizes) <= 1


def test_config_validation():
    from paper_2408_09229_b200 import ContractViolationError, IntegratorConfig
    IntegratorConfig(n_eval=4)
    for bad in (dict(n_eval=3), dict(n_eval=10, max_it=2, skip=2), dict(n_eval=10, batch_size=0),
                dict(n_eval=10, n_intervals=1), dict(n_eval=10, alpha=-1),
                dict(n_eval=10, beta=-0.1), dict(n_eval=10, workers=0),
                dict(n_eval=10, cube_cap=0)):
        with pytest.raises(ContractViolationError):
            IntegratorConfig(**bad)
    c = IntegratorConfig(n_eval=100)
    assert (c.max_it, c.batch_size, c.n_intervals, c.alpha, c.beta) == (20, 1 << 20, 1024, 0.5, 0.75)


def test_integrate_rejects_config_and_overrides():
    import paper_2408_09229_b200 as P
    with pytest.raises(TypeError):
        P.integrate("gaussian", [(0, 1)] * 4, P.IntegratorConfig(n_eval=100), n_eval=10)


def test_combine_iterations_reference_semantics():
    from paper_2408_09229_b200 import IntegrationError, IterationResult, combine_iterations
    r = [IterationResult(1, 1.0, 0.25, True), IterationResult(2, 2.0, 0.25, True)]
    m, v, chi = combine_iterations(r)
    assert m == 1.5 and v == 0.125 and chi == pytest.approx(2.0)
    assert combine_iterations(list(reversed(r))) == (m, v, chi)
    with pytest.raises(IntegrationError):
        combine_iterations([])
    with pytest.raises(IntegrationError):
        combine_iterations([IterationResult(1, 1.0, 0.0, True), IterationResult(2, 2.0, 0.0, True)])
    assert combine_iterations([IterationResult(1, 3.0, 0.0, True),
                               IterationResult(2, 2.0, 1.0, True)]) == (3.0, 0.0, 0.0)


def test_compute_n_strat_reference_cases():
    from paper_2408_09229_b200 import compute_n_strat
    assert compute_n_strat(2, 10) == 1
    assert compute_n_strat(20_000, 2) == 100
    assert compute_n_strat(10 ** 6, 4) == 26
    assert compute_n_strat(10 ** 8, 8) == 5
    assert compute_n_strat(10 ** 8, 4) == 32
    assert compute_n_strat(10 ** 9, 6) == 10
    assert compute_n_strat(4 * 10 ** 9, 20) == 2


def test_registry_matches_reference_values():
    import oracle
    import paper_2408_09229_b200 as P
    # vp/tests/test_integrands.py:27-30: available() is exactly the reference registry
    assert P.available() == sorted([
        "sinexp", "linear", "cosine", "exponential", "roos_arnold",
        "morokoff", "gaussian", "ridge", "asian_option", "path_integral"])
    names = P.available_all()
    for n in ("multipeak8", "genz_oscillatory6", "genz_productpeak6", "gaussian20", "constant"):
        assert n in names
    assert P.lookup("gaussian").reference_value == 1.0
    from oracle import integrands_np as I
    assert P.lookup("multipeak8").reference_value == pytest.approx(I.multipeak8_reference(), rel=1e-15)
    assert P.lookup("genz_oscillatory6").reference_value == pytest.approx(0.12339809, rel=1e-7)
    assert P.lookup("genz_productpeak6").reference_value == pytest.approx(0.14749933, rel=1e-7)
    assert P.lookup("gaussian20").reference_value == pytest.approx(0.99998853, rel=1e-7)
    g = np.load(os.path.join(ROOT, "tests", "golden", "integrands.npz"))
    assert P.lookup("ridge").reference_value == pytest.approx(float(g["ridge_reference"][0]),
                                                              rel=1e-15)
    with pytest.raises(P.UnknownIntegrandError):
        P.lookup("nope")
    with pytest.raises(ValueError):
        P.lookup("gaussian", dim=3)


def test_device_params_match_oracle_constants():
    # the device parameter blobs are built with the reference's expressions
    import oracle
    import paper_2408_09229_b200 as P
    pd = P.lookup("gaussian").evaluate_batch.params(4)
    po = oracle.integrand_params("gaussian", 4)
    assert pd[0] == po[0] and pd[2] == po[2] and pd[3] == po[3] and pd[4] == 1.0 / po[3]
    pd = P.lookup("multipeak8").evaluate_batch.params(8)
    po = oracle.integrand_params("multipeak8", 8)
    assert pd[2] == po[2] and pd[3] == po[3] and list(pd[7:10]) == list(po[5:8])


def test_python_callable_rejected():
    import paper_2408_09229_b200 as P
    from paper_2408_09229_b200.integrands import resolve
    with pytest.raises(P.ContractViolationError):
        resolve(lambda x: x.sum(axis=1))


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist

    import oracle as O
    from paper_2408_09229_b200.distributed import partition_runs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    g = np.random.default_rng(5)
    n_h = g.integers(2, 400, 4 ** 3)
    off = O.build_run_plan(n_h)
    edges = np.sort(g.random((3, 33)), axis=1)
    edges[:, 0], edges[:, -1] = 0.0, 1.0
    lo, hi = partition_runs(int(off[-1]), world)[rank]
    mw, mc, s1, s2, cnt = O.fill(off, edges, 4, 11, 1000, 17, "gaussian", run_lo=lo, run_hi=hi)
    bufs = [torch.from_numpy(np.ascontiguousarray(a)) for a in (mw, mc, s1, s2, cnt)]
    for b in bufs:
        dist.all_reduce(b)
    if rank == 0:
        whole = O.fill(off, edges, 4, 11, 1000, 17, "gaussian")
        ok = (np.array_equal(bufs[1].numpy(), whole[1]) and np.array_equal(bufs[4].numpy(), whole[4])
              and np.allclose(bufs[0].numpy(), whole[0], rtol=1e-12)
              and np.allclose(bufs[2].numpy(), whole[2], rtol=1e-12, atol=1e-290))
        q.put(ok)
    dist.destroy_process_group()


def test_sharded_fill_merge_gloo_world2():
    """Rank shards by the reference partition rule + sum all-reduce reproduce
    the single-process fill (the merge the NCCL path performs on device)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert q.get(timeout=10) is True


def test_reference_arm_under_torchrun_world2():
    """The driver's N>1 launch of the reference arm: rank 0 alone prints the
    one JSON line, the other rank exits 0 without work."""
    env = dict(os.environ, VPB_REF_SAMPLE="100000")
    port = str(29600 + os.getpid() % 300)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                          "--master-port", port, os.path.join(ROOT, "bench.py"), "--impl",
                          "reference", "--gpus", "2", "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0


def test_reference_arm_json_line():
    env = dict(os.environ, VPB_REF_SAMPLE="200000")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                         env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
