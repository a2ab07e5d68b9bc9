"""Multi-process pipeline logic on CPU (gloo, world size 2 and 3).

The per-rank solve is replaced by a deterministic fake so the scatter /
solve / gather / report / failure paths of run_pipeline are exercised
without a GPU; the device solver itself is covered by tests/test_gpu_*.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2003_12677_b200 import (ScanGeometry, SinogramStack, SolverConfig,
                                   WorkerFailureError, run_pipeline)
from paper_2003_12677_b200.pipeline import rank_ranges, unit_slices

Y = X = 8
T, P = 5, 8


def _fake_solver(bad_unit=None, offset=0):
    """rec[slice] = slice mean + slice-local index ramp; per-unit reports."""
    def run(data):
        a = np.asarray(data, dtype=np.float64)
        n = a.shape[0]
        rec = np.empty((n, Y, X))
        for k in range(n):
            rec[k] = a[k].mean() + np.arange(Y * X).reshape(Y, X) * 1e-3
        units = (n + 1) // 2
        final = [float(a[2 * u:2 * u + 2].sum()) for u in range(units)]
        iters = [3 + (u % 2) for u in range(units)]
        conv = [True] * units
        stat = [0] * units
        return rec, final, iters, conv, stat
    return run


def _stack(n_z, seed=0):
    geom = ScanGeometry(n_p=P, n_theta=T, n_z=n_z)
    data = np.random.default_rng(seed).standard_normal((n_z, T, P))
    return SinogramStack(data=data, geometry=geom)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_z, bad_global_unit, out_q, mode="local", out_path=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        stack = _stack(n_z) if (mode != "scatter" or rank == 0) else None
        out = None
        if mode == "out":
            out = np.memmap(out_path, dtype=np.float32, mode="r+", shape=(n_z, Y, X))
        n_units = (n_z + 1) // 2
        u0 = rank_ranges(n_units, world)[rank][0]

        def solver(data):
            rec, final, iters, conv, stat = _fake_solver()(data)
            if bad_global_unit is not None and u0 <= bad_global_unit < u0 + len(stat):
                stat[bad_global_unit - u0] = 7  # SPTB_ERR_NONFINITE
            return rec, final, iters, conv, stat

        try:
            vol, rep = run_pipeline(stack, SolverConfig(algorithm="sirt", max_iter=3), solver=solver,
                                    out=out)
            out_q.put((rank, "ok", None if vol is None else np.array(vol.data), rep.residual_history,
                       rep.iterations_run, rep.converged))
        except WorkerFailureError as e:
            out_q.put((rank, "fail", e.slice_range, str(e.cause), 0, False))
    finally:
        dist.destroy_process_group()


def _run(world, n_z, bad=None, mode="local", out_path=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_z, bad, q, mode, out_path))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return {r[0]: r for r in res}


def test_rank_ranges_partition_units():
    for n_units in range(1, 40):
        for world in range(1, 9):
            rr = rank_ranges(n_units, world)
            assert len(rr) == world
            cur = 0
            for start, ln in rr:
                assert start == cur
                cur += ln
            assert cur == n_units
            lens = [ln for _, ln in rr]
            assert max(lens) - min(lens) <= max(1, -(-n_units // world))
    assert unit_slices(2, 3, 9) == (4, 9)


@pytest.mark.parametrize("mode", ["local", "scatter", "out"])
@pytest.mark.parametrize("world,n_z", [(2, 7), (2, 8), (3, 11)])
def test_distributed_matches_single_process(world, n_z, mode, tmp_path):
    """Per-rank solve of contiguous pair-unit ranges reproduces the
    single-process result bit for bit, and the report aggregates units in
    slice order (pipeline.py:223-234), for every data path: each rank loads
    its own slices ("local"), rank 0 scatters over the process group
    ("scatter", other ranks pass no stack), each rank writes its own slices
    into a shared memory-mapped volume ("out")."""
    single_vol, single_rep = run_pipeline(_stack(n_z), SolverConfig(algorithm="sirt", max_iter=3),
                                          solver=_fake_solver())
    out_path = None
    if mode == "out":
        out_path = str(tmp_path / "vol.f32")
        np.memmap(out_path, dtype=np.float32, mode="w+", shape=(n_z, Y, X)).flush()
    res = _run(world, n_z, mode=mode, out_path=out_path)
    rank0 = res[0]
    assert rank0[1] == "ok"
    # the fake solver runs per rank on float32-transported data: compare to the
    # single-process run on the same float32-rounded stack
    ref_vol, ref_rep = run_pipeline(
        SinogramStack(data=_stack(n_z).data.astype(np.float32).astype(np.float64),
                      geometry=_stack(n_z).geometry),
        SolverConfig(algorithm="sirt", max_iter=3), solver=_fake_solver())
    np.testing.assert_allclose(rank0[2], ref_vol.data, rtol=0, atol=1e-6)
    np.testing.assert_allclose(rank0[3], ref_rep.residual_history, rtol=1e-6)
    assert len(rank0[3]) == (n_z + 1) // 2
    assert rank0[4] == max(3 + (u % 2) for u in range((n_z + 1) // 2))
    assert rank0[5] is True
    for r in range(1, world):
        assert res[r][1] == "ok" and res[r][2] is None
    assert single_vol.data.shape == (n_z, Y, X)


def test_distributed_failure_reports_rank_slice_range():
    """A non-finite unit on rank 1 raises WorkerFailureError on every rank with
    that rank's slice range (pipeline.py:166-176, 215-217)."""
    n_z, world = 8, 2
    res = _run(world, n_z, bad=3)        # unit 3 = slices 6, 7 -> rank 1 owns units 2, 3
    lo, hi = unit_slices(*rank_ranges(4, 2)[1], n_z)
    for r in range(world):
        assert res[r][1] == "fail"
        assert res[r][2] == (lo, hi)
        assert "NonFinite" in res[r][3]


def test_single_process_failure_range():
    """Without a process group the failing unit maps onto the reference's task
    range for (workers, max_per_pass)."""
    def solver(data):
        rec, final, iters, conv, stat = _fake_solver()(data)
        stat[0] = 7
        return rec, final, iters, conv, stat
    with pytest.raises(WorkerFailureError) as err:
        run_pipeline(_stack(8), SolverConfig(algorithm="tv", max_iter=2), workers=2,
                     solver=solver)
    assert err.value.slice_range == (0, 4)
    assert "NonFinite" in str(err.value.cause)
