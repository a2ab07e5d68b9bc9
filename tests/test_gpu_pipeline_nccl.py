"""run_pipeline over 2 GPUs with NCCL (one process per GPU, pipeline.py:179-235):
each data path -- every rank loads its own slices ("local"), rank 0
scatters over NCCL ("scatter"), each rank writes its own slices into a shared
memory-mapped volume ("out") -- gives the single-GPU result bit for bit (same
launch batch on every rank, fixed-order reductions).  The NCCL cases are
skipped on boxes with fewer than 2 GPUs; the gloo cases run two ranks on
cuda:0 with the device solver (test_pipeline_dist.py covers the logic on
CPU)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NZ, N, T = 11, 64, 48


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _stack():
    import paper_2003_12677_b200 as sb
    from oracle import shepp_logan
    geom = sb.ScanGeometry(n_p=N, n_theta=T, n_z=NZ)
    ops = sb.build_operators(sb.ScanGeometry(n_p=N, n_theta=T), filter_kind="hamming")
    rng = np.random.default_rng(2)
    base = ops.radon(shepp_logan(N)[0])
    data = np.stack([base * (1 - 0.03 * k) + 0.01 * rng.standard_normal(base.shape) for k in range(NZ)])
    return sb.SinogramStack(data=data.astype(np.float32), geometry=geom)


def _worker(rank, world, port, mode, out_path, q, backend="nccl"):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    if backend == "gloo":  # both ranks on cuda:0: the host-side data paths
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
    else:
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        import paper_2003_12677_b200 as sb
        stack = _stack() if (mode != "scatter" or rank == 0) else None
        out = np.memmap(out_path, dtype=np.float32, mode="r+", shape=(NZ, N, N)) if mode == "out" else None
        ops = sb.build_operators(sb.ScanGeometry(n_p=N, n_theta=T), filter_kind="hamming")
        vol, rep = sb.run_pipeline(stack, sb.SolverConfig(algorithm="sirt", max_iter=6), ops=ops, out=out)
        q.put((rank, None if vol is None else np.array(vol.data, dtype=np.float32),
               rep.residual_history, rep.iterations_run))
    finally:
        dist.destroy_process_group()


def _run_two(tmp_path, mode, backend):
    import torch.multiprocessing as mp
    import paper_2003_12677_b200 as sb
    ops = sb.build_operators(sb.ScanGeometry(n_p=N, n_theta=T), filter_kind="hamming")
    ref, ref_rep = sb.run_pipeline(_stack(), sb.SolverConfig(algorithm="sirt", max_iter=6), ops=ops)
    out_path = str(tmp_path / "vol.f32")
    np.memmap(out_path, dtype=np.float32, mode="w+", shape=(NZ, N, N)).flush()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, out_path, q, backend)) for r in range(2)]
    for p in procs:
        p.start()
    res = {r[0]: r for r in (q.get(timeout=300) for _ in procs)}
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    vol = res[0][1]
    np.testing.assert_array_equal(vol, ref.data.astype(np.float32))
    np.testing.assert_array_equal(res[0][2], ref_rep.residual_history)
    assert res[0][3] == ref_rep.iterations_run and res[1][1] is None


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("mode", ["local", "scatter", "out"])
def test_two_gpu_pipeline_bitwise(tmp_path, mode):
    _run_two(tmp_path, mode, "nccl")


@pytest.mark.parametrize("mode", ["local", "scatter", "out"])
def test_two_ranks_one_gpu_pipeline_bitwise(tmp_path, mode):
    """The same with both ranks on cuda:0 over gloo: the device solver under
    run_pipeline's multi-rank host paths on a one-GPU box."""
    _run_two(tmp_path, mode, "gloo")
