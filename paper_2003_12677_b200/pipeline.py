"""Slice-parallel pipeline (API of sptomo/pipeline.py) over GPUs.

The reference packs slices (2k, 2k+1) into one complex sinogram and farms
pair units out to a fork pool (pipeline.py:137-235).  Here a unit is one
complex vector of a device batch, and the "workers" are GPUs: one process per
GPU under torch.distributed.  Rank 0 owns the stack; its pair-unit ranges are
scattered to the ranks with NCCL point-to-point sends, every rank solves its
range with the batched device solver (no collective inside iterations), and
the reconstructed slices plus per-unit reports are gathered back to rank 0.
Units never span ranks, so every slice's floating-point path is independent
of the GPU count (same launch batch on every rank).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from .errors import ShapeMismatchError, WorkerFailureError
from .geometry import ScanGeometry

PAIRING_TOL = 1e-5


@dataclass(frozen=True)
class SinogramStack:
    """(n_z, n_theta, n_p) real stack plus geometry (pipeline.py:35-54)."""

    data: np.ndarray
    geometry: ScanGeometry

    def __post_init__(self):
        # float32 / float64 arrays (and memory maps of volume files) are kept
        # as they are -- a 512-slice 2048 x 1536 stack is 6.4 GB in float32;
        # anything else becomes float64 like the reference's
        d = self.data
        if not (isinstance(d, np.ndarray) and d.dtype in (np.float32, np.float64)):
            d = np.asarray(d, dtype=np.float64)
        if d.ndim != 3:
            raise ShapeMismatchError(f"sinogram stack must be 3D, got {d.shape}")
        want = (self.geometry.n_z,) + tuple(self.geometry.sino_shape)
        if d.shape != want:
            raise ShapeMismatchError(f"sinogram stack shape {d.shape} != geometry {want}")
        object.__setattr__(self, "data", d)

    @property
    def n_z(self) -> int:
        return self.data.shape[0]


@dataclass(frozen=True)
class TomogramStack:
    """(n_z, n_y, n_x) real stack (pipeline.py:57-71)."""

    data: np.ndarray

    def __post_init__(self):
        d = np.asarray(self.data)
        if d.ndim != 3:
            raise ShapeMismatchError(f"tomogram stack must be 3D, got {d.shape}")
        object.__setattr__(self, "data", d)

    @property
    def n_z(self) -> int:
        return self.data.shape[0]


@dataclass(frozen=True)
class ChunkPlan:
    """Passes x workers -> (start, length), in order (pipeline.py:74-94)."""

    worker_count: int
    max_slices_per_worker_pass: int
    passes: tuple
    halo: int = 0

    @property
    def n_passes(self) -> int:
        return len(self.passes)

    def nonempty_ranges(self):
        return [r for row in self.passes for r in row if r[1] > 0]


def plan_chunks(n_z: int, workers: int, max_per_pass: int = 8) -> ChunkPlan:
    """ceil(n_z / (workers*max_per_pass)) passes; inside a pass lengths differ
    by at most one and the short ones trail (pipeline.py:97-119)."""
    for name, v, lo in (("n_z", n_z, 1), ("workers", workers, 1), ("max_per_pass", max_per_pass, 1)):
        if v < lo:
            raise ValueError(f"{name} must be >= {lo}, got {v}")
    cap = workers * max_per_pass
    rows, cursor = [], 0
    for _ in range(math.ceil(n_z / cap)):
        todo = min(cap, n_z - cursor)
        q, r = divmod(todo, workers)
        row = []
        for w in range(workers):
            ln = q + (w < r)
            row.append((cursor, ln))
            cursor += ln
        rows.append(tuple(row))
    return ChunkPlan(worker_count=workers, max_slices_per_worker_pass=max_per_pass,
                     passes=tuple(rows))


def pair_complex(a, b) -> np.ndarray:
    """a + i b (pipeline.py:122-128)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ShapeMismatchError(f"pair shapes differ: {a.shape} vs {b.shape}")
    return a + 1j * b


def unpair(u):
    """(Re u, Im u) as contiguous real arrays (pipeline.py:131-134)."""
    u = np.asarray(u)
    return np.ascontiguousarray(u.real), np.ascontiguousarray(u.imag)


# ------------------------------------------------------------------ helpers


def unit_slices(u0: int, ulen: int, n_z: int):
    """Slice range [lo, hi) covered by pair units [u0, u0+ulen)."""
    return 2 * u0, min(2 * (u0 + ulen), n_z)


def rank_ranges(n_units: int, world: int):
    """Contiguous pair-unit range per rank: plan_chunks semantics in one pass
    (equal lengths, trailing ranks one shorter)."""
    per = max(1, math.ceil(n_units / world))
    return list(plan_chunks(n_units, world, per).passes[0])


def _failure(stat, n_units, n_z, workers, max_per_pass, causes):
    """First failing unit -> WorkerFailureError over the task holding it
    (pipeline.py:166-176, 215-217)."""
    bad = [u for u in range(n_units) if stat[u] != 0]
    if not bad:
        return None
    u = bad[0]
    plan = plan_chunks(n_units, workers, max(1, max_per_pass // 2))
    for start, ln in plan.nonempty_ranges():
        if start <= u < start + ln:
            return WorkerFailureError(unit_slices(start, ln, n_z), causes.get(u, "failed"))
    return WorkerFailureError(unit_slices(u, 1, n_z), causes.get(u, "failed"))


def _cause(code: int, algo: str) -> str:
    from . import _lib
    name = {_lib.ERR_DIVERGENCE: "DivergenceError", _lib.ERR_NONFINITE: "NonFiniteError"}.get(
        code, "SptomoError")
    return f"{name}('{algo} failed on the device (status {code})')"


def _device_solver(ops, cfg):
    """(slices tensor/array (k, T, P)) -> (rec, final residual, iters, conv, status) per unit."""
    from .solvers import solve_batch

    def run(data, out=None):
        rec, reps, stat = solve_batch(data, ops, cfg, raise_on_failure=False, out=out)
        final = [r.residual_history[-1] if r.residual_history else 0.0 for r in reps]
        iters = [r.iterations_run for r in reps]
        conv = [r.converged for r in reps]
        return rec, final, iters, conv, stat
    run.batch_units = ops.plan.max_batch
    return run


def run_pipeline(stack: SinogramStack, cfg, workers: int = 1, ops=None, max_per_pass: int = 8,
                 *, group=None, solver=None, out=None):
    """Reconstruct every slice (pipeline.py:179-235).

    Single process: all pair units go through the device solver in batches
    (``workers`` / ``max_per_pass`` only define the task ranges reported by
    WorkerFailureError, exactly as in the reference).  Under an initialised
    torch.distributed group of size G > 1, rank r solves its contiguous unit
    range on its own GPU:

    * input: when every rank passes the stack (e.g. a memory map of the same
      SPTOMO01 file), each rank copies only its own slices host -> device over
      its own PCIe link; otherwise rank 0's stack is scattered with NCCL
      point-to-point sends (other ranks may pass ``stack=None``);
    * output: when every rank passes ``out`` (a host (n_z, n_y, n_x) array all
      ranks can write, e.g. a memory-mapped output volume), each rank writes
      its own slices device -> host; otherwise the slices are gathered to
      rank 0 over NCCL.

    Rank 0 returns the assembled stack (``out`` when given); other ranks
    return ``(None, report)``.  ``solver`` overrides the per-rank solve (used
    by the CPU multi-process tests).
    """
    t0 = time.perf_counter()
    dist = _dist_group(group)
    if dist is None:
        if stack is None:
            raise ValueError("run_pipeline needs a stack outside a process group")
        geom = stack.geometry
        if ops is None and solver is None:
            from .operators import build_operators
            ops = build_operators(geom, filter_kind=cfg.filter_kind())
        solve_fn = solver or _device_solver(ops, cfg)
        n_z = stack.n_z
        n_units = (n_z + 1) // 2
        direct = solver is None and isinstance(stack.data, np.ndarray) and _cuda_ok()
        if direct:
            # host stack on a GPU: chunked, copies overlapped with the solve,
            # results straight into ``out`` (e.g. a memory-mapped volume) or a
            # new float64 stack
            import torch
            dev = torch.device("cuda", torch.cuda.current_device())
            f64 = ops.plan.precision == _f64_precision()
            dt = torch.float64 if f64 else torch.float32
            Y, X = geom.grid_shape
            dst = out if out is not None else np.empty((n_z, Y, X), dtype=np.float64)
            chunk = 2 * _stream_units(solve_fn)
            final, iters, conv, stat = _streamed(stack.data, 0, n_z, solve_fn, dev, dt, chunk,
                                                 _host_sink(dst, dev, dt, chunk, (Y, X)))
            rec = dst
        else:
            rec, final, iters, conv, stat = solve_fn(stack.data)
        bad = [u for u in range(n_units) if stat[u] != 0]
        if bad and workers == 1:
            # one worker: the reference solves in-process, so the solver's own
            # exception reaches the caller (pipeline.py:201-204)
            from .solvers import _EXC
            u = bad[0]
            lo, hi = unit_slices(u, 1, n_z)
            raise _EXC.get(stat[u], RuntimeError)(
                f"{cfg.algorithm} failed on slices [{lo}, {hi}) (device status {stat[u]})")
        err = _failure(stat, n_units, n_z, workers, max_per_pass,
                       {u: _cause(stat[u], cfg.algorithm) for u in range(n_units)})
        if err is not None:
            raise err
        if out is not None:
            if not direct:
                out[...] = np.asarray(rec.cpu().numpy() if hasattr(rec, "cpu") else rec)
            vol = out
        elif direct:
            vol = rec
        else:
            vol = np.asarray(rec.cpu().numpy() if hasattr(rec, "cpu") else rec, dtype=np.float64)
        from .solvers import SolverReport
        rep = SolverReport(residual_history=[float(f) for f in final],
                           iterations_run=int(max(iters)) if iters else 0,
                           converged=all(conv), wall_time=time.perf_counter() - t0)
        return TomogramStack(data=vol), rep
    if ops is None and solver is None:
        from .operators import build_operators
        ops = build_operators(stack.geometry if stack is not None else _bcast_geometry(None, dist),
                              filter_kind=cfg.filter_kind())
    solve_fn = solver or _device_solver(ops, cfg)
    f64 = ops is not None and ops.plan.precision == _f64_precision()
    return _run_distributed(stack, cfg, solve_fn, dist, t0, workers, max_per_pass, f64, out)


def _cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def _stream_units(solve_fn):
    """Units (complex pairs) per streamed chunk: the solver's launch batch."""
    return max(1, int(getattr(solve_fn, "batch_units", 32)))


def _f64_precision():
    from . import _lib
    return _lib.PREC_F64


def _dist_group(group):
    try:
        import torch.distributed as tdist
    except Exception:
        return None
    if not (tdist.is_available() and tdist.is_initialized()):
        return None
    if tdist.get_world_size(group) <= 1:
        return None
    return group if group is not None else tdist.group.WORLD


def _bcast_geometry(stack, group):
    """Rank 0's (n_z, n_theta, n_p, n_y, n_x, center) and angles to every rank."""
    import torch
    import torch.distributed as tdist
    dev = _dist_device(group)
    hdr = torch.zeros(6, dtype=torch.float64, device=dev)
    if tdist.get_rank(group) == 0:
        g = stack.geometry
        hdr[:] = torch.tensor([stack.n_z, g.n_theta, g.n_p, g.n_y, g.n_x, g.center], dtype=torch.float64)
    tdist.broadcast(hdr, _root(group), group)
    n_z, T, P, Y, X, c = hdr.tolist()
    ang = torch.empty(int(T), dtype=torch.float64, device=dev)
    if tdist.get_rank(group) == 0:
        ang.copy_(torch.as_tensor(np.asarray(stack.geometry.angles, dtype=np.float64)))
    tdist.broadcast(ang, _root(group), group)
    return ScanGeometry(n_p=int(P), n_theta=int(T), angles=ang.cpu().numpy(), n_z=int(n_z), n_x=int(X),
                        n_y=int(Y), center=float(c))


def _root(group):
    import torch.distributed as tdist
    return tdist.get_global_rank(group, 0) if group is not None and group != tdist.group.WORLD else 0


def _dist_device(group):
    import torch
    import torch.distributed as tdist
    if tdist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _h2d(host, lo, hi, dtype, dev):
    """Slices [lo, hi) of a host stack -> device tensor (pinned staging)."""
    import torch
    part = np.ascontiguousarray(host[lo:hi], dtype=np.float64 if dtype == torch.float64 else np.float32)
    t = torch.from_numpy(part)
    if dev.type == "cuda":
        return t.pin_memory().to(dev, non_blocking=True)
    return t.clone()


def _streamed(host, lo, hi, solve_fn, dev, dt, chunk, sink):
    """Solve slices [lo, hi) of a host stack chunk by chunk with the copies
    off the critical path: the next chunk's host -> pinned -> device copy and
    the previous chunk's device -> host store run on side streams from two
    helper threads while the current chunk is solved (the ctypes call
    releases the GIL).  ``sink(a, b, rec)`` receives each chunk's device
    result on the helper thread after its solve.  Returns the per-unit
    (final, iters, conv, stat) lists in slice order."""
    import concurrent.futures as cf
    import torch
    np_dt = np.float64 if dt == torch.float64 else np.float32
    bounds = [(a, min(a + chunk, hi)) for a in range(lo, hi, chunk)]
    T, P = host.shape[1:]
    pins = [torch.empty((min(chunk, hi - lo), T, P), dtype=dt, pin_memory=True) for _ in range(2)]
    h2d = torch.cuda.Stream(dev)
    cur = torch.cuda.current_stream(dev)

    def load(i):  # helper thread: its CUDA device must be set explicitly
        a, b = bounds[i]
        buf = pins[i % 2][: b - a]
        np.copyto(buf.numpy(), np.asarray(host[a:b]), casting="same_kind")
        with torch.cuda.device(dev), torch.cuda.stream(h2d):
            d = buf.to(dev, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(h2d)
        return d, ev

    meta = ([], [], [], [])
    stores = []
    with cf.ThreadPoolExecutor(1) as ex_in, cf.ThreadPoolExecutor(1) as ex_out:
        nxt = ex_in.submit(load, 0)
        for i, (a, b) in enumerate(bounds):
            d, ev = nxt.result()
            if i + 1 < len(bounds):
                nxt = ex_in.submit(load, i + 1)
            cur.wait_event(ev)
            rec, final, iters, conv, stat = solve_fn(d)
            for acc, v in zip(meta, (final, iters, conv, stat)):
                acc.extend(v)
            done = torch.cuda.Event()
            done.record(cur)
            if len(stores) >= 2:
                stores[-2].result()  # bound the results in flight
            stores.append(ex_out.submit(sink, a, b, rec, done))
        for f in stores:
            f.result()
    return meta


def _host_sink(out, dev, dt, chunk, T_shape):
    """sink for _streamed: device result -> pinned -> host volume ``out``."""
    import torch
    d2h = torch.cuda.Stream(dev)
    # two buffers: _streamed keeps at most two stores in flight
    pins = [torch.empty((chunk,) + tuple(T_shape), dtype=dt, pin_memory=True) for _ in range(2)]
    count = [0]

    def sink(a, b, rec, done):  # helper thread
        buf = pins[count[0] % 2][: b - a]
        count[0] += 1
        with torch.cuda.device(dev), torch.cuda.stream(d2h):
            d2h.wait_event(done)
            buf.copy_(rec, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(d2h)
        ev.synchronize()
        out[a:b] = buf.numpy()
    return sink


def _run_distributed(stack, cfg, solve_fn, group, t0, workers, max_per_pass, f64=False, out=None):
    import torch
    import torch.distributed as tdist

    from .solvers import SolverReport

    rank, world = tdist.get_rank(group), tdist.get_world_size(group)
    root = _root(group)
    dev = _dist_device(group)
    dt = torch.float64 if f64 else torch.float32
    # every rank learns the geometry and which side holds the data
    flags = torch.tensor([1.0 if stack is not None else 0.0, 1.0 if out is not None else 0.0],
                         dtype=torch.float64, device=dev)
    tdist.all_reduce(flags, op=tdist.ReduceOp.MIN, group=group)
    local_in, local_out = flags[0].item() > 0, flags[1].item() > 0
    geom = stack.geometry if local_in else _bcast_geometry(stack, group)
    n_z = stack.n_z if local_in else geom.n_z
    n_units = (n_z + 1) // 2
    T, P = geom.sino_shape
    Y, X = geom.grid_shape
    ranges = rank_ranges(n_units, world)
    spans = [unit_slices(u0, ul, n_z) if ul > 0 else (0, 0) for u0, ul in ranges]
    lo, hi = spans[rank]

    # ---- input: own range over this rank's PCIe link, or rank 0 -> ranks over NCCL
    streamed = local_in and dev.type == "cuda" and isinstance(stack.data, np.ndarray)
    if streamed:
        # copies overlapped with the solve, chunk by chunk (results either
        # straight to ``out`` or into this rank's device range for the gather)
        mine = None
    elif local_in:
        mine = _h2d(stack.data, lo, hi, dt, dev)
    else:
        mine = torch.empty((hi - lo, T, P), dtype=dt, device=dev)
        ops_ = []
        if rank == 0:
            for r in range(1, world):
                a, b = spans[r]
                if b > a:
                    ops_.append(tdist.P2POp(tdist.isend, _h2d(stack.data, a, b, dt, dev),
                                            tdist.get_global_rank(group, r) if group is not tdist.group.WORLD else r,
                                            group))
            mine.copy_(_h2d(stack.data, lo, hi, dt, dev))
        elif hi > lo:
            ops_.append(tdist.P2POp(tdist.irecv, mine, root, group))
        if ops_:
            for w in tdist.batch_isend_irecv(ops_):
                w.wait()

    # ---- solve (no collective inside)
    ul = ranges[rank][1]
    if ul > 0 and streamed:
        chunk = 2 * _stream_units(solve_fn)
        if local_out:
            sink = _host_sink(out, dev, dt, chunk, (Y, X))
            rec = None
        else:
            rec = torch.empty((hi - lo, Y, X), dtype=dt, device=dev)

            def sink(a, b, r, done, _rec=rec):  # helper thread
                with torch.cuda.device(dev):
                    torch.cuda.current_stream(dev).wait_event(done)
                    _rec[a - lo:b - lo].copy_(r)
        final, iters, conv, stat = _streamed(stack.data, lo, hi, solve_fn, dev, dt, chunk, sink)
        if rec is None:
            rec = torch.empty((0, Y, X), dtype=dt, device=dev)
    elif ul > 0:
        rec, final, iters, conv, stat = solve_fn(mine)
        rec = torch.as_tensor(rec, device=dev).to(dt)
    else:
        rec = torch.empty((0, Y, X), dtype=dt, device=dev)
        final, iters, conv, stat = [], [], [], []
    meta = torch.tensor([[f, i, float(c), float(s)] for f, i, c, s in zip(final, iters, conv, stat)],
                        dtype=torch.float64, device=dev).reshape(-1, 4)

    # ---- output: own range device -> host, or ranks -> rank 0 over NCCL
    vol = None
    if local_out and not streamed:
        if hi > lo:
            out[lo:hi] = rec.cpu().numpy()
    ops_ = []
    metas = [None] * world
    if rank == 0:
        if not local_out:
            vol = torch.empty((n_z, Y, X), dtype=dt, device=dev)
            vol[lo:hi].copy_(rec)
        metas[0] = meta
        for r in range(1, world):
            a, b = spans[r]
            if b > a:
                src = tdist.get_global_rank(group, r) if group is not tdist.group.WORLD else r
                if not local_out:
                    ops_.append(tdist.P2POp(tdist.irecv, vol[a:b], src, group))
                metas[r] = torch.empty((ranges[r][1], 4), dtype=torch.float64, device=dev)
                ops_.append(tdist.P2POp(tdist.irecv, metas[r], src, group))
    elif hi > lo:
        if not local_out:
            ops_.append(tdist.P2POp(tdist.isend, rec.contiguous(), root, group))
        ops_.append(tdist.P2POp(tdist.isend, meta, root, group))
    if ops_:
        for w in tdist.batch_isend_irecv(ops_):
            w.wait()
    if local_out:
        tdist.barrier(group)  # every rank's slices are in ``out``

    # ---- failure decision is shared so every rank raises the same error
    flag = torch.zeros(3, dtype=torch.float64, device=dev)
    if rank == 0:
        allm = torch.cat([m for m in metas if m is not None]).cpu().numpy()
        stat_all = allm[:, 3].astype(int)
        bad = np.flatnonzero(stat_all)
        if bad.size:
            u = int(bad[0])
            r = next(i for i, (u0, ln) in enumerate(ranges) if u0 <= u < u0 + ln)
            flag[0], flag[1], flag[2] = 1.0, float(r), float(stat_all[u])
    tdist.broadcast(flag, root, group)
    if flag[0].item() > 0:
        r = int(flag[1].item())
        raise WorkerFailureError(spans[r], _cause(int(flag[2].item()), cfg.algorithm))
    if rank != 0:
        return None, SolverReport(wall_time=time.perf_counter() - t0)
    rep = SolverReport(residual_history=[float(v) for v in allm[:, 0]],
                       iterations_run=int(allm[:, 1].max()) if len(allm) else 0,
                       converged=bool(np.all(allm[:, 2] > 0)),
                       wall_time=time.perf_counter() - t0)
    data = out if local_out else vol.cpu().numpy().astype(np.float64)
    return TomogramStack(data=data), rep
