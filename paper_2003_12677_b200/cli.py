"""``recon`` on the B200 operators (the reference's ``sptomo recon``,
cli.py:66-81,129-161): SPTOMO01 sinogram volume in, tomogram volume out.

    python -m paper_2003_12677_b200 recon --in SINO --out TOMO [--algo sirt]
        [--iters K] [--filter F] [--center C] [--kernel kb|gauss] [--kw W]
        [--cache DIR] [--workers P] [--metrics-out JSON] [--seed S]

Same flags, exit codes (0 ok, 2 error, messages on stderr as
``error: ...``), file format and metrics record as the reference's command
(results within the operators' and solvers' parity bars).  The volume is
never loaded whole: the input is memory-mapped and the output written into a
pre-sized memory-mapped file, so each GPU copies only its slices.  Under
``torchrun --nproc-per-node N`` every rank maps both files, reconstructs its
contiguous slice range on its own GPU and writes it in place (run_pipeline,
no data-path collective); rank 0 renames the finished file.  Intensity
volumes are converted to line integrals -log(I / I0) (I0 = 1, counts clamped
at 1e-9 max I) slice range by slice range, as the reference's normalize
does (io.py:92-106).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

EXIT_OK = 0
EXIT_ERROR = 2
CLAMP_EPS_REL = 1e-9


def build_parser() -> argparse.ArgumentParser:
    from .operators import FILTER_KINDS
    from .solvers import ALGORITHMS
    ap = argparse.ArgumentParser(prog="paper_2003_12677_b200",
                                 description="B200 sparse-matrix tomography (recon)")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("recon", help="reconstruct a sinogram volume")
    p.add_argument("--in", dest="infile", required=True, metavar="FILE")
    p.add_argument("--out", required=True, metavar="FILE")
    p.add_argument("--algo", choices=ALGORITHMS, default="fbp")
    p.add_argument("--iters", type=int, default=10, metavar="K")
    p.add_argument("--filter", choices=FILTER_KINDS, default=None,
                   help="Fourier filter (default: the algorithm's)")
    p.add_argument("--center", type=float, default=None, metavar="C",
                   help="rotation centre override (default: the file's)")
    p.add_argument("--workers", type=int, default=1, metavar="P",
                   help="task ranges for failure reports (the GPUs are the workers)")
    p.add_argument("--cache", default=None, metavar="DIR",
                   help="SGCSR001 matrix cache (default $SPTOMO_CACHE_DIR)")
    p.add_argument("--metrics-out", default=None, metavar="FILE")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--kernel", choices=("kb", "gauss"), default="kb")
    p.add_argument("--kw", type=int, default=3, metavar="W")
    return ap


def _line_integrals(vol):
    """Intensity volume -> line integrals -log(max(I, 1e-9 max I)) (flat
    field 1), slice by slice (two passes over the mapped payload)."""
    from .errors import InvalidFlatFieldError
    peak = 0.0
    for z in range(vol.data.shape[0]):
        peak = max(peak, float(np.max(vol.data[z])))
    clamp = CLAMP_EPS_REL * peak
    if clamp <= 0:
        raise InvalidFlatFieldError("intensity stack has no positive counts")
    out = np.empty(vol.data.shape, dtype=np.float64)
    for z in range(vol.data.shape[0]):
        out[z] = -np.log(np.maximum(np.asarray(vol.data[z], dtype=np.float64), clamp))
    return out


def _dist():
    try:
        import torch.distributed as tdist
    except Exception:
        return None
    if int(os.environ.get("WORLD_SIZE", "1")) <= 1:
        return None
    if not tdist.is_initialized():
        import torch
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return tdist


def cmd_recon(args) -> int:
    from . import io as vio
    from .errors import SptomoError
    from .geometry import KernelSpec, ScanGeometry
    from .operators import build_operators
    from .pipeline import SinogramStack, run_pipeline
    from .solvers import SolverConfig

    if not os.path.isfile(args.infile):
        raise SptomoError(f"input file not found: {args.infile}")
    vol = vio.read_volume(args.infile)
    if vol.kind == vio.KIND_TOMOGRAM:
        raise SptomoError(f"{args.infile}: expected a sinogram or intensity volume, found a tomogram")
    data = vol.data if vol.kind == vio.KIND_SINOGRAM else _line_integrals(vol)
    n_z, n_a, n_b = data.shape
    center = args.center if args.center is not None else vol.center
    geom = ScanGeometry(n_p=n_b, n_theta=n_a, angles=vol.angles, n_z=n_z, center=center)
    cfg = SolverConfig(algorithm=args.algo, max_iter=args.iters, filter=args.filter, seed=args.seed)
    ops = build_operators(geom, kernel=KernelSpec(family=args.kernel, width=args.kw),
                          filter_kind=cfg.filter_kind(),
                          cache_dir=args.cache if args.cache is not None else os.environ.get("SPTOMO_CACHE_DIR"))
    stack = SinogramStack(data=data, geometry=geom)
    tdist = _dist()
    rank = tdist.get_rank() if tdist else 0
    shape = (n_z,) + geom.grid_shape
    writer = None
    try:
        if rank == 0:
            writer = vio.VolumeWriter(args.out, vio.KIND_TOMOGRAM, shape)
        if tdist:
            tmp = [writer.tmp if writer else None]
            tdist.broadcast_object_list(tmp, src=0)
            out = writer.data if writer else vio.VolumeWriter.attach(tmp[0])
        else:
            out = writer.data
        _, report = run_pipeline(stack, cfg, workers=args.workers, ops=ops, out=out)
        if tdist:
            tdist.barrier()
        if writer is not None:
            writer.close()
    except BaseException:
        if writer is not None:
            writer.abort()
        raise
    if rank == 0:
        if args.metrics_out:
            record = {"algo": args.algo, "iters": report.iterations_run, "snr_db": None,
                      "residual_history": report.residual_history, "wall_time": report.wall_time}
            with open(args.metrics_out, "w") as fh:
                json.dump([record], fh, indent=2)
                fh.write("\n")
        print(f"reconstructed {shape} -> {args.out} (algo={args.algo}, converged={report.converged})")
    return EXIT_OK


def main(argv=None) -> int:
    from .errors import SptomoError
    args = build_parser().parse_args(argv)
    try:
        return {"recon": cmd_recon}[args.command](args)
    except (SptomoError, OSError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_ERROR
