"""Repeat bench.py's SIRT measurement several times in one process."""
import os, sys, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2003_12677_b200 as sb
from oracle import shepp_logan
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
a = types.SimpleNamespace(slices=64, sirt_iters=12, n_p=2048, n_theta=1536)
geom = sb.ScanGeometry(n_p=2048, n_theta=1536)
ops = sb.build_operators(geom, filter_kind="ramlak", max_batch=32)
ph = torch.tensor(shepp_logan(2048)[0], dtype=torch.float32, device=dev)
sino = ops.radon(ph[None].expand(2, -1, -1).contiguous())[0]
sino = (sino[None] * torch.linspace(1.0, 0.8, 64, device=dev)[:, None, None]).contiguous()
for i in range(4):
    r = bench._sirt_rate(sb, geom, sino, a, dev, stream)
    print(round(r["value"]), round(r["ms_per_iteration"], 3), round(r["setup_ms"], 2), flush=True)
