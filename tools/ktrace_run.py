import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from conftest import payload_path
from paper_2010_14962_b200 import Engine
import torch
stem = sys.argv[1]
with Engine(payload_path(stem), device=0, mode="ket") as e:
    for i in range(4):
        e.bench(1, 0, 2 ** e.plan_stats()["n_cut"])
    flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda:0")
    flush.fill_(1.0); torch.cuda.synchronize()
    print("KT ==== last", flush=True)
    e.bench(1, 0, 2 ** e.plan_stats()["n_cut"])
