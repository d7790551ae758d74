"""Co-resident cluster capacity of the cluster split-K GEMM for each cluster size (B200)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2512_23858_b200 import _lib as L
from paper_2512_23858_b200.forward import GemmPlan

L.require_device()
for N, K, M in ((6144, 4096, 50), (4096, 4096, 50), (4096, 14336, 50), (28672, 4096, 50)):
    W = torch.zeros(N, K, dtype=torch.bfloat16, device="cuda")
    X = torch.zeros(M, K, dtype=torch.bfloat16, device="cuda")
    p = GemmPlan(W, X, M, 0)
    out = []
    for cs in range(1, 9):
        rc = L.lib().ygg_gemm_plan_set_cluster(p.handle, cs)
        out.append((cs, rc, L.lib().ygg_last_error().decode() if rc else "ok"))
    print(N, K, M, "tiles", p.tiles, out)
