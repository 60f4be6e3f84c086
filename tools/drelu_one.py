"""One D-ReLU launch per shape (for ncu): python tools/drelu_one.py n D k [tpr]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2508_16769_b200 as dr

n, D, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dr.debug_set("drelu_tpr", int(sys.argv[4]) if len(sys.argv) > 4 else 1)
x = torch.randn(n, D, device="cuda")
for _ in range(3):
    dr.drelu_topk(x, k)
torch.cuda.synchronize()
