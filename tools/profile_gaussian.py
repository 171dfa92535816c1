"""Runs one 4-axis gaussian_filter on the 4D volume (float64) for ncu launch lists."""
import torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_1906_11355_b200 as M
from paper_1906_11355_b200 import datasets
x = datasets.make("4d", seed=0, device="cuda").to(torch.float64)
M.gaussian_filter(x, M.GaussianSpec((1.0, 1.0, 1.0, 1.0)))
torch.cuda.synchronize()
