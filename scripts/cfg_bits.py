"""Dump a layer's output for the current build (compare across compile-time variants)."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2602_07616_b200 import build
from paper_2602_07616_b200.moe import ExpertBank, layer_forward_device
build.build()
g = torch.Generator(device="cuda"); g.manual_seed(7)
bank = ExpertBank.random(128, 0, 2048, 768, seed=11)
x = torch.randn(512, 2048, device="cuda", generator=g).to(torch.bfloat16)
logits = torch.randn(512, 128, device="cuda", generator=g) + torch.randn(128, device="cuda", generator=g)
top = torch.topk(logits, 8, dim=1)
out = layer_forward_device(bank, x, top.indices.to(torch.int32), torch.softmax(top.values, 1))
out.check()
np.save(sys.argv[1], out.y.cpu().numpy())
