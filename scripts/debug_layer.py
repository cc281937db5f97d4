"""Locate wrong outputs of the layer kernel: per-config max error and where it sits."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch
from paper_2602_07616_b200.moe import ExpertBank, layer_forward_device
from test_gpu_layer import _torch_layer_ref

def run(M, K, ns, d_h, d_m, T, beta):
    g = torch.Generator(device="cuda"); g.manual_seed(7)
    bank = ExpertBank.random(M, ns, d_h, d_m, seed=11)
    x = torch.randn(T, d_h, device="cuda", generator=g).to(torch.bfloat16)
    logits = torch.randn(T, M, device="cuda", generator=g) + beta * torch.randn(M, device="cuda", generator=g)
    top = torch.topk(logits, K, dim=1)
    ids = top.indices.to(torch.int32); w = torch.softmax(top.values, dim=1)
    out = layer_forward_device(bank, x, ids, w); out.check()
    ref = _torch_layer_ref(bank, x, ids.long(), w)
    err = (out.y - ref).abs()
    bad = err > 1e-2
    cnt = torch.bincount(ids.flatten().long(), minlength=M)
    rows_bad = bad.any(1).nonzero().flatten().tolist()
    feats_bad = bad.any(0).nonzero().flatten().tolist()
    print(f"M{M} K{K} ns{ns} {d_h}x{d_m} T{T} b{beta}: max {err.max().item():.3e}, bad tokens {len(rows_bad)}, "
          f"bad feats {len(feats_bad)} {feats_bad[:8]}..{feats_bad[-4:] if feats_bad else ''}; max count {cnt.max().item()}")

for cfg in [(64, 6, 0, 2048, 1408, 256, 1.0), (64, 6, 0, 2048, 1408, 64, 0.0), (64, 6, 0, 2048, 1280, 64, 0.0),
            (64, 6, 0, 2048, 1024, 64, 0.0), (64, 6, 0, 2048, 768, 64, 0.0), (64, 6, 0, 1024, 1408, 64, 0.0),
            (128, 8, 0, 2048, 768, 512, 2.0), (16, 8, 0, 1024, 512, 512, 0.0), (4, 2, 0, 1024, 512, 300, 0.0)]:
    run(*cfg)
