import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2602_07616_b200 import build
from paper_2602_07616_b200.moe import route_topk_device
build.build()
M, d_h, K = 128, 2048, 8
w = (torch.randn(M, d_h, device="cuda") / 45).to(torch.bfloat16)
for T in (16, 64, 128, 512):
    x = torch.randn(T, d_h, device="cuda").to(torch.bfloat16)
    ids = torch.empty(T, K, dtype=torch.int32, device="cuda"); wt = torch.empty(T, K, device="cuda")
    for _ in range(5): route_topk_device(w, x, K, out=(ids, wt))
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(50): route_topk_device(w, x, K, out=(ids, wt))
    e.record(); torch.cuda.synchronize()
    print(f"T={T}: {s.elapsed_time(e) / 50 * 1e3:.1f} us per call (incl. python launch)")
# graph-captured
x = torch.randn(512, d_h, device="cuda").to(torch.bfloat16)
ids = torch.empty(512, K, dtype=torch.int32, device="cuda"); wt = torch.empty(512, K, device="cuda")
g = torch.cuda.CUDAGraph()
route_topk_device(w, x, K, out=(ids, wt)); torch.cuda.synchronize()
with torch.cuda.graph(g):
    for _ in range(20): route_topk_device(w, x, K, out=(ids, wt))
g.replay(); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); g.replay(); e.record(); torch.cuda.synchronize()
print(f"graph T=512: {s.elapsed_time(e) / 20 * 1e3:.1f} us per router")
from paper_2602_07616_b200 import _lib
import numpy as np
dbg = torch.zeros(4096 * 8, dtype=torch.int64, device="cuda")
_lib.load().sere_debug_set_route_clocks(dbg.data_ptr())
route_topk_device(w, x, K, out=(ids, wt)); torch.cuda.synchronize()
_lib.load().sere_debug_set_route_clocks(None)
c = dbg.view(-1, 8)[: 32 * 8].cpu().numpy()
c = c[c[:, 0] > 0]
base = c[:, 0].min()
print("phase clocks rel (first 10 CTAs):")
print((c[:10] - base) // 1)
order = [0, 1, 2, 3, 4, 6, 7, 5]
lead = c[c[:, 6] > 0][:, order]
print("phase order", order, "deltas (cycles, CTAs with tokens):", np.diff(lead, axis=1).mean(axis=0).round())
