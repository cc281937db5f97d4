"""Compare the gate/up epilogue output (h_pack in the workspace) with a torch reference, per m-tile."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2602_07616_b200 import _lib
from paper_2602_07616_b200.moe import ExpertBank, layer_forward_device, workspace

def run(M, K, d_h, d_m, T, seed=0):
    bank = ExpertBank.random(M, 0, d_h, d_m, seed=seed)
    g = torch.Generator(device="cuda"); g.manual_seed(seed)
    x = torch.randn(T, d_h, device="cuda", generator=g).to(torch.bfloat16)
    ids = torch.stack([torch.randperm(M, device="cuda", generator=g)[:K] for _ in range(T)]).to(torch.int32)
    w = torch.full((T, K), 1.0 / K, device="cuda")
    out = layer_forward_device(bank, x, ids, w); out.check(); torch.cuda.synchronize()
    ws = workspace(T, K, M, 0, d_h, d_m, bank.device)
    L = _lib.workspace_layout(T, K, M, 0, d_h, d_m)
    base = (ws.data_ptr() + 1023) // 1024 * 1024 - ws.data_ptr()
    raw = ws[base:].cpu().numpy()
    plan = raw[L.off_plan_i32:].view(np.int32)
    G = plan[1]
    gexp = plan[L.plan_group_expert_off:L.plan_group_expert_off + G]
    grow0 = plan[L.plan_group_row0_off:L.plan_group_row0_off + G]
    grows = plan[L.plan_group_rows_off:L.plan_group_rows_off + G]
    row_token = raw[L.off_row_token:].view(np.int32)[: L.r_max]
    kt_n = L.d_m_pad // 64
    hp = raw[L.off_h_pack:L.off_h_pack + kt_n * L.r_max * 128].view(np.uint16).reshape(kt_n, L.r_max, 64)
    # unswizzle: physical chunk c' = c ^ (row & 7)
    h = np.zeros((L.r_max, kt_n * 64), dtype=np.float32)
    rows = np.arange(L.r_max)
    for kt in range(kt_n):
        for c in range(8):
            pc = c ^ (rows & 7)
            vals = hp[kt, rows[:, None], pc[:, None] * 8 + np.arange(8)[None, :]]
            h[:, kt * 64 + c * 8: kt * 64 + c * 8 + 8] = (vals.astype(np.uint32) << 16).view(np.float32)
    wg, wu, wd = bank.unpack()
    xf = x.float()
    bad = {}
    for gi in range(G):
        e = gexp[gi]; r0 = grow0[gi]; n = grows[gi]
        toks = torch.as_tensor(row_token[r0:r0 + n].astype(np.int64), device="cuda")
        ref = (torch.nn.functional.silu(xf[toks] @ wg[e].float()) * (xf[toks] @ wu[e].float())).cpu().numpy()
        got = h[r0:r0 + n, :d_m]
        err = np.abs(got - ref).max(axis=0)  # per feature
        scale = np.abs(ref).max() + 1e-6
        badtiles = sorted(set((np.flatnonzero(err > 0.02 * scale) // 64).tolist()))
        if badtiles:
            bad[int(e)] = (int(n), badtiles)
    print(f"M{M} K{K} {d_h}x{d_m} T{T}: groups {G}, bad groups {len(bad)}: {dict(list(bad.items())[:6])}")

run(4, 1, 256, 384, 16)
run(4, 1, 256, 384, 64)
run(8, 2, 512, 1408, 64)
run(64, 6, 2048, 1408, 64)
run(8, 2, 512, 640, 64)
