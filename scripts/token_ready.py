"""How early could each token be combined? For the last layer of a C4 step: for every token, the
last down-unit ticket among its slots' groups, against the FFN's total ticket count (the combine
could start a token once that ticket's unit is done)."""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2602_07616_b200 import build
from paper_2602_07616_b200 import _lib
from paper_2602_07616_b200.decode import DecodeModel, DecodeStep

build.build()
T, K, Et = 512, 8, 128
for seed in range(3):
    model = DecodeModel(3, 128, 8, 2048, 768, seed=seed, beta=1.0)
    step = DecodeStep(model, T, 1, 0.5, "sere")
    step.set_input(torch.randn(T, 2048, device="cuda", generator=torch.Generator(device="cuda").manual_seed(seed)))
    step.run()
    torch.cuda.synchronize()
    ws_ptr, ws_bytes = step.workspace
    lay = _lib.workspace_layout(T, K, 128, 0, 2048, 768)
    ws = step.ws.view(torch.int32)
    base = (ws_ptr + 1023) // 1024 * 1024 - ws_ptr
    plan = ws[(base + lay.off_plan_i32) // 4:].cpu().numpy()
    slot_row = ws[(base + lay.off_slot_row) // 4:(base + lay.off_slot_row) // 4 + T * K].cpu().numpy().reshape(T, K)
    o_cnt = 16
    o_ge, o_r0, o_rows = o_cnt + Et, o_cnt + 2 * Et, o_cnt + 3 * Et
    o_sched, o_ugu, o_udn = o_cnt + 4 * Et, o_cnt + 5 * Et, o_cnt + 6 * Et + 1
    G, units_gu, units_dn = plan[1], plan[3], plan[4]
    row0 = plan[o_r0:o_r0 + G]
    rows = plan[o_rows:o_rows + G]
    sched = plan[o_sched:o_sched + G]
    udn = plan[o_udn:o_udn + G + 1]
    pos_of = np.empty(G, int)
    pos_of[sched] = np.arange(G)
    last_ticket = units_gu + udn[pos_of + 1] - 1  # per group g
    grp_of_row = np.full(row0.max() + 512, -1)
    for g in range(G):
        grp_of_row[row0[g]:row0[g] + rows[g]] = g
    ready = np.array([last_ticket[grp_of_row[slot_row[t]]].max() for t in range(T)])
    total = units_gu + units_dn
    q = np.percentile(ready, [10, 50, 90, 100])
    print(f"seed {seed}: groups {G}, tickets gu {units_gu} dn {units_dn}; token-ready ticket p10/p50/p90/max "
          f"{q.astype(int)}; tokens ready before the last 148 tickets: {(ready < total - 148).mean():.2f}, "
          f"before the last 296: {(ready < total - 296).mean():.2f}")
