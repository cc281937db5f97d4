"""Wall time of the GPU similarity calibration at the C4 layer shape (1 layer, 2 x 512 tokens)."""
import pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2602_07616_b200 import build, calibrate
from paper_2602_07616_b200.decode import DecodeModel

build.build()
model = DecodeModel(1, 128, 8, 2048, 768, seed=0, beta=0.0)
rng = np.random.default_rng(5)
batches = [rng.standard_normal((512, 2048)) for _ in range(2)]
for metric in ("frobenius", "cosine"):
    calibrate.estimate_similarity(model, batches[:1], metric)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sims = calibrate.estimate_similarity(model, batches, metric)
    torch.cuda.synchronize()
    print(f"{metric}: {time.perf_counter() - t0:.3f} s for 1 layer x 2 batches x 512 tokens (128 experts); "
          f"off-diagonal mean {sims[0][~np.eye(128, dtype=bool)].mean():.3f}")
