"""Which wide-kernel shapes disagree with FP64 beyond the tie zone: d values
with a 3-step remainder (last slice rem >= 11) and with one accumulator
(ns = 33, d = 251..255), for the pre-split (tensor) and converter kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2506_08262_b200 as b200  # noqa: E402

b200.load_library()
eng = b200.engine()
for d in [int(v) for v in os.environ.get("DIAG_D", "75,91,139,250,251,253,255").split(",")]:
    rng = np.random.default_rng(300 + d)
    X = rng.standard_normal((4096 + 77, d))
    U = rng.standard_normal((200, d))
    U /= np.linalg.norm(U, axis=1)[:, None]
    data = b200.Dataset(X)
    z = np.full(d, 0.2)
    y = X @ U.T - (U @ z)[None, :]
    T = (np.abs(y) < 1e-6 * np.maximum(np.linalg.norm(X, axis=1), np.linalg.norm(z))[:, None]).sum(axis=0)
    rle = (y <= 0).sum(axis=0)
    out = []
    for path in ("tensor", "convert", "ffma"):
        eng.set_contract_path(path)
        _, cle, _ = b200.evaluate_directions_counts(z, data, U)
        out.append(f"{path}: max|diff|-T {int(np.max(np.abs(cle - rle) - T))}")
    print(d, " | ".join(out), flush=True)
eng.set_contract_path("auto")
