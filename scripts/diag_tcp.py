"""Effective precision of the wide tensor paths (pre-split contract_tcp vs the
converter contract_tcw): the smallest relative tie zone that explains each
direction's count difference against FP64."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2506_08262_b200 as b200  # noqa: E402

b200.load_library()
eng = b200.engine()
for d in [65, 72, 100, 200]:
    rng = np.random.default_rng(300 + d)
    X = rng.standard_normal((4096 + 77, d)) * rng.uniform(0.1, 10.0, size=d)
    U = rng.standard_normal((200, d))
    U /= np.linalg.norm(U, axis=1)[:, None]
    data = b200.Dataset(X)
    xn = np.linalg.norm(X, axis=1)
    for zi, z in enumerate((X[5], X[9] + 1e-4 * rng.standard_normal(d), np.full(d, 0.2))):
        y = X @ U.T - (U @ z)[None, :]
        scale = np.maximum(xn, np.linalg.norm(z))[:, None]
        rle = (y <= 0).sum(axis=0)
        out = []
        for path in ("tensor", "convert", "ffma"):
            eng.set_contract_path(path)
            _, cle, cge = b200.evaluate_directions_counts(z, data, U)
            # per direction: the tolerance needed = the |y|/scale of the k-th smallest, k = |diff|
            need = 0.0
            r = np.abs(y) / scale
            for j in np.nonzero(cle != rle)[0]:
                k = abs(int(cle[j] - rle[j]))
                need = max(need, np.sort(r[:, j])[k - 1])
            out.append(f"{path}: dirs off {int((cle != rle).sum())}, max |diff| {int(np.abs(cle - rle).max())}, "
                       f"tol needed {need:.2e}")
        print(f"d={d} z{zi}: " + " | ".join(out), flush=True)
eng.set_contract_path("auto")
