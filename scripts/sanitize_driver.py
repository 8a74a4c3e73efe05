"""Small-shape driver for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel of the library runs at least once.

    compute-sanitizer --tool memcheck python scripts/sanitize_driver.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2506_08262_b200 as rrs  # noqa: E402
from paper_2506_08262_b200.synthetic import student_t, toeplitz_gaussian  # noqa: E402

rrs.load_library()
eng = rrs.engine()
cases = [
    # (n, d, notion, contract path, select path)
    (4100, 50, "halfspace", "tensor", "auto"),     # contract_tc + cap_generate_v2 + update
    (4100, 50, "halfspace", "filter", "auto"),     # contract_tcf
    (4100, 80, "halfspace", "tensor", "auto"),     # contract_tcp (pre-split) + presplit + coincide_list32
    (4100, 80, "halfspace", "convert", "auto"),    # contract_tcw (in-kernel converters)
    (4100, 200, "halfspace", "tensor", "auto"),    # contract_tcp, four slices, one accumulator pair
    (1000, 5, "halfspace", "ffma", "auto"),        # contract_kernel<count>
    (1000, 300, "halfspace", "auto", "auto"),      # d > 256: contract64 count
    (5000, 300, "projection", "auto", "auto"),     # d > 256: contract64 store
    (5000, 80, "asym_projection", "auto", "auto"),  # contract_tcp STORE (centred pre-split, 64 < d <= 256)
    (5000, 80, "projection", "convert", "auto"),    # contract_tcw STORE
    (5000, 40, "projection", "tensor", "auto"),    # contract_tc STORE + select v3<256>
    (5000, 40, "asym_projection", "tensor3", "auto"),  # contract_tcs (three-term store)
    (20000, 20, "asym_projection", "ffma", "auto"),  # contract_kernel<store> + select v3<512>
    (20000, 20, "projection", "ffma", "wide"),     # select v3<1024>
    (5000, 20, "projection", "ffma", "radix"),     # select v2<256, smem>
    (60000, 7, "projection", "ffma", "auto"),      # select v5 (rows past shared memory)
    (60000, 7, "projection", "ffma", "radix"),     # select v2<1024, global>
    (60001, 7, "asym_projection", "ffma", "radix"),  # select_kernel (legacy, unaligned rows)
    (500, 30, "projection", "auto", "auto"),       # store64 (FP64 centred store)
]
for n, d, notion, path, sel in cases:
    X = toeplitz_gaussian(d, n, seed=1) if notion == "halfspace" else student_t(d, n, 1.0, seed=1)
    try:
        data = rrs.Dataset(X)
        eng.set_contract_path(path)
        eng.set_select_path(sel)
        cfg = rrs.RrsConfig(total_directions=256, refinements=2, shrink=0.9, notion=notion, seed=1)
        out = rrs.depth_batch_arrays(X[:3], data, cfg, trace=True)
        print(f"n={n} d={d} {notion} {path}/{sel}: depths {np.round(out[0], 6)}", flush=True)
    except (ValueError, RuntimeError) as exc:
        print(f"n={n} d={d} {notion} {path}/{sel}: {type(exc).__name__}: {exc}", flush=True)
eng.set_contract_path("auto")
eng.set_select_path("auto")
# drop-in helpers: FP64 projections / depth_of_projections / cap rows / Philox
X = toeplitz_gaussian(6, 700, seed=2)
U = rrs.generate_batch(rrs.CapSpec(rrs.Pole(np.eye(6)[0]), 0.7), 64, 1, 0).directions
px = rrs.project_parallel(rrs.Dataset(X), U).scores
pz = rrs.project_point(X[0], U)
for notion in ("halfspace", "projection", "asym_projection"):
    print(notion, np.round(rrs.depth_of_projections(notion, px, pz)[:4], 6))
print("sanitize driver done")
