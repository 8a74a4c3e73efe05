"""depthforge direction API on the device (directions.py:76-204).

Pole / CapSpec / DirectionBatch live in config.py; generate_batch in
solver.py.  SubStream, random_sphere and random_sphere_pole run the Philox /
ndtri / pairwise-norm generator kernels of csrc/gen.cu (FP64, -fmad=false, the
reference's operation order), addressed by the same (seed, value, index,
refinement, query) counters.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import CapSpec


def _engine():
    from .solver import _session

    return _session(None)


@dataclass(frozen=True)
class SubStream:
    """Address of one direction's substream: (seed, refinement, query, index)."""

    seed: int
    refinement: int = 0
    query: int = 0
    index: int = 0

    def uniforms(self, count: int, offset: int = 0) -> np.ndarray:
        with _engine() as eng:
            return eng.stream_values(self.seed, self.refinement, self.query, self.index, offset, count, False)

    def normals(self, count: int, offset: int = 0) -> np.ndarray:
        with _engine() as eng:
            return eng.stream_values(self.seed, self.refinement, self.query, self.index, offset, count, True)


def random_sphere(d: int, stream: SubStream) -> np.ndarray:
    """directions.py:138-147: uniform direction on the (d-1)-sphere from
    normalized normals (d = 1 gives exactly +1 or -1)."""
    if d < 1:
        raise ValueError("dimension must be >= 1")
    with _engine() as eng:
        return eng.unit_rows(stream.seed, stream.refinement, stream.query, 1, d, 0, stream.index)[0]


def random_sphere_pole(cap: CapSpec, stream: SubStream) -> np.ndarray:
    """directions.py:185-189: one draw inside the cap; identical to the
    matching generate_batch row."""
    with _engine() as eng:
        return eng.cap_directions(cap.pole.p, cap.epsilon, 1, stream.seed, stream.refinement, stream.query,
                                  index_base=stream.index)[0]
