"""memcolor-b200: B200-native batched local search for deep-learning-guided
memetic graph colouring (arxiv 2109.05948, DLMCOL).

Drop-in replacement for the data-parallel hot path of the reference package
`memcolor` (`pkg/src/memcolor/localsearch.py`, `crossover.py:14-93`,
`distance.py`): the same operator API, backed by hand-written sm_100a CUDA
kernels behind a C ABI (`include/memcolor_b200.h`).  See DESIGN.md.
"""

__version__ = "0.1.0"

from .coloring import Coloring, col_conflicts, wvcp_score  # noqa: F401
from .graph import WeightedGraph, rand_graph  # noqa: F401
from .rng import Stream, stream_key  # noqa: F401
