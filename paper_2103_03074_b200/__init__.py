"""B200-native executor for big-batch tensor-network contraction
(arxiv 2103.03074, Pan & Zhang), drop-in for the reference ``tncut``
engine API (tncut/engine.py).  See DESIGN.md.
"""

__version__ = "0.1.0"

from .engine import (  # noqa: F401
    AmplitudeTable,
    EngineStats,
    HeadVector,
    Program,
    clear_cache,
    compute_head_vector,
    compute_tail_amplitudes,
    contract_tree,
    flop_estimate,
    head_program,
    reduce_partials,
    set_device,
    set_flags,
    set_reorder,
    set_slice_batch,
    tail_amplitudes_unchecked,
)
from .errors import (  # noqa: F401
    ProvenanceMismatch,
    RangeGap,
    RangeOutOfBounds,
    RangeOverlap,
    ShapeMismatch,
    TncutError,
)
from . import analytics  # noqa: F401  (on-device analytics.py drop-in)
from .io import read_head_vector, write_amplitude_tsv, write_head_vector  # noqa: F401
from .provenance import normalize_s1, provenance_hash  # noqa: F401
from .workloads import load_workload  # noqa: F401
