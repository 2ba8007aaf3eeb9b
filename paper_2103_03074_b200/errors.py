"""Exception classes of the drop-in engine.

When the reference package ``tncut`` is importable the engine raises ITS
classes (errors.py:11-128), so existing ``except tncut.errors.X`` handlers
keep working.  Otherwise identical stand-ins with the same names and
hierarchy are defined here.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on the environment
    from tncut.errors import (  # type: ignore
        CannotReachCap,
        ProvenanceMismatch,
        RangeGap,
        RangeOutOfBounds,
        RangeOverlap,
        ShapeMismatch,
        TncutError,
    )
except Exception:  # tncut not installed (e.g. the GPU box)

    class TncutError(Exception):
        """Base class for all package errors (errors.py:11-12)."""

    class ShapeMismatch(TncutError):
        """Internal tensor-shape inconsistency (errors.py:83-84)."""

    class RangeOutOfBounds(TncutError):
        pass

    class RangeGap(TncutError):
        pass

    class RangeOverlap(TncutError):
        pass

    class ProvenanceMismatch(TncutError):
        """Inputs were produced from different circuits, orders or modes."""

    class CannotReachCap(TncutError):
        """Slicing every contracted index still misses the space target (errors.py:77-78)."""


class BlockTooWide(ShapeMismatch):
    """A batched-slice block would need intermediates above the executor's
    rank limit (slice_batch.batched_plan); callers fall back to narrower
    blocks.  A ShapeMismatch subclass, so reference handlers still match."""


__all__ = ["BlockTooWide", "TncutError", "ShapeMismatch", "RangeOutOfBounds", "RangeGap", "RangeOverlap",
           "ProvenanceMismatch", "CannotReachCap"]
