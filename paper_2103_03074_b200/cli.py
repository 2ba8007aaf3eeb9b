"""Run the reference's own command line (``tncut``, cli.py:109-597) on this
executor: ``python -m paper_2103_03074_b200.cli run circuit.qsim order.json
-o amps.tsv --precision single`` behaves exactly like ``tncut run ...`` with
the engine hot path (``compute_head_vector``, ``compute_tail_amplitudes``,
``reduce_partials``, ``contract_tree``; cli.py:38-47, pipeline.py:14-19) and
the analytics (cli.py:29-36) bound to the B200 implementations.  Everything
else -- parsing, ordering, slicing, file formats, exit codes (cli.py:82-97) --
is the reference's code, so existing scripts and partial files keep working.

Requires the reference package (``tncut``) to be importable; this module is
the switch a user of the reference flips, not a reimplementation of its CLI.
"""

from __future__ import annotations

import sys

ENGINE_NAMES = ("compute_head_vector", "compute_tail_amplitudes", "reduce_partials", "contract_tree")
IO_NAMES = ("write_amplitude_tsv",)  # byte-identical, formatted on all host threads (io.py)
ANALYTICS_NAMES = ("xeb", "histogram", "postselect_curve", "mixed_xeb", "marginal_and_conditional",
                   "ks_to_porter_thomas")


def b200_select_slices(tn, tree, target_space, reconfigure=True, leaf_limit=60):
    """``select_slices`` (slicing.py:76-82 signature) backed by the plan
    co-optimiser: head tree + sliced set searched jointly for total head
    work, then the B200 time-model polish (treeopt.py).  ``reconfigure`` /
    ``leaf_limit`` tune the reference's own greedy rebuild and have no
    counterpart here."""
    from .treeopt import select_slices_b200

    return select_slices_b200(tn, tree, target_space, objective="b200")


def bind(slicer: bool | None = None) -> dict:
    """Rebind the engine/analytics names inside the reference's cli and
    pipeline modules (they import them by name) to this package's; with
    ``slicer`` (default: env TNB_CLI_SLICER=b200) also ``tncut slice``'s
    ``select_slices`` to the plan co-optimiser.
    Worker threads of ``tncut run --threads`` are spread over the visible
    GPUs round-robin.  Returns {module.name: previous object} so callers can
    restore."""
    import os

    import tncut.cli as cli
    import tncut.pipeline as pipeline

    from . import analytics, engine, io

    previous = {"paper_2103_03074_b200.engine._thread_devices": engine._thread_devices}
    # `tncut run --threads T` (cli.py:367-380) fans ranges out over T threads:
    # each thread is bound to the next GPU round-robin (engine.set_thread_devices)
    engine.set_thread_devices(True)
    if slicer is None:
        slicer = os.environ.get("TNB_CLI_SLICER", "") == "b200"
    if slicer:
        previous["tncut.cli.select_slices"] = cli.select_slices
        cli.select_slices = b200_select_slices
    for mod in (cli, pipeline):
        for name in ENGINE_NAMES:
            if hasattr(mod, name):
                previous[f"{mod.__name__}.{name}"] = getattr(mod, name)
                setattr(mod, name, getattr(engine, name))
        for name in ANALYTICS_NAMES:
            if hasattr(mod, name):
                previous[f"{mod.__name__}.{name}"] = getattr(mod, name)
                setattr(mod, name, getattr(analytics, name))
        for name in IO_NAMES:
            if hasattr(mod, name):
                previous[f"{mod.__name__}.{name}"] = getattr(mod, name)
                setattr(mod, name, getattr(io, name))
    return previous


def unbind(previous: dict) -> None:
    import importlib

    for key, obj in previous.items():
        mod_name, name = key.rsplit(".", 1)
        setattr(importlib.import_module(mod_name), name, obj)


def main(argv=None) -> int:
    import tncut.cli as cli

    previous = bind()
    try:
        cli.main(args=list(sys.argv[1:] if argv is None else argv), standalone_mode=True)
    except SystemExit as exc:  # click exits with the reference's exit codes
        return int(exc.code or 0)
    finally:
        unbind(previous)
    return 0


if __name__ == "__main__":
    sys.exit(main())
