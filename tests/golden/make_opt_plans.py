"""Freeze co-optimised plans (paper_2103_03074_b200.treeopt) as fixtures.

For each entry, the base fixture's network and circuit are copied and the
head tree + sliced set chosen by ``select_slices_b200`` replace the
reference planner's; the tail and the root step are the reference's.
``make_goldens.py <name>`` then drives the unmodified reference engine on
the new plan (its known-answer vectors).  Deterministic: per-trial seeds,
no wall-clock cut-off at the budgets below.

    python tests/golden/make_opt_plans.py [name ...]
"""

from __future__ import annotations

import json
import math
import os
import shutil
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2103_03074_b200 import treeopt  # noqa: E402
from paper_2103_03074_b200.types import tree_to_doc  # noqa: E402
from paper_2103_03074_b200.workloads import load_workload  # noqa: E402

# name: (base fixture, space target, objective, extra optimiser options
#        [, reference-planner fixture the savings are quoted against])
PLANS = {
    "c1_opt": ("c1", 8, "mults", {}),
    "s8_opt": ("s8", 18, "mults", {}),
    "c4_opt": ("c4", 30, "mults", {"restarts": 16}),
    # c4_opt's tree + slices, then the B200 polish (time-model subtree DP)
    "c4_opt_b200": ("c4_opt", 30, "b200", {"trials": 0, "keep_top": 0, "slice_repeats": 1}, "c4"),
    # space target 2^31 (the executor runs rank-32 intermediates; C4 at 2^31:
    # fewer, bigger slices), then the B200 polish
    "c4_opt31": ("c4", 31, "mults", {"restarts": 16}),
    "c4_opt31_b200": ("c4_opt31", 31, "b200", {"trials": 0, "keep_top": 0, "slice_repeats": 1}, "c4"),
    # C2 (m=12, t=2^28) and C3 (m=14, t=2^30): co-optimised + B200 polish
    "c2_opt_b200": ("c2", 28, "b200", {"restarts": 4}),
    "c3_opt_b200": ("c3", 30, "b200", {"restarts": 4}),
    "c2_opt_b200_alt": ("c2", 28, "b200", {"restarts": 2, "seed": 100}),
    # a second, independent C3 plan (other seeds): its full slice sum must
    # equal c3_opt_b200's (plan independence of the complete contraction)
    "c3_opt_b200_alt": ("c3", 30, "b200", {"restarts": 2, "seed": 100}),
    # the reference plan's OWN sliced set (same slices, same partial head
    # vectors), head tree re-ordered: exact DP, then the B200 polish
    "c4_reordered": ("c4", 30, "b200", {"keep_slices": True}),
    "c5_26_reordered": ("c5_26", 26, "b200", {"keep_slices": True}),
    "c5_28_reordered": ("c5_28", 28, "b200", {"keep_slices": True}),
    "c5_32_reordered": ("c5_32", 32, "b200", {"keep_slices": True}),
}


def make(name: str) -> dict:
    base, target, objective, extra = PLANS[name][:4]
    w = load_workload(base)
    ref = load_workload(PLANS[name][4]) if len(PLANS[name]) > 4 else w
    st: dict = {}
    t0 = time.time()
    kw = dict(objective=objective, seed=0, time_budget_s=3600.0,
              initial_slices=w.sliced if w.target_space == target else None)
    kw.update(extra)
    plan, tree = treeopt.select_slices_b200(w.tn, w.tree, target, stats=st, **kw)
    dt = time.time() - t0
    doc = tree_to_doc(tree, circuit_sha256=w.doc["circuit_sha256"],
                      open_qubits=w.doc["open_qubits"], slices=plan.sliced_indices,
                      subtask=treeopt.plan_subtask(w.tn, tree, plan))
    ref_total = math.log2(ref.tc_per_slice) + ref.n_e
    new_total = math.log2(plan.per_subtask.tc) + len(plan.sliced_indices)
    doc["planner"] = {"tool": "paper_2103_03074_b200.treeopt.select_slices_b200",
                      "base": base, "target_space": target, "objective": objective,
                      "options": {k: v for k, v in kw.items() if k != "initial_slices"},
                      "seconds": round(dt, 1),
                      "reference_plan": {"name": ref.name, "n_e": ref.n_e,
                                         "tc_log2": math.log2(ref.tc_per_slice),
                                         "total_log2": ref_total},
                      "log2_total_work_saved": ref_total - new_total,
                      "stats": st}
    d = os.path.join(HERE, name)
    os.makedirs(d, exist_ok=True)
    for f in ("circuit.qsim", "network.json"):
        shutil.copyfile(os.path.join(HERE, base, f), os.path.join(d, f))
    with open(os.path.join(d, "order.json"), "w") as fh:
        json.dump(doc, fh, indent=1, sort_keys=True)
    print(f"[{name}] n_e {ref.n_e} -> {len(plan.sliced_indices)}, tc/slice 2^{math.log2(ref.tc_per_slice):.2f}"
          f" -> 2^{math.log2(plan.per_subtask.tc):.2f}, total 2^{ref_total:.2f} -> 2^{new_total:.2f}"
          f" ({dt:.0f}s)", flush=True)
    return doc


if __name__ == "__main__":
    for n in sys.argv[1:] or list(PLANS):
        make(n)
