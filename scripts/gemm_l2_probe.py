"""One big contraction step (2-leaf program) for ncu DRAM-traffic experiments.

    TNB_L2_PROMO=0|64|128|256 TNB_GROUP_M=n python scripts/gemm_l2_probe.py ma nb kb
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.gemm_probe import two_leaf  # noqa: E402

from paper_2103_03074_b200.engine import Program  # noqa: E402

ma, nb, kb = (int(x) for x in sys.argv[1:4])
rng = np.random.default_rng(0)
leaves, steps, out, A, B = two_leaf(ma, nb, kb, rng, tiled=True)
p = Program(leaves, steps, [], out, "single", 0)
p.set_timing(True)
for _ in range(2):
    p.update_leaves([(0, leaves[0][1], leaves[0][2] * (1.0 + 1e-7 * np.random.rand()))])
    p.run_range(0, 1)
    t = p.timing()
    fl = 8.0 * 2.0 ** (ma + nb + kb)
    print(f"promo={os.environ.get('TNB_L2_PROMO')} group_m={os.environ.get('TNB_GROUP_M')} "
          f"gemm {t['gemm_ms']:.2f} ms -> {fl / t['gemm_ms'] / 1e9:.1f} TFLOP/s", flush=True)
