"""fold_schedule alone on multi-block cases, repeated (the cooperative scheduler's
depth walk: tree-like batches (exchange slots) and DAGs (pending counts, overflow rounds)):

    python tools/sanitize_sched.py

Prints whether a default-grid and a 3-CTA schedule of each case are identical (the oracle
comparison is in tests/test_gpu_schedule.py)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import foldgen  # noqa: E402
from paper_1702_02181_b200 import fold  # noqa: E402
from tests.helpers import random_dag  # noqa: E402


def main():
    torch.cuda.set_device(0)
    rng = np.random.default_rng(11)
    cases = [("c2 B=32", foldgen.make_config("c2", 32)), ("c4 B=16", foldgen.make_config("c4", 16)),
             ("c3 B=128", foldgen.make_config("c3", 128)), ("dag 9000", random_dag(rng, 9000, 50))]
    for name, gr in cases:
        op, child, token, root = fold.graphs_to_device(gr, "cuda:0")
        a = fold.schedule(op, child, token, root, gr.vocab).to_numpy()
        b = fold.schedule(op, child, token, root, gr.vocab, max_blocks=3).to_numpy()
        same = all(np.array_equal(np.asarray(a[k]), np.asarray(b[k])) for k in a if isinstance(a[k], np.ndarray))
        print(f"sanitize_sched {name}: N={gr.n_nodes} levels={a['n_levels']} repeat identical={same}")


if __name__ == "__main__":
    main()
