"""Print the bf16 path's normwise errors against the fp64 oracle (the margin under the 1e-2
tolerance) for a few shapes; uses the parity tests' own helpers."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import foldgen
from tests import test_gpu_parity as T

for name, gr, S in (("C2 B=2", foldgen.make_config("c2", 2), 1024), ("C3 B=16", foldgen.make_config("c3", 16), 300),
                    ("C4 B=2", foldgen.make_config("c4", 2), 1024), ("C5-shape B=4", foldgen.make_config("c5", 4), 256)):
    e = T._check_bwd(gr, "treelstm", "bf16", S)
    print(name, {k: f"{v:.2e}" for k, v in e.items()}, flush=True)
