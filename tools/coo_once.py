#!/usr/bin/env python
"""One device pauli_sum_to_coo of the TFIM chain (n from argv) for profiling."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_14167_b200 import engine  # noqa: E402
from paper_2602_14167_b200 import qforge as qf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
ctx = engine.default_context(0)
obs = qf.tfim_terms(qf.build_lattice("chain", [n], [False]), 1.0).observable(ctx)
rows, cols, vals = engine.pauli_sum_to_coo(ctx, obs, 26, device=True)
torch.cuda.synchronize()
print("nnz", vals.numel())
