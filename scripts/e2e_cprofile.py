"""cProfile of run_sequence over host inputs (C3, 12 systems): where the host
time outside the kernels goes. python scripts/e2e_cprofile.py   (GPU box)"""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_05820_b200 as pk  # noqa: E402
from paper_1512_05820_b200.problems import elasticity_sequence  # noqa: E402

seq = elasticity_sequence((64, 64, 64), p=12)
specs = list(seq)
cfg = pk.SolverConfig(truncation=pk.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=60,
                                                     max_dim=60), mode="cg")
jac = lambda A: pk.build_preconditioner("jacobi", A)  # noqa: E731
hseq = pk.SystemSequence(seq.n, specs, C=seq.C)
pk.run_sequence(pk.SystemSequence(seq.n, specs[:3], C=seq.C), cfg, precond_factory=jac)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
pk.run_sequence(hseq, cfg, precond_factory=jac)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(22)
