"""sha256 of the numpy iso-parametric assembly (tests/iso_assembly.py) of the
C4 recipe at small N: checks that the host generator is bitwise reproducible
across host CPUs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from golden_util import csr_hash
from iso_assembly import assemble
from paper_2506_08284_b200.assembly import config_draws
from paper_2506_08284_b200.inputs import make_config
for N in (8, 12):
    cfg, sigma, jitter, rng = config_draws("C4", N)
    A_e, S, A_n, D = assemble(N, sigma, False, jitter)
    print("iso", N, [csr_hash(M)[:16] for M in (A_e, S, A_n, D)])
s, rhs, cfg = make_config("C3", 16)
print("host C3@16", [csr_hash(M)[:16] for M in (s.A_e, s.S, s.A_n, s.D)])
