"""Golden values of the reference's coverage models (run here, where /root/reference exists).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_coverage.py

Writes tests/golden/coverage_sampled.json: moesim.coverage.sample_activation
on fixed seeds (numba backend) and the closed forms, for the parity tests of
paper_2510_08055_b200/coverage.py.
"""
import json
import os

import numpy as np
from moesim import coverage as cov

CASES = [(8, 8, 128, 0.0, 0, 2000), (32, 8, 128, 0.0, 1, 500), (576, 8, 128, 0.0, 2, 50), (64, 2, 16, 0.0, 3, 300),
         (8, 8, 128, 1.2, 4, 300), (100, 8, 128, 0.5, 5, 40)]

out = {"sampled": [], "uniform": [], "table": []}
for batch, k, E, skew, seed, trials in CASES:
    r = cov.sample_activation(batch, k, E, skew, np.random.default_rng(seed), trials)
    out["sampled"].append({"batch": batch, "top_k": k, "num_experts": E, "skew": skew, "seed": seed,
                           "trials": trials, "coverage_fraction": r.coverage_fraction,
                           "experts_activated": r.experts_activated,
                           "tokens_per_active_expert": r.tokens_per_active_expert})
for b in (0, 1, 8, 12, 32, 100, 576, 8224):
    out["uniform"].append([b, cov.UniformAnalytic(8, 128).coverage(b)])
    out["table"].append([b, cov.EmpiricalTable().coverage(b)])
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "coverage_sampled.json")
json.dump(out, open(path, "w"), indent=1)
print(path)
