"""The experiments library (exp_lib/liblbm19_exp.so, built with
-DLBM_EXPERIMENTS: the measured-slower dense variants moved out of the
product library) still reproduces the oracle bitwise.  Runs in a subprocess
with LBM_LIB pointing at it; skipped when that library was not built
(python -m paper_2108_13241_b200.build --experiments)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXP = os.path.join(ROOT, "exp_lib", "liblbm19_exp.so")

SCRIPT = r"""
import numpy as np, os, sys
sys.path.insert(0, os.path.join(sys.argv[1], "tests"))
sys.path.insert(0, sys.argv[1])
import paper_2108_13241_b200 as lb
from helpers import oracle_sim, random_mixed_geometry3, to_geometry
c = random_mixed_geometry3(3, n=(64, 12, 10), periodic_z=True)
omega = 1.0 / (3 * 0.08 + 0.5)
params = lb.FlowParams.from_viscosity(U=0.1, L=10, nu=(1.0 / omega - 0.5) / 3.0)
ref = oracle_sim(c, params.omega, np.float32)
ref.initialize(1.0)
ref.step(9)
for scheme, variants in (("ab", ("1", "2", "3", "8")), ("aa", ("12",))):
    for v in variants:
        os.environ["LBM_STEP_VARIANT"] = v
        sim = lb.Simulation(to_geometry(c), params, scalar=np.float32, scheme=scheme)
        sim.initialize(1.0)
        sim.step(9)
        assert np.array_equal(sim.canonical_state(), ref.pre), (scheme, v)
        sim.close()
print("experiments ok")
"""


@pytest.mark.skipif(not os.path.exists(EXP), reason="experiments library not built")
def test_experiment_variants_bitwise_vs_oracle():
    env = dict(os.environ, LBM_LIB=EXP)
    out = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], capture_output=True, text=True, env=env,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    assert "experiments ok" in out.stdout
