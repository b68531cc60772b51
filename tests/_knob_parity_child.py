"""Child process of test_gpu_knobs.py: one reduced C3 / C5 / B1-P5 run under the knob
environment the parent set (knobs are read once per process), compared with the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.core import OracleSEM  # noqa: E402
from paper_2104_08416_b200 import meshgen as mg  # noqa: E402
from paper_2104_08416_b200 import sem as S  # noqa: E402

worst = 0.0
with S.SemContext(0) as ctx:
    for name, scale, deg in (("C3", 10, None), ("C5", 64, None), ("B1", 25, 5)):
        pb = mg.config(name, scale, degree=deg) if deg else mg.config(name, scale)
        pb = mg.Problem(**{**pb.__dict__, "t0": 10 * pb.dt, "f0": 1.0 / (8 * pb.dt)})
        m = pb.mesh
        o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
        Uo, _ = o.leapfrog(pb.dt, 60, src=pb.src_vertex, A=1.0, f0=pb.f0, t0=pb.t0)
        ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P)
        ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
        ctx.sem_step_n(60)
        Ug, n = ctx.sem_read_field()
        assert n == 60
        err = float(np.linalg.norm(Ug - Uo) / np.linalg.norm(Uo))
        worst = max(worst, err)
print("REL_L2 %.3e" % worst)
