"""Child process of test_gpu_knobs.py::test_k8_variants_bitwise: 80 steps of reduced C3 and C5
meshes and a P5 mesh under the K8 knob environment the parent set; prints the SHA-256 of the
fields (internal numbering is the same in every child: the knobs do not touch the reordering)."""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_08416_b200 import meshgen as mg  # noqa: E402
from paper_2104_08416_b200 import sem as S  # noqa: E402

h = hashlib.sha256()
with S.SemContext(0) as ctx:
    for name, scale, deg in (("C3", 10, None), ("C5", 64, None), ("B1", 25, 5)):
        pb = mg.config(name, scale, degree=deg) if deg else mg.config(name, scale)
        pb = mg.Problem(**{**pb.__dict__, "t0": 10 * pb.dt, "f0": 1.0 / (8 * pb.dt)})
        m = pb.mesh
        ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P)
        ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
        ctx.sem_step_n(80)
        Ug, n = ctx.sem_read_field()
        assert n == 80 and np.all(np.isfinite(Ug))
        h.update(np.ascontiguousarray(Ug, dtype=np.float64).tobytes())
print("DIGEST", h.hexdigest())
