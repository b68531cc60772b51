"""B1 at P5 under the Heun integrator (the paper's Benchmark 1 workload): a few steps, for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_08416_b200 import meshgen as mg, sem as S
pb = mg.config("B1", 1, degree=5); m = pb.mesh
with S.SemContext(0) as ctx:
    ctx.sem_set_integrator(S.SEM_INTEGRATOR_HEUN)
    ctx.sem_mesh_reorder(m.vxy, m.tri, 5)
    ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt * 0.2)
    ctx.sem_step_n(8); ctx.sem_sync()
print("ok")
