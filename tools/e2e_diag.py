"""Why is the e2e leg slower after the other bench legs?  Times sem_mesh_reorder
and sem_read_field of C4 before and after heavy legs (SEM_TRACE=1 for phases)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2104_08416_b200 import meshgen as mg, sem as S
torch.cuda.set_device(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
pb = mg.config("C4"); m = pb.mesh
out = torch.zeros(40_000_000, dtype=torch.float64).pin_memory()

def e2e(tag):
    t0 = time.time(); ctx = S.SemContext(0, stream=st.cuda_stream)
    r = ctx.sem_mesh_reorder(m.vxy, m.tri, 3); t1 = time.time()
    ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt); ctx.sem_step_n(10); ctx.sem_sync(); t2 = time.time()
    ctx.sem_read_field(out=out.numpy()[: r["n_nodes"]]); t3 = time.time()
    ctx.close(); t4 = time.time()
    print("%-20s reorder %.3f build+10 %.3f read %.3f close %.3f" % (tag, t1 - t0, t2 - t1, t3 - t2, t4 - t3), flush=True)

e2e("first")
e2e("second")
for P in (5, 7):
    b1 = mg.config("B1", 1, degree=P)
    with S.SemContext(0, stream=st.cuda_stream) as ctx:
        ctx.sem_mesh_reorder(b1.mesh.vxy, b1.mesh.tri, P)
        ctx.sem_build_operators(b1.c, b1.src_vertex, b1.f0, b1.t0, 1.0, b1.dt); ctx.sem_step_n(20); ctx.sem_sync()
    e2e("after P%d" % P)
b1 = mg.config("B1", 1, degree=5)
with S.SemContext(0, stream=st.cuda_stream) as ctx:
    ctx.sem_set_integrator(S.SEM_INTEGRATOR_HEUN)
    ctx.sem_mesh_reorder(b1.mesh.vxy, b1.mesh.tri, 5)
    ctx.sem_build_operators(b1.c, b1.src_vertex, b1.f0, b1.t0, 1.0, b1.dt * 0.2); ctx.sem_step_n(20); ctx.sem_sync()
e2e("after heun P5")
with S.SemContext(0, stream=st.cuda_stream) as ctx:
    for eo, no in ((S.SEM_ORDER_CONN, S.SEM_NODES_VISIT), (S.SEM_ORDER_DIST, S.SEM_NODES_VISIT)):
        ctx.sem_mesh_reorder(m.vxy, m.tri, 3, eo, no)
e2e("after conn/dist")
print("torch reserved %.1f GB, mem_get_info free %.1f GB" % (torch.cuda.memory_reserved() / 1e9, torch.cuda.mem_get_info()[0] / 1e9))
