"""Step time of the leapfrog at P2 (C5/4), P5 and P7 (B1) for A/B library builds (SEM_LIB)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_08416_b200 import meshgen as mg, sem as S
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for P in [int(x) for x in (sys.argv[1:] or ["2", "5", "7"])]:
    pb = mg.config("B1", 1, degree=P) if P != 2 else mg.config("C5", 4)
    m = pb.mesh
    with S.SemContext(0, stream=st.cuda_stream) as ctx:
        ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P); ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
        ctx.sem_step_n(10); ctx.sem_sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); ctx.sem_step_n(200); e1.record(st); torch.cuda.synchronize()
        print(os.path.basename(os.environ.get("SEM_LIB", "libsem.so")), "P%d %s E=%d step %.4f ms" % (P, pb.name, m.ne, e0.elapsed_time(e1) / 200), flush=True)
