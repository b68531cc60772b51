import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np
from paper_2104_08416_b200 import meshgen as mg, sem as S
pb = mg.config("C4"); m = pb.mesh
for i in range(3):
    t0=time.time(); ctx = S.SemContext(0); t1=time.time()
    ctx.sem_mesh_reorder(m.vxy, m.tri, 3); t2=time.time()
    ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt); t3=time.time()
    ctx.close(); t4=time.time()
    print('create %.3f reorder %.3f build %.3f free %.3f' % (t1-t0, t2-t1, t3-t2, t4-t3), flush=True)
