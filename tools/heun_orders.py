"""Heun (the paper's integrator) on the Benchmark 1 mesh (1M elements) at
orders 5 and 7: ms per step and element-updates/s, one B200.  The consumer threads per
element of P5 come from SEM_HEUN_G5 (read once per process: run one process per value)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_08416_b200 import meshgen as mg  # noqa: E402
from paper_2104_08416_b200 import sem as S  # noqa: E402

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
for P in [int(x) for x in (sys.argv[1:] or ["5", "7"])]:
    pb = mg.config("B1", 1, degree=P)
    m = pb.mesh
    with S.SemContext(0, stream=stream.cuda_stream) as ctx:
        ctx.sem_set_integrator(S.SEM_INTEGRATOR_HEUN)
        ctx.sem_mesh_reorder(m.vxy, m.tri, P)
        ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, mg.heun_h(pb))
        ctx.sem_step_n(10)
        ctx.sem_sync()
        K = 200
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        ctx.sem_step_n(K)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        U, _ = ctx.sem_read_field()
        print("heun P%d G5=%s B1 %d elements: %.4f ms/step, %.3e element-updates/s, finite %s" %
              (P, os.environ.get("SEM_HEUN_G5", "1"), m.ne, ms, m.ne / (ms * 1e-3), bool(torch.isfinite(
                  torch.from_numpy(U)).all())), flush=True)
