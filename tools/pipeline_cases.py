"""Small runs of every step kernel for the checked build.

    SEM_LIB=paper_2104_08416_b200/libsem_checked.so SEM_K7_GRID=2 python tools/pipeline_cases.py

(compute-sanitizer is closed on this GPU pool: tools/checked_build.sh runs these cases and the
GPU test-suite against a -DSEM_CHECKED build instead.)
Each case is tiny (a few thousand elements) and, with the grid capped, walks several
chunks per persistent CTA, so the pipeline's stage reuse (empty / wempty / idb
mbarrier waits and parity flips) runs under the checks.  Kernels covered: K7 at P2, P3,
P5, P7 (k7_step), K8 (k8_fix), the fused-K8 variant, Heun KH7 / KH8 (k_heun,
k_heun_fix) at P3 and P5, and the multi-rank interface kernels (loopback group).
Every case also checks its field against the oracle, so a checked run that changes
timing cannot hide a wrong answer.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.core import OracleSEM  # noqa: E402
from paper_2104_08416_b200 import meshgen as mg  # noqa: E402
from paper_2104_08416_b200 import sem as S  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def leapfrog(pb, P, steps, fuse=False):
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, P, pb.c)
    rng = np.random.default_rng(P)
    U0 = rng.standard_normal(o.N)
    Up = U0 + 0.1 * rng.standard_normal(o.N)
    Uo, _ = o.leapfrog(pb.dt, steps, src=pb.src_vertex, A=1.0, f0=pb.f0, t0=0.0, U=U0, Uprev=Up, step0=2)
    if fuse:
        os.environ["SEM_FUSE_K8"] = "1"
    try:
        with S.SemContext(0) as ctx:
            ctx.sem_mesh_reorder(m.vxy, m.tri, P)
            ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, 0.0, 1.0, pb.dt)
            ctx.sem_write_state(U0, Up)
            ctx.sem_set_step(2)
            ctx.sem_step_n(steps)
            Ug, _ = ctx.sem_read_field()
            nch = ctx.sem_get_info()["n_chunks"]
    finally:
        os.environ.pop("SEM_FUSE_K8", None)
    e = rel(Ug, Uo)
    print("leapfrog P%d%s chunks=%d steps=%d rel=%.2e" % (P, " fused-K8" if fuse else "", nch, steps, e), flush=True)
    assert e <= 1e-12


def heun(pb, P, steps):
    m = pb.mesh
    h = mg.heun_h(pb)
    o = OracleSEM(m.vxy, m.tri, P, pb.c)
    rng = np.random.default_rng(10 + P)
    U0 = rng.standard_normal(o.N)
    V0 = rng.standard_normal((m.ne, o.Np, 2))
    Uo, Vo = o.heun(h, steps, src=pb.src_vertex, A=1.0, f0=pb.f0, t0=0.0, U=U0, V=V0, step0=1)
    with S.SemContext(0) as ctx:
        ctx.sem_set_integrator(S.SEM_INTEGRATOR_HEUN)
        ctx.sem_mesh_reorder(m.vxy, m.tri, P)
        ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, 0.0, 1.0, h)
        ctx.sem_write_state(U0, None)
        ctx.sem_write_velocity(V0)
        ctx.sem_set_step(1)
        ctx.sem_step_n(steps)
        Ug, _ = ctx.sem_read_field()
        Vg, _ = ctx.sem_read_velocity()
    print("heun P%d steps=%d relU=%.2e relV=%.2e" % (P, steps, rel(Ug, Uo), rel(Vg, Vo)), flush=True)
    assert rel(Ug, Uo) <= 1e-12 and rel(Vg, Vo) <= 1e-12


def loopback(pb, world, steps):
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    rng = np.random.default_rng(3)
    U0 = rng.standard_normal(o.N)
    Uo, _ = o.leapfrog(pb.dt, steps, src=pb.src_vertex, A=1.0, f0=pb.f0, t0=0.0, U=U0, Uprev=U0, step0=0)
    g = S.LoopbackGroup(world)
    try:
        g.sem_mesh_reorder(m.vxy, m.tri, pb.P)
        g.sem_build_operators(pb.c, pb.src_vertex, pb.f0, 0.0, 1.0, pb.dt)
        g.sem_write_state(U0, U0)
        g.sem_step_n(steps)
        Ug, _ = g.sem_read_field()
    finally:
        g.close()
    print("loopback G=%d steps=%d rel=%.2e" % (world, steps, rel(Ug, Uo)), flush=True)
    assert rel(Ug, Uo) <= 1e-12


def main():
    which = sys.argv[1:] or ["lf", "heun", "mr"]
    steps = int(os.environ.get("SAN_STEPS", "2"))
    if "lf" in which:
        leapfrog(mg.config("C5", 512), 2, steps)        # 2048 P2 elements, 8 chunks
        leapfrog(mg.config("C2", 16), 3, steps)         # 2048 P3 elements, 8 chunks
        leapfrog(mg.config("C2", 16), 3, steps, fuse=True)
        leapfrog(mg.config("B1", 40, degree=5), 5, steps)  # 25 x 12 cells, 600 elements, 5 chunks
        leapfrog(mg.config("B1", 40, degree=7), 7, steps)  # 10 chunks of 64
    if "heun" in which:
        heun(mg.config("C2", 16), 3, steps)
        heun(mg.config("B1", 40, degree=5), 5, steps)
        heun(mg.config("B1", 40, degree=7), 7, steps)  # tensor-core Heun, chunks of 64
    if "mr" in which:
        loopback(mg.config("C2", 16), 2, steps)
    print("pipeline_cases ok", flush=True)


if __name__ == "__main__":
    main()
