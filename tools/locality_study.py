"""GPU analog of the paper's memory study (Table mem_data_exp_1:
LLC misses and stalled memory slots per ordering): DRAM traffic and L2 hit rate
of the step kernels under each ordering, same C4 mesh.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
        -k regex:"k7_step|k8_fix" --csv --log-file gpurun_out/locality.csv python tools/locality_study.py
    python tools/locality_study.py --summarise gpurun_out/locality.csv > profiles/r1s2_locality.md

Each ordering runs STEPS steps after a 2-step warm-up, in the order of ORDERINGS;
the summariser maps launches back to orderings by that order.
"""
import csv
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ORDERINGS = ["hilbert", "hilbert_degree", "hilbert_canonical", "conn", "dist", "natural", "random"]
WARM, STEPS = 2, 3


def run():
    from paper_2104_08416_b200 import meshgen as mg, sem as S
    pb = mg.config("C4")
    table = {
        "hilbert": (pb.mesh, pb.c, S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH),
        "hilbert_degree": (pb.mesh, pb.c, S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH_DEGREE),
        "hilbert_canonical": (pb.mesh, pb.c, S.SEM_ORDER_HILBERT, S.SEM_NODES_CANONICAL),
        "conn": (pb.mesh, pb.c, S.SEM_ORDER_CONN, S.SEM_NODES_VISIT),
        "dist": (pb.mesh, pb.c, S.SEM_ORDER_DIST, S.SEM_NODES_VISIT),
        "natural": (pb.natural, pb.c_natural, S.SEM_ORDER_INPUT, S.SEM_NODES_CANONICAL),
        "random": (pb.mesh, pb.c, S.SEM_ORDER_INPUT, S.SEM_NODES_CANONICAL),
    }
    with S.SemContext(0) as ctx:
        for name in ORDERINGS:
            m, c, eo, no = table[name]
            ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P, eo, no)
            src = pb.src_vertex if m is pb.mesh else int(pb.mesh.vert_perm[pb.src_vertex])
            ctx.sem_build_operators(c, src, pb.f0, pb.t0, 1.0, pb.dt)
            ctx.sem_step_n(WARM + STEPS)
            ctx.sem_sync()
            print(name, "done", flush=True)


UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0,
        "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "%": 1.0}


def summarise(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, ii, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    launches = collections.OrderedDict()
    for r in rows[1:]:
        key = (int(r[ii]), r[ki].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1])
        launches.setdefault(key, {})[r[mi]] = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
    seq = list(launches.items())
    per = 2 * (WARM + STEPS)  # k7_step + k8_fix per step
    print("| ordering | K7 DRAM MB / step | K8 DRAM MB / step | K7 L2 hit % | K7 us | K8 us |")
    print("|---|---|---|---|---|---|")
    for o, name in enumerate(ORDERINGS):
        block = seq[o * per:(o + 1) * per][2 * WARM:]
        k7 = [v for (i, k), v in block if k == "k7_step"]
        k8 = [v for (i, k), v in block if k == "k8_fix"]
        avg = lambda L, m: sum(x[m] for x in L) / max(len(L), 1)
        dram = lambda L: avg(L, "dram__bytes_read.sum") + avg(L, "dram__bytes_write.sum")
        print("| %s | %.1f | %.1f | %.1f | %.1f | %.1f |" % (
            name, dram(k7) / 1e6, dram(k8) / 1e6, avg(k7, "lts__t_sector_hit_rate.pct"),
            avg(k7, "gpu__time_duration.sum"), avg(k8, "gpu__time_duration.sum")))


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--summarise":
        summarise(sys.argv[2])
    else:
        run()
