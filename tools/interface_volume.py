"""Interface exchange volume of the C4 weak-scaling partitions:
per rank, interface nodes, neighbours and bytes sent per step, from the host
partition (sem_debug_partition) of the Hilbert-ordered global mesh.

    python tools/interface_volume.py [scale] > profiles/r1s2_interface_volume.md
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import core
from paper_2104_08416_b200 import meshgen as mg
from paper_2104_08416_b200 import sem as S

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 1
print("| GPUs | elements (global) | per-rank interface nodes (max) | neighbours (max) | bytes sent per step per rank (max) | K7 bytes per step per rank |")
print("|---|---|---|---|---|---|")
for G in (2, 4, 8):
    t0 = time.time()
    pb = mg.config("C4", scale, gpus=G)
    m = pb.mesh
    t = core.orient(m.vxy, m.tri)
    mu, N = core.canonical_nodes(t, m.nv, pb.P)
    _, perm, _ = core.hilbert_order(m.vxy, m.tri)
    _, mu_ft = core.first_touch(mu[perm], N)
    nif, nn, sent = [], [], []
    for r in range(G):
        d = S.sem_debug_partition(mu_ft, N, r, G)
        nif.append(len(d["if_glob"]))
        nn.append(len(d["nbr"]))
        sent.append(8 * len(d["send_glob"]))
    E = m.ne
    k7 = E / G * (4 * 10 + 24) + 32 * N / G
    print("| %d | %d | %d | %d | %d | %.3g |" % (G, E, max(nif), max(nn), max(sent), k7), flush=True)
    print("(G=%d built in %.0f s)" % (G, time.time() - t0), file=sys.stderr, flush=True)
