"""CPU fp64 ORACLE for the SFC-reordered SEM leapfrog step (arxiv 2104.08416).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import, call,
link or execute anything under ``oracle/``.  The product path
(``paper_2104_08416_b200``) never touches it and shares no code with it.

Layout
------
* ``refelem.py``   exact (sympy) reference-triangle tables: nodes, nodal basis,
                   quadrature weights, derivative tables.
* ``listing1.py``  the paper's Listing 1 Hilbert generator, executed verbatim
                   in spirit -- used only as a pin.
* ``sem_oracle.c`` plain C (gcc -O2 -fopenmp, no fast-math): generalized
                   Hilbert path + literal SFC ordering,
                   canonical SEM nodes, first-touch renumbering
                   (PAPER.md:312-321), geometry, lumped mass,
                   Algorithms 1-3 composed into the leapfrog
                   update of the north_star (reading R1).
* ``core.py``      ctypes wrapper around ``liboracle.so``.

Parity status per function:
* reference tables, SFC ordering on 2^k grids, first-touch, canonical nodes,
  geometry, lumped mass, stiffness, leapfrog: pinned by tests/test_oracle_*.py.
* generalized Hilbert curve on non-power-of-two rectangles: "parity unpinned"
  beyond bijection/adjacency invariants (the paper only cites Cerveny 2020).
* P3 Lobatto edge-node positions and the P2 HRZ mass weights: "parity
  unpinned" (readings R3/R4; the paper does not print them).
"""
