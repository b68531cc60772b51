"""B200-native Hilbert-reordered SEM leapfrog step (arxiv 2104.08416).

The product path is the CUDA C-ABI library ``libsem.so`` (csrc/) reached
through the thin ctypes binding in ``sem.py``.  ``meshgen`` holds the seeded
synthetic inputs.  There is no CPU fallback.
"""
