"""Paper Listing 1 (standard Hilbert generator), PAPER.md:51-88 -- TEST PIN ONLY.

The listing's body is restated here as a closure instead of module globals; the
garbled line PAPER.md:64 (`print("`) is read as "emit the current (x0, x1)"
(SURVEY.md P-1).  Starting state x0, x1, distance = -1, 0, 0 and the initial
`step(0)` are as printed, so the first emitted cell is (0, 0).
"""
from __future__ import annotations


def listing1_path(order: int):
    """Cells (x0, x1) in the order Listing 1 visits them, for a 2^order square."""
    state = {"x0": -1, "x1": 0, "distance": 0}
    out = []

    def step(direction):
        direction = direction & 3
        if direction == 0:
            state["x0"] += 1
        if direction == 1:
            state["x1"] += 1
        if direction == 2:
            state["x0"] -= 1
        if direction == 3:
            state["x1"] -= 1
        out.append((state["x0"], state["x1"]))  # PAPER.md:64 (garbled print)
        state["distance"] += 1

    def hilbert(direction, rotation, order):
        if order == 0:
            return
        direction = direction + rotation
        hilbert(direction, -rotation, order - 1)
        step(direction)
        direction = direction - rotation
        hilbert(direction, rotation, order - 1)
        step(direction)
        hilbert(direction, rotation, order - 1)
        direction = direction - rotation
        step(direction)
        hilbert(direction, -rotation, order - 1)

    step(0)
    hilbert(0, 1, order)
    return out
