"""CPU oracle for the Lina expert-parallel MoE layer — TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct definition of what the CUDA
path computes, written from PAPER.md (arXiv 2210.17223).  It is used only by
``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl
reference`` legs of ``bench.py``.  The product path (``paper_2210_17223_b200``)
never imports it, and it never imports the product path; the only shared module
is ``lina_inputs`` (seeded random draws, no method arithmetic).

Precision: fp64 accumulation everywhere.  On the bf16 path the oracle rounds to
bf16 at exactly the points where the CUDA path stores bf16 tensors (h, o, y in
forward; dO, dH, dXe, dX, dW in backward — DESIGN.md R8), so residual
differences come from fp32-vs-fp64 accumulation order only.

Modules
-------
moe        : gating, capacity routing, expert FFN,
             combine, backward.
placement  : Eq. (1) replica counts, first-fit-decreasing packing and the
             per-replica token split.
popularity : sample-path profiles Ψ, phase-one popularity estimation and the
             phase-two top-2k check.

Parity pins (tests/test_oracle_*.py): every function here is pinned by at
least one check that does not re-type its formula — integer arithmetic for the
logits, closed forms for softmax/gates, brute force for top-k and capacity,
identity/dense special cases for the FFN and combine, central finite
differences for the backward, hand-evaluated Eq. (1) cases for placement,
the generator's closed-form transition rows and hand-evaluated estimates for
popularity (tests/test_popularity.py).
No function is "parity unpinned".
"""
