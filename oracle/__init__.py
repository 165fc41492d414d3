"""CPU oracle for the hipBone hot path (arXiv 2202.12477) -- TEST INFRASTRUCTURE ONLY.

This package is a plain, slow, obviously-correct fp64 implementation of what the
paper's hot path computes. It exists to check the CUDA path, nothing else:

* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
  ``--impl reference`` legs may import it. The product package
  ``paper_2202_12477_b200`` never imports it, and it never imports the product.
* It shares no code, headers, tables or constants with the CUDA path. Random
  inputs come from ``tests/inputs.py`` (seeded generators, no method arithmetic);
  the forcing hash is re-implemented independently on each side.
* Every function cites the passage of ``PAPER.md`` (``P:<line>``) it follows, or the
  SURVEY.md §8(c) reading ("c<k>") where the paper is silent.

Modules
  basis      GLL nodes/weights and the 1-D derivative matrix D
  mesh       box numbering, counts, W/B, geometric factors G         (c4, c7)
  partition  rank grid, ownership, halo/interior split, plans        (c8-c11)
  forcing    splitmix64 hash forcing                                 (c12)
  operator   element operator (explicit and sum-factorised), assembly,
             dense A
  cg         Algorithm 1, fixed-iteration and tolerance modes
  ledger     FLOP / byte / roofline formulas

Parity status: every function is pinned by ``tests/test_oracle_*.py`` (closed forms,
invariants, brute force, golden values), including the parity checkers apply_abs,
apply_abs_explicit and apply_entries and the owner rule; see DESIGN.md section 7 and
reading R5. There is no "parity unpinned" function in this package.
"""
