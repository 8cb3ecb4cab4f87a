"""CPU oracle for ChunkAttention decode attention — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg and
`--impl reference` arm may import anything under oracle/.  The product path
(paper_2402_15220_b200/) never imports it and shares no code with it.

  attention.py   C1 fp64 attention over materialised per-sequence KV, and the
                 C2 literal Eqn 1 / Eqn 2 / Alg 1 / Alg 2 emulator.
  tree_model.py  C3 prefix-tree replay model emitting the canonical tables.
  sharing.py     order-free definition of which sequences share which chunk.
  reference.py   the oracle decode step used by bench.py (CPU timing arm).
  prefill.py     C4 causal prefill attention with prefix lookup (row f1).

Every function cites the PAPER.md passage it follows; pins live in
tests/test_oracle_*.py.
"""
