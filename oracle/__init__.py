"""fp64 CPU oracle of the SOR stress-majorization layout -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import, call, link or execute anything under
oracle/.  The product path (paper_1711_01228_b200) never does; the two share no
code, header, table or constant.

Pinned functions (see tests/test_oracle_pins.py and DESIGN.md §5):
  core.stress, core.ly_rows, core.lw_rows, core.dominant_value,
  core.hop_rows/hop_matrix, core.lw_red_dense/lw_red_matvec/lw_diag,
  layout.Problem.H / solve_reduced, layout.run_algorithm1/run_algorithm2,
  layout.sor_combine, layout.cap_step (special cases only: inf and finite),
  strategies.roulette.
End-to-end traces on the C1..C5 graphs have no value printed by the paper:
"parity unpinned" beyond the invariants the pins check.
"""
