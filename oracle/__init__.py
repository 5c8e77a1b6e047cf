"""CPU ORACLE for arXiv 2102.11536 — TEST INFRASTRUCTURE ONLY.

Plain, slow, fp64 NumPy/SciPy implementation of what the CUDA hot path
computes, written from PAPER.md (cited as P:line) and the readings listed in
DESIGN.md "Readings of the paper".  It shares no code with
`paper_2102_11536_b200` (the product): only `tests/`, `__graft_entry__.smoke()`
and bench.py's `cpu_baseline` / `--impl reference` legs may import it.  The
product path never routes through this package.

Modules
  splines     knot vector, Cox-de Boor basis and derivatives
  assembly    Gauss quadrature, geometry, M, K (scalar/elastic), Dirichlet,
              multi-patch gluing
  params      generalized-alpha parameters, both readings
  integrator  initial chain and the order-2k step
  spectral    amplification matrix by stepping unit vectors
  precond     Kronecker / additive-Schwarz preconditioner, PCG

Parity status: every function is pinned by tests/test_oracle_*.py against
values or properties the paper or mathematics fix; see DESIGN.md
"Oracle pins".  `assembly.operator_rows` (sampled rows for full-size checks)
is pinned by agreement with the assembled matrices at small size.
"""
