"""fp64 CPU oracle for the lambda-coupled electrostatics step (arXiv 2410.01626).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import or execute
anything in this package.  The product path (`paper_2410_01626_b200`, the CUDA
library behind `include/cph.h`) never imports it and shares no code with it:
no kernels, constants, tables or helpers.  The only common dependency is the
data-only input generator in `synthetic/`.

Each function cites the PAPER.md passage (P:<line>) or the DESIGN.md reading
(R<n>) it follows.  Everything is plain numpy in float64 except the pair-list
decision, which DESIGN.md R14/R15 fixes in float32 round-to-nearest.

Pins (tests/test_oracle_*.py, `-m "not gpu"`): NaCl/CsCl Madelung constants
(Ewald real+reciprocal+self), PME -> direct Ewald convergence, the
E_rec = (f/2) sum q_i phi_i identity, central finite differences of the energy
for forces and dV/dlambda, charge-conservation and sum-of-weights invariants,
closed-form bias values (SPEC examples), PFC against the Henderson-Hasselbalch
population, Philox4x32-10 known-answer vectors, integrator free flight,
equipartition and electrostatics-off H-H/Hill sampling, fit recovery.
Functions without such a pin say "parity unpinned" in their docstring.
"""
