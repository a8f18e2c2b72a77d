"""ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (numpy, complex128 / float64) of
what the product path computes, written from PAPER.md (arxiv 2208.01498, Wahl &
Strelchuk).  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import it.  It shares no code with the CUDA/C++ path
(paper_2208_01498_b200/); the only common module is tn_inputs/ (seeded circuits).

Modules
  rng         SplitMix64 counter-based generator (same generator the C++ side
              implements independently) for the randomized steps of Algorithm 1.
  network     circuit -> closed tensor network for <x|C|0> (Theorem 2 proof,
              PAPER.md l.121-125; absorption PAPER.md l.116).
  ssa         Sphere Separator Algorithm (SM Algorithm 1),
              separator checks Eqs. (1)-(2) (l.45-49), boundary assignment
              (Theorem 1 proof, l.79), recursive hierarchy (l.80, Fig. 2), greedy
              leaf planner (SM "Numerical implementation", l.217), index slicing.
  contract    naive pairwise contraction along the order; Eq. (3) operation count.
  statevector brute-force state-vector simulation (independent check).
  bounds      Theorem 1 / 2 closed forms and constants (l.57, l.94, l.109, l.118).

Parity status: every function is pinned by tests in tests/test_oracle.py and
tests/test_oracle_ssa_pins.py (mutation check: scripts/oracle_mutations.sh) against
brute force, closed forms and invariants.
"""
