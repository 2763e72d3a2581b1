"""cuTAMP hot-path ORACLE -- test infrastructure only.

A plain, slow, float64 CPU implementation of what the hot path computes
(Eq. 2-4, Algorithm 1's InitializeParticles / OptimizeParticles /
IsGoalSatisfied), written from the paper and SURVEY.md §8(c).  It shares no
code with the CUDA path (`paper_2411_11833_b200/`) and never imports it.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import or execute anything under `oracle/`.
The product path must never route through it.

Parity pins: every function is checked by `tests/test_oracle_*.py` against
closed forms, library routines (scipy Rotation, torch.optim.Adam), central
finite differences and the paper's/SPEC's worked examples.  Parity unpinned:
none of the functions in this package.
"""
