"""CPU fp64 oracle for the SEM Ax + dssum + Jacobi-PCG hot path (arXiv 2405.05640).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_2405_05640_b200`` (the CUDA product
path) and neither package imports the other.

Contents
--------
``sem_oracle.c``  plain C (gcc -O2 -ffp-contract=off, OpenMP over elements):
                  GLL (O1), D (O2), geometry (O4), local Ax (O5), dssum (O7),
                  multiplicity (O7), mask (O8), Jacobi (O9), PCG (O10).
``oracle.py``     ctypes marshalling + the oracle's own node numbering (O6):
                  lattice ids for box meshes, geometric matching for general
                  meshes; the time-step driver (O17).
``hsmg.py``       the pressure preconditioner of f2 (reading R16): hybrid-
                  Schwarz multigrid V-cycle and flexible GMRES, numpy/scipy
                  steps over the C pieces (import ``oracle.hsmg``).

Pins (what fixes each function independently of itself) live in
``tests/test_oracle_*.py``; see DESIGN.md "Oracle pins".  Parity status per
function: every function is pinned except throughput (P16, "parity unpinned":
the paper prints no throughput for this path).
"""
from .oracle import *  # noqa: F401,F403
