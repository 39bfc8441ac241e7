"""oracle/ -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the SPASE hot path computes.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it.  The product package ``paper_2309_01226_b200`` never
imports it, and this package never imports the product: the two share no code.  The only
common module is ``synth`` (seeded input generators, no SPASE arithmetic).

Pieces:
  O1 decoder + O2 brute force  -- saturn_oracle.c via ctypes            (decoder.py)
  O3 validator, O5 lower bound -- plain Python                          (checks.py)
  O4a time-indexed exact solver -- plain Python DFS                     (exact.py)
  O4b the paper's MILP, Eqs. 1-11 with readings A1-A3, solved by HiGHS  (milp.py)
  O6 Philox4x32-10 and the genome (un)ranking                           (philox.py, decoder.py)
  a7 GA operator replay                                                 (ga.py)
  f2 the paper's baseline heuristics                                    (baselines.py)

Parity status per function is listed in DESIGN.md ("Oracle pins").
"""
from .decoder import (  # noqa: F401
    Compacted, compact, decode, decode_batch, decode_batch_nodes, brute_force, brute_force_node_gene,
    space_size, unrank, rank, build_library,
)
from .checks import validate, lower_bound  # noqa: F401
