"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the SPASE method (no compaction, no decoding, no
search).  It only draws inputs: dense runtime tables shaped like the paper's workloads
(Table 2) and random genomes.  Both the oracle side
(`oracle/`) and the CUDA side (`paper_2309_01226_b200/`) consume what it produces; neither
side's code lives here.
"""
from .workloads import (  # noqa: F401
    UPPS, DDP, FSDP, PIPE, SPILL, Instance,
    tiny, txt, img, mix, sweep, tiny_variant, lr_sweep, random_tiny, by_name, CONFIG_NAMES,
    random_genomes,
)
