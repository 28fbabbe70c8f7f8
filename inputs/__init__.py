"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA-side tests/bench.

This package holds NO arithmetic of the method (no seeding of T, no products, no
closure): it only builds CNF grammars and labelled edge lists.  Both `oracle/`
and the CUDA path consume its output; neither imports the other.
"""
from .generators import *  # noqa: F401,F403
