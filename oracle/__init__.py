"""CPU oracle for the vitertile hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker (or the timed CPU
baseline).  The product package ``paper_2011_13579_b200`` never imports it.
"""
from .oracle import *  # noqa: F401,F403
