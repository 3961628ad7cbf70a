"""fp64 CPU oracle for fKK-EC -- TEST INFRASTRUCTURE ONLY.

Allowed importers: tests/, __graft_entry__.smoke(), bench.py (cpu_baseline / --impl reference).
The product package paper_2005_07132_b200 never imports this package and shares no code with it.
"""
from .fkk_oracle import *  # noqa: F401,F403
from .fkk_oracle import Params  # noqa: F401
