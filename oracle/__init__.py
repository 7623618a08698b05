"""fp64 CPU oracle of the memory step -- TEST INFRASTRUCTURE ONLY (see vi_oracle.py).

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs.  The product package never imports it.
"""
from .vi_oracle import *  # noqa: F401,F403
from . import vi_oracle  # noqa: F401
