"""Test infrastructure: the fp64 CPU oracle of the MoEBlaze layer (see moe_oracle.py).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  It shares no code with
paper_2601_05296_b200 and imports nothing from it.
"""
from .moe_oracle import *  # noqa: F401,F403
from .moe_oracle import __all__  # noqa: F401
