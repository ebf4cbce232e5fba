"""fp64 CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_2503_15078_b200) never imports, links or executes it, and this package
never imports the product path: the two share no code.
"""
from .oracle import *  # noqa: F401,F403
