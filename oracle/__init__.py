"""Oracle package: test infrastructure only (see graf_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.
"""
from .graf_oracle import *  # noqa: F401,F403
